timeout 900 env SFLSQR_SELL_A=1 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "config3 or config4 or full_size" > gpurun_out/pytest_sella.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sella.log
for r in 1 2; do
for v in 0 1; do
SFLSQR_SELL_A=$v timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_sa$v.$r.log 2>&1
SFLSQR_SELL_A=$v timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_sa$v.$r.log 2>&1
done; done
SFLSQR_SELL_A=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && SFLSQR_SELL_A=1 timeout 900 ncu --set full --clock-control none -k regex:"spmv" -s 4 -c 2 -o gpurun_out/prof_sella python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_sella.log 2>&1
