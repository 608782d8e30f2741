timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gkb.py tests/test_gpu_flsqr.py tests/test_gpu_sharded.py -q -x -p no:cacheprovider > gpurun_out/pytest_sell.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sell.log
for r in 1 2; do
for v in 0 1; do
SFLSQR_SELL=$v timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_sell$v.$r.log 2>&1
done; done
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none -k regex:"spmv" -s 4 -c 2 -o gpurun_out/prof_sell python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_sell.log 2>&1
