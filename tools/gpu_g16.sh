timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gkb.py tests/test_gpu_flsqr.py -q -x -p no:cacheprovider > gpurun_out/pytest_g16.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g16.log
for r in 1 2; do
for v in 0 1; do
SFLSQR_GATHER16=$v timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_g$v.$r.log 2>&1
done; done
SFLSQR_GATHER16=1 timeout 900 python bench.py --method lsqr --no-cpu-baseline --no-e2e > gpurun_out/bench_c4lsqr_g1.log 2>&1
SFLSQR_GATHER16=0 timeout 900 python bench.py --method lsqr --no-cpu-baseline --no-e2e > gpurun_out/bench_c4lsqr_g0.log 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none -k regex:"spmv" -s 4 -c 2 -o gpurun_out/prof_g16 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_g16.log 2>&1
