timeout 900 env SFLSQR_PAIR_LANES=8 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "config3 or config4 or pair" > gpurun_out/pytest_l8.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_l8.log
for r in 1 2; do
for v in 16 8; do
SFLSQR_PAIR_LANES=$v timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_l$v.$r.log 2>&1
SFLSQR_PAIR_LANES=$v timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_l$v.$r.log 2>&1
done; done
