timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "config3 or config4 or graph" > gpurun_out/pytest_sk.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sk.log
SFLSQR_SKETCH_SIDE=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "config3 or config4 or graph" > gpurun_out/pytest_sk1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sk1.log
for r in 1 2; do
for v in 0 1; do
SFLSQR_SKETCH_SIDE=$v timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-profile > gpurun_out/bench_c4_sk$v.$r.log 2>&1
SFLSQR_SKETCH_SIDE=$v timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/bench_c3_sk$v.$r.log 2>&1
SFLSQR_SKETCH_SIDE=$v timeout 900 python bench.py --config 2 --steps 95 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/bench_c2_sk$v.$r.log 2>&1
done; done
