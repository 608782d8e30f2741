timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_fused.log 2>&1
SFLSQR_FUSE_SKETCH=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_unfused.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --config 3 > gpurun_out/bench_c3.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --config 3 --method sflsmr > gpurun_out/bench_c3m.log 2>&1
