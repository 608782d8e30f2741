timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --config 3 > gpurun_out/bench_c3.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --config 1 --steps 35 > gpurun_out/bench_c1.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --config 2 --steps 95 > gpurun_out/bench_c2.log 2>&1
