timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "config3 or config4 or graph or config1" > gpurun_out/pytest_gemv4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemv4.log
for r in 1 2; do
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_gv.$r.log 2>&1
timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_gv.$r.log 2>&1
done
