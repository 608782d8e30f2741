timeout 1200 python -m pytest tests/test_gpu_gkb.py tests/test_gpu_sharded.py -q -x -p no:cacheprovider > gpurun_out/pytest_epi.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_epi.log
for r in 1 2; do
for c in "--config 4 --method lsqr" "--config 3 --method lsqr" "--config 4"; do
  tag=$(echo $c | tr -d ' -')
  timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-profile $c > gpurun_out/bench_epi_$tag.$r.log 2>&1
done; done
