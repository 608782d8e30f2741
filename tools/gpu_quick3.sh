timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in "--config 8 --steps 90 --warmup 5" "--config 3" "--config 3 --method sflsmr" "--config 6 --steps 45 --warmup 3" "--config 4"; do
  tag=$(echo $c | tr -d ' -')
  timeout 900 python bench.py --no-cpu-baseline --no-e2e $c > gpurun_out/bench_$tag.log 2>&1
done
