timeout 1500 python -m pytest tests/test_gpu_gkb.py tests/test_gpu_sharded.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_sellepi.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sellepi.log
for c in "--config 4 --method lsqr" "--config 4 --method lsmr"; do
  tag=$(echo $c | tr -d ' -')
  timeout 900 python bench.py --no-cpu-baseline --no-e2e $c > gpurun_out/bench_se_$tag.log 2>&1
done
