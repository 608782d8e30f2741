timeout 1500 python -m pytest tests/test_gpu_flsqr.py tests/test_gpu_gaussian.py tests/test_gpu_lowrank.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_cgssel.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cgssel.log
for v in 1 0; do
for c in "--config 4 --method flsqr" "--config 4 --method flsmr" "--config 3 --method flsqr" "--config 6 --steps 45 --warmup 3 --no-profile"; do
  tag=$(echo $c | tr -d ' -')
  SFLSQR_CGS_SELECTIVE=$v timeout 900 python bench.py --no-cpu-baseline --no-e2e $c > gpurun_out/bench_cs${v}_$tag.log 2>&1
done; done
