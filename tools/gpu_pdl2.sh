timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "config3 or config4 or graph or config1 or config2" > gpurun_out/pytest_pdl2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pdl2.log
for r in 1 2; do
for c in "--config 4" "--config 3" "--config 2 --steps 95" "--config 1 --steps 35"; do
  tag=$(echo $c | tr -d ' -')
  timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-profile $c > gpurun_out/bench_trig_$tag.$r.log 2>&1
done; done
