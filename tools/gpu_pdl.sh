timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_pdl.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pdl.log
for r in 1 2; do
for v in 0 1; do
for c in "--config 4" "--config 3" "--config 2 --steps 95" "--config 1 --steps 35"; do
  tag=$(echo $c | tr -d ' -')
  SFLSQR_PDL=$v timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-profile $c > gpurun_out/bench_pdl${v}_$tag.$r.log 2>&1
done; done; done
