# z normalisation fused into the A product: new tests, full GPU suite, A/B vs --knobs znorm_sep
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2aa_build.log 2>&1 || { tail gpurun_out/r2aa_build.log; exit 1; }
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2aa_smoke.log 2>&1; echo "smoke rc=$?"
timeout -s KILL 900 python -m pytest tests/test_gpu_tma.py -m gpu -q > gpurun_out/r2aa_pytest_tma.log 2>&1; echo "pytest tma rc=$?"; tail -15 gpurun_out/r2aa_pytest_tma.log
for rep in 1 2; do
for v in def sep; do
  case $v in def) K="";; sep) K="--knobs znorm_sep";; esac
  for a in "--config 3 --steps 100" "--config 4 --steps 60" "--config 1 --steps 36"; do
    tag=$(echo "$a $v r$rep" | tr -d ' -')
    timeout -s KILL 600 python bench.py $a $K --no-cpu-baseline --no-e2e --no-windows > gpurun_out/r2aa_bench_$tag.log 2>&1; echo "$tag rc=$?"
  done
done
done
timeout -s KILL 2700 python -m pytest tests -m gpu -q > gpurun_out/r2aa_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2aa_pytest.log
echo done
