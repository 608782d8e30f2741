# deferred stop: new tests, full GPU suite, A/B (default = deferred vs --knobs stop_inline)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2w_build.log 2>&1 || { tail gpurun_out/r2w_build.log; exit 1; }
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2w_smoke.log 2>&1; echo "smoke rc=$?"
timeout -s KILL 900 python -m pytest tests/test_gpu_schedule.py -m gpu -q -x > gpurun_out/r2w_pytest_sched.log 2>&1; echo "pytest sched rc=$?"; tail -15 gpurun_out/r2w_pytest_sched.log
for rep in 1 2; do
for v in def inl; do
  case $v in def) K="";; inl) K="--knobs stop_inline";; esac
  for a in "--config 4 --steps 40" "--config 4 --steps 100 --warmup 100" "--config 3 --steps 100" "--config 3 --steps 100 --method sflsmr"; do
    tag=$(echo "$a $v r$rep" | tr -d ' -')
    timeout -s KILL 600 python bench.py $a $K --no-cpu-baseline --no-e2e --no-windows > gpurun_out/r2w_bench_$tag.log 2>&1; echo "$tag rc=$?"
  done
done
done
timeout -s KILL 2700 python -m pytest tests -m gpu -q -x > gpurun_out/r2w_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2w_pytest.log
echo done
