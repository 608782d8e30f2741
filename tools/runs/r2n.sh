python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2n_build.log 2>&1 || { tail gpurun_out/r2n_build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "one_launch or knobs_bitwise or config3_reduced or config1" > gpurun_out/r2n_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r2n_pytest.log
for a in "--config 3" "--config 3 --knobs no_pdl_trigger" "--config 3 --knobs unfused_orth" "--config 3 --knobs no_pdl_trigger,unfused_orth" "--config 3 --method sflsmr" "--config 3 --method sflsmr --knobs unfused_orth" "--config 4" "--config 4 --knobs unfused_orth" "--config 4 --knobs no_pdl_trigger,unfused_orth" "--config 1 --steps 35" "--config 1 --steps 35 --knobs no_pdl_trigger,unfused_orth"; do
  tag=$(echo "$a" | tr -d ' -,')
  timeout -s KILL 600 python bench.py $a --no-cpu-baseline --no-e2e --no-windows > gpurun_out/r2n_bench_$tag.log 2>&1
  echo "$tag rc=$?"
done
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2n_pytest_all.log 2>&1
echo "pytest all rc=$?"; tail -3 gpurun_out/r2n_pytest_all.log
