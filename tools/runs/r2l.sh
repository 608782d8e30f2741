python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2l_build.log 2>&1 || { tail gpurun_out/r2l_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -m gpu -q -x -k "full_warp or config3_reduced or colshard or config5_reduced_to or pair or format or knob" > gpurun_out/r2l_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r2l_pytest.log
for kn in "" "half_warp_rows"; do
  for m in sflsqr lsqr; do
  timeout 600 python bench.py --config 3 --method $m --no-cpu-baseline --no-e2e --no-windows --knobs "$kn" > gpurun_out/r2l_bench_c3_${m}_${kn:-def}.log 2>&1
  done
done
echo done
