python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2g_build.log 2>&1 || { tail gpurun_out/r2g_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gkb.py tests/test_gpu_sharded.py tests/test_gpu_flsqr.py -m gpu -q -x -k "ic16 or pair or format or odd or config3_reduced or config1_full or spmv or transpose or gkb_parity or colshard_config3 or peer or knob or config4_reduced" > gpurun_out/r2g_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r2g_pytest.log
for c in 3 4; do
  for kn in "" "no_ic16"; do
    timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --no-windows --knobs "$kn" > gpurun_out/r2g_bench_c${c}_${kn:-def}.log 2>&1
  done
done
echo done
