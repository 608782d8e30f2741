python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2f_build.log 2>&1 || { tail gpurun_out/r2f_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gkb.py tests/test_gpu_sharded.py -m gpu -q -x -k "ic16 or pair or format or odd or config3_reduced or config1_full or spmv or transpose or gkb_parity or colshard_config3 or peer or knob" > gpurun_out/r2f_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r2f_pytest.log
for c in 3 4; do timeout 600 python bench.py --config $c --steps 60 --no-cpu-baseline --no-e2e --no-windows > gpurun_out/r2f_bench_c$c.log 2>&1; done
SFLSQR_X=1 timeout 600 python - > gpurun_out/r2f_ab.log 2>&1 <<'PY'
import json, subprocess, sys
PY
echo done
