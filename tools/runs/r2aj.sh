# Final confirmation of round 2 on HEAD (process transport, NCCL self-test, widened process-rank tests)
# Theorem 2.1 verifiers), smoke, default bench line, config 3 line
T=r2aj
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail gpurun_out/${T}_build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/${T}_gpu.txt
timeout -s KILL 2400 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"
timeout -s KILL 900 python bench.py > gpurun_out/${T}_bench_default.log 2>&1; echo "default rc=$?"
timeout -s KILL 600 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_config3.log 2>&1; echo "c3 rc=$?"
echo done
