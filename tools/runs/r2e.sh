python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2e_build.log 2>&1 || { tail gpurun_out/r2e_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_flsqr.py tests/test_gpu_sharded.py -m gpu -q -x -k "config1 or config3_reduced or edge or tiny or breakdown or k1 or knob or colshard_config3 or selective or config2" > gpurun_out/r2e_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r2e_pytest.log
timeout 600 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/r2e_bench_c3.log 2>&1
timeout 600 python bench.py --config 4 --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/r2e_bench_c4.log 2>&1
timeout 600 python bench.py --config 4 --method flsqr --no-cpu-baseline --no-e2e --no-windows > gpurun_out/r2e_bench_c4flsqr.log 2>&1
timeout 600 python bench.py --config 1 --steps 35 --no-cpu-baseline --no-e2e --no-windows > gpurun_out/r2e_bench_c1.log 2>&1
echo done
