python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2k_build.log 2>&1 || { tail gpurun_out/r2k_build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_flsqr.py tests/test_gpu_sharded.py tests/test_gpu_gkb.py tests/test_gpu_lowrank.py -m gpu -q -x -k "not full_size and not c4_full and not state_injection" > gpurun_out/r2k_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r2k_pytest.log
timeout 600 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/r2k_bench_c3.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2k_bench_c4.log 2>&1
timeout 600 python bench.py --config 1 --steps 35 --no-cpu-baseline --no-e2e > gpurun_out/r2k_bench_c1.log 2>&1
timeout 600 python bench.py --config 4 --method flsqr --no-cpu-baseline --no-e2e --no-windows > gpurun_out/r2k_bench_c4flsqr.log 2>&1
echo done
