# aligned pair-CSR (mode 17) vs 16 vs 14: parity tests and C4/C3 benches
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "pair_csr" > gpurun_out/pytest_pcsr.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pcsr.log
for m in 17 14; do
  SFLSQR_SPMV_MODE=$m timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_m$m.log 2>&1
  SFLSQR_SPMV_MODE=$m timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_m$m.log 2>&1
done
