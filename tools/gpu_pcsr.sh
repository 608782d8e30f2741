# pair-CSR (SpMV mode 16): parity tests, C4/C3 benches mode 14 vs 16 (pair unroll 2, 4)
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "pair_csr or csr16" > gpurun_out/pytest_pcsr.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pcsr.log
SFLSQR_SPMV_MODE=14 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_m14.log 2>&1
for u in 2 4; do
  SFLSQR_PCSR_UNROLL=$u SFLSQR_SPMV_MODE=16 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_m16u$u.log 2>&1
  SFLSQR_PCSR_UNROLL=$u SFLSQR_SPMV_MODE=16 timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_m16u$u.log 2>&1
done
