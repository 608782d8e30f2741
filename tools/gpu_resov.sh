for r in 1 2; do
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_def$r.log 2>&1
SFLSQR_RES_OVERLAP=1 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_resov$r.log 2>&1
done
