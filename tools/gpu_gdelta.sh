for r in 1 2; do
for dlt in 0 1 2; do
SFLSQR_SPMV_GRID_DELTA=$dlt timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-profile > gpurun_out/bench_c4_gd$dlt.$r.log 2>&1
SFLSQR_SPMV_GRID_DELTA=$dlt timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/bench_c3_gd$dlt.$r.log 2>&1
done; done
