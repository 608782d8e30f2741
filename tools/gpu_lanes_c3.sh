for r in 1 2; do
for v in 16 8 32; do
SFLSQR_PAIR_LANES=$v timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_pl$v.$r.log 2>&1
done; done
