for r in 1 2 3; do
for v in 1 0; do
SFLSQR_SKETCH_SIDE=$v timeout 600 python bench.py --config 6 --steps 45 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/bench_c6_sk$v.$r.log 2>&1
done; done
