for r in 1 2 3; do
for v in 1 0; do
SFLSQR_SKETCH_SIDE=$v timeout 900 python bench.py --config 2 --steps 95 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/bench_c2_sk$v.$r.log 2>&1
SFLSQR_SKETCH_SIDE=$v timeout 900 python bench.py --config 1 --steps 35 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/bench_c1_sk$v.$r.log 2>&1
done; done
