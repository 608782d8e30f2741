timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "sflsmr or flsmr or graph or config1" > gpurun_out/pytest_sk.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sk.log
for r in 1 2; do
for v in 0 1; do
SFLSQR_SKETCH_SIDE=$v timeout 900 python bench.py --method sflsmr --no-cpu-baseline --no-e2e --no-profile > gpurun_out/bench_c4mr_sk$v.$r.log 2>&1
SFLSQR_SKETCH_SIDE=$v timeout 900 python bench.py --config 3 --method sflsmr --no-cpu-baseline --no-e2e --no-profile > gpurun_out/bench_c3mr_sk$v.$r.log 2>&1
SFLSQR_SKETCH_SIDE=$v timeout 900 python bench.py --config 1 --method sflsmr --steps 35 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/bench_c1mr_sk$v.$r.log 2>&1
done; done
