bash tools/gpu_run.sh r2c all --steps 20 --warmup 5
for cfg in 3; do timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r2c_bench_c$cfg.log 2>&1; done
timeout 600 python bench.py --config 4 --method flsqr --no-cpu-baseline --no-e2e --no-windows > gpurun_out/r2c_bench_c4flsqr.log 2>&1
timeout 600 python bench.py --config 4 --no-cpu-baseline --no-e2e --no-windows > gpurun_out/r2c_bench_c4_k195.log 2>&1
echo done
