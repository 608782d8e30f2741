# low-rank tau_r (config 8): parity tests, bench, launch list
timeout 900 python -m pytest tests/test_gpu_lowrank.py -q -x -p no:cacheprovider > gpurun_out/pytest_lr.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_lr.log
timeout 600 python bench.py --config 8 --steps 90 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c8.log 2>&1
timeout 600 python bench.py --config 8 --method sflsmr --steps 90 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c8mr.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c8.csv \
  python bench.py --config 8 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c8.log 2>&1
