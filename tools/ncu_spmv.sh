CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv -s 1 -c 2 -o gpurun_out/prof_spmv2 $CMD > gpurun_out/ncu_full2.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_v2.log 2>&1
