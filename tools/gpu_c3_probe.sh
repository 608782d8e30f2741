timeout 600 python tools/spmv_tune.py 3 > gpurun_out/tune_c3.log 2>&1
timeout 600 python tools/spmv_tune.py 4 > gpurun_out/tune_c4.log 2>&1
CMD="python bench.py --config 3 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain_c3.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $CMD > gpurun_out/ncu_launch_c3.log 2>&1
timeout 300 $CMD > gpurun_out/plain_c3b.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmv" -s 10 -c 2 -o gpurun_out/prof_c3 $CMD > gpurun_out/ncu_full_c3.log 2>&1
echo done
