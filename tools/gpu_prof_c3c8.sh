CMD3="python bench.py --config 3 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e"
timeout 300 $CMD3 > gpurun_out/plain3.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $CMD3 > gpurun_out/ncu_l3.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"spmv" -s 10 -c 2 -o gpurun_out/prof_c3 $CMD3 > gpurun_out/ncu_f3.log 2>&1
CMD8="python bench.py --config 8 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD8 > gpurun_out/plain8.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c8.csv $CMD8 > gpurun_out/ncu_l8.log 2>&1
