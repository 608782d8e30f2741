CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-profile"
timeout 300 $CMD > gpurun_out/plain3.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmv" -s 2 -c 2 -o gpurun_out/prof_spmv_tiled $CMD > gpurun_out/ncu_spmv_tiled.log 2>&1
echo done
