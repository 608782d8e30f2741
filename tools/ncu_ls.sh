CMD="python bench.py --steps 150 --warmup 5 --no-cpu-baseline --no-e2e --no-profile"
timeout 300 $CMD > gpurun_out/plain_ls.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ls" -s 140 -c 1 -o gpurun_out/prof_ls $CMD > gpurun_out/ncu_ls.log 2>&1
echo done
