CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
export SFLSQR_FUSE_SKETCH=0
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sketch_partial|k_sketch_finalize|k_ls|k_res_partial|k_mgs_pass" -s 12 -c 10 -o gpurun_out/prof_small $CMD > gpurun_out/ncu_small.log 2>&1
