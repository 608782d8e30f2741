# ncu --set full of the vector / small kernels of config 4 at late iterations (k ~ 150)
CMD="python bench.py --steps 150 --warmup 5 --no-cpu-baseline --no-e2e --no-profile"
timeout 300 $CMD > gpurun_out/plain_vec.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_orth_dots|k_orth_axpy|k_finish_w|k_finish_z|k_sketch_apply|k_ls|k_res_partial" -s 1000 -c 7 -o gpurun_out/prof_vec_c4 $CMD > gpurun_out/ncu_vec_c4.log 2>&1
CMD3="python bench.py --config 3 --steps 140 --warmup 5 --no-cpu-baseline --no-e2e --no-profile"
timeout 300 $CMD3 > gpurun_out/plain_vec3.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_orth_dots|k_orth_axpy|k_finish_w|k_finish_z|k_sketch_apply|k_ls|k_res_partial|k_xupdate|spmv" -s 1200 -c 9 -o gpurun_out/prof_vec_c3 $CMD3 > gpurun_out/ncu_vec_c3.log 2>&1
echo done
