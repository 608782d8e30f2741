# C3 launch list + ncu --set full of the vector kernels and the two products (iterations ~10)
bash tools/ncu_capture.sh r2d_c3vec "k_orth|k_finish|k_stop" 60 10 --config 3 --steps 5 --warmup 5
bash tools/ncu_capture.sh r2d_c3spmv "k_spmv" 20 4 --config 3 --steps 5 --warmup 5
bash tools/ncu_capture.sh r2d_c4spmv "k_spmv" 12 4 --config 4 --steps 3 --warmup 3
echo done
