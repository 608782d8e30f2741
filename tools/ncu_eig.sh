timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_lr_eig|k_lr_cholsolve" -s 6 -c 2 -o gpurun_out/prof_eig \
  python bench.py --config 8 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_eig.log 2>&1
