bash tools/gpu_run.sh r2i all --steps 20 --warmup 5
for c in 3 4 1; do
  for kn in "" "no_fused_dots"; do
    timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --no-windows --knobs "$kn" > gpurun_out/r2i_bench_c${c}_${kn:-def}.log 2>&1
  done
done
timeout 600 python bench.py --config 4 --no-cpu-baseline --no-e2e --no-windows --knobs no_ell_c16 > gpurun_out/r2i_bench_c4_no_ell_c16.log 2>&1
echo done
