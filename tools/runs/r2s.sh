# Re-entry check of the checkpoint + A z wavefront breakdown (C4, C3) for the TMA staging decision
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2s_build.log 2>&1 || { tail gpurun_out/r2s_build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/r2s_gpu.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2s_smoke.log 2>&1; echo "smoke rc=$?"
for a in "--config 4 --steps 40" "--config 3"; do
  tag=$(echo "$a" | tr -d ' -')
  timeout -s KILL 600 python bench.py $a --no-cpu-baseline --no-e2e --no-windows > gpurun_out/r2s_bench_$tag.log 2>&1; echo "$tag rc=$?"
done
CMD="python bench.py --no-cpu-baseline --no-e2e --no-windows --no-profile --config 4 --steps 3 --warmup 3"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_spmv" -s 6 -c 2 -o gpurun_out/r2s_c4 $CMD > gpurun_out/r2s_c4_ncu.log 2>&1; echo "ncu c4 rc=$?"
CMD="python bench.py --no-cpu-baseline --no-e2e --no-windows --no-profile --config 3 --steps 3 --warmup 5"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_spmv" -s 10 -c 2 -o gpurun_out/r2s_c3 $CMD > gpurun_out/r2s_c3_ncu.log 2>&1; echo "ncu c3 rc=$?"
echo done
