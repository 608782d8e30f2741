# Round-2 final captures (fused w normalisation after the rows, TMA opt-in); same recipe as r2q
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2z_build.log 2>&1 || { tail gpurun_out/r2z_build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/r2z_gpu.txt
timeout -s KILL 2400 python -m pytest tests -m gpu -q > gpurun_out/r2z_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r2z_pytest.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2z_smoke.log 2>&1; echo "smoke rc=$?"
timeout -s KILL 900 python bench.py > gpurun_out/r2z_bench_default.log 2>&1; echo "default rc=$?"
timeout -s KILL 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2z_bench_reference.log 2>&1; echo "ref rc=$?"
for a in "--config 3" "--config 3 --method sflsmr" "--config 3 --method flsqr" "--config 3 --method lsqr" "--config 4 --method sflsmr" "--config 4 --method flsqr" "--config 4 --method lsqr" "--config 2 --steps 95" "--config 1 --steps 35" "--config 8 --steps 45" "--config 6 --steps 45 --warmup 3" "--config 7 --steps 45 --warmup 3"; do
  tag=$(echo "$a" | tr -d ' -')
  timeout -s KILL 600 python bench.py $a --no-cpu-baseline --no-e2e > gpurun_out/r2z_bench_$tag.log 2>&1
done
bash tools/ncu_capture.sh r2z_c4 "k_spmv|k_orth|k_finish|k_res|k_sketch_apply|k_ls" 40 16 --config 4 --steps 5 --warmup 3
bash tools/ncu_capture.sh r2z_c3 "k_spmv|k_orth|k_finish|k_res|k_sketch_apply|k_ls|k_xupdate" 20 16 --config 3 --steps 5 --warmup 5
echo done
# summaries on the box (the .ncu-rep files exceed gpurun's 64 MiB return limit)
for c in c4 c3; do
  python tools/ncu_summary.py launches gpurun_out/r2z_${c}_launches.csv > gpurun_out/r2z_launch_share_${c}.md 2>&1
  python tools/ncu_summary.py full gpurun_out/r2z_${c}.ncu-rep > gpurun_out/r2z_ncu_full_${c}_key_metrics.csv 2>&1
  ncu -i gpurun_out/r2z_${c}.ncu-rep --page raw --csv > gpurun_out/r2z_ncu_full_${c}_raw.csv 2>/dev/null
  gzip -f gpurun_out/r2z_ncu_full_${c}_raw.csv
  rm -f gpurun_out/r2z_${c}.ncu-rep
done
du -sh gpurun_out
