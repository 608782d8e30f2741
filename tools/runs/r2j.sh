python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2j_build.log 2>&1 || exit 1
timeout 900 python bench.py > gpurun_out/r2j_bench_default.log 2>&1; echo "default rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2j_bench_reference.log 2>&1; echo "ref rc=$?"
for a in "--config 3" "--config 3 --method sflsmr" "--config 3 --method flsqr" "--config 3 --method lsqr" "--config 4 --method sflsmr" "--config 4 --method flsqr" "--config 4 --method lsqr" "--config 2 --steps 95" "--config 1 --steps 35" "--config 8 --steps 45" "--config 6 --steps 45 --warmup 3"; do
  tag=$(echo "$a" | tr -d ' -')
  timeout 600 python bench.py $a --no-cpu-baseline --no-e2e > gpurun_out/r2j_bench_$tag.log 2>&1
done
bash tools/ncu_capture.sh r2j_c4 "k_spmv|k_orth|k_finish|k_res|k_sketch_apply|k_ls" 40 16 --config 4 --steps 5 --warmup 3
bash tools/ncu_capture.sh r2j_c3 "k_spmv" 20 4 --config 3 --steps 5 --warmup 5
echo done
