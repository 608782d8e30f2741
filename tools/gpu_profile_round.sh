# full GPU tests, smoke, default bench (with cpu_baseline), reference arm, ncu launch list + full capture of the dominant kernel
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_default.log
timeout 900 python bench.py --no-profile --no-cpu-baseline > gpurun_out/bench_graph.log 2>&1
SFLSQR_REF_BUDGET_S=60 timeout 900 python bench.py --impl reference --steps 195 --warmup 5 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
timeout 300 $CMD > gpurun_out/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmv|k_ls|k_sketch_apply|k_res_partial" -s 20 -c 8 -o gpurun_out/prof_r1 $CMD > gpurun_out/ncu_full.log 2>&1
echo done
