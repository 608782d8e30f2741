python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2h_build.log 2>&1 || exit 1
CMD="python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-windows"
timeout 300 $CMD > gpurun_out/r2h_plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_ic16 -s 4 -c 2 -o gpurun_out/r2h_ic16 $CMD > gpurun_out/r2h_ncu.log 2>&1
echo "rc=$?"
