# w normalisation after the rows (tail) instead of before: A/B vs wnorm_sep on configs 4 and 3, tests
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2y_build.log 2>&1 || { tail gpurun_out/r2y_build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests/test_gpu_tma.py tests/test_gpu_parity.py -m gpu -q -x -k "wnorm or knobs or config4 or config3" > gpurun_out/r2y_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2y_pytest.log
for rep in 1 2; do
for v in def sep; do
  case $v in def) K="";; sep) K="--knobs wnorm_sep";; esac
  for a in "--config 4 --steps 60" "--config 3 --steps 100"; do
    tag=$(echo "$a $v r$rep" | tr -d ' -')
    timeout -s KILL 600 python bench.py $a $K --no-cpu-baseline --no-e2e --no-windows > gpurun_out/r2y_bench_$tag.log 2>&1; echo "$tag rc=$?"
  done
done
done
CMD="python bench.py --no-cpu-baseline --no-e2e --no-windows --no-profile --config 4 --steps 3 --warmup 3"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_spmv|k_finish" --csv --log-file gpurun_out/r2y_c4_def.csv $CMD > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_spmv|k_finish" --csv --log-file gpurun_out/r2y_c4_sep.csv $CMD --knobs wnorm_sep > /dev/null 2>&1
echo done
