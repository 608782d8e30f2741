python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2o_build.log 2>&1 || { tail gpurun_out/r2o_build.log; exit 1; }
for rep in 1 2; do
for a in "--config 1 --steps 35" "--config 3" "--config 4" "--config 3 --method sflsmr" "--config 2 --steps 95"; do
  for kn in "no_pdl_trigger" "no_pdl_trigger,unfused_orth"; do
  tag=$(echo "$a $kn $rep" | tr -d ' -,')
  timeout -s KILL 600 python bench.py $a --knobs $kn --no-cpu-baseline --no-e2e --no-windows > gpurun_out/r2o_bench_$tag.log 2>&1
  echo "$tag rc=$?"
  done
done
done
