# W-path residual from the unnormalised w' (forked beside the transpose product): config 3 A/B vs r2ac
T=r2ad
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail gpurun_out/${T}_build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/${T}_gpu.txt
for a in "--config 3" "--config 3 --method sflsmr"; do
  tag=$(echo "$a" | tr -d ' -')
  timeout -s KILL 600 python bench.py $a --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_$tag.log 2>&1; echo "$a rc=$?"
done
timeout -s KILL 2400 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
timeout -s KILL 900 python bench.py > gpurun_out/${T}_bench_default.log 2>&1; echo "default rc=$?"
timeout -s KILL 600 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_config3b.log 2>&1; echo "c3b rc=$?"
echo done
