# All-config bench lines (no CPU baseline, no e2e) for DESIGN.md / BASELINE.md tables
for c in "--config 4" "--config 4 --method flsqr" "--config 4 --method flsmr" "--config 4 --method lsqr" "--config 4 --method lsmr" "--config 4 --method sflsmr" "--config 3" "--config 3 --method sflsmr" "--config 3 --method flsqr" "--config 3 --method lsqr" "--config 2 --steps 95" "--config 1 --steps 35" "--config 6 --steps 45 --warmup 3" "--config 8 --steps 90 --warmup 5" "--config 8 --method sflsmr --steps 90 --warmup 5"; do
  tag=$(echo $c | tr -d ' -')
  timeout 900 python bench.py --no-cpu-baseline --no-e2e $c > gpurun_out/bench_$tag.log 2>&1
done
echo done
