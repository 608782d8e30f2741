# TMA-staged product v2 (gathers of the next chunk in flight): tests + A/B (default, variant 0, 1)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2u_build.log 2>&1 || { tail gpurun_out/r2u_build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests/test_gpu_tma.py -m gpu -q -x > gpurun_out/r2u_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2u_pytest.log
for v in def tma0 tma1 g2 g4; do
  unset SFLSQR_GRAPH_ITERS
  case $v in def) K="";; tma0) K="--knobs tma"; export SFLSQR_TMA_VARIANT=0;; tma1) K="--knobs tma"; export SFLSQR_TMA_VARIANT=1;; g2) K=""; export SFLSQR_GRAPH_ITERS=2;; g4) K=""; export SFLSQR_GRAPH_ITERS=4;; esac
  for a in "--config 3 --steps 100" "--config 4 --steps 40" "--config 1 --steps 36"; do
    tag=$(echo "$a $v" | tr -d ' -')
    timeout -s KILL 600 python bench.py $a $K --no-cpu-baseline --no-e2e --no-windows > gpurun_out/r2u_bench_$tag.log 2>&1; echo "$tag rc=$?"
  done
done
export SFLSQR_TMA_VARIANT=0; unset SFLSQR_GRAPH_ITERS
CMD="python bench.py --no-cpu-baseline --no-e2e --no-windows --no-profile --config 4 --steps 3 --warmup 3 --knobs tma"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_spmv_tma" -s 3 -c 1 -o gpurun_out/r2u_c4tma $CMD > gpurun_out/r2u_c4_ncu.log 2>&1; echo "ncu c4 rc=$?"
echo done
