# TMA-staged pair-CSR product: GPU tests, same-box A/B on configs 3/4, ncu of the TMA kernel
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2t_build.log 2>&1 || { tail gpurun_out/r2t_build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests/test_gpu_tma.py -m gpu -q -x > gpurun_out/r2t_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2t_pytest.log
for rep in 1 2; do
for v in def tma0 tma1; do
  case $v in def) K="";; tma0) K="--knobs tma"; export SFLSQR_TMA_VARIANT=0;; tma1) K="--knobs tma"; export SFLSQR_TMA_VARIANT=1;; esac
  for a in "--config 3" "--config 4 --steps 40"; do
    tag=$(echo "$a $v r$rep" | tr -d ' -')
    timeout -s KILL 600 python bench.py $a $K --no-cpu-baseline --no-e2e --no-windows > gpurun_out/r2t_bench_$tag.log 2>&1; echo "$tag rc=$?"
  done
done
done
export SFLSQR_TMA_VARIANT=0
CMD="python bench.py --no-cpu-baseline --no-e2e --no-windows --no-profile --config 4 --steps 3 --warmup 3 --knobs tma"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_spmv_tma" -s 3 -c 1 -o gpurun_out/r2t_c4tma $CMD > gpurun_out/r2t_c4_ncu.log 2>&1; echo "ncu c4 rc=$?"
echo done
