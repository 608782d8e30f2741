# A/B of SpMV prologue variants: v0 (HEAD), v1 (singleton prefetch hoisted), v2 (v1 + cross-row row pointers)
K=paper_2605_22281_b200/csrc/sflsqr_kernels.cuh
cp $K /tmp/keep.cuh
for rep in 1 2; do
for v in 0 1 2; do
  cp tools/runs/ab/v$v.cuh $K
  python -c "from paper_2605_22281_b200._build import build_library; build_library()" > gpurun_out/r2p_build_v$v.log 2>&1 || { echo "build v$v failed"; tail -5 gpurun_out/r2p_build_v$v.log; continue; }
  for a in "--config 3" "--config 3 --method lsqr" "--config 4"; do
    tag=$(echo "$a v$v r$rep" | tr -d ' -,')
    timeout -s KILL 600 python bench.py $a --no-cpu-baseline --no-e2e --no-windows > gpurun_out/r2p_bench_$tag.log 2>&1
    echo "$tag rc=$?"
  done
done
done
cp /tmp/keep.cuh $K
python -c "from paper_2605_22281_b200._build import build_library; build_library()" > /dev/null 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gkb.py -m gpu -q -x -k "config3_reduced or knobs or format or warp or pair or gkb_parity or config4_reduced" > gpurun_out/r2p_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r2p_pytest.log
