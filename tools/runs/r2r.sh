# A/B: orthogonalisation kernels at 1024 threads for 76k-303k-element vectors (v1) vs 256 (v0)
K=paper_2605_22281_b200/csrc/sflsqr_kernels.cuh; C=paper_2605_22281_b200/csrc/sflsqr.cu
cp $K /tmp/keepk; cp $C /tmp/keepc
for rep in 1 2; do
for v in 0 1; do
  cp tools/runs/ab/k$v.cuh $K; cp tools/runs/ab/c$v.cu $C
  python -c "from paper_2605_22281_b200._build import build_library; build_library()" > gpurun_out/r2r_build_v$v.log 2>&1 || { echo "build v$v failed"; tail -5 gpurun_out/r2r_build_v$v.log; continue; }
  for a in "--config 3" "--config 3 --method sflsmr" "--config 3 --method flsqr" "--config 8 --steps 45"; do
    tag=$(echo "$a v$v r$rep" | tr -d ' -,')
    timeout -s KILL 600 python bench.py $a --no-cpu-baseline --no-e2e --no-windows > gpurun_out/r2r_bench_$tag.log 2>&1
    echo "$tag rc=$?"
  done
done
done
cp /tmp/keepk $K; cp /tmp/keepc $C
python -c "from paper_2605_22281_b200._build import build_library; build_library()" > /dev/null 2>&1
timeout -s KILL 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_flsqr.py tests/test_gpu_lowrank.py tests/test_gpu_sharded.py -m gpu -q -x > gpurun_out/r2r_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r2r_pytest.log
