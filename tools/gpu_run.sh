#!/bin/bash
# One parameterised GPU-box run (gpurun snapshots the repo; outputs land in gpurun_out/).
#   tools/gpu_run.sh TAG [pytest-k-expr|all|none] [bench args...]
# e.g. gpurun -- 'bash tools/gpu_run.sh r2a all --steps 20 --warmup 5'
TAG=${1:-run}; SEL=${2:-all}; shift 2
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_gpu.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo build failed; tail -20 gpurun_out/${TAG}_build.log; exit 1; }
if [ "$SEL" != "none" ]; then
  if [ "$SEL" = "all" ]; then K=(); else K=(-k "$SEL"); fi
  timeout 3000 python -m pytest tests -m gpu -q -s "${K[@]}" > gpurun_out/${TAG}_pytest.log 2>&1
  echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
fi
if [ $# -gt 0 ] || [ "$SEL" = "all" ]; then
  timeout 900 python bench.py "$@" > gpurun_out/${TAG}_bench.log 2>&1
  echo "bench rc=$?"; tail -c 600 gpurun_out/${TAG}_bench.log
fi
