#!/bin/bash
# ncu on the GPU box, after the same command has exited 0 without ncu (B200_PROFILING.md):
#   tools/ncu_capture.sh TAG KERNEL_REGEX LAUNCH_SKIP LAUNCH_COUNT [bench args...]
# writes gpurun_out/TAG_launches.csv (every launch, gpu__time_duration, clocks unlocked) and
# gpurun_out/TAG.ncu-rep (--set full of the selected launches of KERNEL_REGEX).
TAG=$1; KRX=$2; SKIP=$3; CNT=$4; shift 4
CMD="python bench.py --no-cpu-baseline --no-e2e --no-windows $*"
mkdir -p gpurun_out
timeout 600 $CMD > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/${TAG}_plain.log; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:${KRX}" -s "$SKIP" -c "$CNT" \
  -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu full rc=$?"
