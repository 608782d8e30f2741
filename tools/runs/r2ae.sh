# Process ranks over CUDA IPC (SFLSQR_COMM_IPC) on one GPU, then the whole suite, smoke and bench
T=r2ae
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail gpurun_out/${T}_build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/${T}_gpu.txt
timeout -s KILL 900 python -m pytest tests/test_gpu_ipc_processes.py -m gpu -q -x > gpurun_out/${T}_ipc.log 2>&1
echo "ipc rc=$?"; tail -30 gpurun_out/${T}_ipc.log
timeout -s KILL 600 python -m pytest tests/test_gpu_sharded.py -m gpu -q -x > gpurun_out/${T}_sharded.log 2>&1
echo "sharded rc=$?"; tail -3 gpurun_out/${T}_sharded.log
echo done
