# NCCL transport one-rank self-test (eager + graph capture), then the sharded and process-rank suites
T=r2ah
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail gpurun_out/${T}_build.log; exit 1; }
NCCL_DEBUG=WARN timeout -s KILL 600 python -m pytest tests/test_gpu_sharded.py -m gpu -q -x -k "nccl" > gpurun_out/${T}_nccl.log 2>&1
echo "nccl rc=$?"; tail -15 gpurun_out/${T}_nccl.log
timeout -s KILL 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_ipc_processes.py -m gpu -q > gpurun_out/${T}_sharded.log 2>&1
echo "sharded rc=$?"; tail -3 gpurun_out/${T}_sharded.log
echo done
