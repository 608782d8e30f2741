# The sharded bench branch under torchrun (world 2 and 4) as process ranks over CUDA IPC on one GPU
# (functional check of bench.py's N > 1 path: each rank generates only its rows; not a scaling number)
T=r2af
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail gpurun_out/${T}_build.log; exit 1; }
for N in 2 4; do
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus $N --config 3 --comm ipc --steps 30 --warmup 5 --no-windows > gpurun_out/${T}_bench_c3_ipc$N.log 2> gpurun_out/${T}_bench_c3_ipc$N.err
echo "c3 ipc$N rc=$?"; tail -c 1500 gpurun_out/${T}_bench_c3_ipc$N.log; tail -5 gpurun_out/${T}_bench_c3_ipc$N.err
done
timeout -s KILL 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --gpus 2 --config 4 --comm ipc --steps 20 --warmup 5 --no-windows > gpurun_out/${T}_bench_c4_ipc2.log 2> gpurun_out/${T}_bench_c4_ipc2.err
echo "c4 ipc2 rc=$?"; tail -c 1200 gpurun_out/${T}_bench_c4_ipc2.log; tail -5 gpurun_out/${T}_bench_c4_ipc2.err
echo done
