# N = 2 bench paths on ONE GPU (both ranks on device 0; CF_BENCH_DEVICE): the
# row-band IPC fused-halo path on cfg4 and image-per-rank cfg5.  Proves the
# multi-process plumbing end to end; the numbers are not a scaling result
# (two ranks share one GPU).
O=gpurun_out; TAG=${1:-r02o}
export CF_BENCH_DEVICE=0
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29561 bench.py --gpus 2 --steps 3 --warmup 3 --halo ipc --no-cpu-baseline \
  > $O/bench_n2_ipc_cfg4_$TAG.json 2> $O/bench_n2_ipc_cfg4_$TAG.err; echo "cfg4 n2 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29562 bench.py --gpus 2 --steps 3 --warmup 3 --halo ipc --workload cfg5 \
  --no-cpu-baseline > $O/bench_n2_cfg5_$TAG.json 2> $O/bench_n2_cfg5_$TAG.err; echo "cfg5 n2 rc=$?"
tail -c 400 $O/bench_n2_ipc_cfg4_$TAG.json; tail -c 400 $O/bench_n2_cfg5_$TAG.json
