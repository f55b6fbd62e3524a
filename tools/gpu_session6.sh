O=gpurun_out; TAG=${1:-r02n}
for c in cfg4 cfg5 cfg1_16k; do timeout 600 python bench.py --precision fp64 --workload $c --steps 5 --warmup 3 >> $O/bench_f64_$TAG.jsonl 2>> $O/bench_f64_$TAG.err; echo "f64 $c rc=$?"; done
cat $O/bench_f64_$TAG.jsonl | cut -c1-300
CF_BENCH_DEVICE=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 3 --warmup 3 --halo ipc --workload cfg2 > $O/bench_ipc2_$TAG.json 2> $O/bench_ipc2_$TAG.err; echo "ipc2 rc=$?"; cat $O/bench_ipc2_$TAG.json | cut -c1-600
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$TAG.json 2>$O/bench_$TAG.err; echo "bench rc=$?"; cut -c1-300 $O/bench_$TAG.json
