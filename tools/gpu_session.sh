# One gpurun session: GPU tests, bench lines, reference arm, ncu launch list
# and --set full captures.  Usage (from the repo root on the box):
#   bash tools/gpu_session.sh TAG [tests|bench|ncu|all]
TAG=${1:-r02}
WHAT=${2:-all}
O=gpurun_out
mkdir -p $O
nproc > $O/host_$TAG.txt; lscpu | grep -E 'Model name|^CPU\(s\)' >> $O/host_$TAG.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> $O/host_$TAG.txt
if [ "$WHAT" = tests ] || [ "$WHAT" = all ]; then
  export CF_PARITY_LOG=$O/parity_$TAG.jsonl
  rm -f $CF_PARITY_LOG
  timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > $O/pytest_gpu_$TAG.log 2>&1
  echo "pytest rc=$?"; tail -5 $O/pytest_gpu_$TAG.log
  unset CF_PARITY_LOG
fi
if [ "$WHAT" = bench ] || [ "$WHAT" = all ]; then
  timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_$TAG.json 2> $O/bench_$TAG.err; echo "bench rc=$?"
  cat $O/bench_$TAG.json
  timeout 1500 python bench.py --all $O/bench_all_$TAG.jsonl --steps 10 --warmup 3 > /dev/null 2> $O/bench_all_$TAG.err; echo "bench all rc=$?"
  timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref_$TAG.json 2> $O/bench_ref_$TAG.err; echo "ref rc=$?"
  cat $O/bench_ref_$TAG.json
fi
if [ "$WHAT" = ncu ] || [ "$WHAT" = all ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_cfg4_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch_$TAG.log 2>&1
  echo "ncu launches rc=$?"
  for t in map cfg3 cfg5 cfg4 cfg2; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:wmc_sweeps_kernel -s 1 -c 1 \
      -f -o $O/${TAG}_ncu_$t python tools/ncu_target.py $t 2 > $O/ncu_${t}_$TAG.log 2>&1
    echo "ncu $t rc=$?"
  done
fi
