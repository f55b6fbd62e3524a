# full GPU tests + headline bench + all configs
O=gpurun_out; TAG=${1:-r02l}
export CF_PARITY_LOG=$O/parity_$TAG.jsonl; rm -f $CF_PARITY_LOG
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > $O/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?"; tail -4 $O/pytest_gpu_$TAG.log
unset CF_PARITY_LOG
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_$TAG.json 2> $O/bench_$TAG.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('$O/bench_$TAG.json'));print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['e2e']['value'],d['clocks'])"
timeout 1500 python bench.py --all $O/bench_all_$TAG.jsonl --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2> $O/bench_all_$TAG.err; echo "bench all rc=$?"
python - <<PY
import json
for l in open('$O/bench_all_$TAG.jsonl'):
    d=json.loads(l); print(d['config']['workload'][:40], d['value'], d['roofline']['frac'], d['e2e']['value'])
PY
