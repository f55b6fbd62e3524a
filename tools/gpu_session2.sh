O=gpurun_out; TAG=${1:-r02c}
export CF_PARITY_LOG=$O/parity_$TAG.jsonl; rm -f $CF_PARITY_LOG
timeout 1800 python -m pytest tests/test_gpu_f64.py tests/test_gpu_configs.py -q -p no:cacheprovider --durations=20 > $O/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?"; tail -15 $O/pytest_gpu_$TAG.log
unset CF_PARITY_LOG
timeout 600 python tools/probe_f64.py > $O/probe_f64_$TAG.jsonl 2>&1; echo "probe rc=$?"; cat $O/probe_f64_$TAG.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wmc_f64_kernel -s 3 -c 1 -f -o $O/${TAG}_ncu_f64 python tools/probe_f64.py cfg3 > $O/ncu_f64_$TAG.log 2>&1; echo "ncu rc=$?"
