O=gpurun_out; TAG=${1:-r02h}
timeout 600 python tools/probe_map_variants.py > $O/probe_mapvar_$TAG.jsonl 2>&1; echo "probe rc=$?"; cat $O/probe_mapvar_$TAG.jsonl
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "map or golden or smoke" > $O/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?"; tail -4 $O/pytest_gpu_$TAG.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wmc_map_kernel -s 2 -c 1 -f -o $O/${TAG}_ncu_map python tools/ncu_target.py map 3 > $O/ncu_map_$TAG.log 2>&1; echo "ncu rc=$?"
