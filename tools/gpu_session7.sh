O=gpurun_out; TAG=${1:-r02o}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wmc_f64_kernel -s 5 -c 1 -f -o $O/${TAG}_ncu_f64 python tools/probe_f64.py cfg3 > $O/ncu_f64_$TAG.log 2>&1; echo "ncu rc=$?"
