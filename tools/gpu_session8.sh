# final profile captures of the round (launch list + --set full of each hot kernel)
O=gpurun_out; TAG=${1:-r02z}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_cfg4_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch_$TAG.log 2>&1
echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wmc_sweeps_kernel -s 1 -c 1 -f -o $O/${TAG}_ncu_cfg4 python tools/ncu_target.py cfg4 > $O/ncu_cfg4_$TAG.log 2>&1; echo "cfg4 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wmc_map_kernel -s 2 -c 1 -f -o $O/${TAG}_ncu_map python tools/ncu_target.py map 3 > $O/ncu_map_$TAG.log 2>&1; echo "map rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wmc_f64_kernel -s 5 -c 1 -f -o $O/${TAG}_ncu_f64 python tools/probe_f64.py cfg3 > $O/ncu_f64_$TAG.log 2>&1; echo "f64 rc=$?"
