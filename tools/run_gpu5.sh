set -x
K='regex:router_|route_|dispatch|permute|grouped_tc|select_rows|down_cluster|combine|decode_fused'
timeout 500 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 60 -c 48 --csv --log-file gpurun_out/launches_granite_b256.csv python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu --no-graph > gpurun_out/ncu_g.log 2>&1
python tools/summarize_launches.py gpurun_out/launches_granite_b256.csv 2>&1 | tail -30
timeout 500 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 12 -c 12 --csv --log-file gpurun_out/launches_olmoe_b1.csv python bench.py --workload olmoe --batch 1 --steps 10 --warmup 3 --no-sweep --no-cpu --no-graph > gpurun_out/ncu_o.log 2>&1
python tools/summarize_launches.py gpurun_out/launches_olmoe_b1.csv 2>&1 | tail -12
