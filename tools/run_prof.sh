set -x
timeout 900 python -m pytest tests -m gpu -q -x --timeout 120 2>&1 | tail -15
timeout 500 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"router|route|dispatch|permute|grouped_tc|select|down|combine" -s 60 -c 40 --csv --log-file gpurun_out/l2.csv python bench.py --workload olmoe --batch 1 --steps 10 --warmup 3 --no-sweep --no-cpu --no-graph > gpurun_out/ncu_b.log 2>&1
timeout 500 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"router|route|dispatch|permute|grouped_tc|select|down|combine" -s 60 -c 40 --csv --log-file gpurun_out/l3.csv python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu --no-graph > gpurun_out/ncu_b3.log 2>&1
timeout 300 python bench.py --workload olmoe --batch 1 --no-cpu --no-sweep 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d[\"ms_per_step\"], d[\"roofline\"][\"stage_ms\"], d[\"e2e\"])"
timeout 300 python bench.py --no-cpu --no-sweep 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d[\"ms_per_step\"], d[\"roofline\"][\"stage_ms\"], d[\"e2e\"])"
