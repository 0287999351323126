set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 180 2>&1 | tail -15
timeout 300 python bench.py --workload olmoe --batch 1 --no-cpu --no-sweep > gpurun_out/bench_olmoe_b1.json 2> gpurun_out/bench_olmoe_b1.err; tail -c 3000 gpurun_out/bench_olmoe_b1.json
timeout 400 python bench.py --no-sweep > gpurun_out/bench_granite_b256.json 2> gpurun_out/bench_granite.err; tail -c 3000 gpurun_out/bench_granite_b256.json
