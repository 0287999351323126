mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -x -k "ep_" 2>&1 | tail -5
timeout 600 python bench.py --ep --workload maverick --batch 64 --sparsity 0.9 --steps 50 --warmup 5 --no-cpu > gpurun_out/bench_ep_maverick_w1.json 2> gpurun_out/bench_ep_maverick_w1.err; tail -c 400 gpurun_out/bench_ep_maverick_w1.err; cat gpurun_out/bench_ep_maverick_w1.json | cut -c1-1500
timeout 600 python bench.py --ep --workload gptoss --batch 4096 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_ep_gptoss_w1.json 2> gpurun_out/bench_ep_gptoss_w1.err; tail -c 400 gpurun_out/bench_ep_gptoss_w1.err; cat gpurun_out/bench_ep_gptoss_w1.json | cut -c1-600
timeout 600 python bench.py --workload maverick --batch 64 --sparsity 0.9 --steps 50 --warmup 5 --no-cpu --no-sweep > gpurun_out/bench_maverick_b64.json 2> gpurun_out/bench_maverick_b64.err; tail -c 400 gpurun_out/bench_maverick_b64.err; cat gpurun_out/bench_maverick_b64.json | cut -c1-400
timeout 300 python bench.py --gpus 2 --steps 5 --warmup 3 --no-sweep --no-cpu 2>&1 | tail -5 | cut -c1-400
