mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 -x 2>&1 | tail -4
timeout 600 python bench.py --ep --workload maverick --batch 64 --sparsity 0.9 --steps 50 --warmup 5 --no-cpu > gpurun_out/bench_ep_maverick_w1.json 2> gpurun_out/bench_ep_maverick_w1.err; python -c "
import json; d=json.load(open('gpurun_out/bench_ep_maverick_w1.json')); print('EP maverick w1', d['ms_per_step'], d['roofline']['frac'])"
