mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 -x -k "forward_sparse or fused_decode or invariants" 2>&1 | tail -3
for i in 1 2; do
timeout 600 python bench.py --workload olmoe --batch 1 --no-sweep --no-cpu > gpurun_out/bench_olmoe_b1.json 2> gpurun_out/bench_olmoe_b1.err; tail -c 300 gpurun_out/bench_olmoe_b1.err; python -c "
import json; d=json.load(open('gpurun_out/bench_olmoe_b1.json')); print(d['ms_per_step'], d['layer_frac_of_hbm_roofline'], d['ms_per_step_isolated_launch_dirty_l2'], d['e2e'])"
done
