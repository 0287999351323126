mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 -x -k "forward_sparse or fused_decode or invariants" 2>&1 | tail -4
timeout 600 python bench.py --workload olmoe --batch 1 --no-sweep --no-cpu > gpurun_out/bench_olmoe_b1.json 2> gpurun_out/bench_olmoe_b1.err; tail -c 300 gpurun_out/bench_olmoe_b1.err; python -c "
import json; d=json.load(open('gpurun_out/bench_olmoe_b1.json')); print(d['ms_per_step'], d['layer_frac_of_hbm_roofline'], d['ms_per_step_isolated_launch_dirty_l2'], d['e2e'])"
SKB_DEBUG_TIMING=1 python paper_2605_08575_b200/build.py --force 2>&1 | grep -i error
DBG_TAU=0.2645798623561859 DBG_ROT=5 timeout 120 python tools/dbg_dec.py olmoe 1 > gpurun_out/dbg_olmoe1_thr.txt 2>&1
tail -44 gpurun_out/dbg_olmoe1_thr.txt | head -30 | grep "tma go\|g done\|p2 \|p3\|exit"
