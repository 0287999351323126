mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 180 -k "fused_decode or batch_invariant or falls_back or invariants" 2>&1 | tail -5
for st in 12 6; do
SKB_DEC_STAGES=$st timeout 600 python bench.py --workload olmoe --batch 1 --no-sweep --no-cpu > gpurun_out/bench_olmoe_b1.json 2> gpurun_out/bench_olmoe_b1.err; tail -c 300 gpurun_out/bench_olmoe_b1.err; python -c "
import json; d=json.load(open('gpurun_out/bench_olmoe_b1.json')); print('stages $st', d['ms_per_step'], d['layer_frac_of_hbm_roofline'], d['e2e'])"
done
SKB_DEBUG_TIMING=1 python paper_2605_08575_b200/build.py --force 2>&1 | grep -i error
for st in 12 6; do
SKB_DEC_STAGES=$st timeout 120 python tools/dbg_dec.py olmoe 1 > gpurun_out/dbg_olmoe1_s$st.txt 2>&1
tail -38 gpurun_out/dbg_olmoe1_s$st.txt
done
