# Round-end measurement set: tests, bench lines, ncu launch lists and full captures, sanitizers.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -s --timeout 600 -k "full_shape_outputs or fused_decode_full" 2>&1 | grep -a "max_rel_diff=" | cut -c1-200 > gpurun_out/fullshape_errors.txt; cat gpurun_out/fullshape_errors.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 300 gpurun_out/bench_default.err
timeout 600 python bench.py --workload olmoe --batch 1 --no-sweep > gpurun_out/bench_olmoe_b1.json 2> gpurun_out/bench_olmoe_b1.err
timeout 600 python bench.py --workload qwen35 --batch 64 --no-sweep --no-cpu > gpurun_out/bench_qwen35_b64.json 2> gpurun_out/bench_qwen35_b64.err
timeout 600 python bench.py --workload gptoss --batch 1 --no-sweep --no-cpu > gpurun_out/bench_gptoss_b1.json 2> gpurun_out/bench_gptoss_b1.err
timeout 600 python bench.py --workload gptoss --batch 4096 --steps 20 --warmup 3 --no-sweep --no-cpu > gpurun_out/bench_gptoss_b4096.json 2> gpurun_out/bench_gptoss_b4096.err
timeout 600 python bench.py --workload maverick --batch 1 --sparsity 0.9 --no-sweep --no-cpu > gpurun_out/bench_maverick_b1.json 2> gpurun_out/bench_maverick_b1.err
timeout 600 python bench.py --workload maverick --batch 64 --sparsity 0.9 --steps 50 --no-sweep --no-cpu > gpurun_out/bench_maverick_b64.json 2> gpurun_out/bench_maverick_b64.err
timeout 600 python bench.py --ep --workload maverick --batch 64 --sparsity 0.9 --steps 50 --warmup 5 --no-cpu > gpurun_out/bench_ep_maverick_w1.json 2> gpurun_out/bench_ep_maverick_w1.err
timeout 600 python bench.py --ep --workload gptoss --batch 4096 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_ep_gptoss_w1.json 2> gpurun_out/bench_ep_gptoss_w1.err
timeout 600 python bench.py --ep --peer-dispatch --fused-push --workload maverick --batch 64 --sparsity 0.9 --steps 50 --warmup 5 --no-cpu > gpurun_out/bench_ep_maverick_w1_peer.json 2> gpurun_out/bench_ep_maverick_w1_peer.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
python tools/fused_vs_staged.py olmoe granite qwen gptoss 2>&1 | grep -v "B= [5-8]" > gpurun_out/fused_vs_staged.txt
K='regex:router_|route_|dispatch|permute|grouped_tc|select_rows|down_cluster|combine|decode_fused|ep_'
timeout 500 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 64 -c 48 --csv --log-file gpurun_out/launches_granite_b256.csv python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu --no-graph > gpurun_out/ncu_g.log 2>&1
timeout 500 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 12 -c 12 --csv --log-file gpurun_out/launches_olmoe_b1.csv python bench.py --workload olmoe --batch 1 --steps 10 --warmup 3 --no-sweep --no-cpu --no-graph > gpurun_out/ncu_o.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fused -s 8 -c 1 -o gpurun_out/ncu_full_decode_fused_olmoe_b1 -f python bench.py --workload olmoe --batch 1 --steps 6 --warmup 3 --no-sweep --no-cpu --no-graph > gpurun_out/ncu_full_o.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_tc -s 16 -c 2 -o gpurun_out/ncu_full_grouped_tc_granite_b256 -f python bench.py --steps 6 --warmup 3 --no-sweep --no-cpu --no-graph > gpurun_out/ncu_full_g.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_tc_chunked -s 4 -c 2 -o gpurun_out/ncu_full_chunked_gptoss_b4096 -f python bench.py --workload gptoss --batch 4096 --steps 4 --warmup 3 --no-sweep --no-cpu --no-graph > gpurun_out/ncu_full_p.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"select_rows_warp|router_fused|route_dispatch|combine_rows" -s 8 -c 4 -o gpurun_out/ncu_full_small_granite_b256 -f python bench.py --steps 6 --warmup 3 --no-sweep --no-cpu --no-graph > gpurun_out/ncu_full_s.log 2>&1
python tools/summarize_ncu.py gpurun_out/ncu_full_small_granite_b256.ncu-rep > gpurun_out/ncu_full_small_granite_b256.txt 2>&1
python tools/summarize_ncu.py gpurun_out/ncu_full_decode_fused_olmoe_b1.ncu-rep > gpurun_out/ncu_full_decode_fused_olmoe_b1.txt 2>&1
python tools/summarize_ncu.py gpurun_out/ncu_full_grouped_tc_granite_b256.ncu-rep > gpurun_out/ncu_full_grouped_tc_granite_b256.txt 2>&1
python tools/summarize_ncu.py gpurun_out/ncu_full_chunked_gptoss_b4096.ncu-rep > gpurun_out/ncu_full_chunked_gptoss_b4096.txt 2>&1
python tools/make_traffic_json.py gpurun_out/ncu_traffic.json olmoe:1:decode_fused=gpurun_out/ncu_full_decode_fused_olmoe_b1.ncu-rep:decode_fused "granite:256:gateup=gpurun_out/ncu_full_grouped_tc_granite_b256.ncu-rep:grouped_tc_kernel<128, 0" "gptoss:4096:gateup=gpurun_out/ncu_full_chunked_gptoss_b4096.ncu-rep:grouped_tc_chunked_kernel<128, 0"
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x --timeout 900 -k "fused_decode_matches or batch_invariant or falls_back or forward_sparse_fused or caller_masks or ep_ or compact_active or threshold_mask or forward_topk_vs_oracle or paired or lean_batch" > gpurun_out/sanitizer_memcheck.log 2>&1; tail -4 gpurun_out/sanitizer_memcheck.log
timeout 1100 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x --timeout 900 -k "(fused_decode_matches and (case0 or case3)) or (forward_sparse_fused and case1) or (lean_batch and case0)" > gpurun_out/sanitizer_racecheck.log 2>&1; tail -3 gpurun_out/sanitizer_racecheck.log
timeout 600 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x --timeout 500 -k "fused_decode_matches and case0" > gpurun_out/sanitizer_synccheck.log 2>&1; tail -3 gpurun_out/sanitizer_synccheck.log
python tools/e2e_probe.py 256 > gpurun_out/e2e_probe.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_08575_b200/csrc -o /tmp/silu_check tools/micro/silu_check.cu 2>/dev/null && /tmp/silu_check > gpurun_out/silu_check.txt 2>&1
bash tools/run_dbg_tc.sh > gpurun_out/timeline_granite_b256.txt 2>&1
bash tools/run_staged_points.sh > gpurun_out/staged_points.txt 2>&1
ls -la gpurun_out | tail -40
