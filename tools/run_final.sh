# Round-end measurement set: tests, bench lines, ncu launch lists and full captures.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -q --timeout 180 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 300 gpurun_out/bench_default.err
timeout 600 python bench.py --workload olmoe --batch 1 --no-sweep > gpurun_out/bench_olmoe_b1.json 2> gpurun_out/bench_olmoe_b1.err
timeout 600 python bench.py --workload qwen35 --batch 16 --no-sweep --no-cpu > gpurun_out/bench_qwen35_b16.json 2> gpurun_out/bench_qwen35_b16.err
timeout 600 python bench.py --workload qwen35 --batch 64 --no-sweep --no-cpu > gpurun_out/bench_qwen35_b64.json 2> gpurun_out/bench_qwen35_b64.err
timeout 600 python bench.py --workload gptoss --batch 1 --no-sweep --no-cpu > gpurun_out/bench_gptoss_b1.json 2> gpurun_out/bench_gptoss_b1.err
timeout 600 python bench.py --workload gptoss --batch 4096 --steps 20 --warmup 3 --no-sweep --no-cpu > gpurun_out/bench_gptoss_b4096.json 2> gpurun_out/bench_gptoss_b4096.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
K='regex:router_|route_|dispatch|permute|grouped_tc|select_rows|down_cluster|combine|decode_fused'
timeout 500 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 60 -c 48 --csv --log-file gpurun_out/launches_granite_b256.csv python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu --no-graph > gpurun_out/ncu_g.log 2>&1
timeout 500 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 12 -c 12 --csv --log-file gpurun_out/launches_olmoe_b1.csv python bench.py --workload olmoe --batch 1 --steps 10 --warmup 3 --no-sweep --no-cpu --no-graph > gpurun_out/ncu_o.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fused -s 6 -c 1 -o gpurun_out/prof_decode_olmoe_b1 -f python bench.py --workload olmoe --batch 1 --steps 6 --warmup 3 --no-sweep --no-cpu --no-graph > gpurun_out/ncu_full_o.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_tc -s 12 -c 2 -o gpurun_out/prof_tc_granite_b256 -f python bench.py --steps 6 --warmup 3 --no-sweep --no-cpu --no-graph > gpurun_out/ncu_full_g.log 2>&1
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "fused_decode_matches or batch_invariant or falls_back or forward_topk_vs_oracle or forward_sparse or budget or paired or reference_file or reference_outputs" > gpurun_out/sanitizer_memcheck.log 2>&1; tail -4 gpurun_out/sanitizer_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "fused_decode_matches and (case0 or case3)" > gpurun_out/sanitizer_racecheck.log 2>&1; tail -3 gpurun_out/sanitizer_racecheck.log
timeout 1100 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x --timeout 900 -k "lean_batch or paired_blocks or align_dispatch or forward_budget or forward_sparse_vs" > gpurun_out/sanitizer_racecheck_batch.log 2>&1; tail -3 gpurun_out/sanitizer_racecheck_batch.log
ls -la gpurun_out | tail -30
