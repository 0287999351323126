set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fused -s 6 -c 2 -o gpurun_out/prof_decode_olmoe_b1 -f python bench.py --workload olmoe --batch 1 --steps 6 --warmup 3 --no-sweep --no-cpu --no-graph > gpurun_out/ncu_full_o.log 2>&1
tail -3 gpurun_out/ncu_full_o.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_tc -s 12 -c 2 -o gpurun_out/prof_tc_granite_b256 -f python bench.py --steps 6 --warmup 3 --no-sweep --no-cpu --no-graph > gpurun_out/ncu_full_g.log 2>&1
tail -3 gpurun_out/ncu_full_g.log
ls -la gpurun_out/*.ncu-rep
