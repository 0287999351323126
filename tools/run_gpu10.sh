timeout 900 ncu --set full --clock-control none --import-source on -k regex:"select_rows|dispatch_kernel|combine_rows|route_tokens|permute" -s 15 -c 5 -o gpurun_out/prof_small_granite_b256 -f python bench.py --steps 6 --warmup 3 --no-sweep --no-cpu --no-graph > gpurun_out/ncu_full_s.log 2>&1
tail -2 gpurun_out/ncu_full_s.log | cut -c1-200
