for wl in olmoe granite; do
timeout 300 python bench.py --workload $wl --batch 1 --no-cpu --no-sweep > gpurun_out/bench_${wl}_b1.json 2> gpurun_out/bench_${wl}_b1.err; python -c "
import json; d=json.load(open('gpurun_out/bench_${wl}_b1.json')); print('${wl}', d['ms_per_step'], d['layer_frac_of_hbm_roofline'], d['e2e']['ms_per_step'])"
done
timeout 300 python bench.py --workload olmoe --batch 8 --no-cpu --no-sweep > gpurun_out/bench_olmoe_b8.json 2> gpurun_out/bench_olmoe_b8.err; python -c "
import json; d=json.load(open('gpurun_out/bench_olmoe_b8.json')); print('olmoe b8', d['ms_per_step'], d['layer_frac_of_hbm_roofline'], d['e2e']['ms_per_step'])"
