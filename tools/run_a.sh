mkdir -p gpurun_out
python tools/h_err_probe.py 2>&1 | tail -5
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 -x 2>&1 | tail -4
timeout 900 python bench.py --no-cpu --no-sweep > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 300 gpurun_out/bench_default.err
python -c "
import json; d=json.load(open('gpurun_out/bench_default.json')); print(d['ms_per_step'], d['layer_frac_of_hbm_roofline'], d['roofline']['stage_ms'])"
