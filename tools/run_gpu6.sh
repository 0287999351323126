set -x
mkdir -p gpurun_out
( time timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err ) 2>&1 | tail -4
tail -c 600 gpurun_out/bench_default.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_default.json'))
print({k:d[k] for k in ('value','ms_per_step','layer_frac_of_hbm_roofline','gpu_launches','launches_per_step')})
print(d['roofline']); print(d['e2e']); print(d['cpu_baseline'])
for r in d['sweep']: print(r)
PY
( time timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err ) 2>&1 | tail -4
cat gpurun_out/bench_reference.json | head -c 1500
