timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -8
for b in 256 64; do
python bench.py --batch $b --no-cpu --no-sweep --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('granite B=$b', d['ms_per_step'], d['launches_per_step'], {k: round(v*1e3,1) for k,v in d['roofline']['stage_ms'].items()})"
done
python bench.py --workload qwen35 --batch 64 --no-cpu --no-sweep --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('qwen B=64', d['ms_per_step'], d['launches_per_step'], {k: round(v*1e3,1) for k,v in d['roofline']['stage_ms'].items()})"
