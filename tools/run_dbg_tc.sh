timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash tools/run_pf.sh 2>&1
python bench.py --no-sweep --no-cpu --workload olmoe --batch 16 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.readline()); print('olmoe B=16', d['ms_per_step'], d['roofline']['stage_ms'])"
