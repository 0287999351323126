python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash tools/run_pf.sh 2>&1
python bench.py --no-sweep --no-cpu --batch 512 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.readline()); print('B=512', d['ms_per_step'], d['roofline']['stage_ms'])"
SKB_DEBUG_TIMING=1 python paper_2605_08575_b200/build.py --force 2>&1 | grep -i " error"
timeout 300 python tools/dbg_tc.py granite 256 | tail -18
python paper_2605_08575_b200/build.py --force 2>&1 | grep -i " error"
