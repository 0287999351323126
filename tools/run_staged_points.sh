# staged-path experiment runs: the default workload and the other batch shapes
run() {
  python bench.py --no-sweep --no-cpu "$@" 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.readline())
print('$*', d['ms_per_step'], d['ms_per_step_isolated_launch_dirty_l2'], d['roofline']['stage_ms'])
"
}
run --batch 256
run --batch 64
run --batch 1024
run --workload qwen35 --batch 64
run --workload gptoss --batch 4096 --steps 20
run --workload maverick --batch 64 --steps 20
