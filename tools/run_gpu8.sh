for i in 1 2; do
python bench.py --workload olmoe --batch 1 --no-cpu --no-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sweep  ', d['ms_per_step'], d['roofline']['kernel_ms'])"
SKB_BENCH_READ_SWEEP=0 python bench.py --workload olmoe --batch 1 --no-cpu --no-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nosweep', d['ms_per_step'], d['roofline']['kernel_ms'])"
done
python bench.py --no-cpu --no-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('granite256 sweep  ', d['ms_per_step'], d['roofline']['stage_ms'])"
SKB_BENCH_READ_SWEEP=0 python bench.py --no-cpu --no-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('granite256 nosweep', d['ms_per_step'], d['roofline']['stage_ms'])"
