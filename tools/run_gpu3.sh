set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 120 2>&1 | tail -5
bash tools/run_gpu4.sh
SKB_DEBUG_TIMING=1 python paper_2605_08575_b200/build.py --force 2>&1 | grep -i error
timeout 120 python tools/dbg_dec.py granite 1 | tail -37 | head -21
timeout 120 python tools/dbg_dec.py olmoe 1 | tail -37 | head -21
