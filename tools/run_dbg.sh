set -x
SKB_DEBUG_TIMING=1 python paper_2605_08575_b200/build.py --force > /dev/null 2>&1
python tools/dbg_rf.py
