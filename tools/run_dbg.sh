# in-kernel phase timeline of the fused decode kernel (stamps compiled in with SKB_DEBUG_TIMING)
SKB_DEBUG_TIMING=1 python paper_2605_08575_b200/build.py --force 2>&1 | grep -i error
DBG_ROT=5 timeout 120 python tools/dbg_dec.py olmoe 1 | tail -42 | head -30
python paper_2605_08575_b200/build.py --force 2>&1 | grep -i error
