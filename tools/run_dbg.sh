SKB_DEBUG_TIMING=1 python paper_2605_08575_b200/build.py --force 2>&1 | grep -i error
timeout 120 python tools/dbg_dec.py granite 16 | tail -36 | head -20
