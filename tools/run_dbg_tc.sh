# timeline of the staged batch path (phase stamps compiled in with SKB_DEBUG_TIMING)
SKB_DEBUG_TIMING=1 python paper_2605_08575_b200/build.py --force 2>&1 | grep -i " error"
timeout 300 python tools/dbg_tc.py granite 256 | tail -25
python paper_2605_08575_b200/build.py --force 2>&1 | grep -i " error"
