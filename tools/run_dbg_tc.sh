SKB_DEBUG_TIMING=1 python paper_2605_08575_b200/build.py --force 2>&1 | grep -i " error"
timeout 300 python tools/dbg_tc.py granite 256 | tail -18
python paper_2605_08575_b200/build.py --force 2>&1 | grep -i " error"
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "granite or dense or staged" 2>&1 | tail -2
bash tools/run_pf.sh 2>&1 | head -2
