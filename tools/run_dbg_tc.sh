nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_08575_b200/csrc -o /tmp/silu_check tools/micro/silu_check.cu 2>/dev/null && /tmp/silu_check
SKB_DEBUG_TIMING=1 python paper_2605_08575_b200/build.py --force 2>&1 | grep -i " error"
timeout 300 python tools/dbg_tc.py granite 256 | tail -18
python paper_2605_08575_b200/build.py --force 2>&1 | grep -i " error"
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash tools/run_pf.sh 2>&1
