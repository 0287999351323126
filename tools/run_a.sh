mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 -x -k "forward_sparse" 2>&1 | tail -25
