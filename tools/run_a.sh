mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -x -k "threshold_mask or compact_active" 2>&1 | tail -12
