mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 -x 2>&1 | tail -6
