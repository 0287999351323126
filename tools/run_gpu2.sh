set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 120 2>&1 | tail -40
