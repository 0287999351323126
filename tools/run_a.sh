mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 -x --deselect "tests/test_gpu_parity.py::test_full_shape_outputs_vs_oracle" 2>&1 | tail -15
