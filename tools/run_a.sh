mkdir -p gpurun_out
python tools/h_err_probe.py 2>&1 | tail -5
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -s -k "full_shape_outputs" > gpurun_out/fullshape.log 2>&1
grep -a "max_rel_diff=" gpurun_out/fullshape.log | cut -c1-220
tail -3 gpurun_out/fullshape.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 -x --deselect "tests/test_gpu_parity.py::test_full_shape_outputs_vs_oracle" 2>&1 | tail -5
