mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 -x 2>&1 | tail -6
python tools/fused_vs_staged.py olmoe granite qwen gptoss 2>&1 | grep -v "B= [5-8]" | tee gpurun_out/fused_vs_staged.txt | tail -20
