set -x
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "fused_decode_matches or batch_invariant or falls_back or smoke or forward_topk_vs_oracle" 2>&1 | tail -15
echo "memcheck rc=$?"
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "fused_decode_matches and (case0 or case3)" 2>&1 | tail -15
