"""Paired weight blocks for gate/up and down at the headline point: step time by flag, rotating
over four weight images, back-to-back launches between one event pair."""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2605_08575_b200 as skb
E, K, D, N = 32, 8, 1024, 512
B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cfg = skb.MoEConfig(E, K, D, N, False, 0, True, 64)
layers = [skb.MoELayerWeights.generate_synthetic(cfg, 1, 0.05) for _ in range(4)]
for l in layers: l.reserve(B)
x = torch.randn(B, D, device='cuda'); y = torch.empty_like(x)
st = torch.cuda.Stream()
def run(flags, n=400):
    with torch.cuda.stream(st):
        for i in range(40):
            layers[i % 4].forward_device(x.data_ptr(), y.data_ptr(), B, stream=st.cuda_stream, mode=skb.MODE_TOPK, s_routed=0.5, s_shared=0.0, flags=flags)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for i in range(n):
            layers[i % 4].forward_device(x.data_ptr(), y.data_ptr(), B, stream=st.cuda_stream, mode=skb.MODE_TOPK, s_routed=0.5, s_shared=0.0, flags=flags)
        e1.record(st)
    st.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
for rep in range(2):
    for name, f in (('auto', 0), ('paired', skb.FLAG_PAIRED_BLOCKS), ('unpaired', skb.FLAG_NO_PAIRED_BLOCKS)):
        print(f'B={B} {name:9s} {run(f):7.2f} us')
