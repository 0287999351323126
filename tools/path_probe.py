"""Times the two down-projection paths of the staged kernels on one shape (device entry point,
L2 flushed, CUDA events): the input of the gather/dense choice in csrc/api.cu."""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2605_08575_b200 as skb
E, K, D, N, S, B, s = (int(v) if i < 6 else float(v) for i, v in enumerate(sys.argv[1:8]))
cfg = skb.MoEConfig(E, K, D, N, S > 0, S, True, 64)
layer = skb.MoELayerWeights.generate_synthetic(cfg, 1, 0.05)
layer.reserve(B)
x = torch.randn(B, D, device='cuda'); y = torch.empty_like(x)
flush = torch.empty(512 << 20, dtype=torch.uint8, device='cuda')
for name, flags in (('auto', 0), ('gather', skb.FLAG_GATHER_DOWN), ('dense', skb.FLAG_DENSE_DOWN)):
    ts = []
    for i in range(13):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        layer.forward_device(x.data_ptr(), y.data_ptr(), B, mode=skb.MODE_TOPK, s_routed=s,
                             s_shared=s if S else 0.0, flags=flags,
                             stream=torch.cuda.current_stream().cuda_stream or 1)
        e1.record(); torch.cuda.synchronize()
        if i >= 3: ts.append(e0.elapsed_time(e1) * 1e3)
    print(f'{name:7s} {np.mean(ts):8.1f} us')
