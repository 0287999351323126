"""Fused decode kernel against the staged kernels per (shape, batch): input of the path choice."""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2605_08575_b200 as skb
shapes = {"olmoe": (64, 8, 2048, 1024, 0), "granite": (32, 8, 1024, 512, 0), "qwen": (256, 8, 2048, 512, 512),
          "gptoss": (32, 4, 2880, 2880, 0)}
flush = torch.empty(512 << 20, dtype=torch.uint8, device='cuda')
for name in sys.argv[1:]:
    E, K, D, N, S = shapes[name]
    cfg = skb.MoEConfig(E, K, D, N, S > 0, S, True, 64)
    layer = skb.MoELayerWeights.generate_synthetic(cfg, 1, 0.05)
    layer.reserve(16)
    for B in (1, 2, 3, 4, 5, 6, 7, 8):
        x = torch.randn(B, D, device='cuda'); y = torch.empty_like(x)
        out = []
        for flags in (skb.FLAG_FUSED_DECODE, skb.FLAG_NO_FUSED_DECODE, 0, skb.FLAG_DENSE_DOWN, skb.FLAG_GATHER_DOWN):
            ts = []
            for i in range(23):
                flush.sum()
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                layer.forward_device(x.data_ptr(), y.data_ptr(), B, mode=skb.MODE_TOPK, s_routed=0.5,
                                     s_shared=0.5 if S else 0.0, flags=flags,
                                     stream=torch.cuda.current_stream().cuda_stream or 1)
                e1.record(); torch.cuda.synchronize()
                if i >= 3: ts.append(e0.elapsed_time(e1) * 1e3)
            out.append(float(np.mean(ts)))
        pick = 'fused' if abs(out[2] - out[0]) < abs(out[2] - out[1]) else 'staged'
        best = 'fused' if out[0] <= out[1] else 'staged'
        print(f'{name:8s} B={B:2d}  fused {out[0]:7.1f} us   staged {out[1]:7.1f} us   auto {out[2]:7.1f} us  dense {out[3]:7.1f}  gather {out[4]:7.1f}  picks {pick:6s} best {best:6s} {"" if pick == best or abs(out[0]-out[1]) < 0.03*min(out[:2]) else "<-- WRONG"}')
