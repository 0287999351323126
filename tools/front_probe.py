"""How much of a batch step is the front (router chains, route, dispatch, token copy)?  Times the
Granite-shape step with the exact router, with the parallel (not bit-exact) router, and with
external routing (router skipped), as CUDA-graph replays with L2 flushed."""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2605_08575_b200 as skb
E, K, D, N, S = 32, 8, 1024, 512, 0
cfg = skb.MoEConfig(E, K, D, N, S > 0, S, True, 64)
layer = skb.MoELayerWeights.generate_synthetic(cfg, 1, 0.05)
flush = torch.empty(512 << 20, dtype=torch.uint8, device='cuda')
for B in (64, 256):
    layer.reserve(B)
    x = torch.randn(B, D, device='cuda'); y = torch.empty_like(x)
    ids = torch.stack([torch.randperm(E, device='cuda')[:K] for _ in range(B)]).to(torch.int32).contiguous()
    wts = torch.full((B, K), 1.0 / K, device='cuda')
    for name, kw in (("exact router", dict()), ("parallel router", dict(flags=skb.FLAG_FAST_ROUTER)),
                     ("external routing", dict(ids_in_ptr=ids.data_ptr(), weights_in_ptr=wts.data_ptr()))):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            for _ in range(3):
                layer.forward_device(x.data_ptr(), y.data_ptr(), B, mode=skb.MODE_TOPK, s_routed=0.5,
                                     stream=st.cuda_stream, **kw)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                layer.forward_device(x.data_ptr(), y.data_ptr(), B, mode=skb.MODE_TOPK, s_routed=0.5,
                                     stream=st.cuda_stream, **kw)
        ts = []
        for i in range(40):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
            if i >= 5: ts.append(e0.elapsed_time(e1) * 1e3)
        print(f'B={B:4d} {name:18s} {np.mean(ts):7.1f} us')
