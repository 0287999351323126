"""Where the end-to-end step goes: Python mirror vs the bare C call, pinned buffers, L2 flushed."""
import ctypes as C, sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2605_08575_b200 as skb
from paper_2605_08575_b200 import _lib
E, K, D, N = 32, 8, 1024, 512
cfg = skb.MoEConfig(E, K, D, N, False, 0, True, 64)
layer = skb.MoELayerWeights.generate_synthetic(cfg, 1, 0.05)
flush = torch.empty(512 << 20, dtype=torch.uint8, device='cuda')
L = _lib.load()
for B in (1, 256):
    x = torch.randn(B, D).pin_memory(); y = torch.empty(B, D).pin_memory()
    lvl = skb.SparsityLevel(0.5)
    a = _lib.SkbForwardArgs(); a.batch, a.mode = B, skb.MODE_TOPK; a.s_routed = 0.5
    a.x, a.y = x.data_ptr(), y.data_ptr()
    rep = _lib.SkbReport()
    for name in ("python mirror", "bare C call", "bare C call, no flush"):
        ts = []
        for i in range(60):
            if "no flush" not in name:
                flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if name == "python mirror":
                skb.forward_topk_sparse(layer, x.numpy(), lvl, None, y_out=y.numpy())
            else:
                L.skb_layer_forward(layer._h, C.byref(a), C.byref(rep))
            t1 = time.perf_counter()
            if i >= 10: ts.append((t1 - t0) * 1e6)
        print(f'B={B:4d} {name:24s} {np.mean(ts):7.1f} us  (min {np.min(ts):6.1f})')
    # the copies alone
    d = torch.empty(B, D, device='cuda')
    ts = []
    for i in range(60):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        d.copy_(x, non_blocking=True); y.copy_(d, non_blocking=True); torch.cuda.synchronize()
        t1 = time.perf_counter()
        if i >= 10: ts.append((t1 - t0) * 1e6)
    print(f'B={B:4d} H2D + D2H copies alone     {np.mean(ts):7.1f} us')
