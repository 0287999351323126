"""Phase timeline of the grouped tcgen05 GEMM kernels (build with SKB_DEBUG_TIMING=1)."""
import ctypes as C, numpy as np, sys, os
sys.path.insert(0, '/root/repo')
import torch
import paper_2605_08575_b200 as skb
from paper_2605_08575_b200 import _lib
L = _lib.load()
shape = sys.argv[1] if len(sys.argv) > 1 else "granite"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
shapes = {"olmoe": (64, 8, 2048, 1024, False, 0), "granite": (32, 8, 1024, 512, False, 0),
          "qwen": (256, 8, 2048, 512, True, 512)}
E, K, D, N, hs, S = shapes[shape]
cfg = skb.MoEConfig(E, K, D, N, hs, S, True, 64)
ROT = 4
layers = [skb.MoELayerWeights.generate_synthetic(cfg, 1, 0.05) for _ in range(ROT)]
for l in layers: l.reserve(B)
xd = torch.randn(B, D, device='cuda'); yd = torch.empty_like(xd)
L.skb_debug_tc.argtypes = [C.c_void_p]
for it in range(3):
    for j in range(2 * ROT):
        if j == 2 * ROT - 1:
            torch.cuda.synchronize(); L.skb_debug_tc_clear()
        layers[j % ROT].forward_device(xd.data_ptr(), yd.data_ptr(), B, stream=1, mode=skb.MODE_TOPK,
                                       s_routed=0.5, s_shared=0.5 if hs else 0.0)
    torch.cuda.synchronize()
    out = np.zeros(2 * 1024 * 8, dtype=np.int64)
    L.skb_debug_tc(out.ctypes.data_as(C.c_void_p))
    t = out.reshape(2, 1024, 8).astype(np.float64)
    base = None
    for mode in (0, 1):
        m = t[mode]
        live = m[:, 0] > 0
        if not live.any(): continue
        m = m[live]
        gt0, clk0 = m[:, 0].copy(), m[:, 7].copy()
        if base is None: base = gt0.min()
        names = {0: 'start', 1: 'pdl passed', 3: 'first stage full', 2: 'last tma issue', 4: 'last stage full',
                 5: 'tmem full', 6: 'epilogue done'}
        print(f'--- MODE {mode}: {int(live.sum())} CTAs, {(m[:, 5] > 0).sum()} active')
        for k in (0, 1, 3, 2, 4, 5, 6):
            if k == 0:
                col = gt0 - base
            else:
                nz = m[:, k] > 0
                col = gt0[nz] + (m[nz, k] - clk0[nz]) / 1.965 - base
            if col.size:
                print(f'  {names[k]:18s} n {col.size:4d} min {col.min():8.0f} med {np.median(col):8.0f} '
                      f'p90 {np.percentile(col, 90):8.0f} max {col.max():8.0f} ns')
    if hasattr(L, 'skb_debug_sel') and base is not None:
        so = np.zeros(4096 * 8, dtype=np.int64)
        L.skb_debug_sel.argtypes = [C.c_void_p]
        L.skb_debug_sel(so.ctypes.data_as(C.c_void_p))
        m = so.reshape(4096, 8).astype(np.float64)
        m = m[m[:, 0] > 0]
        gt0, clk0 = m[:, 0].copy(), m[:, 7].copy()
        print(f'--- selection: {m.shape[0]} rows')
        for k, nm in ((0, 'start'), (1, 'tile ready'), (2, 'row loaded'), (3, 'pivot found'), (4, 'stored')):
            col = gt0 - base if k == 0 else gt0 + (m[:, k] - clk0) / 1.965 - base
            print(f'  {nm:18s} n {col.size:4d} min {col.min():8.0f} med {np.median(col):8.0f} '
                  f'p90 {np.percentile(col, 90):8.0f} max {col.max():8.0f} ns')
    if hasattr(L, 'skb_debug_rd'):
        ro = np.zeros(16, dtype=np.int64)
        L.skb_debug_rd.argtypes = [C.c_void_p]
        L.skb_debug_rd(ro.ctypes.data_as(C.c_void_p))
        nm = ['start', 'pdl passed', 'routed', 'barrier passed', 'histograms', 'slots placed', 'tile list', 'permuted']
        print('--- route_dispatch (middle CTA, ns from its start): ' +
              ', '.join(f'{nm[k]} {(ro[k] - ro[0]) / 1.965:.0f}' for k in range(1, 8)))
    if hasattr(L, 'skb_debug_rf'):
        ro = np.zeros(16, dtype=np.int64)
        L.skb_debug_rf.argtypes = [C.c_void_p]
        L.skb_debug_rf(ro.ctypes.data_as(C.c_void_p))
        print('--- router_fused (last CTA to write, ns from its start): ' +
              f'pdl passed {(ro[1]-ro[0])/1.965:.0f}, first sub-chunk in {(ro[8]-ro[0])/1.965:.0f}, '
              f'chains done {(ro[2]-ro[0])/1.965:.0f}, waited on the ring {ro[9]/1.965:.0f}')
