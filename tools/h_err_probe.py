"""Where does the staged (tcgen05) path's output error come from?  h of the device (capture) against
double precision, and outputs against double precision given the DEVICE's h (isolates the down GEMM)."""
import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2605_08575_b200 as skb
from oracle.pyoracle import Config, Oracle
from tests.helpers import SparseSynthModel
o = Oracle.get()
for (E, K, D, N, S, B) in [(32, 8, 1024, 512, 0, 64), (256, 8, 2048, 512, 512, 16), (32, 4, 2880, 2880, 0, 64), (8, 1, 5120, 8192, 0, 32)]:
    cfg = Config(E, K, D, N, S, True)
    layer = skb.MoELayerWeights.generate_synthetic(skb.MoEConfig(E, K, D, N, S > 0, S, True, 64), 1, 0.05)
    x = o.round_bf16(o.generate_tokens(B, D, 5))
    lvl = skb.SparsityLevel(0.5)
    for name, flags in (("staged", skb.FLAG_NO_FUSED_DECODE),):
        rep = skb.forward_topk_sparse(layer, x, lvl, lvl if S else None, capture=True, flags=flags)
        m = SparseSynthModel(o, cfg, 1, 0.05)
        t = 3
        herr = 0.0; yerr_given_h = 0.0
        ysum = np.zeros(D); ysum_h = np.zeros(D)
        for k in range(K):
            e = int(rep.routes.ids[t, k])
            gw, uw, dw = m.expert(e)
            xt = x[t].astype(np.float64)
            g = gw.astype(np.float64) @ xt; u = uw.astype(np.float64) @ xt
            h = g / (1 + np.exp(-g)) * u
            hd = rep.h_routed[t, k].astype(np.float64)[:N]
            herr = max(herr, np.abs(hd - h).max() / np.abs(h).max())
            keep = rep.masks.routed[t, k].astype(bool)
            ysum += rep.routes.weights[t, k] * ((h * keep) @ dw.astype(np.float64))
            ysum_h += rep.routes.weights[t, k] * ((hd * keep) @ dw.astype(np.float64))
        if S:
            gw, uw, dw = m.expert(E)
            g = gw.astype(np.float64) @ xt; u = uw.astype(np.float64) @ xt
            h = g / (1 + np.exp(-g)) * u
            hd = rep.h_shared[t].astype(np.float64)[:S]
            keep = rep.masks.shared[t].astype(bool)
            ysum += (h * keep) @ dw.astype(np.float64); ysum_h += (hd * keep) @ dw.astype(np.float64)
        yd = rep.outputs[t].astype(np.float64)
        sc = np.abs(ysum).max()
        print(f"E{E} K{K} D{D} N{N} S{S} B{B} {name}: h rel err {herr:.2e}; y vs exact {np.abs(yd-ysum).max()/sc:.2e}; y vs exact-given-device-h {np.abs(yd-ysum_h).max()/sc:.2e}; launches {rep.launches}")
    layer.close()
