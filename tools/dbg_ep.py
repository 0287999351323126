import numpy as np, sys
sys.path.insert(0,'/root/repo')
import paper_2605_08575_b200 as skb
full = skb.MoEConfig(16, 4, 256, 192, True, 64, True, 64)
x = np.random.default_rng(3).standard_normal((24, 256)).astype(np.float32)
s16 = skb.MoELayerWeights.synthetic_slice(full, 1, 0.05, 0, 16)
for (lo,hi) in [(0,8),(8,16),(4,8)]:
    sl = skb.MoELayerWeights.synthetic_slice(full, 1, 0.05, lo, hi)
    for flags,name in [(skb.FLAG_GATHER_DOWN,'gather'),(skb.FLAG_DENSE_DOWN,'dense')]:
        for e in [lo, hi-1]:
            ids16 = np.full(24, e, np.int32); idsl = np.full(24, e-lo, np.int32)
            a = skb.forward_routed(s16, x, ids16, s_routed=0.5, flags=flags)
            b = skb.forward_routed(sl, x, idsl, s_routed=0.5, flags=flags)
            print(lo,hi,name,e, float(np.abs(a-b).max()), float(np.abs(a).max()))
    # mixed ids
    rng=np.random.default_rng(0); idsl = rng.integers(0,hi-lo,24).astype(np.int32)
    a = skb.forward_routed(s16, x, idsl+lo, s_routed=0.5); b = skb.forward_routed(sl, x, idsl, s_routed=0.5)
    print(lo,hi,'mixed', float(np.abs(a-b).max()))
    M=11; a = skb.forward_routed(s16, x[:M], idsl[:M]+lo, s_routed=0.5); b = skb.forward_routed(sl, x[:M], idsl[:M], s_routed=0.5)
    print(lo,hi,'mixed M=11', float(np.abs(a-b).max()))
