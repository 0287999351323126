import ctypes as C, numpy as np, sys
sys.path.insert(0,'/root/repo')
import paper_2605_08575_b200 as skb
from paper_2605_08575_b200 import _lib
L=_lib.load()
cfg=skb.MoEConfig(64,8,2048,1024,False,0,True,64)
layer=skb.MoELayerWeights.generate_synthetic(cfg,1,0.05)
x=np.random.default_rng(0).standard_normal((1,2048)).astype(np.float32)
for i in range(3):
    rep=skb.forward_topk_sparse(layer,x,skb.SparsityLevel(0.5))
    out=(C.c_longlong*16)()
    L.skb_debug_rf(out)
    t=list(out)[:10]
    print([t[i]-t[0] for i in range(9)], 'wait', t[9])

for i in range(3):
    rep=skb.forward_topk_sparse(layer,x,skb.SparsityLevel(0.5))
    out=(C.c_longlong*16)()
    L.skb_debug_dn(out)
    t=list(out)[:10]
    print('down', [t[i]-t[0] for i in range(10)])
