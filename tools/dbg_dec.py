import ctypes as C, numpy as np, sys, os
sys.path.insert(0,'/root/repo')
import paper_2605_08575_b200 as skb
from paper_2605_08575_b200 import _lib
L=_lib.load()
shape = sys.argv[1] if len(sys.argv) > 1 else "olmoe"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
shapes = {"olmoe": (64,8,2048,1024,False,0), "granite": (32,8,1024,512,False,0), "qwen": (256,8,2048,512,True,512)}
E,K,D,N,hs,S = shapes[shape]
cfg=skb.MoEConfig(E,K,D,N,hs,S,True,64)
layer=skb.MoELayerWeights.generate_synthetic(cfg,1,0.05)
x=np.random.default_rng(0).standard_normal((B,D)).astype(np.float32)
lvl=skb.SparsityLevel(0.5)
ref=skb.forward_topk_sparse(layer,x,lvl,lvl if hs else None,flags=skb.FLAG_NO_FUSED_DECODE)
import torch
flush=torch.empty(512<<20,dtype=torch.uint8,device='cuda')
ROT=int(os.environ.get('DBG_ROT','0'))  # >0: back-to-back launches rotating over ROT weight images (the bench's timed region)
if ROT:
    layers=[layer]+[skb.MoELayerWeights.generate_synthetic(cfg,1,0.05) for _ in range(ROT-1)]
    xd=torch.from_numpy(x).cuda(); yd=torch.empty_like(xd)
    for l in layers: l.reserve(B)
for i in range(3):
    (flush.zero_() if os.environ.get('DBG_DIRTY') else flush.sum()); torch.cuda.synchronize()
    if ROT:
        for j in range(4*ROT):
            layers[j%ROT].forward_device(xd.data_ptr(), yd.data_ptr(), B, stream=1, **(dict(mode=skb.MODE_THRESHOLD, tau=float(os.environ['DBG_TAU']), flags=skb.FLAG_FUSED_DECODE) if os.environ.get('DBG_TAU') else dict(mode=skb.MODE_TOPK, s_routed=0.5, s_shared=0.5 if hs else 0.0)))
        torch.cuda.synchronize()
    rep=skb.forward_topk_sparse(layer,x,lvl,lvl if hs else None) if not ROT else ref
    print('launches', rep.launches, 'ref launches', ref.launches, 'maxdiff', float(np.abs(rep.outputs-ref.outputs).max()))
    if hasattr(L, 'skb_debug_dec'):
        out=(C.c_longlong*(160*32))()
        L.skb_debug_dec(out)
        t=np.array(list(out)).reshape(160,32)
        # stamps are SM cycle counts: onto the common nanosecond axis through the {globaltimer, clock64} pair of stamp 0
        clk0=t[:,31].copy(); gt0=t[:,0].copy()
        for k in range(1,31):
            nz=t[:,k]>0
            t[nz,k]=gt0[nz]+((t[nz,k]-clk0[nz])/1.965).astype(np.int64)
        names={14:'chain start',15:'chain end',0:'start',1:'p0 done',2:'tables',3:'tma issued',4:'g done',8:'p2 ready',9:'p2 pivot',11:'p2 prefix',12:'p2 list',13:'p2 gather',5:'p2 done',6:'p3 barrier',7:'exit',10:'route done',11:'tma go',16:'x staged',17:'cons go',18:'piece1 done',19:'p3 tables',20:'p3 loaded',21:'polled',22:'cand done',23:'p3 pass1',24:'cand start',25:'cand tok',26:'poll start',27:'probe1 back'}
        for k in (1,26,27,21,24,25,22,2,11,16,17,18,3,14,15,10,4,8,9,12,13,5,19,6,23,20,7):
            col=t[:148,k]-t[:148,0].min()
            col=col[t[:148,k]>0]
            if col.size: print(f'  {names[k]:12s} n {col.size:3d} min {col.min():7d} med {int(np.median(col)):7d} max {col.max():7d}')
        g=t[:148,16:20]*0
        g0=g[:,0].min()
        for k,nm in enumerate(['g start','g p1 done','g p2 ready','g exit']):
            col=g[:,k]; col=col[col>0]-g0
            if col.size: print(f'  {nm:12s} n {col.size:3d} min {col.min():7d} med {int(np.median(col)):7d} max {col.max():7d} (ns)')
        if i == 2:
            ks=(0,1,2,11,18,3,4,8,9,12,13,5,19,6,20,7)
            print('   cta ' + ' '.join(f'{names.get(k,k)[:9]:>9s}' for k in ks))
            for b in (0,1,31,32,63,64,100,127,128,143,144,145,146,147):
                print(f'   {b:3d} ' + ' '.join(f'{(t[b,k]-t[:148,0].min() if t[b,k]>0 else -1):9d}' for k in ks))
