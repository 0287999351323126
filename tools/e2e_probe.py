"""Where the end-to-end time of the host-buffer call goes (Granite shape, batch 256): the PCIe copies
alone, the device stages alone, and the whole call."""
import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2605_08575_b200 as skb
E, K, D, N = 32, 8, 1024, 512
B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cfg = skb.MoEConfig(E, K, D, N, False, 0, True, 64)
layer = skb.MoELayerWeights.generate_synthetic(cfg, 1, 0.05)
layer.reserve(B)
xh = torch.randn(B, D).pin_memory(); yh = torch.empty(B, D).pin_memory()
xd = torch.empty(B, D, device='cuda'); yd = torch.empty(B, D, device='cuda')
lvl = skb.SparsityLevel(0.5)
st = torch.cuda.Stream()
def timeit(fn, n=200, warm=20):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); fn(); ts.append((time.perf_counter() - t0) * 1e6)
    return float(np.median(ts)), float(np.mean(ts))
def copies():
    with torch.cuda.stream(st):
        xd.copy_(xh, non_blocking=True); yh.copy_(yd, non_blocking=True)
    st.synchronize()
def h2d():
    with torch.cuda.stream(st):
        xd.copy_(xh, non_blocking=True)
    st.synchronize()
def dev():
    layer.forward_device(xd.data_ptr(), yd.data_ptr(), B, stream=st.cuda_stream, mode=skb.MODE_TOPK, s_routed=0.5, s_shared=0.0)
    st.synchronize()
def whole():
    skb.forward_topk_sparse(layer, xh.numpy(), lvl, None, y_out=yh.numpy())
xn, yn = xh.numpy(), yh.numpy()
def whole_np():
    skb.forward_topk_sparse(layer, xn, lvl, None, y_out=yn)
for name, fn in (('h2d 1 copy + sync', h2d), ('h2d + d2h + sync', copies), ('device stages + sync', dev), ('forward_topk_sparse (host buffers)', whole), ('... numpy views hoisted', whole_np)):
    med, mean = timeit(fn)
    print(f'{name:40s} median {med:7.1f} us  mean {mean:7.1f} us')
