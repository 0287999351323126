"""cProfile of the Python mirror around the C call (pinned buffers, Granite shape, batch 256)."""
import cProfile, pstats, sys, torch
sys.path.insert(0, '/root/repo')
import paper_2605_08575_b200 as skb
cfg = skb.MoEConfig(32, 8, 1024, 512, False, 0, True, 64)
layer = skb.MoELayerWeights.generate_synthetic(cfg, 1, 0.05)
B = 256
x = torch.randn(B, 1024).pin_memory(); y = torch.empty(B, 1024).pin_memory()
lvl = skb.SparsityLevel(0.5)
xn, yn = x.numpy(), y.numpy()
for _ in range(20):
    skb.forward_topk_sparse(layer, xn, lvl, None, y_out=yn)
pr = cProfile.Profile()
pr.enable()
for _ in range(2000):
    skb.forward_topk_sparse(layer, xn, lvl, None, y_out=yn)
pr.disable()
pstats.Stats(pr).sort_stats('tottime').print_stats(12)
