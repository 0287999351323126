"""Regenerates tests/golden/* with the UNMODIFIED reference (oracle/_ref/libsparsekit_ref.so,
compiled from /root/reference/proj/src by oracle/Makefile).  Run in the build container, where
/root/reference exists:  python tests/golden/make_golden.py

  moe1_e4k2d8n16_seed1.moe     save_weights(generate_synthetic(E4 K2 D8 N16, seed 1, 0.05))
                               -- the reference's own golden configuration (model_test.cpp:70-88)
  moe1_e3k2d8n8s4_seed7.moe    the same with a shared expert (d_shared = 4), renormalize off
  layer_e8k2d96n160s48.npz     synthetic layer (seed 11, 0.1; experts snapped to bf16, router fp32
                               = what skb_layer_create_synthetic holds), tokens
                               generate_tokens(5, 96, 4) rounded to bf16, and the reference's
                               forward_dense, build_topk_masks(0.5, R+S) + forward_masked_dense,
                               forward_sparse(0.05) outputs and report fields
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.pyoracle import Config, Oracle, Ref, RefLayer  # noqa: E402


def main():
    assert Ref.available(), "build oracle/_ref first (python -c 'import __graft_entry__ as g; g.build()')"
    ref = Ref.get()
    for cfg, seed, name in ((Config(4, 2, 8, 16, 0, True), 1, "moe1_e4k2d8n16_seed1.moe"),
                            (Config(3, 2, 8, 8, 4, False), 7, "moe1_e3k2d8n8s4_seed7.moe")):
        layer = RefLayer.synthetic(cfg, seed, 0.05)
        rc = ref.lib.ref_save_weights(layer.h, os.path.join(HERE, name).encode())
        assert rc == 0, ref.last_error()

    cfg = Config(8, 2, 96, 160, 48, True)
    # the operands the device image holds: expert matrices snapped to bf16, router kept fp32
    synth = Oracle.get().generate_synthetic(cfg, 11, 0.1)
    w = synth.rounded_bf16()
    w.router = synth.router
    layer = RefLayer.from_weights(w)
    x = Oracle.get().round_bf16(Oracle.get().generate_tokens(5, cfg.d_model, 4))
    y_dense, rep_dense = layer.forward_dense(x)
    routed, shared = layer.build_topk_masks(x, 0.5, 1)
    y_masked, rep_masked = layer.forward_masked_dense(x, routed, shared)
    y_sparse, rep_sparse = layer.forward_sparse(x, 0.05)
    np.savez_compressed(
        os.path.join(HERE, "layer_e8k2d96n160s48.npz"), x=x, y_dense=y_dense, routed=routed,
        shared=shared, y_masked=y_masked, y_sparse=y_sparse,
        rep_masked=np.array([rep_masked.active_neurons_total], np.uint64),
        rep_sparse=np.array([rep_sparse.gate_macs, rep_sparse.up_macs, rep_sparse.down_macs,
                             rep_sparse.other_macs, rep_sparse.active_neurons_total,
                             rep_sparse.tiles_total, rep_sparse.tiles_skipped], np.uint64))
    print("wrote", sorted(f for f in os.listdir(HERE) if not f.endswith(".py")))


if __name__ == "__main__":
    main()
