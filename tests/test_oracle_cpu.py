"""Pins oracle/moe_oracle.c: the reference's own golden vector and hand cases
(restated from proj/tests/*.cpp, cited per test) and bit-for-bit agreement with
the unmodified reference compiled into oracle/_ref.  CPU only."""
import math

import numpy as np
import pytest

from oracle.pyoracle import Config, RefLayer
from tests.helpers import SplitMix64, max_rel_diff, random_config

PAD = -1


# ---- model / rng ------------------------------------------------------------

def test_golden_router_row0(oracle):
    """proj/tests/golden/gen_e4k2d8n16_seed1_router_row0.txt via model_test.cpp:70-88."""
    golden = [0x3bda1bda, 0x3cc9582a, 0x3d40ec37, 0xbbb652e7, 0xbbb6a233, 0x3cd75cf0, 0x3d1a8fe0,
              0x3b172c4d]
    w = oracle.generate_synthetic(Config(4, 2, 8, 16), 1, 0.05)
    assert [int(v) for v in w.router[0].view(np.uint32)] == golden


def test_synthetic_matches_reference_bitwise(oracle, ref):
    """model.cpp:129-166 fill order, including the jump-ahead offsets."""
    for cfg in (Config(4, 2, 8, 16), Config(5, 3, 7, 9, 6), Config(3, 1, 16, 4, 2, False)):
        mine = oracle.generate_synthetic(cfg, 42, 0.1)
        theirs = RefLayer.synthetic(cfg, 42, 0.1).weights()
        for n in ("router", "gate", "up", "down_t", "shared_gate", "shared_up", "shared_down_t"):
            a, b = getattr(mine, n), getattr(theirs, n)
            if a is None:
                assert b is None
            else:
                assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), n


def test_tokens_match_reference_bitwise(oracle, ref):
    """model.cpp:168-178 + rng.hpp:42-55 (Box-Muller with cached spare)."""
    for B, D, seed in ((1, 8, 2), (3, 5, 99), (4, 64, 7)):
        theirs = np.empty((B, D), np.float32)
        assert ref.lib.ref_generate_tokens(B, D, seed, theirs.reshape(-1)) == 0
        assert np.array_equal(oracle.generate_tokens(B, D, seed).view(np.uint32),
                              theirs.view(np.uint32))


def test_round_bf16(oracle):
    v = np.array([1.0, 1.00390625, 1.005859375, -3.14159, 0.0, 1e-40], np.float32)
    r = oracle.round_bf16(v)
    assert np.all((r.view(np.uint32) & 0xffff) == 0)
    assert r[0] == 1.0 and r[1] == 1.0  # tie to even
    assert r[2] == np.float32(1.0078125)


# ---- router -----------------------------------------------------------------

def test_route_hand_cases(oracle):
    """router_test.cpp:17-53"""
    rc, ids, w = oracle.route(np.array([[0.0, 0.0]]), 2)
    assert rc == 0 and ids.tolist() == [[0, 1]] and np.allclose(w, 0.5, atol=1e-6)
    rc, ids, w = oracle.route(np.array([[1.0, 3.0, 2.0]]), 1)
    assert ids.tolist() == [[1]] and abs(w[0, 0] - 1.0) < 1e-6
    lg = np.array([[0.0, np.log(np.float32(2.0)), 0.0, 0.0]], np.float32)
    rc, ids, w = oracle.route(lg, 2)
    assert ids.tolist() == [[1, 0]]
    assert np.allclose(w, [[2 / 3, 1 / 3]], rtol=1e-5)
    rc, ids, w = oracle.route(lg, 2, renorm=False)
    assert np.allclose(w, [[0.4, 0.2]], rtol=1e-5)
    rc, _, _ = oracle.route(np.zeros((1, 2)), 3)
    assert rc == 2  # ConfigError


def test_align_dispatch_hand_cases(oracle):
    """router_test.cpp:55-78"""
    rc, s, eob = oracle.align_dispatch(np.array([[3]]), 4, 4)
    assert s.tolist() == [0, PAD, PAD, PAD] and eob.tolist() == [3]
    rc, s, eob = oracle.align_dispatch(np.array([[1], [1]]), 4, 2)
    assert s.tolist() == [0, 1] and eob.tolist() == [1]
    rc, _, _ = oracle.align_dispatch(np.array([[7]]), 4, 2)
    assert rc == 3  # IndexError


def test_route_dispatch_property_and_reference(oracle, ref):
    """router_test.cpp:80-127 (permutation property) + bit-equality with the reference."""
    rng = SplitMix64(31)
    for _ in range(200):
        E = 1 + rng.below(12)
        K = 1 + rng.below(min(4, E))
        B = 1 + rng.below(16)
        block = 1 + rng.below(8)
        logits = oracle.fill_symmetric(B * E, rng.next(), 0, 2.0).reshape(B, E)
        rc, ids, w = oracle.route(logits, K)
        assert rc == 0
        rid = np.empty_like(ids)
        rw = np.empty_like(w)
        assert ref.lib.ref_route(logits, B, E, K, 1, rid, rw) == 0
        assert np.array_equal(ids, rid)
        assert np.array_equal(w.view(np.uint32), rw.view(np.uint32))
        for t in range(B):
            assert len(set(ids[t].tolist())) == K
            assert abs(float(w[t].sum()) - 1.0) <= 1e-5
        rc, s, eob = oracle.align_dispatch(ids, E, block)
        assert s.size % block == 0 and s.size <= B * K + E * (block - 1)
        live = s[s != PAD]
        assert sorted(live.tolist()) == list(range(B * K))
        for i, entry in enumerate(s.tolist()):
            if entry != PAD:
                assert ids.reshape(-1)[entry] == eob[i // block]
        cap = B * K + E * (block - 1)
        rs, reob = np.empty(cap, np.int32), np.empty(cap, np.int32)
        import ctypes as C
        npad, nblk = C.c_int32(), C.c_int32()
        assert ref.lib.ref_align_dispatch(ids, B, K, E, block, rs, reob, C.byref(npad),
                                          C.byref(nblk)) == 0
        assert s.tolist() == rs[:npad.value].tolist()
        assert eob.tolist() == reob[:nblk.value].tolist()


def test_combine_matches_reference(oracle, ref):
    """router.cpp:109-132"""
    rng = np.random.default_rng(5)
    B, K, D = 3, 4, 17
    so = rng.standard_normal((B, K, D)).astype(np.float32)
    w = rng.random((B, K)).astype(np.float32)
    ids = np.zeros((B, K), np.int32)
    y = oracle.combine(so, w, D)
    ry = np.empty_like(y)
    assert ref.lib.ref_combine(so.reshape(-1), ids, w, B, K, D, ry) == 0
    assert np.array_equal(y.view(np.uint32), ry.view(np.uint32))


# ---- activation / selection -------------------------------------------------

def test_silu_and_swiglu(oracle, ref):
    """activation_test.cpp:15-43"""
    assert oracle.lib.ork_silu(0.0) == 0.0
    assert abs(oracle.lib.ork_silu(30.0) / 30.0 - 1.0) < 1e-6
    for x in (-3.0, -1.0, 0.5, 2.0, -87.0, 12.5):
        assert oracle.lib.ork_silu(x) == ref.lib.ref_silu(x)
        assert abs(oracle.lib.ork_silu(x) - x / (1 + math.exp(-x))) <= 1e-6 * max(1, abs(x))
    h = oracle.swiglu_rows(np.array([1.0], np.float32), np.array([2.0], np.float32))
    assert abs(h[0] - 2 / (1 + math.exp(-1))) < 1e-6


def test_topk_mask_hand_cases(oracle):
    """activation_test.cpp:45-63"""
    h = np.array([0.1, -0.5, 0.3, 0.05], np.float32)
    assert oracle.topk_mask(h, 0.0)[1].tolist() == [1, 1, 1, 1]
    assert oracle.topk_mask(h, 1.0)[1].tolist() == [0, 0, 0, 0]
    assert oracle.topk_mask(h, 0.5)[1].tolist() == [0, 1, 1, 0]
    assert oracle.topk_mask(np.full(4, 0.2, np.float32), 0.5)[1].tolist() == [0, 0, 1, 1]
    assert oracle.topk_mask(h, 1.5)[0] == 2 and oracle.topk_mask(h, float("nan"))[0] == 2


def test_topk_mask_counts_and_reference(oracle, ref):
    """activation_test.cpp:65-77, budget_test.cpp:139-162"""
    rng = SplitMix64(7)
    for s in (0.0, 0.25, 0.5, 0.9, 1.0):
        for n in range(1, 65):
            h = oracle.fill_symmetric(n, rng.next(), 0, 1.0)
            # inject ties, signed zeros and duplicates of opposite sign
            if n > 4:
                h[1] = -h[0]
                h[3] = 0.0
                h[2] = -0.0
            rc, mask = oracle.topk_mask(h, s)
            assert int((mask == 0).sum()) == int(math.floor(s * n + 0.5))
            rmask = np.empty(n, np.uint8)
            assert ref.lib.ref_topk_mask(h, n, s, rmask) == 0
            assert np.array_equal(mask, rmask)
    rmask = np.empty(3, np.uint8)
    h = np.array([1, -3, 2], np.float32)
    assert ref.lib.ref_apply_budget(h, 3, 2, rmask) == 0
    assert rmask.tolist() == [0, 1, 1] == oracle.mask_smallest(h, 1).tolist()


def test_threshold_mask_and_compact(oracle, ref):
    """activation_test.cpp:79-198"""
    g = np.array([2.0, -2.0, 0.01], np.float32)
    assert oracle.threshold_mask(g, 0.0)[1].tolist() == [1, 1, 1]
    assert oracle.threshold_mask(g, 1e30)[1].tolist() == [0, 0, 0]
    assert oracle.threshold_mask(g, 0.5)[1].tolist() == [1, 0, 0]
    assert oracle.threshold_mask(g, -1.0)[0] == 2
    assert [oracle.lib.ork_default_capacity(*a) for a in ((1, 4), (2, 64), (3, 8), (2, 16))] == \
        [32, 128, 32, 32]

    rc, flat, per, tot = oracle.compact_active([0, 0, 0, 0], [2], 4, 8)
    assert tot == 0 and per.tolist() == [0] and set(flat.tolist()) == {PAD}
    rc, flat, per, tot = oracle.compact_active([1, 0, 1, 0], [2], 4, 32)
    assert tot == 2 and flat[:3].tolist() == [8, 10, PAD]
    rc, flat, per, tot = oracle.compact_active([1, 1, 1, 0], [0], 4, 1)
    assert tot == 1 and per.tolist() == [1] and flat.tolist() == [0]
    rc, flat, per, tot = oracle.compact_active([1, 1, 1, 1], [1, 0], 2, 3)
    assert per.tolist() == [2, 1] and tot == 3 and flat.tolist() == [2, 3, 0]

    import ctypes as C
    rng = SplitMix64(41)
    for _ in range(50):
        K = 1 + rng.below(4)
        N = 1 + rng.below(32)
        cap = oracle.lib.ork_default_capacity(K, N) - (rng.below(3) * 8)
        cap = max(cap, 0)
        masks = np.array([rng.below(2) for _ in range(K * N)], np.uint8)
        ids = np.array([rng.below(8) for _ in range(K)], np.int32)
        rc, flat, per, tot = oracle.compact_active(masks, ids, N, cap)
        rflat, rper, rtot = np.empty(max(cap, 1), np.int32), np.empty(K, np.int32), C.c_int32()
        assert ref.lib.ref_compact_active(masks, ids, K, N, cap, rflat, rper, C.byref(rtot)) == 0
        assert flat.tolist() == rflat[:cap].tolist() and per.tolist() == rper.tolist()
        assert tot == rtot.value


def test_linalg_hand_cases(oracle, ref):
    """linalg_test.cpp hand cases + SPEC examples (matvec / gathered_matvec_T)."""
    assert oracle.matvec([[1, 2], [3, 4]], [1, 1]).tolist() == [3, 7]
    rc, y = oracle.gathered_matvec_t(np.eye(2, dtype=np.float32), [1], [5.0])
    assert y.tolist() == [0, 5]
    rc, y = oracle.gathered_matvec_t([[1, 3], [2, 4]], [0, 1], [1.0, 1.0])
    assert y.tolist() == [3, 7]
    rc, y = oracle.gathered_matvec_t(np.ones((2, 3), np.float32), [], [])
    assert y.tolist() == [0, 0, 0]
    rc, _ = oracle.gathered_matvec_t(np.ones((2, 3), np.float32), [2], [1.0])
    assert rc == 3
    rng = np.random.default_rng(3)
    w = rng.standard_normal((37, 29)).astype(np.float32)
    idx = rng.integers(0, 37, 50).astype(np.int32)
    h = rng.standard_normal(50).astype(np.float32)
    rc, y = oracle.gathered_matvec_t(w, idx, h)
    ry = np.empty_like(y)
    assert ref.lib.ref_gathered_matvec_t(w.reshape(-1), 37, 29, idx, h, 50, ry) == 0
    assert np.array_equal(y.view(np.uint32), ry.view(np.uint32))


# ---- layer ------------------------------------------------------------------

def _rand_case(rng, oracle, allow_shared=True):
    cfg = random_config(rng, allow_shared)
    w = oracle.generate_synthetic(cfg, rng.next(), 0.1)
    B = 1 + rng.below(6)
    x = oracle.generate_tokens(B, cfg.d_model, rng.next())
    return cfg, w, B, x


def test_dense_matches_reference_and_scalar(oracle, ref):
    """engine_test.cpp:69-80, acceptance.cpp:132-147, MAC closed forms :241-265."""
    rng = SplitMix64(91)
    for _ in range(25):
        cfg, w, B, x = _rand_case(rng, oracle)
        y, rep = oracle.forward(w, x)
        rl = RefLayer.from_weights(w)
        ry, rrep = rl.forward_dense(x, threads=3)
        assert np.array_equal(y.view(np.uint32), ry.view(np.uint32))
        assert rep.as_dict() == rrep.as_dict()
        bkdn = B * cfg.top_k * cfg.d_model * cfg.d_ffn
        assert rep.gate_macs == rep.up_macs == rep.down_macs == bkdn
        assert rep.other_macs == B * cfg.n_experts * cfg.d_model + 3 * B * cfg.d_shared * cfg.d_model
        assert max_rel_diff(y, oracle.scalar_forward(w, x)) <= 1e-5
        assert np.array_equal(oracle.scalar_forward(w, x).view(np.uint32),
                              rl.scalar_forward(x).view(np.uint32))


def test_masked_invariants_and_reference(oracle, ref):
    """engine_test.cpp:111-189 (all-true == dense, all-false == shared only, random masks)."""
    rng = SplitMix64(57)
    for _ in range(20):
        cfg, w, B, x = _rand_case(rng, oracle)
        dense, _ = oracle.forward(w, x)
        ones = np.ones((B, cfg.top_k, cfg.d_ffn), np.uint8)
        y1, rep1 = oracle.forward(w, x, ones)
        assert np.array_equal(y1.view(np.uint32), dense.view(np.uint32))
        assert rep1.achieved_routed_sparsity == 0.0
        zeros = np.zeros_like(ones)
        y0, rep0 = oracle.forward(w, x, zeros)
        assert rep0.active_neurons_total == 0 and rep0.achieved_routed_sparsity == 1.0
        if not cfg.has_shared:
            assert not y0.any()
        rl = RefLayer.from_weights(w)
        for s in (0.25, 0.5, 0.9):
            rm, sm = oracle.build_topk_masks(w, x, s, mode=1)
            rrm, rsm = rl.build_topk_masks(x, s, mode=1)
            assert np.array_equal(rm, rrm)
            assert (sm is None and rsm is None) or np.array_equal(sm, rsm)
            y, rep = oracle.forward(w, x, rm, sm)
            ry, rrep = rl.forward_masked_dense(x, rm, sm, threads=2)
            assert np.array_equal(y.view(np.uint32), ry.view(np.uint32))
            assert rep.as_dict() == rrep.as_dict()
            assert max_rel_diff(y, oracle.scalar_forward(w, x, rm, sm)) <= 1e-5
            n_off = oracle.n_off(s, cfg.d_ffn)
            assert rep.active_neurons_total == B * cfg.top_k * (cfg.d_ffn - n_off)


def test_capture_h_matches_masks(oracle):
    rng = SplitMix64(11)
    cfg, w, B, x = _rand_case(rng, oracle)
    y, rep, cap = oracle.forward(w, x, capture=True)
    rm, _ = oracle.build_topk_masks(w, x, 0.5, mode=0)
    for t in range(B):
        for s in range(cfg.top_k):
            assert np.array_equal(oracle.topk_mask(cap["h_routed"][t, s], 0.5)[1], rm[t, s])


def test_forward_sparse_matches_reference(oracle, ref):
    """engine_test.cpp:191-335, acceptance.cpp:78-130: tau=0 == dense to 1e-5, closed forms,
    and the restatement is bit-identical to the reference."""
    rng = SplitMix64(97)
    for _ in range(20):
        cfg, w, B, x = _rand_case(rng, oracle)
        rl = RefLayer.from_weights(w)
        tau = 0.002 + 0.05 * rng.unit()
        for t in (0.0, tau, 1e30):
            rc, y, rep = oracle.forward_sparse(w, x, t)
            ry, rrep = rl.forward_sparse(x, t, threads=2)
            assert rc == 0
            assert np.array_equal(y.view(np.uint32), ry.view(np.uint32))
            assert rep.as_dict() == rrep.as_dict()
        rc, y0, _ = oracle.forward_sparse(w, x, 0.0)
        dense, _ = oracle.forward(w, x)
        assert max_rel_diff(y0, dense) <= 1e-5
        assert oracle.forward_sparse(w, x, -1.0)[0] == 2
        assert oracle.forward_sparse(w, x, float("nan"))[0] == 2


def test_reference_error_codes(ref):
    """errors.hpp:12-43 -> shim codes (1 shape, 2 config)."""
    from oracle.pyoracle import RefError
    rl = RefLayer.synthetic(Config(4, 2, 8, 16), 1, 0.05)
    with pytest.raises(RefError) as ei:
        rl.forward_sparse(np.zeros((1, 8), np.float32), -1.0)
    assert ei.value.code == 2
    with pytest.raises(RefError) as ei:
        rl.build_topk_masks(np.zeros((1, 8), np.float32), 1.5)
    assert ei.value.code == 2
    with pytest.raises(ValueError):
        RefLayer.synthetic(Config(4, 5, 8, 16), 1, 0.05)


def test_sparse_synth_model_matches_the_full_oracle(oracle):
    """The one-expert-at-a-time double-precision checker used by the full-shape GPU tests gives
    the oracle's own answer on a shape small enough to materialise whole."""
    from tests.helpers import SparseSynthModel
    o = oracle
    cfg = Config(8, 2, 48, 40, 24, True)
    w_raw = o.generate_synthetic(cfg, 7, 0.1)
    w = w_raw.rounded_bf16()
    w.router = w_raw.router
    x = o.round_bf16(o.generate_tokens(5, cfg.d_model, 3))
    routed, shared = o.build_topk_masks(w, x, 0.5, 1)
    y_ref, _, cap = o.forward(w, x, routed, shared, capture=True)
    m = SparseSynthModel(o, cfg, 7, 0.1)
    ids, wts = m.routing(x, cfg.top_k)
    np.testing.assert_array_equal(ids, cap["ids"])
    np.testing.assert_array_equal(wts, cap["weights"])
    y = m.scalar_forward(x, ids, wts, routed.reshape(5, 2, 40), shared.reshape(5, 24), tokens=[0, 3, 4])
    assert max_rel_diff(y, y_ref[[0, 3, 4]]) <= 1e-5
    y_scalar = o.scalar_forward(w, x, routed, shared)
    assert max_rel_diff(y, y_scalar[[0, 3, 4]]) <= 1e-6
