"""Shared test helpers (numpy side)."""
import numpy as np

from oracle.pyoracle import Config


class SplitMix64:
    """Python twin of the reference RNG (rng.hpp:16-40) for test-case generation."""
    M = (1 << 64) - 1

    def __init__(self, seed):
        self.s = seed & self.M

    def next(self):
        self.s = (self.s + 0x9E3779B97F4A7C15) & self.M
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.M
        return z ^ (z >> 31)

    def below(self, n):
        return self.next() % n

    def unit(self):
        return (self.next() >> 11) * 2.0 ** -53


def random_config(rng: SplitMix64, allow_shared=True) -> Config:
    """Same shape distribution as proj/tests/support.hpp:154-167."""
    E = 1 + rng.below(16)
    K = 1 + rng.below(min(4, E))
    D = 1 + rng.below(64)
    N = 1 + rng.below(128)
    S = 0
    if allow_shared and rng.below(2) == 0:
        S = 1 + rng.below(32)
    renorm = rng.below(2) == 0
    return Config(E, K, D, N, S, renorm)


def max_rel_diff(a, b):
    """proj/tests/support.hpp:32-42"""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(b))))


def true_rel_err(a, b):
    """max |a - b| / max |b| -- the relative error proper (max_rel_diff above divides by
    max(1, max |b|), which is an absolute error whenever the outputs are below 1)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(1e-30, np.max(np.abs(b))))


class SparseSynthModel:
    """generate_synthetic(cfg, seed, scale) (proj/src/model.cpp:129-166) materialised ONE EXPERT
    AT A TIME through the SplitMix64 jump-ahead offsets of the oracle library -- shapes whose fp32
    model does not fit the host (GPT-OSS: 3.2 GB is fine, Llama-4-Maverick: 64 GB is not) are
    checked on the experts the routing actually touches.  Weights are rounded to bf16 as the
    device image is (router stays fp32)."""

    def __init__(self, oracle, cfg: Config, seed: int, scale: float):
        import ctypes as C
        self.o, self.cfg, self.seed, self.scale = oracle, cfg, seed, scale
        self._c = cfg.c()
        self._C = C
        self._cache = {}
        E, D = cfg.n_experts, cfg.d_model
        self.router = oracle.fill_symmetric(E * D, seed, 0, scale).reshape(E, D)

    def expert(self, e):
        """(gate, up, down_t) of expert e, each [N][D], bf16-rounded fp32; e == n_experts is the
        shared expert ([S][D])."""
        if e in self._cache:
            return self._cache[e]
        o, cfg, C = self.o, self.cfg, self._C
        D = cfg.d_model
        mats = []
        for which in range(3):
            if e == cfg.n_experts:
                off = o.lib.ork_synth_offset_shared(C.byref(self._c), which)
                n = cfg.d_shared
            else:
                off = o.lib.ork_synth_offset_expert(C.byref(self._c), e, which)
                n = cfg.d_ffn
            mats.append(o.round_bf16(o.fill_symmetric(n * D, self.seed, off, self.scale)).reshape(n, D))
        if len(self._cache) >= 2:  # a Maverick expert is 3 x 168 MB
            self._cache.pop(next(iter(self._cache)))
        self._cache[e] = tuple(mats)
        return self._cache[e]

    def routing(self, x, top_k, renorm=True):
        """ids / weights of the reference for these tokens (order-faithful logits)."""
        logits = np.stack([self.o.matvec(self.router, x[t]) for t in range(x.shape[0])])
        _, ids, wts = self.o.route(logits, top_k, renorm)
        return ids, wts

    def scalar_forward(self, x, ids, wts, routed_masks, shared_masks=None, tokens=None):
        """testsupport::scalar_forward (proj/tests/support.hpp:55-152) in double precision on the
        given routing and masks, for the listed tokens only; expert-major so that every expert is
        materialised once.  Returns y[len(tokens)][D] as float64."""
        cfg = self.cfg
        tokens = list(range(x.shape[0])) if tokens is None else list(tokens)
        y = np.zeros((len(tokens), cfg.d_model), np.float64)
        slot_out = {}
        pairs = sorted((int(ids[t, k]), ti, k) for ti, t in enumerate(tokens) for k in range(ids.shape[1]))
        for e, ti, k in pairs:
            g_w, u_w, d_w = self.expert(e)
            xt = x[tokens[ti]].astype(np.float64)
            g = g_w.astype(np.float64) @ xt
            u = u_w.astype(np.float64) @ xt
            h = g / (1.0 + np.exp(-g)) * u
            keep = np.asarray(routed_masks[tokens[ti], k], bool)
            slot_out[(ti, k)] = (h * keep) @ d_w.astype(np.float64)
        for ti, t in enumerate(tokens):
            for k in range(ids.shape[1]):  # combine: slots ascending (router.cpp:119-130)
                y[ti] += float(wts[t, k]) * slot_out[(ti, k)]
        if cfg.d_shared:
            g_w, u_w, d_w = self.expert(cfg.n_experts)
            for ti, t in enumerate(tokens):
                xt = x[t].astype(np.float64)
                g = g_w.astype(np.float64) @ xt
                u = u_w.astype(np.float64) @ xt
                h = g / (1.0 + np.exp(-g)) * u
                if shared_masks is not None:
                    h = h * np.asarray(shared_masks[t], bool)
                y[ti] += h @ d_w.astype(np.float64)  # engine.cpp:55-84: after the routed combine
        return y
