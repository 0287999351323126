"""ctypes doors to the test oracle.  TEST INFRASTRUCTURE ONLY.

Two libraries, both built by ``make -C oracle``:

* ``libmoe_oracle.so``          -- plain-C restatement of the reference layer
  (``Oracle`` class below; always available).
* ``_ref/libsparsekit_ref.so``  -- the unmodified reference compiled from
  /root/reference/proj (``Ref`` class; available when it was built in the
  container -- the file travels to the GPU box with the repo).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs may import
this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libmoe_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsparsekit_ref.so")

f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


class OrkConfig(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "n_experts", "top_k", "d_model", "d_ffn", "has_shared", "d_shared", "renormalize",
        "align_block")]


class OrkWeights(C.Structure):
    _fields_ = [("cfg", OrkConfig)] + [(n, C.c_void_p) for n in (
        "router", "gate", "up", "down_t", "shared_gate", "shared_up", "shared_down_t")]


class OrkReport(C.Structure):
    _fields_ = [("gate_macs", C.c_uint64), ("up_macs", C.c_uint64), ("down_macs", C.c_uint64),
                ("other_macs", C.c_uint64), ("active_neurons_total", C.c_uint64),
                ("achieved_routed_sparsity", C.c_double), ("tiles_total", C.c_uint64),
                ("tiles_skipped", C.c_uint64), ("path_used", C.c_int32)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


@dataclass
class Config:
    n_experts: int
    top_k: int
    d_model: int
    d_ffn: int
    d_shared: int = 0
    renormalize: bool = True
    align_block: int = 64

    @property
    def has_shared(self):
        return self.d_shared > 0

    def c(self) -> OrkConfig:
        return OrkConfig(self.n_experts, self.top_k, self.d_model, self.d_ffn,
                         int(self.has_shared), self.d_shared, int(self.renormalize),
                         self.align_block)


def build(force: bool = False) -> None:
    """Compile the oracle (and oracle/_ref when /root/reference is present)."""
    need = force or not os.path.exists(ORACLE_SO) or (
        os.path.isdir("/root/reference/proj/src") and not os.path.exists(REF_SO))
    if need:
        subprocess.run(["make", "-C", HERE, "-j4"], check=True, capture_output=True)


def _opt(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Weights:
    """Contiguous fp32 weight arrays in the layout moe_oracle.h documents."""

    def __init__(self, cfg: Config, router, gate, up, down_t, sg=None, su=None, sd=None):
        self.cfg = cfg
        self.router, self.gate, self.up, self.down_t = router, gate, up, down_t
        self.shared_gate, self.shared_up, self.shared_down_t = sg, su, sd

    def c(self) -> OrkWeights:
        w = OrkWeights()
        w.cfg = self.cfg.c()
        for n in ("router", "gate", "up", "down_t", "shared_gate", "shared_up", "shared_down_t"):
            a = getattr(self, n)
            setattr(w, n, None if a is None else a.ctypes.data)
        return w

    def rounded_bf16(self) -> "Weights":
        o = Oracle.get()
        arrs = []
        for n in ("router", "gate", "up", "down_t", "shared_gate", "shared_up", "shared_down_t"):
            a = getattr(self, n)
            arrs.append(None if a is None else o.round_bf16(a))
        return Weights(self.cfg, *arrs)


class Oracle:
    _inst = None

    @classmethod
    def get(cls) -> "Oracle":
        if cls._inst is None:
            cls._inst = cls()
        return cls._inst

    def __init__(self):
        build()
        L = self.lib = C.CDLL(ORACLE_SO)
        L.ork_fill_symmetric.argtypes = [f32p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_float]
        L.ork_fill_gaussian.argtypes = [f32p, C.c_uint64, C.c_uint64]
        for fn in (L.ork_synth_offset_router,):
            fn.argtypes = [C.POINTER(OrkConfig)]
            fn.restype = C.c_uint64
        L.ork_synth_offset_expert.argtypes = [C.POINTER(OrkConfig), C.c_int, C.c_int]
        L.ork_synth_offset_expert.restype = C.c_uint64
        L.ork_synth_offset_shared.argtypes = [C.POINTER(OrkConfig), C.c_int]
        L.ork_synth_offset_shared.restype = C.c_uint64
        L.ork_round_bf16.argtypes = [f32p, C.c_uint64]
        L.ork_route.argtypes = [f32p, C.c_int, C.c_int, C.c_int, C.c_int, i32p, f32p]
        L.ork_align_dispatch.argtypes = [i32p, C.c_int, C.c_int, C.c_int, C.c_int, i32p, i32p,
                                         C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.ork_combine.argtypes = [f32p, f32p, C.c_int, C.c_int, C.c_int, f32p]
        L.ork_silu.argtypes = [C.c_float]
        L.ork_silu.restype = C.c_float
        L.ork_swiglu_rows.argtypes = [f32p, f32p, C.c_int, f32p]
        L.ork_n_off.argtypes = [C.c_double, C.c_int]
        L.ork_mask_smallest.argtypes = [f32p, C.c_int, C.c_int, u8p]
        L.ork_topk_mask.argtypes = [f32p, C.c_int, C.c_double, u8p]
        L.ork_threshold_mask.argtypes = [f32p, C.c_int, C.c_float, u8p]
        L.ork_compact_active.argtypes = [u8p, i32p, C.c_int, C.c_int, C.c_int, i32p, i32p,
                                         C.POINTER(C.c_int32)]
        L.ork_matvec.argtypes = [f32p, C.c_int, C.c_int, f32p, f32p]
        L.ork_gathered_matvec_t.argtypes = [f32p, C.c_int, C.c_int, i32p, f32p, C.c_int, f32p]
        L.ork_build_topk_masks.argtypes = [C.POINTER(OrkWeights), f32p, C.c_int, C.c_double,
                                           C.c_int, u8p, C.c_void_p]
        L.ork_forward_masked.argtypes = [C.POINTER(OrkWeights), f32p, C.c_int, C.c_void_p,
                                         C.c_void_p, f32p, C.POINTER(OrkReport), C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p]
        L.ork_forward_sparse.argtypes = [C.POINTER(OrkWeights), f32p, C.c_int, C.c_float, f32p,
                                         C.POINTER(OrkReport)]
        L.ork_scalar_forward.argtypes = [C.POINTER(OrkWeights), f32p, C.c_int, C.c_void_p,
                                         C.c_void_p, f32p]
        L.ork_max_rel_diff.argtypes = [f32p, f32p, C.c_uint64]
        L.ork_max_rel_diff.restype = C.c_double

    # -- generators --------------------------------------------------------
    def fill_symmetric(self, count, seed, offset, scale):
        out = np.empty(count, np.float32)
        self.lib.ork_fill_symmetric(out, count, seed, offset, scale)
        return out

    def generate_tokens(self, batch, d_model, seed):
        out = np.empty(batch * d_model, np.float32)
        self.lib.ork_fill_gaussian(out, out.size, seed)
        return out.reshape(batch, d_model)

    def generate_synthetic(self, cfg: Config, seed: int, scale: float) -> Weights:
        c = cfg.c()
        E, D, N, S = cfg.n_experts, cfg.d_model, cfg.d_ffn, cfg.d_shared
        router = self.fill_symmetric(E * D, seed, 0, scale).reshape(E, D)
        gate = np.empty((E, N, D), np.float32)
        up = np.empty((E, N, D), np.float32)
        down = np.empty((E, N, D), np.float32)
        for e in range(E):
            for which, dst in enumerate((gate, up, down)):
                off = self.lib.ork_synth_offset_expert(C.byref(c), e, which)
                dst[e] = self.fill_symmetric(N * D, seed, off, scale).reshape(N, D)
        sh = [None, None, None]
        if cfg.has_shared:
            for which in range(3):
                off = self.lib.ork_synth_offset_shared(C.byref(c), which)
                sh[which] = self.fill_symmetric(S * D, seed, off, scale).reshape(S, D)
        return Weights(cfg, router, gate, up, down, *sh)

    def round_bf16(self, a):
        out = np.ascontiguousarray(a, dtype=np.float32).copy()
        self.lib.ork_round_bf16(out.reshape(-1), out.size)
        return out

    # -- stages ------------------------------------------------------------
    def route(self, logits, top_k, renorm=True):
        logits = np.ascontiguousarray(logits, np.float32)
        B, E = logits.shape
        ids = np.empty((B, top_k), np.int32)
        wts = np.empty((B, top_k), np.float32)
        rc = self.lib.ork_route(logits, B, E, top_k, int(renorm), ids, wts)
        return rc, ids, wts

    def align_dispatch(self, ids, n_experts, block):
        ids = np.ascontiguousarray(ids, np.int32)
        B, K = ids.shape
        cap = B * K + n_experts * (block - 1)
        sorted_out = np.empty(max(cap, 1), np.int32)
        eob = np.empty(max(cap, 1), np.int32)
        n_padded, n_blocks = C.c_int32(), C.c_int32()
        rc = self.lib.ork_align_dispatch(ids, B, K, n_experts, block, sorted_out, eob,
                                         C.byref(n_padded), C.byref(n_blocks))
        return rc, sorted_out[:n_padded.value].copy(), eob[:n_blocks.value].copy()

    def n_off(self, s, n):
        return self.lib.ork_n_off(s, n)

    def mask_smallest(self, h, count):
        h = np.ascontiguousarray(h, np.float32)
        mask = np.empty(h.size, np.uint8)
        self.lib.ork_mask_smallest(h, h.size, count, mask)
        return mask

    def topk_mask(self, h, s):
        h = np.ascontiguousarray(h, np.float32)
        mask = np.empty(h.size, np.uint8)
        rc = self.lib.ork_topk_mask(h, h.size, s, mask)
        return rc, mask

    def threshold_mask(self, g, tau):
        g = np.ascontiguousarray(g, np.float32)
        mask = np.empty(g.size, np.uint8)
        rc = self.lib.ork_threshold_mask(g, g.size, tau, mask)
        return rc, mask

    def compact_active(self, masks, topk_ids, d_ffn, capacity):
        masks = np.ascontiguousarray(masks, np.uint8).reshape(-1)
        topk_ids = np.ascontiguousarray(topk_ids, np.int32)
        flat = np.empty(max(capacity, 1), np.int32)
        per = np.empty(topk_ids.size, np.int32)
        tot = C.c_int32()
        rc = self.lib.ork_compact_active(masks, topk_ids, topk_ids.size, d_ffn, capacity, flat,
                                         per, C.byref(tot))
        return rc, flat[:capacity], per, tot.value

    def swiglu_rows(self, g, u):
        g = np.ascontiguousarray(g, np.float32)
        u = np.ascontiguousarray(u, np.float32)
        h = np.empty_like(g)
        self.lib.ork_swiglu_rows(g, u, g.size, h)
        return h

    def matvec(self, w, x):
        w = np.ascontiguousarray(w, np.float32)
        y = np.empty(w.shape[0], np.float32)
        self.lib.ork_matvec(w, w.shape[0], w.shape[1], np.ascontiguousarray(x, np.float32), y)
        return y

    def gathered_matvec_t(self, w_t, idx, h):
        w_t = np.ascontiguousarray(w_t, np.float32)
        idx = np.ascontiguousarray(idx, np.int32)
        y = np.empty(w_t.shape[1], np.float32)
        rc = self.lib.ork_gathered_matvec_t(w_t, w_t.shape[0], w_t.shape[1], idx,
                                            np.ascontiguousarray(h, np.float32), idx.size, y)
        return rc, y

    def combine(self, slot_outputs, weights, d_model):
        weights = np.ascontiguousarray(weights, np.float32)
        B, K = weights.shape
        y = np.empty((B, d_model), np.float32)
        self.lib.ork_combine(np.ascontiguousarray(slot_outputs, np.float32).reshape(-1), weights,
                             B, K, d_model, y)
        return y

    # -- layer -------------------------------------------------------------
    def build_topk_masks(self, w: Weights, x, s, mode=1):
        cfg = w.cfg
        x = np.ascontiguousarray(x, np.float32)
        B = x.shape[0]
        routed = np.empty((B, cfg.top_k, cfg.d_ffn), np.uint8)
        shared = np.empty((B, cfg.d_shared), np.uint8) if (mode == 1 and cfg.has_shared) else None
        cw = w.c()
        rc = self.lib.ork_build_topk_masks(C.byref(cw), x, B, s, mode, routed, _opt(shared))
        assert rc == 0, rc
        return routed, shared

    def forward(self, w: Weights, x, routed_masks=None, shared_masks=None, capture=False):
        cfg = w.cfg
        x = np.ascontiguousarray(x, np.float32)
        B = x.shape[0]
        y = np.empty((B, cfg.d_model), np.float32)
        rep = OrkReport()
        cap = {}
        if capture:
            cap["ids"] = np.empty((B, cfg.top_k), np.int32)
            cap["weights"] = np.empty((B, cfg.top_k), np.float32)
            cap["h_routed"] = np.empty((B, cfg.top_k, cfg.d_ffn), np.float32)
            cap["h_shared"] = np.empty((B, cfg.d_shared), np.float32) if cfg.has_shared else None
        cw = w.c()
        rc = self.lib.ork_forward_masked(
            C.byref(cw), x, B, _opt(routed_masks), _opt(shared_masks), y, C.byref(rep),
            _opt(cap.get("ids")), _opt(cap.get("weights")), _opt(cap.get("h_routed")),
            _opt(cap.get("h_shared")))
        assert rc == 0, rc
        return (y, rep, cap) if capture else (y, rep)

    def forward_sparse(self, w: Weights, x, tau):
        x = np.ascontiguousarray(x, np.float32)
        B = x.shape[0]
        y = np.empty((B, w.cfg.d_model), np.float32)
        rep = OrkReport()
        cw = w.c()
        rc = self.lib.ork_forward_sparse(C.byref(cw), x, B, tau, y, C.byref(rep))
        return rc, y, rep

    def scalar_forward(self, w: Weights, x, routed_masks=None, shared_masks=None):
        x = np.ascontiguousarray(x, np.float32)
        y = np.empty((x.shape[0], w.cfg.d_model), np.float32)
        cw = w.c()
        self.lib.ork_scalar_forward(C.byref(cw), x, x.shape[0], _opt(routed_masks),
                                    _opt(shared_masks), y)
        return y

    def max_rel_diff(self, a, b):
        a = np.ascontiguousarray(a, np.float32).reshape(-1)
        b = np.ascontiguousarray(b, np.float32).reshape(-1)
        return self.lib.ork_max_rel_diff(a, b, a.size)


class Ref:
    """The unmodified reference library behind oracle/ref_shim.cpp."""
    _inst = None

    @classmethod
    def available(cls) -> bool:
        build()
        return os.path.exists(REF_SO)

    @classmethod
    def get(cls) -> "Ref":
        if cls._inst is None:
            cls._inst = cls()
        return cls._inst

    def __init__(self):
        build()
        L = self.lib = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_layer_synthetic.argtypes = [C.POINTER(OrkConfig), C.c_uint64, C.c_float]
        L.ref_layer_synthetic.restype = C.c_void_p
        L.ref_layer_from_arrays.argtypes = [C.POINTER(OrkConfig)] + [C.c_void_p] * 7
        L.ref_layer_from_arrays.restype = C.c_void_p
        L.ref_layer_free.argtypes = [C.c_void_p]
        L.ref_layer_round_bf16.argtypes = [C.c_void_p]
        for n in ("ref_layer_router",):
            getattr(L, n).argtypes = [C.c_void_p]
            getattr(L, n).restype = C.POINTER(C.c_float)
        for n in ("ref_layer_gate", "ref_layer_up", "ref_layer_down_t", "ref_layer_shared"):
            getattr(L, n).argtypes = [C.c_void_p, C.c_int]
            getattr(L, n).restype = C.POINTER(C.c_float)
        L.ref_generate_tokens.argtypes = [C.c_int, C.c_int, C.c_uint64, f32p]
        L.ref_save_weights.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_forward_dense.argtypes = [C.c_void_p, f32p, C.c_int, C.c_int, f32p, C.POINTER(OrkReport)]
        L.ref_forward_masked_dense.argtypes = [C.c_void_p, f32p, C.c_int, u8p, C.c_void_p, C.c_int,
                                               f32p, C.POINTER(OrkReport)]
        L.ref_forward_sparse.argtypes = [C.c_void_p, f32p, C.c_int, C.c_float, C.c_int, f32p,
                                         C.POINTER(OrkReport)]
        L.ref_build_topk_masks.argtypes = [C.c_void_p, f32p, C.c_int, C.c_double, C.c_int, u8p,
                                           C.c_void_p]
        L.ref_scalar_forward.argtypes = [C.c_void_p, f32p, C.c_int, C.c_void_p, C.c_void_p, f32p]
        L.ref_calibrate_tau.argtypes = [C.c_void_p, C.c_double, C.c_int, C.c_uint64, C.c_uint64,
                                        C.c_uint64, C.POINTER(C.c_double)]
        f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
        L.ref_sweep_cutoff.argtypes = [C.c_void_p, f32p, C.c_int, f64p, C.c_int, C.c_double, C.c_int,
                                       f64p, C.POINTER(C.c_double), C.c_char_p]
        L.ref_emit_report.argtypes = [f64p, C.c_int, C.c_char_p, C.c_double, C.c_char_p]
        L.ref_route.argtypes = [f32p, C.c_int, C.c_int, C.c_int, C.c_int, i32p, f32p]
        L.ref_align_dispatch.argtypes = [i32p, C.c_int, C.c_int, C.c_int, C.c_int, i32p, i32p,
                                         C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.ref_combine.argtypes = [f32p, i32p, f32p, C.c_int, C.c_int, C.c_int, f32p]
        L.ref_silu.argtypes = [C.c_float]
        L.ref_silu.restype = C.c_float
        L.ref_swiglu_rows.argtypes = [f32p, f32p, C.c_int, f32p]
        L.ref_mask_smallest.argtypes = [f32p, C.c_int, C.c_int, u8p]
        L.ref_topk_mask.argtypes = [f32p, C.c_int, C.c_double, u8p]
        L.ref_apply_budget.argtypes = [f32p, C.c_int, C.c_int, u8p]
        L.ref_threshold_mask.argtypes = [f32p, C.c_int, C.c_float, u8p]
        L.ref_default_capacity.argtypes = [C.c_int, C.c_int]
        L.ref_compact_active.argtypes = [u8p, i32p, C.c_int, C.c_int, C.c_int, i32p, i32p,
                                         C.POINTER(C.c_int32)]
        L.ref_matvec.argtypes = [f32p, C.c_int, C.c_int, f32p, f32p]
        L.ref_gathered_matvec_t.argtypes = [f32p, C.c_int, C.c_int, i32p, f32p, C.c_int, f32p]

    def last_error(self):
        return self.lib.ref_last_error().decode()


class RefLayer:
    """Owns a reference MoELayerWeights instance."""

    def __init__(self, cfg: Config, handle):
        self.cfg = cfg
        self.h = handle
        self.ref = Ref.get()

    @classmethod
    def synthetic(cls, cfg: Config, seed: int, scale: float) -> "RefLayer":
        c = cfg.c()
        h = Ref.get().lib.ref_layer_synthetic(C.byref(c), seed, scale)
        if not h:
            raise ValueError(Ref.get().last_error())
        return cls(cfg, h)

    @classmethod
    def from_weights(cls, w: Weights) -> "RefLayer":
        c = w.cfg.c()
        h = Ref.get().lib.ref_layer_from_arrays(
            C.byref(c), *[_opt(getattr(w, n)) for n in (
                "router", "gate", "up", "down_t", "shared_gate", "shared_up", "shared_down_t")])
        return cls(w.cfg, h)

    def __del__(self):
        try:
            if self.h:
                self.ref.lib.ref_layer_free(self.h)
                self.h = None
        except Exception:
            pass

    def round_bf16(self):
        self.ref.lib.ref_layer_round_bf16(self.h)
        return self

    def _view(self, ptr, shape):
        return np.ctypeslib.as_array(ptr, shape=shape)

    def weights(self) -> Weights:
        """Copy the reference's matrices out into contiguous arrays."""
        cfg, L = self.cfg, self.ref.lib
        E, D, N, S = cfg.n_experts, cfg.d_model, cfg.d_ffn, cfg.d_shared
        router = self._view(L.ref_layer_router(self.h), (E, D)).copy()
        gate = np.stack([self._view(L.ref_layer_gate(self.h, e), (N, D)) for e in range(E)])
        up = np.stack([self._view(L.ref_layer_up(self.h, e), (N, D)) for e in range(E)])
        down = np.stack([self._view(L.ref_layer_down_t(self.h, e), (N, D)) for e in range(E)])
        sh = [None] * 3
        if cfg.has_shared:
            sh = [self._view(L.ref_layer_shared(self.h, i), (S, D)).copy() for i in range(3)]
        return Weights(cfg, router, gate, up, down, *sh)

    def expert_ptrs(self):
        """(gate, up, down_t) arrays of E raw pointers into the reference's storage."""
        L, E = self.ref.lib, self.cfg.n_experts
        out = []
        for fn in (L.ref_layer_gate, L.ref_layer_up, L.ref_layer_down_t):
            arr = (C.c_void_p * E)()
            for e in range(E):
                arr[e] = C.cast(fn(self.h, e), C.c_void_p).value
            out.append(arr)
        return out

    def router_ptr(self):
        return C.cast(self.ref.lib.ref_layer_router(self.h), C.c_void_p)

    def shared_ptr(self, which):
        return C.cast(self.ref.lib.ref_layer_shared(self.h, which), C.c_void_p)

    def _check(self, rc):
        if rc != 0:
            raise RefError(rc, self.ref.last_error())

    def forward_dense(self, x, threads=1):
        x = np.ascontiguousarray(x, np.float32)
        y = np.empty((x.shape[0], self.cfg.d_model), np.float32)
        rep = OrkReport()
        self._check(self.ref.lib.ref_forward_dense(self.h, x, x.shape[0], threads, y, C.byref(rep)))
        return y, rep

    def forward_masked_dense(self, x, routed, shared=None, threads=1):
        x = np.ascontiguousarray(x, np.float32)
        y = np.empty((x.shape[0], self.cfg.d_model), np.float32)
        rep = OrkReport()
        routed = np.ascontiguousarray(routed, np.uint8).reshape(-1)
        shared = None if shared is None else np.ascontiguousarray(shared, np.uint8)
        self._check(self.ref.lib.ref_forward_masked_dense(self.h, x, x.shape[0], routed,
                                                          _opt(shared), threads, y, C.byref(rep)))
        return y, rep

    def forward_sparse(self, x, tau, threads=1):
        x = np.ascontiguousarray(x, np.float32)
        y = np.empty((x.shape[0], self.cfg.d_model), np.float32)
        rep = OrkReport()
        self._check(self.ref.lib.ref_forward_sparse(self.h, x, x.shape[0], tau, threads, y,
                                                    C.byref(rep)))
        return y, rep

    def build_topk_masks(self, x, s, mode=1):
        cfg = self.cfg
        x = np.ascontiguousarray(x, np.float32)
        B = x.shape[0]
        routed = np.empty((B, cfg.top_k, cfg.d_ffn), np.uint8)
        shared = np.empty((B, cfg.d_shared), np.uint8) if (mode == 1 and cfg.has_shared) else None
        self._check(self.ref.lib.ref_build_topk_masks(self.h, x, B, s, mode, routed, _opt(shared)))
        return routed, shared

    def scalar_forward(self, x, routed=None, shared=None):
        x = np.ascontiguousarray(x, np.float32)
        y = np.empty((x.shape[0], self.cfg.d_model), np.float32)
        self._check(self.ref.lib.ref_scalar_forward(self.h, x, x.shape[0], _opt(routed),
                                                    _opt(shared), y))
        return y

    def sweep_cutoff(self, x, targets, retention, mode=1, csv=None):
        """profiler.cpp:152-219 (default metric) -> (points [n][5], cutoff); csv: emit_report path."""
        x = np.ascontiguousarray(x, np.float32)
        t = np.ascontiguousarray(targets, np.float64)
        pts = np.zeros((t.size, 5), np.float64)
        cut = C.c_double()
        self._check(self.ref.lib.ref_sweep_cutoff(self.h, x, x.shape[0], t, t.size, retention, mode,
                                                  pts, C.byref(cut),
                                                  None if csv is None else str(csv).encode()))
        return pts, cut.value

    def calibrate_tau(self, target, calib_batch=16, token_seed=3, sample_cap=1 << 20, seed=4):
        tau = C.c_double()
        self._check(self.ref.lib.ref_calibrate_tau(self.h, target, calib_batch, token_seed,
                                                   sample_cap, seed, C.byref(tau)))
        return tau.value


class RefError(Exception):
    def __init__(self, code, msg):
        super().__init__(f"reference error {code}: {msg}")
        self.code = code
