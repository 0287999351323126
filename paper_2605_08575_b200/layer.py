"""Host-side mirror of the reference layer API over the C ABI (numpy in, numpy out).

Names, argument meaning and error behaviour follow the reference headers
(``proj/include/sparsekit/{model,router,activation,engine,profiler}.hpp``):
``MoEConfig``, ``MoELayerWeights``, ``RouteResult``, ``MaskSet``, ``ForwardReport``,
``SparsityLevel``, ``forward_dense``, ``forward_masked_dense``, ``route``, ``align_dispatch``,
``combine``, ``topk_mask``, ``mask_smallest_magnitudes``, ``build_topk_masks``; plus
``forward_topk_sparse`` -- the fused entry the reference lacks.

Every function runs on the GPU through libsparsekit_b200.so; nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import (FLAG_BF16_H, FLAG_DENSE_DOWN, FLAG_FAST_ROUTER, FLAG_GATHER_DOWN,  # noqa: F401
                   FLAG_FUSED_DECODE, FLAG_NO_FUSED_DECODE, FLAG_NO_PAIRED_BLOCKS, FLAG_PAIRED_BLOCKS, FLAG_NO_PDL, FLAG_SIMT_GATEUP, FLAG_TIME_STAGES,
                   MODE_DENSE, MODE_MASKED, MODE_ROUTE_ONLY, MODE_THRESHOLD, MODE_TOPK, STAGE_NAMES,
                   SkbConfig,
                   SkbForwardArgs,
                   SkbReport)


# ---- error types, proj/include/sparsekit/errors.hpp:12-43 ------------------------------------
class ShapeError(ValueError):
    pass


class ConfigError(ValueError):
    pass


class IndexError_(IndexError):
    pass


class InternalError(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


class FormatError(RuntimeError):
    """File-format violation; carries the byte offset where parsing stopped (errors.hpp:36-43)."""

    def __init__(self, msg: str, offset: int = 0):
        super().__init__(msg)
        self.offset = offset


class IoError(RuntimeError):
    pass


_ERR = {_lib.SKB_ESHAPE: ShapeError, _lib.SKB_ECONFIG: ConfigError, _lib.SKB_EINDEX: IndexError_,
        _lib.SKB_EINTERNAL: InternalError, _lib.SKB_ECUDA: CudaError}


def _check(rc: int) -> None:
    if rc != 0:
        msg = _lib.load().skb_last_error().decode()
        if rc == _lib.SKB_EFORMAT:
            raise FormatError(msg, int(_lib.load().skb_last_error_offset()))
        if rc == _lib.SKB_EIO:
            raise IoError(msg)
        raise _ERR.get(rc, InternalError)(msg)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---- value types ------------------------------------------------------------------------------
@dataclass
class MoEConfig:
    """proj/include/sparsekit/model.hpp:15-29"""
    n_experts: int = 1
    top_k: int = 1
    d_model: int = 1
    d_ffn: int = 1
    has_shared: bool = False
    d_shared: int = 0
    renormalize: bool = True
    align_block: int = 64
    kTile = 64

    def c(self) -> SkbConfig:
        return SkbConfig(self.n_experts, self.top_k, self.d_model, self.d_ffn,
                         int(self.has_shared), self.d_shared, int(self.renormalize),
                         self.align_block)

    def validate(self) -> None:
        cfg = self.c()
        _check(_lib.load().skb_config_validate(C.byref(cfg)))


@dataclass
class SparsityLevel:
    """proj/include/sparsekit/activation.hpp:15-23"""
    s: float = 0.0

    def __post_init__(self):
        if not (0.0 <= self.s <= 1.0):
            raise ConfigError("sparsity must lie in [0, 1]")


@dataclass
class RouteResult:
    """proj/include/sparsekit/router.hpp:20-32"""
    batch: int
    top_k: int
    ids: np.ndarray      # [batch, top_k] int32
    weights: np.ndarray  # [batch, top_k] float32


@dataclass
class DispatchPlan:
    """proj/include/sparsekit/router.hpp:39-44"""
    sorted_token_slots: np.ndarray
    expert_of_block: np.ndarray
    block_size: int
    n_padded: int


@dataclass
class MaskSet:
    """proj/include/sparsekit/engine.hpp:31-34"""
    routed: np.ndarray                      # B*K*d_ffn uint8, slot-major per token
    shared: Optional[np.ndarray] = None     # B*d_shared uint8 or None (dense shared expert)


@dataclass
class MacCounter:
    gate_macs: int = 0
    up_macs: int = 0
    down_macs: int = 0
    other_macs: int = 0

    def total(self) -> int:
        return self.gate_macs + self.up_macs + self.down_macs + self.other_macs


@dataclass
class ForwardReport:
    """proj/include/sparsekit/engine.hpp:19-27"""
    outputs: np.ndarray
    macs: MacCounter
    active_neurons_total: int = 0
    achieved_routed_sparsity: float = 0.0
    tiles_total: int = 0
    tiles_skipped: int = 0
    path_used: int = 0
    routes: Optional[RouteResult] = None
    masks: Optional[MaskSet] = None
    h_routed: Optional[np.ndarray] = None
    h_shared: Optional[np.ndarray] = None
    stage_ms: Optional[dict] = None
    launches: int = 0


SWEEP_ROUTED_ONLY, SWEEP_ROUTED_AND_SHARED = 0, 1


class MoELayerWeights:
    """Device-resident counterpart of MoELayerWeights (proj/include/sparsekit/model.hpp:34-43).

    Holds the opaque ``skb_layer*``; the bf16 weight image lives in HBM for the object's life.
    """

    def __init__(self, config: MoEConfig, handle: int):
        self.config = config
        self._h = C.c_void_p(handle)

    @classmethod
    def from_arrays(cls, config: MoEConfig, router, gate, up, down_t, shared_gate=None,
                    shared_up=None, shared_down_t=None, device: int = 0) -> "MoELayerWeights":
        """gate/up/down_t: [E, N, D] arrays or sequences of E [N, D] matrices (fp32)."""
        L = _lib.load()
        config.validate()
        E, N, D, S = config.n_experts, config.d_ffn, config.d_model, config.d_shared
        keep = []

        def mats(m):
            out = []
            for e in range(E):
                a = np.ascontiguousarray(m[e], dtype=np.float32)
                if a.shape != (N, D):
                    raise ShapeError(f"expert matrix must be {N}x{D}, got {a.shape}")
                keep.append(a)
                out.append(a.ctypes.data)
            return (C.c_void_p * E)(*out)

        r = np.ascontiguousarray(router, dtype=np.float32)
        if r.shape != (E, D):
            raise ShapeError(f"router must be {E}x{D}, got {r.shape}")
        g, u, d = mats(gate), mats(up), mats(down_t)
        sh = [None, None, None]
        if config.has_shared:
            for i, m in enumerate((shared_gate, shared_up, shared_down_t)):
                if m is None:
                    raise ShapeError("shared matrices missing while has_shared is set")
                sh[i] = np.ascontiguousarray(m, dtype=np.float32)
                if sh[i].shape != (S, D):
                    raise ShapeError(f"shared matrix must be {S}x{D}, got {sh[i].shape}")
        cfg = config.c()
        h = C.c_void_p()
        _check(L.skb_layer_create(C.byref(cfg), _ptr(r), g, u, d, _ptr(sh[0]), _ptr(sh[1]),
                                  _ptr(sh[2]), device, C.byref(h)))
        return cls(config, h.value)

    @classmethod
    def load(cls, path, device: int = 0) -> "MoELayerWeights":
        """load_weights (proj/src/model.cpp:218-282) straight into the device image: the "MOE1"
        file is mapped and converted expert by expert, no host copy of the fp32 weights.
        Raises FormatError (with .offset) / IoError like the reference."""
        cfg = SkbConfig()
        h = C.c_void_p()
        _check(_lib.load().skb_layer_load(str(path).encode(), device, C.byref(cfg), C.byref(h)))
        config = MoEConfig(cfg.n_experts, cfg.top_k, cfg.d_model, cfg.d_ffn, bool(cfg.has_shared),
                           cfg.d_shared, bool(cfg.renormalize), cfg.align_block)
        return cls(config, h.value)

    @classmethod
    def generate_synthetic(cls, config: MoEConfig, seed: int, scale: float,
                           device: int = 0) -> "MoELayerWeights":
        """generate_synthetic, proj/src/model.cpp:129-166, evaluated on the device."""
        L = _lib.load()
        cfg = config.c()
        h = C.c_void_p()
        _check(L.skb_layer_create_synthetic(C.byref(cfg), seed & (2 ** 64 - 1), scale, device,
                                            C.byref(h)))
        return cls(config, h.value)

    @classmethod
    def synthetic_slice(cls, full: MoEConfig, seed: int, scale: float, e_lo: int = 0,
                        e_hi: int = 0, shared: bool = False, device: int = 0) -> "MoELayerWeights":
        """Expert-parallel slice of generate_synthetic(full, seed, scale): experts [e_lo, e_hi)
        as a top-1 layer without shared expert, or (shared=True) the shared expert as a
        one-expert layer.  Carries the full router for route_only()."""
        cfg = full.c()
        h = C.c_void_p()
        _check(_lib.load().skb_layer_create_synthetic_slice(
            C.byref(cfg), seed & (2 ** 64 - 1), scale, e_lo, e_hi, 1 if shared else 0, device,
            C.byref(h)))
        if shared:
            loc = MoEConfig(1, 1, full.d_model, full.d_shared, False, 0, full.renormalize,
                            full.align_block)
        else:
            loc = MoEConfig(e_hi - e_lo, 1, full.d_model, full.d_ffn, False, 0, full.renormalize,
                            full.align_block)
        out = cls(loc, h.value)
        out.route_shape = (full.n_experts, full.top_k)
        return out

    def set_router(self, router, top_k: int, renormalize: bool = True) -> None:
        """Attach the full model's router to an expert-parallel slice built from arrays."""
        r = np.ascontiguousarray(router, dtype=np.float32)
        if r.ndim != 2 or r.shape[1] != self.config.d_model:
            raise ShapeError(f"router must be E x {self.config.d_model}, got {r.shape}")
        _check(_lib.load().skb_layer_set_router(self._h, _ptr(r), r.shape[0], top_k,
                                                int(renormalize)))
        self.route_shape = (r.shape[0], top_k)

    def reserve(self, max_batch: int) -> None:
        _check(_lib.load().skb_layer_reserve(self._h, max_batch))

    @property
    def weight_bytes(self) -> int:
        return int(_lib.load().skb_layer_weight_bytes(self._h))

    def stage_times(self) -> list:
        """Milliseconds per stage (STAGE_NAMES order) of the last FLAG_TIME_STAGES forward."""
        ms = (C.c_float * _lib.N_STAGES)()
        _check(_lib.load().skb_layer_stage_times(self._h, ms))
        return [float(v) for v in ms]

    def last_launches(self) -> int:
        return int(_lib.load().skb_layer_last_launches(self._h))

    def close(self) -> None:
        if self._h:
            _lib.load().skb_layer_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- device-pointer entry for the benchmark's value leg and for stream capture --
    def forward_device(self, x_ptr: int, y_ptr: int, batch: int, mode: int = MODE_TOPK,
                       s_routed: float = 0.0, s_shared: float = 0.0, flags: int = 0,
                       stream: int = 0, ids_in_ptr: int = 0, weights_in_ptr: int = 0,
                       tau: float = 0.0) -> None:
        """All pointers are device pointers.  ids_in_ptr: external routing ([batch][top_k] int32
        expert ids of this layer); weights_in_ptr 0 => un-weighted slot outputs."""
        a = SkbForwardArgs()
        a.batch, a.mode, a.flags = batch, mode, flags
        a.s_routed, a.s_shared = s_routed, s_shared
        a.tau = tau  # MODE_THRESHOLD only
        a.x, a.y = x_ptr, y_ptr
        a.ids_in, a.weights_in = ids_in_ptr or None, weights_in_ptr or None
        _check(_lib.load().skb_layer_forward_device(self._h, C.byref(a), C.c_void_p(stream), None))

    def forward_device_rows(self, x_ptr: int, y_rows_ptr: int, batch: int, mode: int = MODE_TOPK,
                            s_routed: float = 0.0, s_shared: float = 0.0, flags: int = 0,
                            stream: int = 0, ids_in_ptr: int = 0, weights_in_ptr: int = 0) -> None:
        """forward_device with one destination per output row: y_rows_ptr is a device array of
        `batch` device pointers (d_model floats each)."""
        a = SkbForwardArgs()
        a.batch, a.mode, a.flags = batch, mode, flags
        a.s_routed, a.s_shared = s_routed, s_shared
        a.x = x_ptr
        a.ids_in, a.weights_in = ids_in_ptr or None, weights_in_ptr or None
        _check(_lib.load().skb_layer_forward_device_rows(self._h, C.byref(a), C.c_void_p(stream),
                                                         C.c_void_p(y_rows_ptr)))

    def route_device(self, x_ptr: int, ids_out_ptr: int, weights_out_ptr: int, batch: int,
                     flags: int = 0, stream: int = 0) -> None:
        """SKB_MODE_ROUTE_ONLY on device pointers: x [batch][D] -> ids / weights [batch][K_route]."""
        a = SkbForwardArgs()
        a.batch, a.mode, a.flags = batch, MODE_ROUTE_ONLY, flags
        a.x = x_ptr
        a.ids_out, a.weights_out = ids_out_ptr, weights_out_ptr
        _check(_lib.load().skb_layer_forward_device(self._h, C.byref(a), C.c_void_p(stream), None))


def _forward(w: MoELayerWeights, x: np.ndarray, mode: int, s_routed=0.0, s_shared=0.0,
             masks: Optional[MaskSet] = None, flags: int = 0, capture: bool = False,
             y_out: Optional[np.ndarray] = None, tau: float = 0.0,
             slot_n_off=None) -> ForwardReport:
    L = _lib.load()
    cfg = w.config
    x = np.ascontiguousarray(x, dtype=np.float32)
    if x.ndim != 2 or x.shape[1] != cfg.d_model:
        # engine.cpp:98-101
        raise ShapeError(f"forward: tokens are B x {x.shape[-1] if x.ndim else 0}, model expects "
                         f"d_model={cfg.d_model}")
    B, K, N, S = x.shape[0], cfg.top_k, cfg.d_ffn, cfg.d_shared
    y = y_out if y_out is not None else np.empty((B, cfg.d_model), np.float32)
    a = SkbForwardArgs()
    a.batch, a.mode, a.flags = B, mode, flags
    a.s_routed, a.s_shared = float(s_routed), float(s_shared)
    a.tau = float(tau)
    a.x, a.y = x.ctypes.data, y.ctypes.data
    keep = [x, y]
    if slot_n_off is not None:
        sn = np.ascontiguousarray(slot_n_off, dtype=np.int32).reshape(-1)
        if sn.size != K:
            raise ShapeError(f"per-slot counts: need top_k={K} entries, got {sn.size}")
        a.slot_n_off = sn.ctypes.data
        keep.append(sn)
    if mode == MODE_MASKED:
        r = np.ascontiguousarray(masks.routed, dtype=np.uint8).reshape(-1)
        a.routed_mask_in, a.routed_mask_len = r.ctypes.data, r.size
        keep.append(r)
        if masks.shared is not None and np.size(masks.shared) > 0:
            sm = np.ascontiguousarray(masks.shared, dtype=np.uint8).reshape(-1)
            a.shared_mask_in, a.shared_mask_len = sm.ctypes.data, sm.size
            keep.append(sm)
    cap = {}
    if capture:
        cap["ids"] = np.empty((B, K), np.int32)
        cap["weights"] = np.empty((B, K), np.float32)
        cap["routed"] = np.empty((B, K, N), np.uint8)
        cap["h_routed"] = np.empty((B, K, N), np.float32)
        a.ids_out, a.weights_out = cap["ids"].ctypes.data, cap["weights"].ctypes.data
        a.routed_mask_out, a.h_routed_out = cap["routed"].ctypes.data, cap["h_routed"].ctypes.data
        if cfg.has_shared:
            cap["shared"] = np.empty((B, S), np.uint8)
            cap["h_shared"] = np.empty((B, S), np.float32)
            a.shared_mask_out, a.h_shared_out = cap["shared"].ctypes.data, cap["h_shared"].ctypes.data
    rep = SkbReport()
    _check(L.skb_layer_forward(w._h, C.byref(a), C.byref(rep)))
    out = ForwardReport(
        outputs=y, macs=MacCounter(rep.gate_macs, rep.up_macs, rep.down_macs, rep.other_macs),
        active_neurons_total=rep.active_neurons_total,
        achieved_routed_sparsity=rep.achieved_routed_sparsity, tiles_total=rep.tiles_total,
        tiles_skipped=rep.tiles_skipped, path_used=rep.path_used,
        launches=L.skb_layer_last_launches(w._h))
    if capture:
        out.routes = RouteResult(B, K, cap["ids"], cap["weights"])
        out.masks = MaskSet(cap["routed"], cap.get("shared"))
        out.h_routed, out.h_shared = cap["h_routed"], cap.get("h_shared")
    if flags & FLAG_TIME_STAGES:
        ms = (C.c_float * _lib.N_STAGES)()
        _check(L.skb_layer_stage_times(w._h, ms))
        out.stage_ms = dict(zip(STAGE_NAMES, [float(v) for v in ms]))
    return out


def route_tokens(w: MoELayerWeights, x) -> RouteResult:
    """route_logits + route (engine.cpp:121-122) with the router attached to `w` (its own, or
    the full model's on an expert-parallel slice); host buffers."""
    L = _lib.load()
    x = np.ascontiguousarray(x, dtype=np.float32)
    if x.ndim != 2 or x.shape[1] != w.config.d_model:
        raise ShapeError(f"route_tokens: tokens must be B x {w.config.d_model}")
    E, K = getattr(w, "route_shape", (w.config.n_experts, w.config.top_k))
    B = x.shape[0]
    ids = np.empty((B, K), np.int32)
    wts = np.empty((B, K), np.float32)
    a = SkbForwardArgs()
    a.batch, a.mode = B, MODE_ROUTE_ONLY
    a.x = x.ctypes.data
    a.ids_out, a.weights_out = ids.ctypes.data, wts.ctypes.data
    _check(L.skb_layer_forward(w._h, C.byref(a), None))
    return RouteResult(B, K, ids, wts)


def forward_routed(w: MoELayerWeights, x, ids, weights=None, s_routed: float = 0.0, *,
                   flags: int = 0) -> np.ndarray:
    """External routing (the owner-rank half of expert parallelism): row t of x goes through
    experts ids[t, :] of THIS layer with combine weights `weights` (None = 1.0, i.e. the
    un-weighted slot output for top_k = 1), top-k selection at s_routed."""
    L = _lib.load()
    cfg = w.config
    x = np.ascontiguousarray(x, dtype=np.float32)
    ids = np.ascontiguousarray(ids, dtype=np.int32).reshape(x.shape[0], cfg.top_k)
    y = np.empty((x.shape[0], cfg.d_model), np.float32)
    a = SkbForwardArgs()
    a.batch, a.mode, a.flags = x.shape[0], MODE_TOPK, flags
    a.s_routed, a.s_shared = float(s_routed), 0.0
    a.x, a.y, a.ids_in = x.ctypes.data, y.ctypes.data, ids.ctypes.data
    keep = [x, y, ids]
    if weights is not None:
        wt = np.ascontiguousarray(weights, dtype=np.float32).reshape(ids.shape)
        a.weights_in = wt.ctypes.data
        keep.append(wt)
    _check(L.skb_layer_forward(w._h, C.byref(a), None))
    return y


def forward_dense(w: MoELayerWeights, x, threads: int = 1, *, flags: int = 0,
                  capture: bool = False) -> ForwardReport:
    """engine.hpp:38-39.  `threads` is accepted for signature parity and ignored."""
    return _forward(w, x, MODE_DENSE, flags=flags, capture=capture)


def forward_masked_dense(w: MoELayerWeights, x, masks: MaskSet, threads: int = 1, *,
                         flags: int = 0, capture: bool = False) -> ForwardReport:
    """engine.hpp:43-44: dense execution with h zeroed where masked (here: rows not gathered)."""
    return _forward(w, x, MODE_MASKED, masks=masks, flags=flags, capture=capture)


def forward_topk_sparse(w: MoELayerWeights, x, s_routed: SparsityLevel,
                        s_shared: Optional[SparsityLevel] = None, threads: int = 1, *,
                        flags: int = 0, capture: bool = False, y_out=None) -> ForwardReport:
    """== forward_masked_dense(w, x, build_topk_masks(w, x, s, mode)) with the selection done on
    the device and masked W_down rows skipped.  s_shared=None => shared expert stays dense
    (SweepMode::kRoutedOnly); pass the same level for kRoutedAndShared."""
    ss = 0.0 if s_shared is None else s_shared.s
    return _forward(w, x, MODE_TOPK, s_routed=s_routed.s, s_shared=ss, flags=flags,
                    capture=capture, y_out=y_out)


def forward_sparse(w: MoELayerWeights, x, threshold: float, threads: int = 1, *, flags: int = 0,
                   capture: bool = False, y_out=None) -> ForwardReport:
    """engine.hpp:46-51 / engine.cpp:229-369: a routed neuron is kept iff |silu(gate)| >= threshold
    (threshold_mask, activation.cpp:62-72); the shared expert stays dense; the report carries
    the reference's 64-neuron tile accounting.  `threads` is accepted and ignored."""
    if not (threshold >= 0.0):  # also rejects NaN, like the reference's !(t >= 0)
        raise ConfigError("forward_sparse: threshold must be >= 0")
    return _forward(w, x, MODE_THRESHOLD, flags=flags, capture=capture, y_out=y_out,
                    tau=float(threshold))


# ---- "MOE1" weight files (model.hpp:59-63, model.cpp:180-282) ---------------------------------
def weight_file_size(config: MoEConfig) -> int:
    cfg = config.c()
    return int(_lib.load().skb_weight_file_size(C.byref(cfg)))


def save_weights(config: MoEConfig, path, router, gate, up, down_t, shared_gate=None,
                 shared_up=None, shared_down_t=None) -> None:
    """save_weights, model.cpp:190-216 (host arrays in, file out; validates the config first)."""
    config.validate()
    E = config.n_experts
    keep = []

    def mats(m):
        ptrs = []
        for e in range(E):
            a = np.ascontiguousarray(m[e], dtype=np.float32)
            keep.append(a)
            ptrs.append(a.ctypes.data)
        return (C.c_void_p * E)(*ptrs)

    r = np.ascontiguousarray(router, dtype=np.float32)
    sh = [None if m is None else np.ascontiguousarray(m, dtype=np.float32)
          for m in (shared_gate, shared_up, shared_down_t)]
    cfg = config.c()
    _check(_lib.load().skb_save_weights(C.byref(cfg), _ptr(r), mats(gate), mats(up), mats(down_t),
                                        _ptr(sh[0]), _ptr(sh[1]), _ptr(sh[2]), str(path).encode()))


# ---- neuron budgets (budget.hpp, budget.cpp) -------------------------------------------------
@dataclass
class BudgetRatios:
    """Distribution ratios of the three router-weight groups (budget.hpp:15-20)."""
    r0: float = 1.0
    r1: float = 1.0
    r2: float = 1.0


@dataclass
class ExpertGroups:
    """Slot indices by router weight: g0 the floor(K/3) heaviest, g1 the next floor(K/3), g2 the
    rest (budget.hpp:22-28)."""
    g0: list = field(default_factory=list)
    g1: list = field(default_factory=list)
    g2: list = field(default_factory=list)


def group_experts(topk_weights) -> ExpertGroups:
    """budget.cpp:15-35: stable descending order, so equal weights keep slot order."""
    wts = [float(v) for v in np.asarray(topk_weights, np.float32).reshape(-1)]
    k = len(wts)
    if k < 1:
        raise ConfigError("group_experts: need at least one slot")
    order = sorted(range(k), key=lambda i: -wts[i])  # sorted() is stable
    third = k // 3
    return ExpertGroups(order[:third], order[third:2 * third], order[2 * third:])


def allocate_budget(top_k: int, d_ffn: int, s_active: float, groups: ExpertGroups,
                    ratios: BudgetRatios):
    """budget.cpp:37-76: per-slot survivor counts for a budget of s_active * K * d_ffn neurons,
    n_e = clamp(floor(budget * r_x / sum_x(r_x |g_x|) + 0.5), 0, d_ffn) for the slots of g_x."""
    import math
    if not (0.0 <= s_active <= 1.0):
        raise ConfigError("allocate_budget: s_active must lie in [0, 1]")
    if ratios.r0 < 0.0 or ratios.r1 < 0.0 or ratios.r2 < 0.0:
        raise ConfigError("allocate_budget: ratios must be non-negative")
    denom = (ratios.r0 * float(len(groups.g0)) + ratios.r1 * float(len(groups.g1)) +
             ratios.r2 * float(len(groups.g2)))
    if not (denom > 0.0):
        raise ConfigError("allocate_budget: no ratio mass on non-empty groups")
    budget = s_active * top_k * d_ffn
    counts = [0] * top_k
    assigned = 0
    for members, ratio in ((groups.g0, ratios.r0), (groups.g1, ratios.r1), (groups.g2, ratios.r2)):
        n_e = min(max(int(math.floor(budget * ratio / denom + 0.5)), 0), d_ffn)
        for slot in members:
            if slot < 0 or slot >= top_k:
                raise IndexError_(f"allocate_budget: slot {slot} outside [0, {top_k})")
            counts[slot] = n_e
            assigned += 1
    if assigned != top_k:
        raise ConfigError("allocate_budget: groups must partition the slots")
    return counts


def apply_budget(h, keep_count: int) -> np.ndarray:
    """budget.cpp:78-85: keep the keep_count largest-|h| entries of one slot (on the device)."""
    n = int(np.size(h))
    if keep_count < 0 or keep_count > n:
        raise ConfigError("apply_budget: keep_count outside [0, N]")
    return mask_smallest_magnitudes(h, n - keep_count)


def forward_budget_sparse(w: MoELayerWeights, x, sparsity: float, ratios: BudgetRatios,
                          mask_shared: bool = False, *, flags: int = 0,
                          capture: bool = False) -> ForwardReport:
    """The reference CLI's budget analysis mode (tools/main.cpp:271-345) as one device forward:
    per routing slot, apply_budget with the count allocate_budget gives its router-weight group
    (slots are in descending router weight, so slot s has rank s for every token); with
    mask_shared the shared expert gets a plain top-k mask at `sparsity` (R+S).  Numerically
    forward_masked_dense on those masks, with masked W_down rows skipped."""
    cfg = w.config
    lvl = SparsityLevel(sparsity)
    groups = group_experts(np.arange(cfg.top_k, 0, -1, dtype=np.float32))  # rank = slot
    counts = allocate_budget(cfg.top_k, cfg.d_ffn, 1.0 - lvl.s, groups, ratios)
    n_off_slots = [cfg.d_ffn - c for c in counts]
    return _forward(w, x, MODE_TOPK, s_routed=lvl.s,
                    s_shared=lvl.s if (mask_shared and cfg.has_shared) else 0.0, flags=flags,
                    capture=capture, slot_n_off=n_off_slots)


# ---- the dense/sparse switch (engine.hpp:52-89, engine.cpp:371-420) ---------------------------
SPARSE_ALWAYS = (1 << 64) - 1  # SwitchTable::kSparseAlways


@dataclass
class SwitchTable:
    """Batches of at least `tipping_batch` take the dense path (engine.hpp:54-61)."""
    tipping_batch: int = SPARSE_ALWAYS

    def use_dense(self, batch: int) -> bool:
        return batch >= self.tipping_batch


class Stopwatch:
    """Injectable monotonic clock in milliseconds (engine.hpp:63-69)."""

    def now_ms(self) -> float:
        raise NotImplementedError


class SteadyStopwatch(Stopwatch):
    """Host wall clock; the forward entry points return after their device work and the copy
    back, so host time is layer time as the caller sees it."""

    def now_ms(self) -> float:
        return time.perf_counter() * 1e3


def generate_tokens(batch: int, d_model: int, seed: int) -> np.ndarray:
    """model.cpp:168-178: standard normals by Box-Muller over SplitMix64 (host libm)."""
    x = np.empty((max(batch, 0), max(d_model, 0)), np.float32)
    _check(_lib.load().skb_generate_tokens(batch, d_model, seed & ((1 << 64) - 1), _ptr(x)))
    return x


def _median(values):
    v = sorted(values)
    n = len(v)
    return v[n // 2] if n % 2 else 0.5 * (v[n // 2 - 1] + v[n // 2])


def profile_tipping(w: MoELayerWeights, threshold: float, batch_grid, repetitions: int = 5,
                    clock: Optional[Stopwatch] = None, token_seed: int = 0) -> SwitchTable:
    """engine.cpp:371-412: the smallest batch of the ascending grid whose dense median is at or
    below the sparse median, else kSparseAlways.  Per grid point `repetitions` sparse runs then
    `repetitions` dense runs, one now_ms() before and after each."""
    grid = [int(b) for b in batch_grid]
    if not grid:
        raise ConfigError("profile_tipping: empty batch grid")
    for i, b in enumerate(grid):
        if b < 1 or (i > 0 and b <= grid[i - 1]):
            raise ConfigError("profile_tipping: grid must be ascending, >= 1")
    if repetitions < 1:
        raise ConfigError("profile_tipping: repetitions must be >= 1")
    clock = clock or SteadyStopwatch()
    for gi, batch in enumerate(grid):
        tokens = generate_tokens(batch, w.config.d_model, token_seed + gi)
        sparse_ms, dense_ms = [], []
        for _ in range(repetitions):
            t0 = clock.now_ms()
            forward_sparse(w, tokens, threshold)
            sparse_ms.append(clock.now_ms() - t0)
        for _ in range(repetitions):
            t0 = clock.now_ms()
            forward_dense(w, tokens)
            dense_ms.append(clock.now_ms() - t0)
        if _median(dense_ms) <= _median(sparse_ms):
            return SwitchTable(batch)
    return SwitchTable(SPARSE_ALWAYS)


def step(w: MoELayerWeights, x, threshold: float, table: SwitchTable,
         threads: int = 1) -> ForwardReport:
    """engine.cpp:414-420: forward_dense when the table says so for this batch, else
    forward_sparse."""
    rows = np.asarray(x).shape[0]
    if table.use_dense(rows):
        return forward_dense(w, x, threads)
    return forward_sparse(w, x, threshold, threads)


def build_topk_masks(w: MoELayerWeights, tokens, s: SparsityLevel,
                     mode: int = SWEEP_ROUTED_AND_SHARED) -> MaskSet:
    """profiler.hpp:71-72 / profiler.cpp:101-150."""
    shared = s if (mode == SWEEP_ROUTED_AND_SHARED and w.config.has_shared) else None
    rep = forward_topk_sparse(w, tokens, s, shared, capture=True)
    return MaskSet(rep.masks.routed, rep.masks.shared if shared is not None else None)


# ---- quality sweep and its report file (profiler.hpp:38-83) ------------------------------------
REPORT_HEADER = "target,achieved_total,achieved_routed,quality,rel_error,path"


@dataclass
class SweepPoint:
    """profiler.hpp:49-56"""
    target: float = 0.0
    achieved_total: float = 0.0
    achieved_routed: float = 0.0
    quality: float = 0.0
    rel_error: float = 0.0
    path: str = ""   # "R" or "R+S"


@dataclass
class SweepResult:
    """profiler.hpp:58-61"""
    points: list = field(default_factory=list)
    cutoff: float = 0.0


def mean_relative_error(outputs, dense_outputs) -> float:
    """profiler.cpp:76-99: mean over tokens of ||y - y_dense|| / ||y_dense|| in double; tokens
    whose dense norm is below 1e-12 are left out; no token left: 0."""
    y = np.asarray(outputs, np.float64)
    d = np.asarray(dense_outputs, np.float64)
    if y.shape != d.shape:
        raise ShapeError("mean_relative_error: shape mismatch")
    ref = np.sqrt((d * d).sum(axis=1))
    err = np.sqrt(((y - d) ** 2).sum(axis=1))
    ok = ref >= 1e-12
    return float((err[ok] / ref[ok]).mean()) if ok.any() else 0.0


def sweep_cutoff(w: MoELayerWeights, eval_tokens, targets: Sequence[float], retention: float,
                 mode: int = SWEEP_ROUTED_AND_SHARED, metric=None) -> SweepResult:
    """profiler.hpp:66-69 / profiler.cpp:152-219: the masked-dense quality sweep, every point one
    fused top-k forward on the device (selection inside the layer instead of build_topk_masks +
    forward_masked_dense; same masks, same outputs)."""
    targets = [float(t) for t in targets]
    if not targets:
        raise ConfigError("sweep_cutoff: no targets")
    for i, t in enumerate(targets):
        if not (0.0 <= t <= 1.0):
            raise ConfigError("sweep_cutoff: targets must lie in [0, 1]")
        if i > 0 and not (t > targets[i - 1]):
            raise ConfigError("sweep_cutoff: targets must be strictly increasing")
    if not (0.0 < retention <= 1.0):
        raise ConfigError("sweep_cutoff: retention must lie in (0, 1]")
    cfg = w.config
    x = np.ascontiguousarray(eval_tokens, np.float32)
    dense = forward_dense(w, x)
    with_shared = mode == SWEEP_ROUTED_AND_SHARED and cfg.has_shared
    label = "R" if mode == SWEEP_ROUTED_ONLY else "R+S"
    B = x.shape[0]

    def evaluate(target: float) -> SweepPoint:
        lvl = SparsityLevel(target)
        rep = forward_topk_sparse(w, x, lvl, lvl if with_shared else None, capture=True)
        rel = mean_relative_error(rep.outputs, dense.outputs)
        masked_shared = int((rep.masks.shared == 0).sum()) if with_shared else 0
        routed_neurons = B * cfg.top_k * cfg.d_ffn
        masked_routed = routed_neurons - rep.active_neurons_total
        per_token = cfg.top_k * cfg.d_ffn + cfg.d_shared
        return SweepPoint(target=target,
                          achieved_total=(masked_routed + masked_shared) / float(B * per_token),
                          achieved_routed=rep.achieved_routed_sparsity,
                          quality=metric(rep.outputs, dense.outputs) if metric else 1.0 - rel,
                          rel_error=rel, path=label)

    baseline = evaluate(0.0)  # the quality floor always refers to the zero-sparsity point
    res = SweepResult()
    for t in targets:
        res.points.append(baseline if t == 0.0 else evaluate(t))
    floor = retention * baseline.quality
    for p in res.points:
        if p.quality >= floor:
            res.cutoff = max(res.cutoff, p.target)
    return res


def emit_report(result: SweepResult, path) -> None:
    """profiler.hpp:79-82 / profiler.cpp:221-243: CSV, 9 significant digits, '# cutoff=' trailer."""
    try:
        with open(path, "w", newline="") as f:
            f.write(REPORT_HEADER + "\n")
            for p in result.points:
                f.write("%.9g,%.9g,%.9g,%.9g,%.9g,%s\n" % (p.target, p.achieved_total,
                                                           p.achieved_routed, p.quality,
                                                           p.rel_error, p.path))
            if result.points:
                f.write("# cutoff=%.9g\n" % result.cutoff)
    except OSError as exc:
        raise IoError(f"cannot open for writing: {path}") from exc


def read_report(path) -> SweepResult:
    """profiler.cpp:245-286; FormatError carries the byte offset of the offending line."""
    try:
        with open(path, "r", newline="") as f:
            text = f.read()
    except OSError as exc:
        raise IoError(f"cannot open for reading: {path}") from exc
    lines = text.split("\n")
    if text.endswith("\n"):
        lines = lines[:-1]
    if not lines or lines[0] != REPORT_HEADER:
        raise FormatError("missing report header", 0)
    offset = len(lines[0]) + 1
    res = SweepResult()
    for line in lines[1:]:
        if line.startswith("# cutoff="):
            res.cutoff = _strtod(line[9:])
        elif line:
            parts = line.split(",", 5)
            if len(parts) < 5:
                raise FormatError("short report row", offset)
            if len(parts) < 6:
                raise FormatError("report row missing path", offset)
            vals = [_strtod(v) for v in parts[:5]]
            res.points.append(SweepPoint(*vals, path=parts[5]))
        offset += len(line) + 1
    return res


def _strtod(text: str) -> float:
    """strtod semantics: the longest numeric prefix, 0.0 when there is none."""
    import re
    m = re.match(r"\s*[-+]?(?:inf(?:inity)?|nan|(?:\d+\.?\d*|\.\d+)(?:[eE][-+]?\d+)?)", text, re.I)
    return float(m.group(0)) if m else 0.0


# ---- stage functions --------------------------------------------------------------------------
def route(logits, top_k: int, renormalize: bool) -> RouteResult:
    """router.hpp:34 / router.cpp:13-68."""
    logits = np.ascontiguousarray(logits, dtype=np.float32)
    if logits.ndim != 2:
        raise ShapeError("route: logits must be batch x n_experts")
    B, E = logits.shape
    ids = np.empty((max(B, 0), max(top_k, 0)), np.int32)
    wts = np.empty((max(B, 0), max(top_k, 0)), np.float32)
    _check(_lib.load().skb_route(_ptr(logits), B, E, top_k, int(renormalize), _ptr(ids), _ptr(wts)))
    return RouteResult(B, top_k, ids, wts)


def align_dispatch(r: RouteResult, n_experts: int, block: int) -> DispatchPlan:
    """router.hpp:46-47 / router.cpp:70-107."""
    ids = np.ascontiguousarray(r.ids, dtype=np.int32).reshape(-1)
    cap = ids.size + n_experts * max(block - 1, 0) + 1
    sorted_out = np.empty(cap, np.int32)
    eob = np.empty(cap, np.int32)
    n_padded, n_blocks = C.c_int32(), C.c_int32()
    _check(_lib.load().skb_align_dispatch(_ptr(ids), r.batch, r.top_k, n_experts, block,
                                          _ptr(sorted_out), _ptr(eob), C.byref(n_padded),
                                          C.byref(n_blocks)))
    return DispatchPlan(sorted_out[:n_padded.value].copy(), eob[:n_blocks.value].copy(), block,
                        n_padded.value)


def combine(slot_outputs, r: RouteResult, d_model: int) -> np.ndarray:
    """router.hpp:52-53 / router.cpp:109-132."""
    so = np.ascontiguousarray(slot_outputs, dtype=np.float32).reshape(-1)
    if so.size != r.batch * r.top_k * d_model:
        raise InternalError(f"combine: got {so.size} values, expected {r.batch * r.top_k * d_model}")
    wts = np.ascontiguousarray(r.weights, dtype=np.float32)
    y = np.empty((r.batch, d_model), np.float32)
    _check(_lib.load().skb_combine(_ptr(so), _ptr(wts), r.batch, r.top_k, d_model, _ptr(y)))
    return y


def mask_smallest_magnitudes(h, count) -> np.ndarray:
    """activation.hpp:35-36.  h: [n] or [rows, n]; count: int or per-row sequence."""
    h = np.ascontiguousarray(h, dtype=np.float32)
    one = h.ndim == 1
    h2 = h.reshape(1, -1) if one else h
    rows, n = h2.shape
    counts = np.ascontiguousarray(np.broadcast_to(np.asarray(count, np.int32), (rows,)))
    mask = np.empty((rows, n), np.uint8)
    _check(_lib.load().skb_mask_smallest(_ptr(h2), rows, n, _ptr(counts), _ptr(mask), None, None))
    return mask[0] if one else mask


def select_survivors(h, count):
    """Like mask_smallest_magnitudes but also returns the ascending survivor lists the
    down-projection consumes: (mask, kept_idx padded with -1, kept_count)."""
    h2 = np.ascontiguousarray(h, dtype=np.float32)
    rows, n = h2.shape
    counts = np.ascontiguousarray(np.broadcast_to(np.asarray(count, np.int32), (rows,)))
    mask = np.empty((rows, n), np.uint8)
    kidx = np.empty((rows, n), np.int32)
    kcnt = np.empty(rows, np.int32)
    _check(_lib.load().skb_mask_smallest(_ptr(h2), rows, n, _ptr(counts), _ptr(mask), _ptr(kidx),
                                         _ptr(kcnt)))
    return mask, kidx, kcnt


def topk_mask(h, s: SparsityLevel) -> np.ndarray:
    """activation.hpp:39 / activation.cpp:54-60."""
    h = np.ascontiguousarray(h, dtype=np.float32)
    one = h.ndim == 1
    h2 = h.reshape(1, -1) if one else h
    mask = np.empty(h2.shape, np.uint8)
    _check(_lib.load().skb_topk_mask(_ptr(h2), h2.shape[0], h2.shape[1], s.s, _ptr(mask)))
    return mask[0] if one else mask


K_PAD_INDEX = -1  # activation.hpp: kPadIndex


@dataclass
class ActiveIndexRow:
    """activation.hpp:41-49: flat[capacity] of expert * d_ffn + neuron, padded with -1."""
    flat: np.ndarray
    active_per_slot: np.ndarray
    total_active: int


def threshold_mask(gate_out, threshold: float) -> np.ndarray:
    """activation.hpp:52 / activation.cpp:62-72: keep iff |silu(g)| >= threshold."""
    g = np.ascontiguousarray(gate_out, dtype=np.float32)
    mask = np.empty(g.shape, np.uint8)
    rows = 1 if g.ndim <= 1 else int(np.prod(g.shape[:-1]))
    n = g.shape[-1] if g.ndim else 1
    _check(_lib.load().skb_threshold_mask(_ptr(g) if g.size else None, rows, n, float(threshold),
                                          _ptr(mask) if g.size else None))
    return mask


def default_capacity(top_k: int, d_ffn: int) -> int:
    """activation.cpp:74-77."""
    return int(_lib.load().skb_default_capacity(top_k, d_ffn))


def compact_active(masks, topk_ids, d_ffn: int, capacity: int):
    """activation.hpp:58-60 / activation.cpp:79-114.  masks: [slots * d_ffn] with topk_ids [slots]
    -> one ActiveIndexRow; masks [batch, slots, d_ffn] with topk_ids [batch, slots] -> a list."""
    masks = np.ascontiguousarray(masks, dtype=np.uint8)
    ids = np.ascontiguousarray(topk_ids, dtype=np.int32)
    one = ids.ndim == 1
    ids2 = ids.reshape(1, -1) if one else ids
    batch, K = ids2.shape
    cap = max(int(capacity), 0)
    flat = np.empty((batch, cap), np.int32)
    per = np.empty((batch, K), np.int32)
    tot = np.empty(batch, np.int32)
    _check(_lib.load().skb_compact_active(_ptr(masks) if masks.size else None, masks.size,
                                          _ptr(ids2) if ids2.size else None, batch, K, d_ffn,
                                          int(capacity), _ptr(flat) if flat.size else None,
                                          _ptr(per) if per.size else None, _ptr(tot)))
    rows = [ActiveIndexRow(flat[t], per[t], int(tot[t])) for t in range(batch)]
    return rows[0] if one else rows


def n_off(s: float, n: int) -> int:
    out = C.c_int32()
    _check(_lib.load().skb_n_off(s, n, C.byref(out)))
    return out.value


def device_count() -> int:
    return _lib.load().skb_device_count()
