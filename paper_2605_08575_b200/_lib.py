"""ctypes binding of libsparsekit_b200.so (include/sparsekit_b200.h).

Loading fails loudly: there is no fallback implementation of any entry point.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libsparsekit_b200.so")

SKB_OK, SKB_ESHAPE, SKB_ECONFIG, SKB_EINDEX, SKB_EINTERNAL, SKB_ECUDA, SKB_EFORMAT, SKB_EIO = range(8)
MODE_DENSE, MODE_TOPK, MODE_MASKED, MODE_ROUTE_ONLY, MODE_THRESHOLD = 0, 1, 2, 3, 4
FLAG_FAST_ROUTER, FLAG_SIMT_GATEUP, FLAG_TIME_STAGES, FLAG_NO_PDL = 1, 2, 4, 8
FLAG_GATHER_DOWN, FLAG_DENSE_DOWN, FLAG_BF16_H, FLAG_NO_FUSED_DECODE = 16, 32, 64, 128
FLAG_FUSED_DECODE = 256
FLAG_NO_PAIRED_BLOCKS = 0x200
FLAG_PAIRED_BLOCKS = 0x400
N_STAGES = 6
STAGE_NAMES = ("router", "dispatch", "gateup", "select", "down", "combine")

# every symbol include/sparsekit_b200.h declares
EXPORTS = (
    "skb_last_error", "skb_abi_version", "skb_device_count", "skb_config_validate",
    "skb_layer_create", "skb_layer_create_synthetic", "skb_layer_create_synthetic_slice",
    "skb_layer_set_router", "skb_layer_destroy", "skb_layer_reserve",
    "skb_layer_forward", "skb_layer_forward_device", "skb_layer_stage_times",
    "skb_layer_last_launches", "skb_layer_weight_bytes", "skb_route", "skb_align_dispatch",
    "skb_combine", "skb_mask_smallest", "skb_topk_mask", "skb_n_off", "skb_generate_tokens",
    "skb_layer_load", "skb_save_weights", "skb_weight_file_size", "skb_last_error_offset",
    "skb_threshold_mask", "skb_default_capacity", "skb_compact_active",
    "skb_ep_row_stride", "skb_ep_plan", "skb_ep_pack", "skb_ep_unpack", "skb_ep_combine",
    "skb_ep_symm_alloc", "skb_ep_symm_free", "skb_ep_ipc_export", "skb_ep_ipc_import",
    "skb_ep_ipc_close", "skb_ep_push_back", "skb_ep_combine_symm", "skb_ep_push_rows",
    "skb_ep_unpack_symm", "skb_ep_back_ptrs", "skb_ep_signal_back", "skb_layer_forward_device_rows",
)


class SkbConfig(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "n_experts", "top_k", "d_model", "d_ffn", "has_shared", "d_shared", "renormalize",
        "align_block")]


class SkbReport(C.Structure):
    _fields_ = [("gate_macs", C.c_uint64), ("up_macs", C.c_uint64), ("down_macs", C.c_uint64),
                ("other_macs", C.c_uint64), ("active_neurons_total", C.c_uint64),
                ("achieved_routed_sparsity", C.c_double), ("tiles_total", C.c_uint64),
                ("tiles_skipped", C.c_uint64), ("path_used", C.c_int32), ("reserved", C.c_int32)]


class SkbForwardArgs(C.Structure):
    _fields_ = [
        ("batch", C.c_int32), ("mode", C.c_int32), ("flags", C.c_uint32), ("reserved", C.c_int32),
        ("s_routed", C.c_double), ("s_shared", C.c_double),
        ("x", C.c_void_p), ("y", C.c_void_p),
        ("routed_mask_in", C.c_void_p), ("routed_mask_len", C.c_uint64),
        ("shared_mask_in", C.c_void_p), ("shared_mask_len", C.c_uint64),
        ("ids_out", C.c_void_p), ("weights_out", C.c_void_p),
        ("routed_mask_out", C.c_void_p), ("shared_mask_out", C.c_void_p),
        ("h_routed_out", C.c_void_p), ("h_shared_out", C.c_void_p),
        ("ids_in", C.c_void_p), ("weights_in", C.c_void_p),
        ("tau", C.c_float), ("reserved2", C.c_int32), ("slot_n_off", C.c_void_p),
    ]


_lib = None


def load() -> C.CDLL:
    """Returns the loaded library; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no non-CUDA implementation of this package)")
    L = C.CDLL(LIB_PATH)
    vp, i32, u64 = C.c_void_p, C.c_int32, C.c_uint64
    L.skb_last_error.restype = C.c_char_p
    L.skb_abi_version.restype = C.c_int
    L.skb_device_count.restype = C.c_int
    L.skb_config_validate.argtypes = [C.POINTER(SkbConfig)]
    L.skb_layer_create.argtypes = [C.POINTER(SkbConfig), vp, vp, vp, vp, vp, vp, vp, C.c_int,
                                   C.POINTER(vp)]
    L.skb_layer_create_synthetic.argtypes = [C.POINTER(SkbConfig), u64, C.c_float, C.c_int,
                                             C.POINTER(vp)]
    L.skb_layer_create_synthetic_slice.argtypes = [C.POINTER(SkbConfig), u64, C.c_float, C.c_int,
                                                   C.c_int, C.c_int, C.c_int, C.POINTER(vp)]
    L.skb_layer_set_router.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int]
    L.skb_layer_destroy.argtypes = [vp]
    L.skb_layer_destroy.restype = None
    L.skb_layer_reserve.argtypes = [vp, C.c_int]
    L.skb_layer_forward.argtypes = [vp, C.POINTER(SkbForwardArgs), C.POINTER(SkbReport)]
    L.skb_layer_forward_device.argtypes = [vp, C.POINTER(SkbForwardArgs), vp, C.POINTER(SkbReport)]
    L.skb_layer_stage_times.argtypes = [vp, C.POINTER(C.c_float)]
    L.skb_layer_last_launches.argtypes = [vp]
    L.skb_layer_weight_bytes.argtypes = [vp]
    L.skb_layer_weight_bytes.restype = u64
    L.skb_route.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp]
    L.skb_align_dispatch.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp,
                                     C.POINTER(i32), C.POINTER(i32)]
    L.skb_combine.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int, vp]
    L.skb_mask_smallest.argtypes = [vp, C.c_int, C.c_int, vp, vp, vp, vp]
    L.skb_topk_mask.argtypes = [vp, C.c_int, C.c_int, C.c_double, vp]
    L.skb_n_off.argtypes = [C.c_double, C.c_int, C.POINTER(i32)]
    L.skb_generate_tokens.argtypes = [C.c_int32, C.c_int32, C.c_uint64, vp]
    L.skb_layer_load.argtypes = [C.c_char_p, C.c_int, C.POINTER(SkbConfig), C.POINTER(vp)]
    L.skb_save_weights.argtypes = [C.POINTER(SkbConfig), vp, vp, vp, vp, vp, vp, vp, C.c_char_p]
    L.skb_weight_file_size.argtypes = [C.POINTER(SkbConfig)]
    L.skb_weight_file_size.restype = C.c_uint64
    L.skb_last_error_offset.argtypes = []
    L.skb_last_error_offset.restype = C.c_uint64
    L.skb_threshold_mask.argtypes = [vp, C.c_int, C.c_int, C.c_float, vp]
    L.skb_default_capacity.argtypes = [C.c_int, C.c_int]
    L.skb_compact_active.argtypes = [vp, C.c_uint64, vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp]
    L.skb_ep_row_stride.argtypes = [C.c_int]
    L.skb_ep_plan.argtypes = [vp, C.c_int, C.c_int, vp, C.c_int, vp, vp, vp, vp]
    L.skb_ep_pack.argtypes = [vp, vp, vp, C.c_int, C.c_int, C.c_int, vp, vp]
    L.skb_ep_unpack.argtypes = [vp, C.c_int, C.c_int, vp, vp, vp]
    L.skb_ep_combine.argtypes = [vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, vp, vp]
    L.skb_ep_symm_alloc.argtypes = [C.c_uint64, C.POINTER(vp)]
    L.skb_ep_symm_free.argtypes = [vp]
    L.skb_ep_ipc_export.argtypes = [vp, vp]
    L.skb_ep_ipc_import.argtypes = [vp, C.POINTER(vp)]
    L.skb_ep_ipc_close.argtypes = [vp]
    L.skb_ep_push_back.argtypes = [vp, C.c_int, C.c_int, vp, C.c_int, C.c_int, vp, vp, vp, vp, vp]
    L.skb_ep_back_ptrs.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp]
    L.skb_ep_signal_back.argtypes = [vp, C.c_int, C.c_int, vp, vp, vp]
    L.skb_layer_forward_device_rows.argtypes = [vp, C.POINTER(SkbForwardArgs), vp, vp]
    L.skb_ep_push_rows.argtypes = [vp, vp, vp, C.c_int, C.c_int, C.c_int, vp, C.c_int, C.c_int, vp, vp, vp,
                                   vp]
    L.skb_ep_unpack_symm.argtypes = [vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp]
    L.skb_ep_combine_symm.argtypes = [vp, vp, vp, C.c_int, vp, vp, vp, C.c_int, C.c_int, C.c_int,
                                      vp, vp]
    _lib = L
    return L
