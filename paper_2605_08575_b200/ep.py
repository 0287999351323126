"""Expert parallelism for the activation-sparse MoE layer: one process per GPU, experts sharded
across ranks, token dispatch and combine as all-to-all over NCCL (NVLink / NVSwitch).

The reference is single-process and has no communication backend; the
partitioning follows from its structure: experts are independent given their routed tokens
(proj/src/engine.cpp:132-165 touches only gate[e]/up[e]/down_t[e] per dispatch block) and the
combine is a per-token sum over slots (proj/src/router.cpp:119-130).

Per forward, rank r ("home" of its own tokens x_r):
  1. route:    ids, weights = route(route_logits(x_r))            full router, replicated
  2. dispatch: all-to-all-v of the routed token rows to the ranks that own ids // E_local
               (counts first, then rows + local expert ids), rows sorted by destination
  3. experts:  un-weighted slot outputs of the received rows through the local experts
               (external routing, top-k neuron selection at s_routed)
  4. combine:  all-to-all-v back, un-sort, y = sum_s w_s * out_s in ascending slot order with
               multiply and add rounded separately (router.cpp:119-130), then the shared
               expert's output (replicated, computed at home with its own ratio) last
               (engine.cpp:168-173)

Selection and routing are per-(token, slot) local, so expert ids and masks are identical to the
single-GPU layer; outputs agree to the fp32 tolerance (the single-GPU kernels fold the weights
into a different, equally fixed, reduction tree).

`Backend` isolates the three local computations so that the host-side logic (sorting, counts,
all-to-all, un-sorting, combine order) is exercised by multi-process gloo tests on CPU tensors
with an oracle backend, and by the CUDA backend (the C ABI) on the device.
"""
from __future__ import annotations

from typing import Optional, Protocol

import torch
import torch.distributed as dist


class Backend(Protocol):
    n_experts: int       # E of the full model
    top_k: int
    e_lo: int            # this rank owns experts [e_lo, e_hi)
    e_hi: int
    has_shared: bool

    def route(self, x: torch.Tensor):  # -> ids [B, K] int32, weights [B, K] float32
        ...

    def experts(self, rows: torch.Tensor, local_ids: torch.Tensor, s: float) -> torch.Tensor:
        ...  # rows [M, D], local_ids [M] int32 in [0, e_hi - e_lo) -> un-weighted outputs [M, D]

    def shared(self, x: torch.Tensor, s: float) -> torch.Tensor:
        ...  # [B, D] -> shared-expert output [B, D]


def owner_ranges(n_experts: int, world: int):
    """Contiguous expert ranges, remainder spread over the first ranks."""
    base, rem = divmod(n_experts, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < rem else 0)
        out.append((lo, hi))
        lo = hi
    return out


class ExpertParallelLayer:
    def __init__(self, backend: Backend, group: Optional[dist.ProcessGroup] = None):
        self.b = backend
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.ranges = owner_ranges(backend.n_experts, self.world)
        assert self.ranges[self.rank] == (backend.e_lo, backend.e_hi), \
            "backend expert range does not match owner_ranges()"
        # expert id -> owner rank
        owner = torch.empty(backend.n_experts, dtype=torch.int64)
        for r, (lo, hi) in enumerate(self.ranges):
            owner[lo:hi] = r
        self._owner_cpu = owner
        self._owner = {}
        self.last_stats = {}

    def _owner_on(self, device):
        if device not in self._owner:
            self._owner[device] = self._owner_cpu.to(device)
        return self._owner[device]

    def _all_to_all(self, send: torch.Tensor, send_counts, recv_counts) -> torch.Tensor:
        recv = send.new_empty((int(sum(recv_counts)),) + tuple(send.shape[1:]))
        if self.world == 1:
            recv.copy_(send)
            return recv
        dist.all_to_all_single(recv, send, output_split_sizes=list(recv_counts),
                               input_split_sizes=list(send_counts), group=self.group)
        return recv

    def forward(self, x: torch.Tensor, s_routed: float, s_shared: float = 0.0) -> torch.Tensor:
        b, K = self.b, self.b.top_k
        B, D = x.shape
        dev = x.device
        ids, w = b.route(x)                                   # [B, K]
        flat = ids.reshape(-1).to(torch.int64)                # flat slot i = t * K + s
        dest = self._owner_on(dev)[flat]
        order = torch.argsort(dest, stable=True)              # slots grouped by owner rank
        send_counts = torch.bincount(dest, minlength=self.world)
        # counts exchange (tiny), then the rows and their local expert ids
        if self.world > 1:
            recv_counts = torch.empty_like(send_counts)
            dist.all_to_all_single(recv_counts, send_counts, group=self.group)
        else:
            recv_counts = send_counts.clone()
        sc, rc = send_counts.tolist(), recv_counts.tolist()
        tok = torch.div(order, K, rounding_mode="floor")
        rows = x.index_select(0, tok)                         # [B*K, D] sorted by destination
        lo_of_dest = torch.tensor([r[0] for r in self.ranges], device=dev)[dest[order]]
        local = (flat[order] - lo_of_dest).to(torch.int32)
        rows_in = self._all_to_all(rows, sc, rc)
        ids_in = self._all_to_all(local, sc, rc)
        out_in = b.experts(rows_in, ids_in, s_routed) if rows_in.shape[0] else rows_in
        out_sorted = self._all_to_all(out_in, rc, sc)         # back to the home ranks
        slot_out = torch.empty_like(out_sorted)
        slot_out[order] = out_sorted                          # un-sort to flat slot order
        slot_out = slot_out.view(B, K, D)
        y = torch.zeros((B, D), dtype=x.dtype, device=dev)
        for s in range(K):                                    # ascending slots, mul then add
            y = y + w[:, s:s + 1] * slot_out[:, s, :]
        if b.has_shared:
            y = y + b.shared(x, s_shared)
        self.last_stats = {"sent_rows": sc, "recv_rows": rc,
                           "dispatch_bytes": int(sum(sc)) * D * x.element_size(),
                           "combine_bytes": int(sum(rc)) * D * x.element_size()}
        return y


class CudaBackend:
    """The C-ABI layer as EP backend: an experts slice + (optionally) a shared-expert slice of
    generate_synthetic(full, seed, scale), both resident on this rank's GPU."""

    def __init__(self, skb, full_cfg, seed: int, scale: float, rank: int, world: int,
                 device: int = 0, max_rows: int = 1024):
        self.skb = skb
        self.n_experts, self.top_k = full_cfg.n_experts, full_cfg.top_k
        self.e_lo, self.e_hi = owner_ranges(full_cfg.n_experts, world)[rank]
        self.has_shared = bool(full_cfg.has_shared)
        self.D = full_cfg.d_model
        self.slice = skb.MoELayerWeights.synthetic_slice(full_cfg, seed, scale, self.e_lo,
                                                         self.e_hi, device=device)
        self.slice.reserve(max_rows)
        self.shared_slice = None
        if self.has_shared:
            self.shared_slice = skb.MoELayerWeights.synthetic_slice(full_cfg, seed, scale,
                                                                    shared=True, device=device)
            self.shared_slice.reserve(max_rows)
        self._zero_ids = {}

    def _stream(self):
        # the C ABI reads a NULL stream as "the layer's own stream"; torch's default stream has
        # handle 0, so name it explicitly (cudaStreamLegacy == 0x1)
        return torch.cuda.current_stream().cuda_stream or 1

    def route(self, x):
        B = x.shape[0]
        ids = torch.empty((B, self.top_k), dtype=torch.int32, device=x.device)
        w = torch.empty((B, self.top_k), dtype=torch.float32, device=x.device)
        self.slice.reserve(B)
        self.slice.route_device(x.data_ptr(), ids.data_ptr(), w.data_ptr(), B, stream=self._stream())
        return ids, w

    def experts(self, rows, local_ids, s):
        M = rows.shape[0]
        rows = rows.contiguous()
        y = torch.empty_like(rows)
        self.slice.reserve(M)
        self.slice.forward_device(rows.data_ptr(), y.data_ptr(), M, mode=self.skb.MODE_TOPK,
                                  s_routed=s, stream=self._stream(),
                                  ids_in_ptr=local_ids.contiguous().data_ptr())
        return y

    def shared(self, x, s):
        B = x.shape[0]
        if B not in self._zero_ids:
            self._zero_ids[B] = torch.zeros(B, dtype=torch.int32, device=x.device)
        y = torch.empty_like(x)
        self.shared_slice.reserve(B)
        self.shared_slice.forward_device(x.data_ptr(), y.data_ptr(), B, mode=self.skb.MODE_TOPK,
                                         s_routed=s, stream=self._stream(),
                                         ids_in_ptr=self._zero_ids[B].data_ptr())
        return y
