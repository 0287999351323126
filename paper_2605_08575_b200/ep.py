"""Expert parallelism for the activation-sparse MoE layer: one process per GPU, experts sharded
across ranks, token dispatch and combine as all-to-all over NCCL (NVLink / NVSwitch).

The reference is single-process and has no communication backend; the
partitioning follows from its structure: experts are independent given their routed tokens
(proj/src/engine.cpp:132-165 touches only gate[e]/up[e]/down_t[e] per dispatch block) and the
combine is a per-token sum over slots (proj/src/router.cpp:119-130).

Per forward, rank r ("home" of its own tokens x_r):
  1. route:    ids, weights = route(route_logits(x_r))            full router, replicated
  2. plan:     all-gather of the ids (B*K*4 bytes per rank); every rank then derives the WHOLE
               send/receive matrix on the device (csrc/ep.cu: ep_plan_kernel) -- no count
               exchange; the matrix crosses to the host once, because NCCL's all-to-all-v takes
               its split sizes from the host (the one synchronisation of the step)
  3. dispatch: ONE all-to-all-v of packed rows [D bf16 | int32 local expert id], grouped by
               destination rank, ascending flat slot inside a group (ep_pack_kernel)
  4. experts:  un-weighted slot outputs of the received rows through the local experts
               (external routing, top-k neuron selection at s_routed)
  5. combine:  ONE all-to-all-v back (fp32: the 1e-5 parity mode), then y = sum_s w_s * out_s in
               ascending slot order with multiply and add rounded separately
               (router.cpp:119-130) and the shared expert's output (replicated, computed at home
               with its own ratio) last (engine.cpp:168-173) -- ep_combine_kernel

Tokens cross the wire as bf16 (what the device image of the layer multiplies anyway: the expert
GEMMs round their operands to bf16), so results equal the single-GPU layer's on bf16-representable
tokens.  Selection and routing are per-(token, slot) local, so expert ids and masks are identical
to the single-GPU layer; outputs agree to the fp32 tolerance (the single-GPU kernels fold the
weights into a different, equally fixed, reduction tree).

`Backend` isolates the local computations so that the host-side logic (plan, split sizes,
all-to-all, combine order) is exercised by multi-process gloo tests on CPU tensors with an
oracle backend, and by the CUDA backend (the C ABI) on the device.
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

    def plan(self, ids_all: torch.Tensor, expert_lo: torch.Tensor, rank: int):
        ...  # ids_all [W, Bmax*K] int32 -> counts [W, W] int32, pos [Bmax*K] int32, local [Bmax*K] int32

    def pack(self, x: torch.Tensor, pos: torch.Tensor, local: torch.Tensor, n_send: int) -> torch.Tensor:
        ...  # -> uint8 [n_send, row_stride] packed bf16 rows + local expert ids

    def unpack(self, recv: torch.Tensor, d_model: int):
        ...  # uint8 [M, row_stride] -> rows [M, D] float32, local_ids [M] int32

    def experts(self, rows: torch.Tensor, local_ids: torch.Tensor, s: float) -> torch.Tensor:
        ...  # rows [M, D], local_ids [M] int32 in [0, e_hi - e_lo) -> un-weighted outputs [M, D]

    def shared(self, x: torch.Tensor, s: float) -> torch.Tensor:
        ...  # [B, D] -> shared-expert output [B, D]

    def combine(self, back: torch.Tensor, pos: torch.Tensor, w: torch.Tensor,
                shared: Optional[torch.Tensor]) -> torch.Tensor:
        ...  # back [n_send, D], pos [B*K], w [B, K] -> y [B, D]


def owner_ranges(n_experts: int, world: int):
    """Contiguous expert ranges, remainder spread over the first ranks."""
    base, rem = divmod(n_experts, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < rem else 0)
        out.append((lo, hi))
        lo = hi
    return out


def row_stride(d_model: int) -> int:
    """Bytes of one packed dispatch row: [D bf16][int32 local expert id], padded to 16."""
    return (d_model * 2 + 4 + 15) // 16 * 16


class ExpertParallelLayer:
    def __init__(self, backend: Backend, group: Optional[dist.ProcessGroup] = None,
                 max_batch: Optional[int] = None, peer_combine: bool = False,
                 peer_rows: int = 0, peer_dispatch: bool = False, fused_push: bool = False):
        """`max_batch`: the largest home batch of any rank (all ranks pass the same value); the
        all-gathered ids are padded to it.  None: every rank's batch has the same size.
        `peer_combine`: the combine direction without a collective -- expert
        ranks write their row outputs straight into the home ranks' peer-mapped buffers (room
        for `peer_rows` rows) and the home combine waits on counters; CUDA backend only."""
        self.b = backend
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.max_batch = max_batch
        self.ranges = owner_ranges(backend.n_experts, self.world)
        assert self.ranges[self.rank] == (backend.e_lo, backend.e_hi), \
            "backend expert range does not match owner_ranges()"
        self._lo_cpu = torch.tensor([r[0] for r in self.ranges] + [backend.n_experts], dtype=torch.int32)
        self._lo = {}
        self.last_stats = {}
        self.peer = None
        # `fused_push` (with peer_combine): the expert layer's combine kernel writes each output
        # row into the home rank's buffer directly instead of a separate push pass
        self.fused_push = bool(fused_push)
        assert not fused_push or peer_combine, "fused_push rides on the peer_combine setup"
        self.peer_dispatch = bool(peer_dispatch)
        if peer_combine or peer_dispatch:
            # `peer_dispatch`: the dispatch direction without a collective either -- the home rank
            # packs its token rows straight into the owners' receive buffers (needs peer_combine's
            # buffers too: both directions share the setup)
            assert peer_combine, "peer_dispatch rides on the peer_combine setup"
            self.peer = backend.symm_setup(peer_rows, self.world, self.rank, group,
                                           **({"dispatch": True} if peer_dispatch else {}))

    def _lo_on(self, device):
        if device not in self._lo:
            self._lo[device] = self._lo_cpu.to(device)
        return self._lo[device]

    def _all_to_all(self, send: torch.Tensor, send_counts, recv_counts) -> torch.Tensor:
        recv = send.new_empty((int(sum(recv_counts)),) + tuple(send.shape[1:]))
        if self.world == 1:
            recv.copy_(send)
            return recv
        dist.all_to_all_single(recv, send, output_split_sizes=list(recv_counts),
                               input_split_sizes=list(send_counts), group=self.group)
        return recv

    def forward(self, x: torch.Tensor, s_routed: float, s_shared: float = 0.0) -> torch.Tensor:
        b, K, W = self.b, self.b.top_k, self.world
        B, D = x.shape
        dev = x.device
        ids, w = b.route(x)                                   # [B, K]
        Bmax = self.max_batch if self.max_batch is not None else B
        assert B <= Bmax
        mine = ids.reshape(-1)
        if B < Bmax:                                          # short batch: pad with -1
            mine = torch.cat([mine, mine.new_full(((Bmax - B) * K,), -1)])
        if W > 1:
            flat_all = torch.empty(W * Bmax * K, dtype=torch.int32, device=dev)
            dist.all_gather_into_tensor(flat_all, mine.contiguous(), group=self.group)
            ids_all = flat_all.view(W, Bmax * K)
        else:
            ids_all = mine.reshape(1, -1)
        counts, pos, local = b.plan(ids_all, self._lo_on(dev), self.rank)
        cm = counts.cpu()                                     # the step's one host synchronisation
        sc, rc = cm[self.rank].tolist(), cm[:, self.rank].tolist()
        if self.peer_dispatch:
            b.push_rows(x, pos, local, counts, self.peer, self.rank)   # no first collective
            sh = b.shared(x, s_shared) if b.has_shared else None
            rows_in, ids_in = b.unpack_symm(self.peer, counts, self.rank, int(sum(rc)), D)
        else:
            send = b.pack(x, pos, local, int(sum(sc)))
            # the shared expert does not depend on the exchange: enqueue it before the all-to-all
            # so that it runs under the transfer (replicated weights, own sparsity ratio)
            sh = b.shared(x, s_shared) if b.has_shared else None
            recv = self._all_to_all(send, sc, rc)
            rows_in, ids_in = b.unpack(recv, D)
        if self.peer is not None and self.fused_push:
            # the expert layer's last kernel writes into the home ranks' buffers itself
            b.experts_to_peers(rows_in, ids_in, s_routed, counts, self.peer, self.rank)
            y = b.combine_symm(self.peer, pos, w, sh)
        elif self.peer is not None:                           # no second collective
            out_in = b.experts(rows_in, ids_in, s_routed) if rows_in.shape[0] else rows_in
            b.push_back(out_in, counts, self.peer, self.rank)
            y = b.combine_symm(self.peer, pos, w, sh)
        else:
            out_in = b.experts(rows_in, ids_in, s_routed) if rows_in.shape[0] else rows_in
            back = self._all_to_all(out_in, rc, sc)           # back to the home ranks, send order
            y = b.combine(back, pos, w, sh)
        self.last_stats = {"sent_rows": sc, "recv_rows": rc,
                           "dispatch_bytes": int(sum(sc)) * row_stride(D),
                           "combine_bytes": int(sum(rc)) * D * 4,
                           "host_syncs": 1,
                           "collectives": (1 if W > 1 else 0) +
                           (2 - (self.peer is not None) - self.peer_dispatch) * (W > 1)}
        return y


class CudaBackend:
    """The C-ABI layer as EP backend: an experts slice + (optionally) a shared-expert slice of
    generate_synthetic(full, seed, scale), both resident on this rank's GPU; plan / pack / unpack
    / combine are the kernels of csrc/ep.cu."""

    def __init__(self, skb, full_cfg, seed: int, scale: float, rank: int, world: int,
                 device: int = 0, max_rows: int = 1024):
        from . import _lib
        self.skb = skb
        self.L = _lib.load()
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

    def _ok(self, rc, what):
        if rc != 0:
            raise RuntimeError(f"{what} failed with status {rc}")

    def route(self, x):
        B = x.shape[0]
        ids = torch.empty((B, self.top_k), dtype=torch.int32, device=x.device)
        w = torch.empty((B, self.top_k), dtype=torch.float32, device=x.device)
        self.slice.reserve(B)
        self.slice.route_device(x.data_ptr(), ids.data_ptr(), w.data_ptr(), B, stream=self._stream())
        return ids, w

    def plan(self, ids_all, expert_lo, rank):
        W, slots = ids_all.shape
        dev = ids_all.device
        counts = torch.empty((W, W), dtype=torch.int32, device=dev)
        pos = torch.empty(slots, dtype=torch.int32, device=dev)
        local = torch.empty(slots, dtype=torch.int32, device=dev)
        self._ok(self.L.skb_ep_plan(ids_all.contiguous().data_ptr(), W, slots, expert_lo.data_ptr(),
                                    rank, counts.data_ptr(), pos.data_ptr(), local.data_ptr(),
                                    self._stream()), "skb_ep_plan")
        return counts, pos, local

    def pack(self, x, pos, local, n_send):
        B, D = x.shape
        send = torch.empty((n_send, row_stride(D)), dtype=torch.uint8, device=x.device)
        self._ok(self.L.skb_ep_pack(x.contiguous().data_ptr(), pos.data_ptr(), local.data_ptr(),
                                    B * self.top_k, self.top_k, D, send.data_ptr(), self._stream()),
                 "skb_ep_pack")
        return send

    def unpack(self, recv, d_model):
        M = recv.shape[0]
        rows = torch.empty((M, d_model), dtype=torch.float32, device=recv.device)
        ids = torch.empty(M, dtype=torch.int32, device=recv.device)
        self._ok(self.L.skb_ep_unpack(recv.data_ptr(), M, d_model, rows.data_ptr(), ids.data_ptr(),
                                      self._stream()), "skb_ep_unpack")
        return rows, ids

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

    def combine(self, back, pos, w, shared):
        B, K = w.shape
        D = back.shape[1] if back.dim() == 2 else self.D
        y = torch.empty((B, D), dtype=torch.float32, device=w.device)
        self._ok(self.L.skb_ep_combine(back.contiguous().data_ptr(), pos.data_ptr(),
                                       w.contiguous().data_ptr(),
                                       shared.data_ptr() if shared is not None else None,
                                       B, K, D, y.data_ptr(), self._stream()), "skb_ep_combine")
        return y

    # ---- exchange over peer-mapped buffers (csrc/ep.cu: ep_push_back_kernel, ep_combine_symm_kernel,
    # ep_push_rows_kernel, ep_unpack_symm_kernel)
    def symm_setup(self, max_rows, world, rank, group=None, dispatch=False):
        """One `back` buffer [max_rows][D] fp32 and `world` cumulative counters per rank -- and, for
        the dispatch direction, one `recv` buffer [max_rows][row_stride] with counters of its own
        -- exported through CUDA IPC and mapped by every peer (world 1: the rank maps itself)."""
        import ctypes as C
        L, D = self.L, self.D
        rows = max(1, max_rows)
        bufs = [("back", rows * D * 4), ("flag", 8 * 16)]
        if dispatch:
            bufs += [("recv", rows * row_stride(D)), ("dflag", 8 * 16)]
        local = {}
        for name, nbytes in bufs:
            p = C.c_void_p()
            self._ok(L.skb_ep_symm_alloc(nbytes, C.byref(p)), "skb_ep_symm_alloc")
            local[name] = p
        peers = {name: [local[name].value] * world for name, _ in bufs}
        dev = torch.device("cuda", torch.cuda.current_device())
        if world > 1:
            nb = 64 * len(bufs)
            h = torch.zeros(nb, dtype=torch.uint8)
            for i, (name, _) in enumerate(bufs):
                self._ok(L.skb_ep_ipc_export(local[name], h.data_ptr() + 64 * i), "skb_ep_ipc_export")
            allh = torch.empty(world * nb, dtype=torch.uint8, device=dev)
            dist.all_gather_into_tensor(allh, h.to(dev), group=group)
            allh = allh.cpu()
            for r in range(world):
                if r == rank:
                    continue
                for i, (name, _) in enumerate(bufs):
                    pp = C.c_void_p()
                    self._ok(L.skb_ep_ipc_import(allh[r * nb + 64 * i:].data_ptr(), C.byref(pp)),
                             "skb_ep_ipc_import")
                    peers[name][r] = pp.value
        out = {"back": local["back"].value, "flag": local["flag"].value, "max_rows": max_rows,
               "peer_back": torch.tensor(peers["back"], dtype=torch.int64, device=dev),
               "peer_flag": torch.tensor(peers["flag"], dtype=torch.int64, device=dev),
               "expect": torch.zeros(16, dtype=torch.int64, device=dev),
               "done": torch.zeros(1, dtype=torch.int32, device=dev), "world": world}
        if dispatch:
            out.update({"recv": local["recv"].value, "dflag": local["dflag"].value,
                        "peer_recv": torch.tensor(peers["recv"], dtype=torch.int64, device=dev),
                        "peer_dflag": torch.tensor(peers["dflag"], dtype=torch.int64, device=dev),
                        "dexpect": torch.zeros(16, dtype=torch.int64, device=dev),
                        "ddone": torch.zeros(1, dtype=torch.int32, device=dev)})
        return out

    def push_rows(self, x, pos, local, counts, peer, rank):
        """pack + dispatch in one kernel: token rows straight into the owners' receive buffers"""
        B, D = x.shape
        self._ok(self.L.skb_ep_push_rows(x.contiguous().data_ptr(), pos.data_ptr(), local.data_ptr(),
                                         B * self.top_k, self.top_k, D, counts.data_ptr(),
                                         peer["world"], rank, peer["peer_recv"].data_ptr(),
                                         peer["peer_dflag"].data_ptr(), peer["ddone"].data_ptr(),
                                         self._stream()), "skb_ep_push_rows")

    def unpack_symm(self, peer, counts, rank, n_rows, d_model):
        """wait for the peers' rows (cumulative counters), then unpack"""
        dev = counts.device
        rows = torch.empty((n_rows, d_model), dtype=torch.float32, device=dev)
        ids = torch.empty(n_rows, dtype=torch.int32, device=dev)
        assert n_rows <= max(1, peer["max_rows"]), "peer receive buffer too small for this step"
        self._ok(self.L.skb_ep_unpack_symm(peer["recv"], peer["dflag"], peer["dexpect"].data_ptr(),
                                           counts.data_ptr(), peer["world"], rank, n_rows, d_model,
                                           rows.data_ptr(), ids.data_ptr(), self._stream()),
                 "skb_ep_unpack_symm")
        return rows, ids

    def experts_to_peers(self, rows, local_ids, s, counts, peer, rank):
        """The expert layer writes every output row straight into its home rank's back buffer
        (skb_ep_back_ptrs + skb_layer_forward_device_rows), then the counters move
        (skb_ep_signal_back): no output tensor, no copy pass."""
        M = rows.shape[0]
        if M:
            rows = rows.contiguous()
            ptrs = torch.empty(M, dtype=torch.int64, device=rows.device)
            self._ok(self.L.skb_ep_back_ptrs(counts.data_ptr(), peer["world"], rank, M, self.D,
                                             peer["peer_back"].data_ptr(), ptrs.data_ptr(),
                                             self._stream()), "skb_ep_back_ptrs")
            self.slice.reserve(M)
            self.slice.forward_device_rows(rows.data_ptr(), ptrs.data_ptr(), M, mode=self.skb.MODE_TOPK,
                                           s_routed=s, stream=self._stream(),
                                           ids_in_ptr=local_ids.contiguous().data_ptr())
        self._ok(self.L.skb_ep_signal_back(counts.data_ptr(), peer["world"], rank,
                                           peer["peer_flag"].data_ptr(), peer["expect"].data_ptr(),
                                           self._stream()), "skb_ep_signal_back")

    def push_back(self, out_rows, counts, peer, rank):
        M = out_rows.shape[0]
        self._ok(self.L.skb_ep_push_back(out_rows.contiguous().data_ptr() if M else None, M, self.D,
                                         counts.data_ptr(), peer["world"], rank,
                                         peer["peer_back"].data_ptr(), peer["peer_flag"].data_ptr(),
                                         peer["expect"].data_ptr(), peer["done"].data_ptr(),
                                         self._stream()), "skb_ep_push_back")

    def combine_symm(self, peer, pos, w, shared):
        B, K = w.shape
        y = torch.empty((B, self.D), dtype=torch.float32, device=w.device)
        self._ok(self.L.skb_ep_combine_symm(peer["back"], peer["flag"], peer["expect"].data_ptr(),
                                            peer["world"], pos.data_ptr(), w.contiguous().data_ptr(),
                                            shared.data_ptr() if shared is not None else None,
                                            B, K, self.D, y.data_ptr(), self._stream()),
                 "skb_ep_combine_symm")
        return y
