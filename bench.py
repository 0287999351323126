#!/usr/bin/env python
"""bench.py -- MoE-layer tokens/s and achieved HBM GB/s vs intra-expert sparsity (decode).

Contract (driver): ``python bench.py --gpus N --steps K --warmup W [--impl reference]`` prints
ONE JSON line on rank 0.  A "step" is one forward of the activation-sparse MoE FFN layer over
one batch of synthetic tokens.

  value     tokens/s of the whole job with tokens resident in HBM (device entry point of the
            C ABI, CUDA-graph replay, L2 flushed between steps, CUDA events per step).
  e2e       the same metric through the host-buffer entry point skb_layer_forward (the call a
            user of the reference's forward_* makes): pinned host tokens in, host outputs out,
            H2D/D2H inside the timed region.
  roofline  dominant kernel (gate/up grouped GEMM): algorithmic weight bytes of the launch
             / its CUDA-event duration, against MEASURED_PEAKS.json's HBM GB/s.
  sweep     tokens/s, layer GB/s and roofline fraction at s in {0,.25,.5,.75,.9} plus the
            north-star point (OLMoE shape, batch 1, s=0.5).
  cpu_baseline / --impl reference
            the UNMODIFIED reference (oracle/_ref/libsparsekit_ref.so: build_topk_masks +
            forward_masked_dense, the path this layer replaces) on the host cores.

The oracle is imported only by the cpu_baseline / reference legs.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

# shape table: BASELINE.json configs (d_model / d_shared as assumed in SURVEY.md 8d)
WORKLOADS = {
    "olmoe": dict(name="OLMoE-1B-7B", E=64, K=8, D=2048, N=1024, S=0),
    "granite": dict(name="Granite-1B-A400M", E=32, K=8, D=1024, N=512, S=0),
    "qwen35": dict(name="Qwen3.5-35B-A3B", E=256, K=8, D=2048, N=512, S=512),
    "gptoss": dict(name="GPT-OSS-20B", E=32, K=4, D=2880, N=2880, S=0),
    "maverick": dict(name="Llama-4-Maverick", E=128, K=1, D=5120, N=8192, S=8192),
}
SEED, SCALE = 1, 0.05          # generate_synthetic defaults of the reference CLI (tools/main.cpp:157)
# calibrate_tau(target 0.5) of the unmodified reference on generate_synthetic(seed 1, 0.05) rounded
# to bf16 (oracle/_ref in the build container: RefLayer.calibrate_tau(0.5), defaults of
# tools/main.cpp: 16 calibration tokens seed 3, sample cap 2^20, sampler seed 4)
THRESHOLD_TAU = {"granite": 0.2473328560590744, "olmoe": 0.2645798623561859}


def calibrated_tau(workload, use_reference):
    """tau for a 0.5 routed-sparsity target: the reference's own calibrate chain, run here on the
    host cores (oracle/_ref, cpu_baseline leg) when allowed and present; else the value it gave
    in the build container (above)."""
    if use_reference:
        try:
            lay, _ = _ref_layer(WORKLOADS[workload])
            if lay is not None:
                return float(lay.calibrate_tau(0.5)), "reference calibrate_tau(0.5), this run"
        except Exception as exc:  # the baseline leg must not take the bench down
            print(f"[bench] calibrate_tau failed ({exc}); using the recorded value", file=sys.stderr)
    return THRESHOLD_TAU[workload], "reference calibrate_tau(0.5), recorded in the build container"
SWEEP_S = (0.0, 0.25, 0.5, 0.75, 0.9)
W_BYTES = 2                    # bf16 weight image


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def tensor_peak():
    """Dense bf16 TFLOP/s: the sustained figure (the kernel is timed inside a long step)."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        if "bf16_tflops_sustained" in d:
            return float(d["bf16_tflops_sustained"]), "measured sustained (MEASURED_PEAKS.json)"
    return 1400.0, "fallback (B200_PROFILING.md)"


def n_off(s, n):
    # topk_mask, proj/src/activation.cpp:54-60
    return int(min(max(np.floor(s * n + 0.5), 0), n))


_TOKEN_SOURCE = [None]  # (batch, d_model, seed) -> float32 [batch, d_model]


def make_tokens(B, D, seed):
    """generate_tokens(B, D, seed) of the reference (proj/src/model.cpp:168-178; seed
    2 + iteration) rounded to bf16-representable fp32, so that both arms see the same operands.
    Our arm draws them through the C ABI's host function skb_generate_tokens, the reference arm
    through the reference's own generate_tokens (bit-identical: tests/test_oracle_cpu.py)."""
    x = np.ascontiguousarray(_TOKEN_SOURCE[0](B, D, seed), dtype=np.float32).reshape(B, D).copy()
    u = x.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).reshape(B, D)


def algorithmic_bytes(shape, B, ids, routed_mask, shared_mask):
    """SURVEY.md 8d, computed exactly from the realised routing and masks (integers)."""
    E, K, D, N, S = (shape[k] for k in "EKDNS")
    ids = np.asarray(ids).reshape(B, K)
    routed_mask = np.asarray(routed_mask).reshape(B * K, N)
    flat = ids.reshape(-1)
    experts = np.unique(flat)
    r_down = 0
    for e in experts:
        r_down += int(np.count_nonzero(routed_mask[flat == e].any(axis=0)))
    router = E * D * W_BYTES
    gateup = len(experts) * 2 * N * D * W_BYTES
    down = r_down * D * W_BYTES
    sh_gateup = sh_down = 0
    if S:
        sh_gateup = 2 * S * D * W_BYTES
        if shared_mask is None:
            r_sh = S
        else:
            r_sh = int(np.count_nonzero(np.asarray(shared_mask).reshape(B, S).any(axis=0)))
        sh_down = r_sh * D * W_BYTES
    io = B * D * (4 + 4)
    return dict(total=router + gateup + down + sh_gateup + sh_down + io,
                gateup=gateup + sh_gateup, down=down + sh_down, router=router, io=io,
                distinct_experts=int(len(experts)), r_down=r_down)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.lines, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms",
                 "50", "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._pump, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            f = [v.strip() for v in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "samples": len(sm),
                "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------------
L2_BYTES = 126 << 20


class Point:
    """One (shape, batch, sparsity) measurement set-up on the current device.

    L2 policy of the timed region ("inputs larger than L2"): the steps run back to back over a
    ROTATION of identical weight images (``layers``), image r with token batch r, sized so that
    between two uses of one image the other images stream at least twice the L2 capacity --
    every weight byte of a step comes out of HBM, and the lines it evicts are clean, as they are
    when a model's layers follow each other.  (A memset flush leaves the L2 full of dirty lines
    whose write-back rides on every miss of the next kernel: tools/micro/burst.cu measures a
    64 MB burst at 14.4 us after a memset against 12.2 us after a read sweep.)"""

    RING = 8

    def __init__(self, skb, torch, layer, shape, B, make_layer=None):
        self.skb, self.torch, self.layer, self.shape, self.B = skb, torch, layer, shape, B
        self.make_layer = make_layer
        self.layers = [layer]
        D = shape["D"]
        self.x_host = [make_tokens(B, D, 2 + i) for i in range(self.RING)]
        self.x_ring = [torch.from_numpy(x).cuda() for x in self.x_host]
        self.x = torch.empty((B, D), dtype=torch.float32, device="cuda")
        self.y = torch.empty((B, D), dtype=torch.float32, device="cuda")
        self.flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
        layer.reserve(B)

    def rotation(self, bytes_per_step):
        """Grow the rotation so that (R - 1) * bytes_per_step >= 2 * L2 (bounded by memory)."""
        want = 1 + int(np.ceil(2.0 * L2_BYTES / max(1.0, bytes_per_step)))
        free, _ = self.torch.cuda.mem_get_info()
        room = int((free - (8 << 30)) // max(1, self.layer.weight_bytes))
        want = max(1, min(want, 1 + max(0, room), 16))
        while len(self.layers) < want and self.make_layer is not None:
            lay = self.make_layer(self.shape)
            lay.reserve(self.B)
            self.layers.append(lay)
        return len(self.layers)

    def bytes_for(self, s):
        """Exact algorithmic bytes per ring slot (one capture forward each; untimed)."""
        skb, S = self.skb, self.shape["S"]
        lvl = skb.SparsityLevel(s)
        out = []
        for x in self.x_host:
            rep = skb.forward_topk_sparse(self.layer, x, lvl, lvl if S else None, capture=True)
            out.append(algorithmic_bytes(self.shape, self.B, rep.routes.ids, rep.masks.routed,
                                         rep.masks.shared if S else None))
        return out

    def _enqueue(self, s, flags=0, layer=None, x=None):
        S = self.shape["S"]
        layer = layer if layer is not None else self.layer
        x = x if x is not None else self.x
        if isinstance(s, tuple):  # ("tau", value): the threshold runtime path, forward_sparse
            layer.forward_device(x.data_ptr(), self.y.data_ptr(), self.B,
                                 mode=self.skb.MODE_THRESHOLD, tau=s[1], flags=flags,
                                 stream=self.torch.cuda.current_stream().cuda_stream or 1)
            return
        layer.forward_device(x.data_ptr(), self.y.data_ptr(), self.B,
                             mode=self.skb.MODE_TOPK, s_routed=s, s_shared=s if S else 0.0,
                             flags=flags,
                             # NULL would mean "the layer's own stream": name torch's
                             # default stream explicitly (cudaStreamLegacy == 0x1)
                             stream=self.torch.cuda.current_stream().cuda_stream or 1)

    def time_device(self, s, steps, warmup, use_graph=True, flags=0):
        """Milliseconds per step of the device entry point: `steps` forwards back to back inside
        ONE CUDA-event pair, rotating over the weight images (see the class comment).  Returns
        (ms_per_step, graphed)."""
        torch = self.torch
        R = len(self.layers)
        xs = [self.x_ring[r % self.RING] for r in range(R)]
        single, full = None, None
        if use_graph:
            try:
                side = torch.cuda.Stream()
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(side):
                    for r in range(R):  # warm (module load, attribute set) before capture
                        self._enqueue(s, flags, self.layers[r], xs[r])
                torch.cuda.current_stream().wait_stream(side)
                torch.cuda.synchronize()
                single = []
                for r in range(R):
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g):
                        self._enqueue(s, flags, self.layers[r], xs[r])
                    single.append(g)
                if R > 1:
                    full = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(full):
                        for r in range(R):
                            self._enqueue(s, flags, self.layers[r], xs[r])
            except Exception as exc:  # capture unsupported: direct launches
                print(f"[bench] CUDA graph capture failed ({exc}); timing direct launches",
                      file=sys.stderr)
                single, full = None, None
                torch.cuda.synchronize()

        def run(n):
            i = 0
            while i < n:
                if full is not None and n - i >= R:
                    full.replay()
                    i += R
                    continue
                r = i % R
                if single is not None:
                    single[r].replay()
                else:
                    self._enqueue(s, flags, self.layers[r], xs[r])
                i += 1

        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        self.flush.zero_()
        run(-(-max(warmup, R) // R) * R)  # whole rotations, so that the timed run starts at image 0
        e0.record()
        run(steps)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps, single is not None

    def time_isolated(self, s, steps, warmup):
        """The same forward timed alone: one CUDA-event pair per step around a graph replay on an
        idle GPU, 512 MiB memset before each (dirty L2).  Includes the ~5 us an isolated launch
        costs between two events; reported beside the back-to-back figure."""
        torch = self.torch
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self._enqueue(s)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            self._enqueue(s)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
        for i in range(warmup + steps):
            self.x.copy_(self.x_ring[i % self.RING])
            self.flush.zero_()
            if i >= warmup:
                ev[i - warmup][0].record()
            graph.replay()
            if i >= warmup:
                ev[i - warmup][1].record()
        torch.cuda.synchronize()
        return float(np.mean([a.elapsed_time(b) for a, b in ev]))

    def time_stages(self, s, steps, warmup):
        """Per-stage CUDA-event times (ms, mean over steps), stages serialised (no PDL)."""
        torch, skb = self.torch, self.skb
        acc = np.zeros(len(skb.STAGE_NAMES))
        for i in range(warmup + steps):
            self.x.copy_(self.x_ring[i % self.RING])
            self.flush.zero_()
            torch.cuda.synchronize()  # stage events must not straddle the flush
            self._enqueue(s, flags=skb.FLAG_TIME_STAGES)
            ms = self.layer.stage_times()
            if i >= warmup:
                acc += np.asarray(ms)
        return dict(zip(skb.STAGE_NAMES, (acc / steps).tolist()))

    def time_e2e(self, s, steps, warmup):
        """Wall-clock per-step times (ms) of the host-buffer entry point (H2D + stages + D2H +
        synchronise inside), pinned host buffers, L2 flushed between steps."""
        torch, skb, S = self.torch, self.skb, self.shape["S"]
        D = self.shape["D"]
        xin = [torch.from_numpy(x).pin_memory() for x in self.x_host]
        yout = torch.empty((self.B, D), dtype=torch.float32).pin_memory()
        lvl = skb.SparsityLevel(s)
        times = []
        for i in range(warmup + steps):
            self.flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            skb.forward_topk_sparse(self.layer, xin[i % self.RING].numpy(), lvl,
                                    lvl if S else None, y_out=yout.numpy())
            t1 = time.perf_counter()
            if i >= warmup:
                times.append((t1 - t0) * 1e3)
        return times, self.B * D * 4, self.B * D * 4


def run_ep(args, torch, dist, skb, rank, world, local):
    """Expert-parallel arm (north-star: GPT-OSS and Maverick shapes): experts sharded over the
    ranks, tokens home-sharded, dispatch/combine as NCCL all-to-all-v (paper_2605_08575_b200/ep.py).
    With one rank the same code path runs with local slicing instead of the collective."""
    from paper_2605_08575_b200 import ep
    shape = WORKLOADS[args.workload]
    B, s = args.batch, args.sparsity
    hbm_peak, peak_src = peaks()
    cfg = skb.MoEConfig(shape["E"], shape["K"], shape["D"], shape["N"], shape["S"] > 0, shape["S"],
                        True, 64)
    if world > 1:
        assert dist.get_world_size() == world and dist.get_backend() == "nccl", \
            "the expert-parallel arm needs the NCCL process group of all ranks"
    backend = ep.CudaBackend(skb, cfg, SEED, SCALE, rank, world, device=local,
                             max_rows=max(64, 4 * B * shape["K"]))
    layer = ep.ExpertParallelLayer(backend, peer_combine=args.peer_combine or args.peer_dispatch or args.fused_push,
                                   peer_dispatch=args.peer_dispatch, fused_push=args.fused_push,
                                   peer_rows=world * B * shape["K"])
    xs = [torch.from_numpy(make_tokens(B, shape["D"], 2 + 17 * rank + i)).cuda() for i in range(8)]
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    ssh = s if shape["S"] else 0.0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(args.warmup + args.steps):
        flush.zero_()
        if i >= args.warmup:
            ev[i - args.warmup][0].record()
        y = layer.forward(xs[i % 8], s, ssh)
        if i >= args.warmup:
            ev[i - args.warmup][1].record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = float(sum(a.elapsed_time(b) for a, b in ev))
    if world > 1:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms = total_ms / args.steps
    # end to end: pinned host tokens in, host outputs out, per step
    xin = [x.cpu().pin_memory() for x in xs]
    yout = torch.empty((B, shape["D"]), dtype=torch.float32).pin_memory()
    xdev = torch.empty_like(xs[0])
    e2e_t = []
    for i in range(3 + min(args.steps, 50)):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        xdev.copy_(xin[i % 8], non_blocking=True)
        yout.copy_(layer.forward(xdev, s, ssh), non_blocking=True)
        torch.cuda.synchronize()
        if i >= 3:
            e2e_t.append((time.perf_counter() - t0) * 1e3)
    e2e_ms = float(np.mean(e2e_t))
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    # algorithmic bytes of this rank's step (upper bound on the union of kept rows)
    ids, _ = backend.route(xs[0])
    torch.cuda.synchronize()
    idn = ids.cpu().numpy().reshape(-1)
    keep_r = shape["N"] - n_off(s, shape["N"])
    keep_s = shape["S"] - n_off(ssh, shape["S"]) if shape["S"] else 0
    cnt = np.bincount(idn, minlength=shape["E"])
    r_down = int(np.minimum(shape["N"], cnt * keep_r).sum())
    D = shape["D"]
    bytes_alg = (shape["E"] * D * 2 + int((cnt > 0).sum()) * 2 * shape["N"] * D * 2 + r_down * D * 2
                 + (2 * shape["S"] * D * 2 + min(shape["S"], B * keep_s) * D * 2 if shape["S"] else 0)
                 + B * D * 8)
    clocks = sampler.stop() if rank == 0 else None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        # the reference CPU layer beside it, on a bounded sample of this rank's batch
        cpu = cpu_reference(shape, min(B, 256), s, reps=1)
    if rank == 0:
        gbs = bytes_alg / (ms * 1e-3) / 1e9
        print(json.dumps({
            "metric": "MoE-layer tokens/s (decode) at intra-expert sparsity s; HBM GB/s in roofline/sweep",
            "value": round(world * B / (ms * 1e-3), 1), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": {"workload": f"{shape['name']} shape, E={shape['E']} top-{shape['K']} "
                                   f"d_model={D} d_ffn={shape['N']} d_shared={shape['S']}, "
                                   f"batch {B} decode per GPU, top-k neuron selection s={s}",
                       "sparsity": s, "batch_per_gpu": B,
                       "parallelism": f"expert parallel x{world}: experts sharded, ids all-gathered, " +
                                      ("packed bf16 rows stored into the owners' peer-mapped "
                                       "receive buffers (no collective) and "
                                       if args.peer_dispatch else "one packed bf16 all-to-all-v out and ") +
                                      ("peer-memory stores back (no second collective)"
                                       if (args.peer_combine or args.peer_dispatch or args.fused_push)
                                       else "one fp32 all-to-all-v back") +
                                      (" written by the expert layer's last kernel" if args.fused_push else "") +
                                      " over NCCL / NVLink, shared expert replicated",
                       "l2": "512 MiB memset between steps (inside the timed pair is only the "
                             "layer) + ring of 8 token batches",
                       "launch": "direct launches; the send/receive matrix crosses to the host "
                                 "once per step (NCCL takes split sizes from the host)"},
            "bytes_alg_per_step_rank0_upper_bound": int(bytes_alg),
            "roofline": {"bound": "hbm", "kernel": "whole EP step (rank 0)", "achieved": round(gbs, 1),
                         "peak": hbm_peak, "unit": "GB/s", "frac": round(gbs / hbm_peak, 4),
                         "traffic": None, "peak_source": peak_src},
            "e2e": {"value": round(world * B / (e2e_ms * 1e-3), 1), "unit": "tokens/s",
                    "ms_per_step": round(e2e_ms, 5), "h2d_bytes_per_step": B * D * 4,
                    "d2h_bytes_per_step": B * D * 4},
            "gpu_launches": None, "clocks": clocks, "cpu_baseline": cpu,
            "ep_stats": layer.last_stats}))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (this layer has no CPU path)")
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2605_08575_b200 as skb
    _TOKEN_SOURCE[0] = skb.generate_tokens

    if args.ep or (world > 1 and args.workload in ("maverick", "gptoss")):
        return run_ep(args, torch, dist, skb, rank, world, local)

    shape = WORKLOADS[args.workload]
    B, s = args.batch, args.sparsity
    hbm_peak, peak_src = peaks()

    def mk_layer(sh):
        cfg = skb.MoEConfig(sh["E"], sh["K"], sh["D"], sh["N"], sh["S"] > 0, sh["S"], True, 64)
        return skb.MoELayerWeights.generate_synthetic(cfg, SEED, SCALE, device=local)

    layer = mk_layer(shape)
    pt = Point(skb, torch, layer, shape, B, make_layer=mk_layer)
    bytes_ring = pt.bytes_for(s)
    n_rot = pt.rotation(float(np.mean([b["total"] for b in bytes_ring])))

    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()

    # ---- headline: device-resident value ----
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms_dev, graphed = pt.time_device(s, args.steps, args.warmup, use_graph=not args.no_graph)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = ms_dev * args.steps
    if world > 1:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = world * B / (ms_per_step * 1e-3)

    # ---- dominant kernel, live: per-stage events ----
    stage_steps = max(10, min(args.steps, 50))
    stages = pt.time_stages(s, stage_steps, 3)
    launches_per_step = layer.last_launches()
    mean_bytes = {k: float(np.mean([b[k] for b in bytes_ring])) for k in bytes_ring[0]}
    if launches_per_step == 1:
        # decode batches: the whole layer is ONE persistent launch (decode_fused_kernel); its
        # algorithmic bytes are the layer's, its duration the single stage the library reports
        dom, dom_name, dom_bytes = "gateup", "decode_fused_kernel", mean_bytes["total"]
        stages = dict(stages)
        stages["gateup_isolated_launch"] = stages["gateup"]
        stages["gateup"] = ms_per_step  # the launch IS the step: its back-to-back duration
    else:
        dom = max(("gateup", "down"), key=lambda k: stages[k])
        dom_name = {"gateup": "grouped_tc_kernel<TN,0> (gate/up + SwiGLU)",
                    "down": "grouped_tc_kernel<TN,1> / down_cluster_kernel"}[dom]
        dom_bytes = mean_bytes[dom]
    dom_gbs = dom_bytes / (stages[dom] * 1e-3) / 1e9
    # DRAM traffic of that kernel from the committed ncu --set full capture of this workload
    traffic, traffic_src = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        key = f"{args.workload}:{B}:{'decode_fused' if launches_per_step == 1 else dom}"
        if key in tr and abs(s - 0.5) < 1e-9:
            traffic, traffic_src = int(tr[key]["bytes"]), tr[key]["capture"]
    except (OSError, ValueError, KeyError):
        pass
    # algorithmic FLOPs of that kernel: gate/up 2 * rows * 2N * D, down 2 * kept * D
    rows_r, rows_s = B * shape["K"], (B if shape["S"] else 0)
    if launches_per_step == 1:
        dom_flops = None
    elif dom == "gateup":
        dom_flops = 2.0 * (rows_r * 2 * shape["N"] + rows_s * 2 * shape["S"]) * shape["D"]
    else:
        dom_flops = 2.0 * (rows_r * (shape["N"] - n_off(s, shape["N"])) +
                           rows_s * (shape["S"] - n_off(s, shape["S"]))) * shape["D"]
    tf_peak, tf_src = tensor_peak()
    tensor_bound = dom_flops is not None and dom_flops / (tf_peak * 1e12) > dom_bytes / (hbm_peak * 1e9)
    if tensor_bound:
        dom_tf = dom_flops / (stages[dom] * 1e-3) / 1e12
        roofline = {"bound": "tensor", "kernel": dom_name, "achieved": round(dom_tf, 1),
                    "peak": tf_peak, "unit": "TFLOP/s", "frac": round(dom_tf / tf_peak, 4),
                    "traffic": None, "traffic_source": None, "peak_source": tf_src,
                    "algorithmic_flops_per_launch": int(dom_flops),
                    "algorithmic_bytes_per_launch": int(dom_bytes),
                    "hbm_frac": round(dom_gbs / hbm_peak, 4),
                    "kernel_ms": round(stages[dom], 5),
                    "stage_ms": {k: round(v, 5) for k, v in stages.items()}}
    else:
        roofline = {"bound": "hbm", "kernel": dom_name,
                    "achieved": round(dom_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                    "frac": round(dom_gbs / hbm_peak, 4), "traffic": traffic,
                    "traffic_source": traffic_src, "peak_source": peak_src,
                    "algorithmic_bytes_per_launch": int(dom_bytes),
                    "kernel_ms": round(stages[dom], 5),
                    "stage_ms": {k: round(v, 5) for k, v in stages.items()}}
    if roofline["bound"] == "hbm" and roofline["frac"] > 1.0:
        roofline["note"] = ("above 1: the peak is the measured COPY bandwidth (reads + writes); a "
                            "read-only weight stream can exceed it (B200 spec 8 TB/s)")
    layer_gbs = mean_bytes["total"] / (ms_per_step * 1e-3) / 1e9
    # the same step timed alone after a memset flush (what round 1 reported)
    iso_ms = pt.time_isolated(s, max(10, min(args.steps, 50)), 3)

    # ---- end to end through the host-buffer entry point ----
    e2e_steps = max(10, min(args.steps, 100))
    e2e_times, h2d, d2h = pt.time_e2e(s, e2e_steps, args.warmup)
    e2e_ms = float(np.mean(e2e_times))
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": round(world * B / (e2e_ms * 1e-3), 1), "unit": "tokens/s",
           "ms_per_step": round(e2e_ms, 5), "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}

    # ---- sparsity sweep on this workload + the north-star point ----
    sweep = []

    def entry(point, sh, bb, ss, br=None, flags=0, **extra):
        br = br if br is not None else point.bytes_for(ss)
        tot = float(np.mean([b["total"] for b in br]))
        point.rotation(tot)
        m, _ = point.time_device(ss, sw_steps, 3, use_graph=not args.no_graph, flags=flags)
        return {"workload": sh["name"], "batch": bb, "sparsity": ss, "ms_per_step": round(m, 5),
                "tokens_per_s": round(bb / (m * 1e-3), 1), "bytes_alg": int(tot),
                "layer_gbs": round(tot / (m * 1e-3) / 1e9, 1),
                "layer_frac_of_hbm_roofline": round(tot / (m * 1e-3) / 1e9 / hbm_peak, 4),
                "weight_images_in_rotation": len(point.layers), **extra}

    if not args.no_sweep and rank == 0:
        sw_steps = max(20, min(args.steps, 100))
        for ss in SWEEP_S:
            sweep.append(entry(pt, shape, B, ss, bytes_ring if ss == s else None))
        # the 1e-2 (bf16) parity mode: h rounded to bf16 before the down projection
        sweep.append(entry(pt, shape, B, s, bytes_ring, flags=skb.FLAG_BF16_H,
                           accumulation="bf16 h (1e-2 parity mode, SKB_FLAG_BF16_H)"))
        # the threshold runtime path (forward_sparse) on the same workload,
        # tau = the reference's calibrate_tau for a 0.5 target on these synthetic weights
        if args.workload in THRESHOLD_TAU:
            tau, tau_src = calibrated_tau(args.workload, not args.no_cpu and world == 1)
            m, _ = pt.time_device(("tau", tau), sw_steps, 3, use_graph=not args.no_graph)
            rep = skb.forward_sparse(layer, pt.x_host[0], tau)
            ent = {"workload": shape["name"], "batch": B, "mode": "threshold (forward_sparse)",
                   "tau": tau, "tau_source": tau_src,
                   "achieved_routed_sparsity": round(rep.achieved_routed_sparsity, 4),
                   "ms_per_step": round(m, 5), "tokens_per_s": round(B / (m * 1e-3), 1),
                   "tiles_skipped_frac": round(rep.tiles_skipped / max(1, rep.tiles_total), 4)}
            if not args.no_cpu and world == 1:
                ent["cpu_reference"] = cpu_reference_sparse(shape, B, tau)
            sweep.append(ent)
        # the other batch sizes of this workload's range (configs[1]: batch 1-256), s = 0.5
        for bb in (1, 16, 64):
            if bb == B:
                continue
            pb = Point(skb, torch, layer, shape, bb, make_layer=mk_layer)
            pb.layers = list(pt.layers)
            for lay in pb.layers:
                lay.reserve(bb)
            sweep.append(entry(pb, shape, bb, 0.5))
            pt.layers = list(pb.layers)  # keep images the larger rotation added
            del pb
        if args.workload != "olmoe" or B != 1:
            sh = WORKLOADS["olmoe"]
            l2 = mk_layer(sh)
            p2 = Point(skb, torch, l2, sh, 1, make_layer=mk_layer)
            for ss in SWEEP_S:
                e = entry(p2, sh, 1, ss)
                if ss == 0.5:
                    e["north_star_point"] = True
                    e["ms_per_step_isolated_launch_dirty_l2"] = round(p2.time_isolated(ss, sw_steps, 3), 5)
                sweep.append(e)
            # the threshold runtime path on the same point (fused decode kernel: the gate rows
            # stream alone, W_up / W_down rows are gathered for the survivors): algorithmic bytes
            # = router + gate of the routed experts + 2 x surviving rows + token/output rows
            tau, tau_src = calibrated_tau("olmoe", not args.no_cpu and world == 1)
            tb = []
            for xh in p2.x_host:
                rp = skb.forward_sparse(l2, xh, tau, capture=True)
                kept = int(np.asarray(rp.masks.routed).sum())
                nexp = len(np.unique(np.asarray(rp.routes.ids)))
                tb.append(sh["E"] * sh["D"] * W_BYTES + nexp * sh["N"] * sh["D"] * W_BYTES +
                          2 * kept * sh["D"] * W_BYTES + sh["D"] * 8)
            tot = float(np.mean(tb))
            p2.rotation(tot)
            m, _ = p2.time_device(("tau", tau), sw_steps, 3, use_graph=not args.no_graph)
            sweep.append({"workload": sh["name"], "batch": 1, "mode": "threshold (forward_sparse)",
                          "tau": tau, "tau_source": tau_src,
                          "achieved_routed_sparsity": round(rp.achieved_routed_sparsity, 4),
                          "ms_per_step": round(m, 5), "tokens_per_s": round(1 / (m * 1e-3), 1),
                          "bytes_alg": int(tot), "layer_gbs": round(tot / (m * 1e-3) / 1e9, 1),
                          "layer_frac_of_hbm_roofline": round(tot / (m * 1e-3) / 1e9 / hbm_peak, 4),
                          "weight_images_in_rotation": len(p2.layers)})
            # decode batch sizes on the same shape, s = 0.5
            for bb in (2, 4, 8, 16):
                pb = Point(skb, torch, l2, sh, bb, make_layer=mk_layer)
                pb.layers = list(p2.layers)
                for lay in pb.layers:
                    lay.reserve(bb)
                sweep.append(entry(pb, sh, bb, 0.5))
                del pb
            del p2, l2

    clocks = sampler.stop() if rank == 0 else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_reference(shape, B, s, reps=2)

    if rank == 0:
        line = {
            "metric": "MoE-layer tokens/s (decode) at intra-expert sparsity s; HBM GB/s in roofline/sweep",
            "value": round(value, 1), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"{shape['name']} shape, E={shape['E']} top-{shape['K']} "
                                   f"d_model={shape['D']} d_ffn={shape['N']} d_shared={shape['S']}, "
                                   f"batch {B} decode per GPU, top-k neuron selection s={s}",
                       "sparsity": s, "batch_per_gpu": B,
                       "weights": f"generate_synthetic(seed={SEED}, scale={SCALE}) as bf16 image",
                       "parallelism": "single GPU" if world == 1 else f"token-sharded replicas x{world}",
                       "l2": f"inputs larger than L2: steps rotate over {n_rot} identical weight "
                             f"images ({n_rot - 1} x {int(mean_bytes['total']) >> 20} MB of other "
                             "weights stream between two uses of an image; L2 = 126 MB), image r "
                             "with token batch r",
                       "timing": "steps back to back inside one CUDA-event pair",
                       "launch": "CUDA graph replay" if graphed else "direct launches + PDL",
                       "accumulation": "fp32 (h kept fp32; 1e-5 parity mode)"},
            "layer_gbs": round(layer_gbs, 1), "layer_frac_of_hbm_roofline": round(layer_gbs / hbm_peak, 4),
            "ms_per_step_isolated_launch_dirty_l2": round(iso_ms, 5),
            "bytes_alg_per_step": int(mean_bytes["total"]),
            "roofline": roofline, "e2e": e2e, "gpu_launches": int(launches_per_step * args.steps),
            "launches_per_step": int(launches_per_step), "clocks": clocks,
            "cpu_baseline": cpu, "sweep": sweep,
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------------------------
# the reference's CPU implementation (oracle/_ref, built from /root/reference unmodified)
# ---------------------------------------------------------------------------------------------
def _ref_layer(shape):
    from oracle.pyoracle import Config, Ref, RefLayer
    if not Ref.available():
        return None, None
    cfg = Config(shape["E"], shape["K"], shape["D"], shape["N"], shape["S"], True)
    lay = RefLayer.synthetic(cfg, SEED, SCALE).round_bf16()
    return lay, cfg


def _ref_step(lay, x, s, shared, threads):
    routed, sh = lay.build_topk_masks(x, s, 1 if shared else 0)
    lay.forward_masked_dense(x, routed, sh, threads=threads)


def cpu_reference(shape, B, s, reps):
    """build_topk_masks + forward_masked_dense of the unmodified reference on the host cores."""
    cores = os.cpu_count() or 1
    fp32_bytes = (shape["E"] * 3 * shape["N"] + 3 * shape["S"]) * shape["D"] * 4
    if fp32_bytes > 24 << 30:
        return {"value": None, "unit": "tokens/s", "cores": cores, "kind": "reference",
                "sample": "skipped: fp32 model does not fit the bounded-sample budget"}
    lay, _ = _ref_layer(shape)
    if lay is None:
        return {"value": None, "unit": "tokens/s", "cores": cores, "kind": "reference",
                "sample": "oracle/_ref/libsparsekit_ref.so missing"}
    x = make_tokens(B, shape["D"], 2)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        _ref_step(lay, x, s, shape["S"] > 0, cores)
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    return {"value": round(B / t, 2), "unit": "tokens/s", "cores": cores, "kind": "reference",
            "ms_per_step": round(t * 1e3, 2),
            "sample": f"full batch {B}, build_topk_masks(s={s}) + forward_masked_dense, "
                      f"threads={cores}, median of {reps}"}


def cpu_reference_sparse(shape, B, tau):
    """forward_sparse of the unmodified reference on the host cores (one timed call)."""
    cores = os.cpu_count() or 1
    lay, _ = _ref_layer(shape)
    if lay is None:
        return None
    x = make_tokens(B, shape["D"], 2)
    t0 = time.perf_counter()
    lay.forward_sparse(x, tau, threads=cores)
    t = time.perf_counter() - t0
    return {"value": round(B / t, 2), "unit": "tokens/s", "cores": cores, "kind": "reference",
            "ms_per_step": round(t * 1e3, 2), "sample": f"full batch {B}, forward_sparse, one call"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from oracle.pyoracle import Oracle
    _TOKEN_SOURCE[0] = Oracle.get().generate_tokens
    shape = WORKLOADS[args.workload]
    B, s = args.batch, args.sparsity
    cores = os.cpu_count() or 1
    lay, _ = _ref_layer(shape)
    if lay is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libsparsekit_ref.so missing"}))
        return
    steps, warmup = min(args.steps, 5), min(args.warmup, 1)
    xs = [make_tokens(B, shape["D"], 2 + i) for i in range(8)]
    ts = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        _ref_step(lay, xs[i % 8], s, shape["S"] > 0, cores)
        if i >= warmup:
            ts.append(time.perf_counter() - t0)
    ms = float(np.mean(ts)) * 1e3
    val = round(B / (ms * 1e-3), 2)
    line = {
        "impl": "reference",
        "metric": "MoE-layer tokens/s (decode) at intra-expert sparsity s; HBM GB/s in roofline/sweep",
        "value": val, "unit": "tokens/s", "n_gpus": world, "steps": steps, "warmup": warmup,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{shape['name']} shape, E={shape['E']} top-{shape['K']} "
                               f"d_model={shape['D']} d_ffn={shape['N']} d_shared={shape['S']}, "
                               f"batch {B} decode per GPU, top-k neuron selection s={s}",
                   "sparsity": s, "batch_per_gpu": B,
                   "note": "reference CPU layer (unmodified sources), rank 0 only; steps capped at 5"},
        "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": cores, "kind": "reference",
                         "sample": f"full batch {B}, build_topk_masks + forward_masked_dense, "
                                   f"threads={cores}, mean of {steps}"},
        "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="granite", choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--sparsity", type=float, default=0.5)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ep", action="store_true", help="expert-parallel arm (ep.py) at any rank count")
    ap.add_argument("--peer-combine", action="store_true",
                    help="--ep: combine through peer-mapped buffers instead of the second all-to-all")
    ap.add_argument("--fused-push", action="store_true",
                    help="--ep --peer-combine: the expert layer's last kernel writes into the home buffers")
    ap.add_argument("--peer-dispatch", action="store_true",
                    help="--ep: both directions through peer-mapped buffers (no data-path collective)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        # started as a plain process: become N ranks (one per GPU) through torch.distributed.run,
        # the way the driver launches the multi-GPU runs.  NCCL's communicator log goes to stderr.
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd, env=env))
    if args.gpus > 1 and args.impl == "ours":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        if world != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
