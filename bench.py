#!/usr/bin/env python
"""Dion2 optimizer-step benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (N = 1): BASELINE configs[1], the 1B-class transformer matrix set
(24 layers of Wq, Wk, Wv, Wo 2048x2048, W_up 8192x2048, W_down 2048x8192;
144 matrices, 1.208 B parameters), fp32 W / M / G, alpha = 0.25, auto axis,
5 Newton-Schulz steps on the tcgen05 path (fp16 operands, fp32 accumulation;
DESIGN.md R24).  One "step" = one Dion2
update of every matrix (Alg. 1 over the whole model).  Synthetic data:
W0 ~ N(0, 1/n), G ~ N(0, 1) from a seeded generator, M0 = 0.  The inputs
(14.5 GB touched per step) are far larger than L2 (126 MB), so no flush is
needed between steps.  The same library at alpha = 1 (full Muon) is timed
beside it, as is the fp64 oracle on the host cores (cpu_baseline).

Prints ONE JSON line (rank 0); per-phase times and the sweeps go to the sidecar
gpurun_out/bench_details_<config>_n<N>.json.  `--gpus N` without torchrun re-launches
this script under torch.distributed.run (one rank per GPU, owner-compute step).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


def model_shapes(name: str, layers: int = 0):
    from synth import layer_set_1b, layer_set_8b
    if name == "1b":
        return layer_set_1b(layers or 24)
    if name == "1b16":
        return layer_set_1b(16)
    if name == "8b":
        return layer_set_8b(32)
    if name == "stress":  # configs[4]: embedding-like and MLP stress shapes (run at alpha = 0.0625)
        return [(4096, 32768), (28672, 8192)]
    raise ValueError(name)


LAYER_MATS = {"1b": 6, "1b16": 6, "8b": 7, "stress": 2}  # matrices per layer (the oracle's sample unit)
CONFIG_LABEL = {"1b": "configs[1]", "1b16": "configs[1], 16-layer variant (paper Table 1 depth)",
                "8b": "configs[3] matrix set on one GPU", "stress": "configs[4] stress shapes on one GPU"}


def ns_uses_gram_form(p, q, ns_form="auto"):
    """The library's choice (dion2_api.cu build_layout, reading R23): Gram space iff the
    256-padded wide X has q >= 2p or the unpadded one does (AUTO; per matrix here, per shape
    group in the library, identical for the benchmark sets)."""
    if ns_form != "auto":
        return ns_form == "gram"
    pad = lambda v: (v + 255) // 256 * 256  # noqa: E731
    return pad(q) >= 2 * pad(p) or q >= 2 * p


def ns_segments(steps=5, a=3.4445, growth=64.0):
    """Restart segment lengths of the Gram-space form (dion2_api.cu ns_segments, reading R24):
    [3, 2] for the default quintic at T = 5."""
    segs, cur, prod = [], 0, 1.0
    for _ in range(steps):
        if cur and prod * a > growth:
            segs.append(cur)
            cur, prod = 0, 1.0
        cur += 1
        prod *= a
    segs.append(cur)
    return segs


def work_model(shapes, alpha, steps=5, mt=False, ns_form="auto"):
    """Algorithmic work per Dion2 step and per-phase algorithmic HBM bytes.
    NS FLOPs of the form the library evaluates (full products; symmetric tiles not credited):
      direct: T(4p^2 q + 2p^3)  -- gram 2p^2q, poly 2p^3, apply 2p^2q per iteration
      Gram space with restarts (R23, R24): per segment of Ts iterations a gram and an apply
      (4p^2 q) and (4 Ts - 3) p x p products (Ts polys, 3 Ts - 3 products C.Q / C.A / C.(CA)):
      8p^2 q + 28 p^3 at T = 5 (segments 3 + 2)."""
    ns_flops = {"ns_gram": 0.0, "ns_poly": 0.0, "ns_apply": 0.0, "ns_mul": 0.0}
    byts = {"momentum_score": 0.0, "momentum_score_mt": 0.0}
    for ph in ("gather", "gather_rows", "gather_cols", "scatter", "scatter_rows", "scatter_cols"):
        byts[ph] = 0.0
    segs = ns_segments(steps)
    for (m, n) in shapes:
        rows = m <= n
        d, o = (m, n) if rows else (n, m)
        k = max(1, min(d, int(math.floor(alpha * d + 0.5))))
        p, q = min(k, o), max(k, o)
        if ns_uses_gram_form(p, q, ns_form):
            for ts in segs:
                ns_flops["ns_gram"] += 2.0 * p * p * q
                ns_flops["ns_poly"] += ts * 2.0 * p ** 3
                ns_flops["ns_mul"] += max(0, 3 * ts - 3) * 2.0 * p ** 3
                ns_flops["ns_apply"] += 2.0 * p * p * q
        else:
            ns_flops["ns_gram"] += steps * 2.0 * p * p * q
            ns_flops["ns_poly"] += steps * 2.0 * p ** 3
            ns_flops["ns_apply"] += steps * 2.0 * p * p * q
        k1 = "momentum_score_mt" if (mt and not rows) else "momentum_score"
        byts[k1] += m * n * 12.0 + d * 4.0                    # read G, read M, write M, write scores
        # the library's path choice (dion2_api.cu build_layout)
        if rows and k <= n:
            sfx = "_rows"
        elif (not rows) and k <= m and k <= 1024:
            sfx = "_cols"
        else:
            sfx = ""
        gsfx = "_rows" if (mt and not rows) else sfx           # transposed M: row gather of M^T
        byts["gather" + gsfx] += k * o * (4.0 + 4.0 + 2.0)    # read M[K], write mu*M[K], write fp16 X
        byts["scatter" + sfx] += k * o * (2.0 + 4.0 + 4.0)    # read fp16 O, read+write W[K]
    return ns_flops, byts


def mma_flops(shapes, alpha, steps=5, ns_form="auto"):
    """FLOPs the tensor cores actually execute per step: padded dims (p_pad, q_pad multiples of
    256) and, for the symmetric products (gram, poly, Gram-space p x p products), only the
    upper-triangle 256 x 256 tiles: T(T+1)/2 of T^2 with T = p_pad / 256.  The apply is a full
    product.  (work_model's counts are unpadded full products.)"""
    pad = lambda v: (v + 255) // 256 * 256  # noqa: E731
    tot = 0.0
    segs = ns_segments(steps)
    for (m, n) in shapes:
        d, o = (m, n) if m <= n else (n, m)
        k = max(1, min(d, int(math.floor(alpha * d + 0.5))))
        p, q = pad(min(k, o)), pad(max(k, o))
        T = p // 256
        sym = T * (T + 1) / 2 / (T * T)
        if ns_uses_gram_form(min(k, o), max(k, o), ns_form):
            for ts in segs:
                tot += sym * 2.0 * p * p * q + 2.0 * p * p * q + sym * (ts + max(0, 3 * ts - 3)) * 2.0 * p ** 3
        else:
            tot += steps * (sym * 2.0 * p * p * q + sym * 2.0 * p ** 3 + 2.0 * p * p * q)
    return tot


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------- our arm

def build_state(shapes, device, seed=0, fan_in=None, m_transposed=None):
    """Flat fp32 W / M / G buffers with one row-major view per matrix (W0 ~ N(0, 1/fan-in));
    M[i] is a (cols, rows) view when m_transposed[i] (column-mode matrices)."""
    import torch
    total = sum(m * n for m, n in shapes)
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    W = torch.empty(total, dtype=torch.float32, device=device)
    G = torch.empty(total, dtype=torch.float32, device=device)
    M = torch.zeros(total, dtype=torch.float32, device=device)
    W.normal_(0.0, 1.0, generator=gen)
    G.normal_(0.0, 1.0, generator=gen)
    Ws, Ms, Gs, off = [], [], [], 0
    for i, (m, n) in enumerate(shapes):
        Ws.append(W[off:off + m * n].view(m, n).mul_(1.0 / math.sqrt(fan_in[i] if fan_in else n)))
        mt = bool(m_transposed[i]) if m_transposed else False
        Ms.append(M[off:off + m * n].view((n, m) if mt else (m, n)))
        Gs.append(G[off:off + m * n].view(m, n))
        off += m * n
    return (W, M, G), Ws, Ms, Gs


def time_steps(opt, Ws, Ms, Gs, steps, warmup, dist_barrier=None):
    import torch
    if getattr(opt, "cuda_graph", False):
        warmup = max(warmup, 2)  # graph mode captures on a key's second call: keep it untimed
    for _ in range(warmup):
        opt.step(Ws, Ms, Gs)
    torch.cuda.synchronize()
    if dist_barrier:
        dist_barrier()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        opt.step(Ws, Ms, Gs)
    e1.record(s)
    torch.cuda.synchronize()
    if dist_barrier:
        dist_barrier()
    return e0.elapsed_time(e1) / steps


def cpu_oracle_baseline(shapes, alpha, budget_s=20.0, per_layer=6):
    """Time the fp64 oracle (as it stands) on a bounded sample of the workload:
    whole layers (per_layer matrices each) until ~budget_s; scaled to ms per model step."""
    import oracle as O
    from synth import gen_grad, gen_w0
    per_layer = min(per_layer, len(shapes))
    layers = len(shapes) // per_layer
    cfg = O.OracleConfig(alpha=alpha)
    t_used, done = 0.0, 0
    for L in range(layers):
        mats = shapes[L * per_layer:(L + 1) * per_layer]
        data = [(gen_w0(m, n, 0, L * per_layer + i).astype(np.float64), np.zeros((m, n)),
                 gen_grad(m, n, 0, L * per_layer + i, 0).astype(np.float64)) for i, (m, n) in enumerate(mats)]
        t0 = time.perf_counter()
        for (W, M, G) in data:
            O.dion2_step(W, M, G, cfg)
        t_used += time.perf_counter() - t0
        done += 1
        if t_used >= budget_s:
            break
    ms_model = t_used / done * layers * 1e3
    cores = len(os.sched_getaffinity(0))
    return {"value": ms_model, "unit": "ms/step", "cores": cores, "kind": "oracle",
            "sample": f"{done} of {layers} layers ({done * per_layer} matrices) at alpha={alpha}, one step, "
                      f"fp64 NumPy; scaled x{layers / done:.1f} to the whole model"}


def select_counts(shapes, alpha):
    ks = []
    for (m, n) in shapes:
        d = m if m <= n else n
        ks.append(max(1, min(d, int(math.floor(float(np.float32(alpha)) * d + 0.5)))))
    return ks


def e2e_run(opt, Ws, Ms, Gs, G_flat, steps, ks):
    """End to end through the public API: pinned host G -> device, the step, and the
    selected index sets + status word read back, every step, inside the timed region."""
    import torch
    host_G = torch.empty(G_flat.numel(), dtype=G_flat.dtype, pin_memory=True)
    host_G.copy_(G_flat.cpu())
    sel_dev = torch.empty(sum(ks), dtype=torch.int32, device=G_flat.device)
    sel_views, off = [], 0
    for k in ks:
        sel_views.append(sel_dev[off:off + k])
        off += k
    sel_host = torch.empty(sum(ks), dtype=torch.int32, pin_memory=True)
    # per-matrix views of the pinned host buffer (the user's host gradients)
    host_views, off = [], 0
    for g in Gs:
        host_views.append(host_G[off:off + g.numel()].view(g.shape))
        off += g.numel()
    pipelined = hasattr(opt, "step_host")
    for _ in range(2):  # untimed: plans and, in graph mode, the captures (a key's second call)
        if pipelined:
            opt.step_host(Ws, Ms, Gs, host_views, sel_out=sel_views)
        else:
            opt.step(Ws, Ms, Gs, sel_out=sel_views)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        if pipelined:  # host-to-device upload chunk by chunk, overlapped with the earlier chunks' steps
            opt.step_host(Ws, Ms, Gs, host_views, sel_out=sel_views)
        else:
            G_flat.copy_(host_G, non_blocking=True)
            opt.step(Ws, Ms, Gs, sel_out=sel_views)
        sel_host.copy_(sel_dev, non_blocking=True)
    e1.record(s)
    torch.cuda.synchronize()
    rc, _ = opt.status()
    return e0.elapsed_time(e1) / steps, G_flat.numel() * G_flat.element_size(), sum(ks) * 4, rc


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2512_16928_b200 import Dion2, get_phase_times, last_launch_count, set_phase_timing
    from paper_2512_16928_b200 import dion2 as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # DION2_BENCH_DIST=1 runs the owner-compute path even at N = 1 (single-rank NCCL group)
    use_dist = world > 1 or os.environ.get("DION2_BENCH_DIST") == "1"
    if use_dist and world == 1:  # one-rank NCCL group without torchrun
        for k, v in (("RANK", "0"), ("WORLD_SIZE", "1"), ("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29531")):
            os.environ.setdefault(k, v)
    torch.cuda.set_device(local)
    if use_dist:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    barrier = (lambda: dist.barrier()) if world > 1 else None

    shapes = model_shapes(args.config, args.layers)
    n_params = sum(m * n for m, n in shapes)
    if use_dist:
        # owner-compute over all ranks: every matrix sharded along its non-selection axis
        # column-mode shards keep their momentum transposed (local to each rank), as on one GPU
        info0 = D.dist_info(shapes, world, rank, alpha=args.alpha)
        mts = [(not args.no_mt) and ax == 1 for ax in info0["axis"]]
        info = D.dist_info(shapes, world, rank, alpha=args.alpha, m_transposed=mts)
        bufs, Ws, Ms, Gs = build_state(info["shard"], dev, seed=rank, fan_in=[n for (_, n) in shapes],
                                       m_transposed=mts)
        # pieces by direct peer stores / loads over NCCL symmetric memory (DION2_FLAG_DIST_DIRECT:
        # K3 pushes into the owner's window, K7 pulls O; the library falls back to NCCL send /
        # recv where that is unavailable); DION2_BENCH_DIRECT=0 forces send / recv
        direct = os.environ.get("DION2_BENCH_DIRECT", "1") == "1"
        make_opt = lambda a, graph=True: D.Dion2Dist(shapes, alpha=a, axis="auto", precision="bf16",  # noqa: E731
                                                      ns_form=args.ns_form, m_transposed=mts, dist_direct=direct,
                                                      cuda_graph=graph and not args.no_graph)
    else:
        info = None
        # optimizer-state layout: momentum of column-mode matrices stored transposed (the
        # column gather of M[:, K] becomes a contiguous row gather of M^T); --no-mt disables
        mts = [(not args.no_mt) and m > n for (m, n) in shapes]
        bufs, Ws, Ms, Gs = build_state(shapes, dev, seed=rank, m_transposed=mts)
        make_opt = lambda a, graph=True: Dion2(alpha=a, axis="auto", precision="bf16", m_transposed=mts,  # noqa: E731
                                               ns_form=args.ns_form, cuda_graph=graph and not args.no_graph)
    opt = make_opt(args.alpha)

    with ClockSampler(local) as clk:
        ms = time_steps(opt, Ws, Ms, Gs, args.steps, args.warmup, barrier)
    launches = last_launch_count() * args.steps
    rc, bad = opt.status()
    # the exchange the distributed plan actually uses (direct peer memory, or NCCL send / recv)
    xmode = ("direct peer-memory" if opt.exchange_mode() == "direct" else "NCCL send/recv") if use_dist else None
    if rc != 0:
        raise RuntimeError(f"status {rc} (matrix {bad})")

    # the same step without the CUDA graph (every step's launches enqueued by the host)
    ms_eager = None
    if not args.no_graph:
        opt_e = make_opt(args.alpha, graph=False)
        ms_eager = time_steps(opt_e, Ws, Ms, Gs, args.steps, args.warmup, barrier)
        del opt_e

    # per-phase device time (CUDA events on the launching stream around every launch)
    opt_iso = make_opt(args.alpha, graph=False)  # eager: the phase events are recorded per host launch
    opt_iso.step(Ws, Ms, Gs)  # build the plan outside the timed pass
    set_phase_timing(True)
    ms_timed = time_steps(opt_iso, Ws, Ms, Gs, args.steps, 0, None)
    phases = get_phase_times()
    set_phase_timing(False)
    del opt_iso
    torch.cuda.empty_cache()

    peaks, peak_src = load_peaks()
    ns_flops, byts = work_model(shapes, args.alpha, mt=not args.no_mt, ns_form=args.ns_form)
    if use_dist:  # this rank's share: 1/world of every streaming pass, NS of its owned matrices
        owned = [s for s, o in zip(shapes, info["owner"]) if o == rank]
        ns_flops = work_model(owned, args.alpha, ns_form=args.ns_form)[0] if owned else {k: 0.0 for k in ns_flops}
        byts = {k: v / world for k, v in byts.items()}
    per_phase = {}
    for name, (t_ms, cnt) in phases.items():
        if cnt == 0:
            continue
        t = t_ms / args.steps
        ent = {"ms_per_step": t, "launches_per_step": cnt / args.steps}
        if name in ns_flops:
            ent["tflops"] = ns_flops[name] / (t * 1e-3) / 1e12
            ent["frac_bf16_burst"] = ent["tflops"] / peaks["bf16_tflops"]
        if name in byts:
            ent["gbs"] = byts[name] / (t * 1e-3) / 1e9
            ent["frac_hbm"] = ent["gbs"] / peaks["hbm_gbs"]
        per_phase[name] = ent
    ns_ms = sum(per_phase[p]["ms_per_step"] for p in ns_flops if p in per_phase)
    ns_total = sum(ns_flops.values())
    ns_tflops = ns_total / (ns_ms * 1e-3) / 1e12 if ns_ms > 0 else 0.0
    # SURVEY 8(d)'s standard count T(4p^2 q + 2p^3) of the direct iteration: the Gram-space form
    # (R23) computes the same map with fewer FLOPs, so this "equivalent" rate can exceed the peak
    owned_shapes = shapes if not use_dist else [s for s, o in zip(shapes, info["owner"]) if o == rank]
    ns_std = sum(work_model(owned_shapes, args.alpha, ns_form="direct")[0].values()) if owned_shapes else 0.0
    ns_std_tflops = ns_std / (ns_ms * 1e-3) / 1e12 if ns_ms > 0 else 0.0
    ns_mma = mma_flops(owned_shapes, args.alpha, ns_form=args.ns_form) if owned_shapes else 0.0
    # dominant kernel (largest per-step device time)
    dom = max(per_phase, key=lambda p: per_phase[p]["ms_per_step"])
    de = per_phase[dom]
    if dom in ns_flops:
        roof = {"kernel": dom, "bound": "tensor", "achieved": de["tflops"], "peak": peaks["bf16_tflops"],
                "unit": "TFLOP/s", "frac": de["frac_bf16_burst"], "traffic": None,
                "per_launch": f"{ns_flops[dom] / de['launches_per_step'] / 1e12:.4f} TFLOP"}
    else:
        roof = {"kernel": dom, "bound": "hbm", "achieved": de["gbs"], "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": de["frac_hbm"], "traffic": None,
                "per_launch": f"{byts[dom] / de['launches_per_step'] / 1e9:.3f} GB"}
    roof["peak_source"] = f"MEASURED_PEAKS.json ({peak_src}, burst)"
    roof["timing"] = "CUDA events around each launch on the launching stream, separate K-step pass"
    trafp = os.path.join(ROOT, "profiles", "traffic.json")
    # the committed ncu traffic is per launch of the single-GPU 1B step (one launch per phase)
    if os.path.exists(trafp) and not use_dist and args.config == "1b" and not args.layers \
            and de["launches_per_step"] == 1:
        with open(trafp) as f:
            tr = json.load(f)
        if dom in tr:
            roof["traffic"] = tr[dom]

    # alpha = 1 (full Muon, same library)
    ms_a1 = None
    if not args.no_alpha1 and args.alpha != 1.0:
        del opt
        torch.cuda.empty_cache()
        opt1 = make_opt(1.0)
        ms_a1 = time_steps(opt1, Ws, Ms, Gs, max(2, min(args.steps, 5)), max(1, min(args.warmup, 2)), barrier)
        del opt1
        torch.cuda.empty_cache()
        opt = make_opt(args.alpha)
        opt.step(Ws, Ms, Gs)

    # BASELINE configs[1]: the alpha sweep and the forced row / column modes (single GPU; a few
    # steps each; the momentum buffer is re-viewed in W's layout for the forced modes)
    sweep = None
    if not args.no_sweep and not use_dist:
        del opt
        torch.cuda.empty_cache()
        sweep = {"alpha_ms_per_step": {}, "axis_ms_per_step": {}, "steps": 3}
        for a in (1.0, 0.5, 0.25, 0.125):
            if a == 1.0 and ms_a1 is not None:
                sweep["alpha_ms_per_step"]["1.0"] = ms_a1
                continue
            if a == args.alpha:
                sweep["alpha_ms_per_step"][str(a)] = ms
                continue
            o_ = make_opt(a)
            sweep["alpha_ms_per_step"][str(a)] = time_steps(o_, Ws, Ms, Gs, 3, 1, None)
            del o_
            torch.cuda.empty_cache()
        Ms_w, off = [], 0
        for (m, n) in shapes:
            Ms_w.append(bufs[1][off:off + m * n].view(m, n))
            off += m * n
        for ax in ("rows", "cols"):
            o_ = Dion2(alpha=args.alpha, axis=ax, precision="bf16", ns_form=args.ns_form)
            sweep["axis_ms_per_step"][ax] = time_steps(o_, Ws, Ms_w, Gs, 3, 1, None)
            del o_
            torch.cuda.empty_cache()
        # the column-mode matrices (fan-out > fan-in) stored (in, out) as JAX / Flax kernels are
        # (ABI v5 storage_transposed): every selection is then a contiguous row selection
        sts = [m > n for (m, n) in shapes]
        Wt, Mt, Gt, off = [], [], [], 0
        for (m, n), st in zip(shapes, sts):
            sh = (n, m) if st else (m, n)
            Wt.append(bufs[0][off:off + m * n].view(*sh))
            Mt.append(bufs[1][off:off + m * n].view(*sh))
            Gt.append(bufs[2][off:off + m * n].view(*sh))
            off += m * n
        o_ = Dion2(alpha=args.alpha, axis="auto", precision="bf16", ns_form=args.ns_form, storage_transposed=sts)
        sweep["row_selection_layout_ms_per_step"] = time_steps(o_, Wt, Mt, Gt, 3, 1, None)
        if not args.no_e2e:  # its end-to-end time (host G upload: PCIe-bound like the default layout's)
            sweep["row_selection_layout_e2e_ms_per_step"] = e2e_run(o_, Wt, Mt, Gt, bufs[2], 2,
                                                                    select_counts(shapes, args.alpha))[0]
        del o_
        torch.cuda.empty_cache()
        # the same step with bf16 gradients (mixed-precision training): K1 reads 10 B/param
        Gb = bufs[2].to(torch.bfloat16)
        Gbs, off = [], 0
        for (m, n) in shapes:
            Gbs.append(Gb[off:off + m * n].view(m, n))
            off += m * n
        o_ = make_opt(args.alpha)
        sweep["bf16_grad_ms_per_step"] = time_steps(o_, Ws, Ms, Gbs, 3, 1, None)
        del o_, Gbs, Gb
        torch.cuda.empty_cache()
        opt = make_opt(args.alpha)
        opt.step(Ws, Ms, Gs)

    # end to end through the public API (host G)
    e2e_ms, h2d, d2h = None, None, None
    e2e_bf16 = None
    if not args.no_e2e:
        e2e_ms, h2d, d2h, _ = e2e_run(opt, Ws, Ms, Gs, bufs[2], max(2, min(args.steps, 5)),
                                      select_counts(shapes, args.alpha))
        if not use_dist:
            # the same with bf16 gradients (mixed-precision training): half the PCIe bytes
            Gb = bufs[2].to(torch.bfloat16)
            Gbs, off = [], 0
            for (m, n) in shapes:
                Gbs.append(Gb[off:off + m * n].view(m, n))
                off += m * n
            ms_b, h2d_b, _, _ = e2e_run(opt, Ws, Ms, Gbs, Gb, max(2, min(args.steps, 5)),
                                        select_counts(shapes, args.alpha))
            e2e_bf16 = {"value": ms_b, "unit": "ms/step", "h2d_bytes_per_step": h2d_b}
            del Gb, Gbs
            torch.cuda.empty_cache()
    comm = None
    if use_dist:
        opt.step(Ws, Ms, Gs)
        comm = {"sent_bytes_per_step_rank": opt.last_comm_bytes,
                "analytic_piece_bytes_per_step_rank": 2 * sum(info["send_bytes"][o] for o in range(world) if o != rank),
                # the NVLink floor of those bytes (each exchange sends and receives concurrently at
                # 900 GB/s per direction; C2 and C3 follow each other)
                "nvlink_floor_ms": opt.last_comm_bytes / 900e9 * 1e3,
                "exchange": xmode,
                "note": "gather-to-owner + scatter-back of k x (o/P) fp16 pieces, plus the score all-gather"}

    # max over ranks
    if world > 1:
        t = torch.tensor([ms, e2e_ms or 0.0], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e_ms = t.tolist()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_oracle_baseline(shapes, args.alpha, budget_s=args.cpu_budget, per_layer=LAYER_MATS[args.config])

    if rank == 0:
        ns_std_frac = ns_std_tflops / peaks["bf16_tflops"]
        details = {
            "configs1_sweep": sweep,
            "ns_tflops_evaluated": ns_tflops,
            "ns_evaluated_note": "the evaluated form's FLOPs (Gram space with restarts: per segment of Ts "
                                 "iterations 4p^2q + (4Ts-3)2p^3, full products) over the NS kernels' time",
            "ns_frac_bf16_sustained": ns_tflops / peaks["bf16_tflops_sustained"],
            "ns_mma_tflops": ns_mma / (ns_ms * 1e-3) / 1e12 if ns_ms > 0 else 0.0,
            "ns_mma_note": "FLOPs the tensor cores execute (padded dims, upper-triangle tiles of the symmetric "
                           "products) over the NS kernels' time",
            "ns_standard_tflop_per_step": ns_std / 1e12,
            "ns_standard_equiv_tflops": ns_std_tflops,
            "ns_standard_equiv_frac_bf16_burst": ns_std_frac,
            "ns_ms_per_step": ns_ms,
            "e2e_bf16_grad": e2e_bf16,
            "ms_per_step_eager": ms_eager,
            "ms_per_step_with_phase_events": ms_timed,
            "phases_note": "per-kernel times (CUDA events around every launch) from a separate K-step pass",
            "phases": per_phase,
        }
        det_path = None
        if not args.no_details:
            det_dir = os.path.join(ROOT, "gpurun_out")
            os.makedirs(det_dir, exist_ok=True)
            det_path = os.path.join(det_dir, f"bench_details_{args.config}_n{world}.json")
            with open(det_path, "w") as f:
                json.dump(details, f, indent=1)
        out = {
            "metric": "Dion2 optimizer-step ms per model at alpha=0.25 vs alpha=1; NS tensor-peak fraction",
            "value": ms,
            "unit": "ms/step",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": False,
            "scaling": "weak" if world == 1 else "strong",
            "vs_baseline": None,
            "dtype": "f32 state; fp16 NS operands, f32 accumulate",
            "data": "synthetic (W0~N(0,1/n), G~N(0,1), M0=0; seeded device RNG)",
            "config": {"workload": f"{args.config}-set Dion2 step ({CONFIG_LABEL[args.config]})",
                       "matrices": len(shapes), "params": n_params, "alpha": args.alpha, "ns_steps": 5,
                       "ns_form": args.ns_form,
                       "l2_flush": f"not needed: {12 * n_params / 1e9:.1f} GB touched per step >> 126 MB L2",
                       "parallelism": "single GPU" if not use_dist else
                       f"owner-compute over {world} GPUs ({xmode} exchange; shards along the non-selection axis)",
                       "step_mode": "CUDA graph" if not args.no_graph else "eager"},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_ms, "unit": "ms/step", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if comm:
            out["comm"] = comm
        if det_path:
            out["details"] = os.path.relpath(det_path, ROOT)
        # the gate numbers last (BASELINE metric: alpha = 0.25 vs alpha = 1, NS tensor-peak fraction)
        out["alpha1_ms_per_step"] = ms_a1
        out["speedup_vs_alpha1"] = (ms_a1 / ms) if ms_a1 else None
        out["ns_frac_bf16_burst"] = ns_tflops / peaks["bf16_tflops"]
        out["ns_frac_flops"] = "evaluated form (Gram space with restarts), full products"
        out["ns_mma_frac_bf16_burst"] = (ns_mma / (ns_ms * 1e-3) / 1e12 / peaks["bf16_tflops"]) if ns_ms > 0 else 0.0
        print(json.dumps(out))
    if use_dist:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------------- reference arm

def run_reference(args):
    """The reference arm for this tier is the fp64 oracle on the host cores, on our
    arm's config/metric: each step is a bounded sample (one transformer layer of the
    set), reported scaled to ms per whole-model step."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import oracle as O
    from synth import gen_grad, gen_w0
    shapes = model_shapes(args.config)
    per_layer = min(LAYER_MATS[args.config], len(shapes))
    layer = shapes[:per_layer]
    layers = len(shapes) // per_layer
    cfg = O.OracleConfig(alpha=args.alpha)
    data = [(gen_w0(m, n, 0, i).astype(np.float64), np.zeros((m, n)), gen_grad(m, n, 0, i, 0).astype(np.float64))
            for i, (m, n) in enumerate(layer)]
    for _ in range(args.warmup):
        for (W, M, G) in data:
            O.dion2_step(W, M, G, cfg)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for (W, M, G) in data:
            O.dion2_step(W, M, G, cfg)
    dt = (time.perf_counter() - t0) / args.steps
    ms = dt * layers * 1e3
    cores = len(os.sched_getaffinity(0))
    out = {"impl": "reference",
           "metric": "Dion2 optimizer-step ms per model at alpha=0.25 vs alpha=1; NS tensor-peak fraction",
           "value": ms, "unit": "ms/step", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": ms, "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (W0~N(0,1/n), G~N(0,1), M0=0; seeded host RNG)",
           "config": {"workload": f"{args.config}-set Dion2 step ({CONFIG_LABEL[args.config]})", "alpha": args.alpha, "axis": "auto",
                      "ns_steps": 5},
           "cpu_baseline": {"value": ms, "unit": "ms/step", "cores": cores, "kind": "oracle",
                            "sample": f"1 of {layers} layers ({per_layer} matrices) per step, fp64 NumPy, scaled x{layers}"},
           "e2e": {"value": ms, "unit": "ms/step", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def relaunch(n: int) -> int:
    """`python bench.py --gpus N` without torchrun: re-run this command under
    torch.distributed.run with N ranks on this node (rank 0 prints the line)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--alpha", type=float, default=0.25)
    ap.add_argument("--config", default="1b")
    ap.add_argument("--no-alpha1", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--layers", type=int, default=0, help="override the layer count (profiling only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="eager steps (default: Dion2(cuda_graph=True), the step replayed as a CUDA graph)")
    ap.add_argument("--no-sweep", action="store_true", help="skip the alpha sweep / forced axis modes")
    ap.add_argument("--no-mt", action="store_true", help="keep column-mode momentum in W's layout")
    ap.add_argument("--ns-form", choices=["auto", "direct", "gram"], default="auto",
                    help="Newton-Schulz evaluation form (DESIGN.md reading R23)")
    ap.add_argument("--no-details", action="store_true", help="do not write gpurun_out/bench_details_*.json")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args.gpus))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
