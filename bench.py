#!/usr/bin/env python
"""Benchmark of Streaming DiLoCo's per-fragment outer synchronization on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload 1B] [--impl ours|reference]

One process per GPU (torchrun for N > 1), replica m = rank, M = N replicas.
A step is one pass of the whole hot path for the
next fragment on the calendar: schedule -> k_quantize -> NCCL all-gather ->
block-receive -> k_apply (decode + fp32 mean + Nesterov + alpha-merge),
cycling through all P fragments of the workload (1B: 8 fragments of
151M-217M fp32 params, arrays > L2, so no flush is needed).  Inputs are
resident in HBM (synthetic, seeded, synth/); `e2e` repeats the steps through
the same C-ABI calls with the fragment's parameters coming from and going
back to pinned host memory inside the timed region.

Timing: W untimed warm-up steps, then exactly K steps between a barrier +
cuda synchronize on both sides, CUDA events on the compute stream, max over
ranks.  Rank 0 prints one JSON line.  `--impl reference` times the CPU
oracle (oracle/, single thread) on bounded samples of the same workload.
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
sys.path.insert(0, ROOT)

BASELINE = json.load(open(os.path.join(ROOT, "BASELINE.json")))
METRIC = BASELINE["metric"]
UNIT = "params/s"


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        j = json.load(open(path))
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=512)
    ap.add_argument("--warmup", type=int, default=16)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="1B", choices=["toy", "35M", "1B", "4B"])
    ap.add_argument("--scale-block", type=int, default=1024)
    ap.add_argument("--tau", type=int, default=None, help="override the workload's tau (configs[4] sweep)")
    ap.add_argument("--fragment-size", type=int, default=None, help="override |p| in layers (configs[4] sweep)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU time of the cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-m-sweep", action="store_true")
    ap.add_argument("--serial", action="store_true", help="no send/receive pipelining across fragments")
    ap.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                    help="replay each step as a CUDA graph (auto: single GPU, L2-resident small configs)")
    ap.add_argument("--gather", choices=["auto", "ce", "push", "pull", "mc"], default="auto",
                    help="all-gather: NCCL copy engines (ce), fused into the quantize kernel (push) or into "
                         "the merge kernel (pull), one copy-engine write through the NVLS multicast alias (mc), "
                         "or libsd's choice (auto)")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 100 ms, host-stamped."""

    FIELDS = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_index: int):
        self.samples = []
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(gpu_index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                try:
                    self.samples.append((time.time(), float(parts[0]), float(parts[1]), float(parts[2]), parts[3:7]))
                except ValueError:
                    pass

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0: float, t1: float):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "note": "nvidia-smi unavailable"}
        win = [s for s in self.samples if t0 <= s[0] <= t1]
        window = "timed region"
        if len(win) < 3:
            win = [s for s in self.samples if s[3] > 0] or self.samples
            window = "whole GPU phase (timed region shorter than 3 samples)"
        reasons = sorted({self.NAMES[i] for s in win for i, v in enumerate(s[4]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(s[1] for s in win), "sm_max_mhz": max(s[2] for s in win),
                "reasons": reasons, "samples": len(win), "window": window}


# --------------------------------------------------------------------------- host link
def pcie_probe(host, dev_buf, s_in, s_out, reps=5):
    """The host link's ceiling for e2e: pinned H2D alone, D2H alone, and both
    at once on two streams (full duplex), best of `reps`, GB/s per direction."""
    import torch
    nbytes = 4 * host.numel()
    res = {}
    for kind in ("h2d", "d2h", "duplex"):
        best = 0.0
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            if kind in ("h2d", "duplex"):
                s_in.wait_event(a)
                with torch.cuda.stream(s_in):
                    dev_buf.copy_(host, non_blocking=True)
            if kind in ("d2h", "duplex"):
                tmp = host if kind == "d2h" else _probe_pinned(host)
                s_out.wait_event(a)
                with torch.cuda.stream(s_out):
                    tmp.copy_(dev_buf if kind == "d2h" else _probe_dev(dev_buf), non_blocking=True)
            torch.cuda.current_stream().wait_stream(s_in)
            torch.cuda.current_stream().wait_stream(s_out)
            b.record()
            torch.cuda.synchronize()
            best = max(best, nbytes / (a.elapsed_time(b) / 1e3) / 1e9)
        res[kind + "_gbs"] = best
    return res


_PROBE = {}


def _probe_pinned(like):
    import torch
    if "h" not in _PROBE:
        _PROBE["h"] = torch.empty_like(like, pin_memory=True)
    return _PROBE["h"]


def _probe_dev(like):
    import torch
    if "d" not in _PROBE:
        _PROBE["d"] = torch.empty_like(like)
    return _PROBE["d"]


# --------------------------------------------------------------------------- workload
def algorithmic_bytes(n: int, M: int, B: int):
    """quantize reads theta, A (8 B) and writes 0.5 B of codes
    + 4/B of scales; apply reads A, v, theta (12 B) + M payloads and writes
    A, v, theta (12 B).  B = 0: one scale per fragment."""
    nb = 1 if B == 0 else -(-n // B)
    pay = n / 2 + 4 * nb
    return 8 * n + pay, 24 * n + M * pay


def calendar_sends(sd, cfg, count: int):
    """The first `count` (fragment, send step) events from t = H on (libsd's scheduler)."""
    out, t = [], cfg.H
    while len(out) < count:
        send, _ = sd.sd_fragment_schedule(cfg, t)
        out.extend((p, t) for p in send)
        t += 1
    return out[:count]


def workload_with_overrides(wl, args):
    import dataclasses

    kw = {}
    if args.tau is not None:
        kw["tau"] = args.tau
    if args.fragment_size is not None:
        kw["fragment_size"] = args.fragment_size
    return dataclasses.replace(wl, **kw) if kw else wl


def make_cfg(sd, wl, B):
    return sd.sd_config_default(wl.layers, wl.fragment_size, wl.H, tau=wl.tau, alpha=wl.alpha, outer_lr=wl.lr,
                                outer_momentum=wl.mu, scale_block=B)


def workload_config(wl, B, world):
    return {"workload": wl.describe() + f"; M = {world} replica(s), one per GPU; E3M0 B={B}",
            "fragments": None, "l2": "inputs > L2 (fragments of 0.6-0.9 GB per fp32 array, cycled); no flush",
            "parallelism": f"diloco-replicas{world}"}



# --------------------------------------------------------------------------- oracle timing
_SAMPLES = {}


def oracle_sample_rate(wl, B, M, p, segs, S, reps=1):
    """Runs the CPU oracle's full round (or_round: quantize M replicas, mean,
    Nesterov, merge M replicas) on the first S elements of fragment p.
    Inputs are generated once per (fragment, size) and reused (the round
    updates them in place, as successive rounds would).
    Returns (seconds per round, elements per round)."""
    import numpy as np

    import oracle
    import synth

    key = (p, S, M)
    if key not in _SAMPLES:
        A = synth.host_init(segs, p, 0, S)
        thetas = [synth.host_apply_window(A.copy(), segs, p, m, 1) for m in range(M)]
        _SAMPLES[key] = (A, thetas, [t.copy() for t in thetas], np.zeros(S, np.float32))
    A, thetas, merges, v = _SAMPLES[key]
    t0 = time.perf_counter()
    for _ in range(reps):
        oracle.round_(thetas, merges, A, v, B=B, lr=wl.lr, mu=wl.mu, alpha=wl.alpha)
    return (time.perf_counter() - t0) / reps, S


def cpu_baseline(wl, B, M, order, segs, n, target_s):
    """The oracle's full round (all M replicas) over the fragments of the
    calendar in order, whole fragments until ~target_s of CPU time (the last
    one cut to fit), single thread."""
    import oracle  # noqa: F401  (test infrastructure, allowed in this leg only)

    S0 = min(n[order[0]], 1 << 20)
    dt0, _ = oracle_sample_rate(wl, B, M, order[0], segs[order[0]], S0)
    rate = S0 / max(dt0, 1e-9)                       # elements per second, estimate
    budget = rate * target_s
    total_t, total_e, used = 0.0, 0, []
    for p in order:
        S = int(min(n[p], budget - total_e))
        S -= S % 1024
        if S < (1 << 20) and total_e > 0:  # not worth another fragment's input generation
            break
        S = max(S, min(n[p], 1024))
        dt, _ = oracle_sample_rate(wl, B, M, p, segs[p], S)
        total_t += dt
        total_e += S
        used.append(f"{S} of fragment {p}")
        if total_e >= budget:
            break
    _SAMPLES.clear()
    return {"value": total_e * M / total_t, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"or_round on {', '.join(used)} (calendar order), all M={M} replicas: {total_e} elements "
                      f"in {total_t:.2f} s, single thread, -O2 -ffp-contract=off"}


# --------------------------------------------------------------------------- reference arm
def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return 0
    import synth
    from synth.workloads import WORKLOADS
    from paper_2501_18512_b200 import sd

    wl = workload_with_overrides(WORKLOADS[args.workload], args)
    B = args.scale_block
    cfg = make_cfg(sd, wl, B)
    P = sd.sd_fragment_count(cfg)
    lay = [sd.sd_fragment_layout(cfg, p) for p in range(P)]
    segs = [wl.segments(b, e) for b, _, e in lay]
    M = world
    nmin = min(synth.segments_numel(s) for s in segs)
    dt, _ = oracle_sample_rate(wl, B, M, 0, segs[0], min(1 << 18, nmin))
    per_step = min(2.0, 90.0 / max(1, args.steps + args.warmup))
    S = int(min(nmin, max(1 << 16, min(1 << 18, nmin) * per_step / max(dt, 1e-6))))
    S -= S % 1024 if S > 1024 else 0
    events = calendar_sends(sd, cfg, args.warmup + args.steps)
    for p, _ in events[:args.warmup]:
        oracle_sample_rate(wl, B, M, p, segs[p], S)
    total = 0.0
    for p, _ in events[args.warmup:]:
        dt, _ = oracle_sample_rate(wl, B, M, p, segs[p], S)
        total += dt
    value = args.steps * S * M / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(wl, B, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"per step: or_round on the first {S} elements of the calendar's fragment, "
                                   f"all M={M} replicas, single thread"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# --------------------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import synth
    from synth.workloads import WORKLOADS
    from paper_2501_18512_b200 import FragmentSync, sd

    rank, local, world = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    wl = workload_with_overrides(WORKLOADS[args.workload], args)
    B = args.scale_block
    M = world
    cfg = make_cfg(sd, wl, B)
    P = sd.sd_fragment_count(cfg)
    lay = [sd.sd_fragment_layout(cfg, p) for p in range(P)]
    segs = [wl.segments(b, e) for b, _, e in lay]
    n = [synth.segments_numel(s) for s in segs]

    # outer-state store (a2): every fragment's anchor, momentum and live params resident in HBM
    A = [synth.dev_init(torch.empty(n[p], device=dev), segs[p], p) for p in range(P)]
    v = [torch.zeros(n[p], device=dev) for p in range(P)]
    theta = []
    for p in range(P):
        th = A[p].clone()
        synth.dev_apply_window(th, segs[p], p, rank, 1)
        theta.append(th)
    sync = FragmentSync(cfg, n, rank, world, local,
                        gather_mode={"auto": sd.SD_GATHER_AUTO, "ce": sd.SD_GATHER_COPY_ENGINE,
                                     "push": sd.SD_GATHER_PUSH, "pull": sd.SD_GATHER_PULL,
                                     "mc": sd.SD_GATHER_MULTICAST}[args.gather])
    torch.cuda.synchronize()

    K, W = args.steps, max(1, args.warmup)
    events = calendar_sends(sd, cfg, W + K)
    sampler = ClockSampler(local)

    def one_step(p, t, ev=None):
        """Serialized round of fragment p: quantize, gather, block-receive, apply."""
        ctx = sync.ctx
        if ev is not None:
            ev[0].record()
        ctx.sd_outer_grad_quantize(p, t, theta[p], A[p], sync.slot(p), n[p])     # a1 + a3
        if ev is not None:
            ev[1].record()
        ctx.sd_fragment_sync(p, t, sync.gather[p], n[p])                          # a4
        ctx.sd_fragment_wait(p, t + cfg.tau)                                      # a5
        if ev is not None:
            ev[2].record()
        ctx.sd_merge(p, t + cfg.tau, sync.gather[p], theta[p], A[p], v[p], n[p])  # a6
        if ev is not None:
            ev[3].record()

    pending = []

    def pipe_step(p, t, ev=None):
        """Send of fragment p (quantize + async gather), then the receive of the
        fragment sent one step earlier: its gather ran concurrently with this
        quantize (tau >= 1: the receive comes after later compute)."""
        ctx = sync.ctx
        if ev is not None:
            ev[0].record()
        ctx.sd_outer_grad_quantize(p, t, theta[p], A[p], sync.slot(p), n[p])
        if ev is not None:
            ev[1].record()
        ctx.sd_fragment_sync(p, t, sync.gather[p], n[p])
        if pending:
            pp, tt = pending.pop()
            ctx.sd_fragment_wait(pp, tt + cfg.tau)
            if ev is not None:
                ev[2].record()
            ctx.sd_merge(pp, tt + cfg.tau, sync.gather[pp], theta[pp], A[pp], v[pp], n[pp])
            if ev is not None:
                ev[3].record()
        elif ev is not None:
            ev[2].record()
            ev[3].record()
        pending.append((p, t))

    def drain():
        while pending:
            pp, tt = pending.pop()
            sync.ctx.sd_fragment_wait(pp, tt + cfg.tau)
            sync.ctx.sd_merge(pp, tt + cfg.tau, sync.gather[pp], theta[pp], A[pp], v[pp], n[pp])

    pipelined = P > 1 and not args.serial and cfg.tau > 0  # tau = 0: the receive is in the send's step
    step_fn = pipe_step if pipelined else one_step

    # L2 policy: the 1B/4B state (12 B/param, GBs) streams through HBM; small
    # configs (toy, 35M) would stay L2-resident, so they flush L2 between steps
    # and time only the steps (sum of per-step event intervals).
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = 12 * sum(n) < 4 * l2_bytes
    flush_buf = torch.empty(2 * l2_bytes, dtype=torch.uint8, device=dev) if flush else None

    def timed(evs, fn):
        for p, t in evs[:W]:
            fn(p, t)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        kev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
        sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = sd.sd_kernel_launch_count()
        torch.cuda.synchronize()
        t0 = time.time()
        start.record()
        for i, (p, t) in enumerate(evs[W:]):
            if flush:
                flush_buf.zero_()
                sev[i][0].record()
            fn(p, t, kev[i])
            if flush:
                sev[i][1].record()
        stop.record()
        torch.cuda.synchronize()
        t1 = time.time()
        nl = sd.sd_kernel_launch_count() - l0
        drain()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        total = sum(a.elapsed_time(b) for a, b in sev) if flush else start.elapsed_time(stop)
        return total, kev, nl, t0, t1

    ms, kev, launches, w0, w1 = timed(events, step_fn)
    remeasured = False
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    if bad & set(sampler.summary(w0, w1).get("reasons", [])):
        # a throttled timed region is not a valid number: take it once more
        more_ev = calendar_sends(sd, cfg, 7 * (W + K))[6 * (W + K):]
        ms, kev, launches, w0, w1 = timed(more_ev, step_fn)
        events = more_ev
        remeasured = True
    launches0 = 0
    ms_eager = None
    use_graph = args.graph == "on" or (args.graph == "auto" and flush and world == 1)
    if use_graph:
        # Launch-bound small fragments: capture one serialized step per fragment of a
        # calendar cycle as a CUDA graph (libsd's calls are stream-ordered and
        # capturable; the host-side schedule/state checks run once, at capture),
        # then replay one graph per step.  Timed exactly like the eager loop.
        ms_eager = ms
        gev = calendar_sends(sd, cfg, 2 * (W + K) + 2 * P)[2 * (W + K):]
        graphs = []
        for p, t in gev[:P]:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                one_step(p, t)
            graphs.append(g)
        for i in range(W):
            graphs[i % P].replay()
        torch.cuda.synchronize()
        sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.time()
        start.record()
        for i in range(K):
            if flush:
                flush_buf.zero_()
            sev[i][0].record()
            graphs[i % P].replay()
            sev[i][1].record()
        stop.record()
        torch.cuda.synchronize()
        w1 = time.time()
        ms = sum(a.elapsed_time(b) for a, b in sev) if flush else start.elapsed_time(stop)
        applied_g = [gev[i % P] for i in range(K)]
        launches = 2 * K if args.scale_block in (256, 512, 1024) else 3 * K
    q_ms = [e[0].elapsed_time(e[1]) for e in kev]
    a_ms = [e[2].elapsed_time(e[3]) for e in kev]
    if world > 1:
        tms = torch.tensor([ms], device=dev)
        dist.all_reduce(tms, op=dist.ReduceOp.MAX)
        ms = float(tms.item())
    ms_serial = None
    if pipelined and world > 1:
        ser_events = calendar_sends(sd, cfg, 4 * (W + K) + 12)[3 * (W + K) + 12:]
        ms_serial, _, _, _, _ = timed(ser_events, one_step)
        tms = torch.tensor([ms_serial], device=dev)
        dist.all_reduce(tms, op=dist.ReduceOp.MAX)
        ms_serial = float(tms.item())
    st, fb = sync.check()
    if st != sd.SD_OK:
        raise SystemExit(f"libsd reported {sd.STATUS_NAMES[st]} (first bad index {fb})")

    applied = events[W - 1:W + K - 1] if pipelined else events[W:]
    elems_eager = sum(n[p] for p, _ in applied)
    if use_graph:
        applied = applied_g
    elems = sum(n[p] for p, _ in applied)                # fragment elements per replica over K steps
    value = elems * world / (ms / 1e3)                   # whole job: all replicas' elements / max time
    qb = sum(algorithmic_bytes(n[p], M, B)[0] for p, _ in events[W:])
    ab = sum(algorithmic_bytes(n[p], M, B)[1] for p, _ in applied)
    q_gbs = qb / (sum(q_ms) / 1e3) / 1e9
    a_gbs = ab / (sum(a_ms) / 1e3) / 1e9
    peak, peak_src = peaks()
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        tj = json.load(open(tpath)).get(f"k_apply/{args.workload}/M{M}/B{B}")
        if tj:
            traffic = tj["dram_bytes_per_launch"]

    # ---- end to end: the same calls, parameters from / to pinned host memory
    e2e = None
    if not args.no_e2e:
        host = [torch.empty(n[p], dtype=torch.float32, pin_memory=True) for p in range(P)]
        for p in range(P):
            host[p].copy_(theta[p])
        e_events = calendar_sends(sd, cfg, W + K + W + K)[W + K:]
        # Host copies are double-buffered across fragments: while fragment k
        # runs on the compute stream, fragment k+1's parameters come in on
        # one copy engine and fragment k-1's go out on the other (PCIe is
        # full duplex); events order copy -> step -> copy per fragment.
        cs = torch.cuda.current_stream()
        h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
        in_ev = [torch.cuda.Event() for _ in range(P)]
        step_ev = [torch.cuda.Event() for _ in range(P)]
        out_ev = [torch.cuda.Event() for _ in range(P)]

        def h2d(p):
            with torch.cuda.stream(h2d_s):
                h2d_s.wait_event(out_ev[p])          # the previous D2H of this fragment is done
                theta[p].copy_(host[p], non_blocking=True)
                in_ev[p].record(h2d_s)

        def run(evs):
            h2d(evs[0][0])
            for i, (p, t) in enumerate(evs):
                if i + 1 < len(evs):
                    h2d(evs[i + 1][0])
                cs.wait_event(in_ev[p])
                one_step(p, t)
                step_ev[p].record(cs)
                with torch.cuda.stream(d2h_s):
                    d2h_s.wait_event(step_ev[p])
                    host[p].copy_(theta[p], non_blocking=True)
                    out_ev[p].record(d2h_s)
            cs.wait_stream(d2h_s)

        for e in out_ev:
            e.record(cs)
        run(e_events[:W])
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(e_events[W:])
        e1.record()
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if world > 1:
            tms = torch.tensor([ems], device=dev)
            dist.all_reduce(tms, op=dist.ReduceOp.MAX)
            ems = float(tms.item())
        eel = sum(n[p] for p, _ in e_events[W:])
        e2e = {"value": eel * world / (ems / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": 4 * eel // K, "d2h_bytes_per_step": 4 * eel // K,
               "ms_per_step": ems / K, "path": ("pinned host theta -> H2D -> sd_* C-ABI calls -> D2H for every step's fragment; "
                        "copies of neighbouring fragments overlap (two copy streams)"),
               "link_gbs_each_way": 4 * eel / (ems / 1e3) / 1e9,
               "pcie_probe": pcie_probe(host[0], theta[0], h2d_s, d2h_s)}
    sampler.stop()
    clocks = sampler.summary(w0, w1)
    clocks["remeasured_after_throttle"] = remeasured

    # ---- gather hidden behind tau synthetic inner steps? (N > 1 only)
    overlap = None
    if world > 1 and cfg.tau > 0:
        overlap = {}
        for i, kind in enumerate(("adamw", "gemm")):
            base = 5 * (W + K) + 40 * i
            evs = calendar_sends(sd, cfg, base + 40)[base:]
            overlap[kind] = overlap_run(torch, dist, sd, synth, sync, cfg, theta, A, v, n, P, rank, world, evs, dev,
                                        kind=kind)

    # ---- per-GPU kernel work at M = 1/2/4/8 replicas, emulated on this GPU (1 fragment)
    m_sweep = None
    if world == 1 and not args.no_m_sweep:
        m_sweep = m_sweep_run(torch, sd, synth, cfg, segs[0], n[0], B, dev, peak)

    # ---- NEXT-1: the inner AdamW step before a send, separate vs fused with the quantize
    fused = None
    if world == 1 and not args.no_m_sweep:
        fused = fused_inner_run(torch, sd, sync, cfg, theta[0], A[0], n[0], B, dev, peak)

    # ---- NEXT-3: host-offloaded outer state -- transfer cost of one fragment's A, v
    offload = None
    if world == 1 and not args.no_e2e:
        offload = offload_run(torch, sync, A[0], v[0], n, P, dev)

    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl, B, M, [p for p, _ in events[:P]], segs, n, args.cpu_seconds)

    if rank == 0:
        avg_a = statistics.fmean(a_ms)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (seeded counter-based generator, synth/; Chinchilla-shaped fragments)",
            "config": dict(workload_config(wl, B, world), fragments=[int(x) for x in n],
                           gather=("none (M = 1: no collective)" if world == 1 else
                                   "copy engine writes each payload once through the NVLS multicast alias "
                                   "(NVSwitch replicates), flag handshake" if args.gather == "mc" else
                                   "fused into k_apply: NVLink loads of the peers' payloads + flag handshake"
                                   if (args.gather == "pull" or (args.gather == "auto" and cfg.tau == 0 and
                                                                 world in (4, 8))) else
                                   "fused into k_quantize: NVLink stores to the peers' symmetric buffers + "
                                   "flag handshake" if (args.gather == "push" or
                                                        (args.gather == "auto" and cfg.tau == 0)) else
                                   "NCCL in-place all-gather on copy engines (symmetric window, zero CTAs)"),
                           l2=("state (12 B/param) fits in ~4x L2: L2 flushed (2x L2 written) between steps, "
                               "only the steps are timed" if flush else
                               "inputs > L2 (fragments of %.0f-%.0f MB per fp32 array, cycled); no flush"
                               % (4 * min(n) / 1e6, 4 * max(n) / 1e6))),
            "per_gpu_value": value / world,
            "schedule": ("serialized step replayed as a CUDA graph (one per fragment of the cycle)" if use_graph else
                         "pipelined: each step sends fragment k (quantize + async NCCL all-gather) and receives "
                         "fragment k-1 (block-receive + apply), so a gather overlaps the next step's kernels "
                         "(tau >= 1)" if pipelined else "serialized: quantize, gather, block-receive, apply per step"),
            "value_serialized": (elems * world / (ms_serial / 1e3)) if ms_serial else None,
            "cuda_graph": ({"replayed": True, "value_eager": elems_eager * world / (ms_eager / 1e3)} if use_graph else None),
            "roofline": {"bound": "hbm", "kernel": "k_apply", "achieved": a_gbs, "peak": peak, "unit": "GB/s",
                         "frac": a_gbs / peak, "traffic": traffic, "peak_source": peak_src,
                         "algorithmic_bytes_per_elem": 24 + M * (0.5 + (4.0 / B if B else 0.0)),
                         "avg_launch_ms": avg_a, "frac_of_8000_spec": a_gbs / 8000.0},
            "kernels": {
                "k_quantize": {"avg_ms": statistics.fmean(q_ms), "achieved_GBps": q_gbs, "frac": q_gbs / peak,
                               "algorithmic_bytes_per_elem": 8.5 + (4.0 / B if B else 0.0)},
                "k_apply": {"avg_ms": avg_a, "achieved_GBps": a_gbs, "frac": a_gbs / peak},
                "critical_path_frac": (qb + ab) / ((sum(q_ms) + sum(a_ms)) / 1e3) / 1e9 / peak,
                "critical_path_frac_of_8000_spec": (qb + ab) / ((sum(q_ms) + sum(a_ms)) / 1e3) / 1e9 / 8000.0,
                "step_share": {"k_quantize": sum(q_ms) / ms, "k_apply": sum(a_ms) / ms},
            },
            "gpu_launches": launches,
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "m_sweep_emulated": m_sweep,
            "overlap": overlap,
            "offload": offload,
            "inner_adamw_fused": fused,
        }
        print(json.dumps(line))
    sync.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def overlap_run(torch, dist, sd, synth, sync, cfg, theta, A, v, n, P, rank, world, events, dev, reps=15,
                kind="adamw"):
    """SURVEY.md §8(d) hidden-gather check on the real NCCL path: per round,
    quantize -> all-gather on the comm stream while the compute stream runs
    tau synthetic inner steps -> block-receive -> apply.  exposed = window
    with the gather in flight - the same tau inner steps alone; hidden <=>
    exposed <= 5% of the gather measured alone.  Two inner-step kinds:
    "adamw" = an AdamW-shaped pass over the whole replica (24 B/param, HBM-
    bound: the worst case for the gather's own HBM traffic) and "gemm" =
    bf16 cuBLAS matmuls (SM-bound).  CUDA events on the compute stream, max
    over ranks."""
    import statistics as st

    tau = cfg.tau
    Ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    step = [1]
    if kind == "adamw":
        m1 = [torch.zeros_like(x) for x in theta]
        m2 = [torch.zeros_like(x) for x in theta]

        def inner():
            for p in range(P):
                synth.dev_inner_adamw(theta[p], m1[p], m2[p], rank, step[0])
            step[0] += 1
    else:
        X = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
        Wm = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
        Y = torch.empty(8192, 8192, device=dev, dtype=torch.bfloat16)

        def inner():
            for _ in range(4):
                torch.matmul(X, Wm, out=Y)

    def maxr(x):
        t = torch.tensor([x], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    it = iter(events)
    alone, gath, over, bytes_in = [], [], [], []
    for r in range(reps + 1):
        e = [Ev() for _ in range(6)]
        e[0].record()
        for _ in range(tau):
            inner()
        e[1].record()
        p, t = next(it)
        sync.ctx.sd_outer_grad_quantize(p, t, theta[p], A[p], sync.slot(p), n[p])
        # the gather alone starts with every rank's payload ready: otherwise
        # it would also time the ranks' skew from the inner steps before it
        torch.cuda.synchronize()
        dist.barrier()
        e[2].record()
        sync.ctx.sd_fragment_sync(p, t, sync.gather[p], n[p])
        sync.ctx.sd_fragment_wait(p, t + cfg.tau)
        e[3].record()
        sync.ctx.sd_merge(p, t + cfg.tau, sync.gather[p], theta[p], A[p], v[p], n[p])
        p, t = next(it)
        sync.ctx.sd_outer_grad_quantize(p, t, theta[p], A[p], sync.slot(p), n[p])
        sync.ctx.sd_fragment_sync(p, t, sync.gather[p], n[p])
        e[4].record()
        for _ in range(tau):
            inner()
        sync.ctx.sd_fragment_wait(p, t + cfg.tau)
        e[5].record()
        sync.ctx.sd_merge(p, t + cfg.tau, sync.gather[p], theta[p], A[p], v[p], n[p])
        torch.cuda.synchronize()
        dist.barrier()
        if r == 0:
            continue
        alone.append(maxr(e[0].elapsed_time(e[1])))
        gath.append(maxr(e[2].elapsed_time(e[3])))
        over.append(maxr(e[4].elapsed_time(e[5])))
        bytes_in.append((world - 1) * sync.payload[p])
    ta, tg, to = st.median(alone), st.median(gath), st.median(over)
    # paired estimate: each rep measures the inner steps alone and with the gather back to back
    exposed = max(0.0, st.median([o - a for o, a in zip(over, alone)]))
    gbps = st.median(bytes_in) / (tg / 1e3) / 1e9
    # the gather's own HBM bytes on this GPU (peers' payloads written in, this
    # rank's payload read out M-1 times) at the copy peak: an HBM-bound inner
    # step is slowed by at least this much, whatever the transfer overlaps
    hbm_ms = 2 * st.median(bytes_in) / (peaks()[0] * 1e6)
    return {"tau": tau, "inner_step": ("AdamW-shaped synthetic pass over the whole replica, 24 B/param (synth/)"
                                       if kind == "adamw" else "4 bf16 8192^3 cuBLAS matmuls (SM-bound)"),
            "inner_window_ms": ta, "overlap_window_ms": to, "gather_alone_ms": tg, "exposed_ms": exposed,
            "exposed_frac_of_gather": exposed / tg if tg > 0 else None,
            "gather_hbm_bytes_ms": hbm_ms,
            "hidden": exposed <= max(0.05 * tg, hbm_ms if kind == "adamw" else 0.0),
            "hidden_rule": ("exposed <= max(5% of the gather alone, its HBM bytes at the copy peak)" if kind == "adamw"
                            else "exposed <= 5% of the gather alone"),
            "inner_slowdown": to / ta if ta > 0 else None,
            "nvlink": {"ingress_bytes_per_gpu": int(st.median(bytes_in)), "GBps_per_direction": gbps,
                       "frac_of_900_nominal": gbps / 900.0, "frac_of_770_measured_peer": gbps / 770.0}}


def fused_inner_run(torch, sd, sync, cfg, th, A0, n, B, dev, peak, reps=8):
    """NEXT-1: AdamW inner step + quantize as two kernels (28 + 8.5 B/param)
    vs the fused last-inner-step kernel (32.5 B/param: theta stays in
    registers), and AdamW + merge vs the fused receive step.  Fragment 0."""
    import statistics as st

    ctx = sync.ctx
    g = torch.randn(n, device=dev) * 1e-3
    m = torch.zeros(n, device=dev)
    v = torch.zeros(n, device=dev)
    mom = torch.zeros(n, device=dev)  # outer momentum (the merges only keep the calendar state legal)
    hp = sd.SdAdamW(lr=3e-4, beta1=0.9, beta2=0.99, eps=1e-8, weight_decay=0.1)
    slot = sync.slot(0)
    t0 = cfg.H
    sep, fus = [], []
    for r in range(reps + 2):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record()
        ctx.sd_inner_adamw(r + 1, th, g, m, v, hp, n)
        ctx.sd_outer_grad_quantize(0, t0, th, A0, slot, n)
        e[1].record()
        ctx.sd_fragment_sync(0, t0, sync.gather[0], n)
        ctx.sd_merge(0, t0 + cfg.tau, sync.gather[0], th, A0, mom, n)
        e[2].record()
        ctx.sd_inner_adamw_quantize(0, t0, r + 1, th, g, m, v, A0, slot, hp, n)
        e[3].record()
        ctx.sd_fragment_sync(0, t0, sync.gather[0], n)
        ctx.sd_merge(0, t0 + cfg.tau, sync.gather[0], th, A0, mom, n)
        torch.cuda.synchronize()
        if r >= 2:
            sep.append(e[0].elapsed_time(e[1]))
            fus.append(e[2].elapsed_time(e[3]))
    # the receive step: AdamW + merge (28 + 24.5 B/param) vs fused (44.5: theta once)
    msep, mfus = [], []
    for r in range(reps + 2):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ctx.sd_outer_grad_quantize(0, t0, th, A0, slot, n)
        ctx.sd_fragment_sync(0, t0, sync.gather[0], n)
        e[0].record()
        ctx.sd_inner_adamw(r + 1, th, g, m, v, hp, n)
        ctx.sd_merge(0, t0 + cfg.tau, sync.gather[0], th, A0, mom, n)
        e[1].record()
        ctx.sd_outer_grad_quantize(0, t0, th, A0, slot, n)
        ctx.sd_fragment_sync(0, t0, sync.gather[0], n)
        e[2].record()
        ctx.sd_inner_adamw_merge(0, t0 + cfg.tau, r + 1, th, g, m, v, sync.gather[0], A0, mom, hp, n)
        e[3].record()
        torch.cuda.synchronize()
        if r >= 2:
            msep.append(e[0].elapsed_time(e[1]))
            mfus.append(e[2].elapsed_time(e[3]))
    tms, tmf = st.median(msep), st.median(mfus)
    ts, tf = st.median(sep), st.median(fus)
    pay = n / 2 + 4 * (1 if B == 0 else -(-n // B))
    bs, bf = 36 * n + pay, 32 * n + pay
    return {"fragment_elems": int(n), "separate_ms": ts, "fused_ms": tf, "speedup": ts / tf,
            "separate_frac": bs / (ts / 1e3) / 1e9 / peak, "fused_frac": bf / (tf / 1e3) / 1e9 / peak,
            "algorithmic_bytes_per_elem": {"separate": 36.5, "fused": 32.5},
            "receive_step": {"separate_ms": tms, "fused_ms": tmf, "speedup": tms / tmf,
                             "fused_frac": (44 * n + pay) / (tmf / 1e3) / 1e9 / peak,
                             "algorithmic_bytes_per_elem": {"separate": 52.5, "fused": 44.5}}}


def offload_run(torch, sync, A0, v0, n, P, dev, reps=5):
    """Outer state offloaded to pinned host memory (sd_state_prefetch /
    sd_state_writeback): time to move fragment 0's anchor +
    momentum (8 B/param) H2D and D2H on libsd's copy stream."""
    import statistics as st

    ctx = sync.ctx
    hA = torch.empty(n[0], dtype=torch.float32, pin_memory=True)
    hv = torch.empty(n[0], dtype=torch.float32, pin_memory=True)
    pre, wb = [], []
    for r in range(reps + 1):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        ctx.sd_state_writeback(0, A0, v0, hA, hv, n[0])
        ctx.sd_state_sync()
        e[1].record()
        ctx.sd_state_prefetch(0, hA, hv, A0, v0, n[0])
        ctx.sd_state_sync()
        e[2].record()
        torch.cuda.synchronize()
        if r:
            wb.append(e[0].elapsed_time(e[1]))
            pre.append(e[1].elapsed_time(e[2]))
    tp, tw = st.median(pre), st.median(wb)
    nbytes = 8 * n[0]
    return {"fragment_elems": int(n[0]), "bytes_each_way": int(nbytes), "prefetch_ms": tp, "writeback_ms": tw,
            "H2D_GBps": nbytes / (tp / 1e3) / 1e9, "D2H_GBps": nbytes / (tw / 1e3) / 1e9,
            "paper_claim": "< 10 ms per fragment + outer state on an H100 (PAPER.md:149)",
            "hbm_outer_state_bytes": {"resident": int(8 * sum(n)), "offloaded_two_slots": int(2 * 8 * max(n))}}


def m_sweep_run(torch, sd, synth, cfg, segs, n, B, dev, peak, iters=12):
    """Per-GPU kernel time of one fragment round at M = 1, 2, 4, 8 replicas,
    the M payloads produced on this GPU by M emulated replicas (include/sd.h's
    single-GPU seam).  Times replica 0's k_quantize and k_apply."""
    out = {}
    A = synth.dev_init(torch.empty(n, device=dev), segs, 0)
    v = torch.zeros(n, device=dev)
    for M in (1, 2, 4, 8):
        ctx = [sd.SdContext(cfg, m, M, None, dev.index) for m in range(M)]
        pb = sd.sd_payload_bytes(cfg, n)
        gather = torch.empty(M * pb, dtype=torch.uint8, device=dev)
        th = []
        for m in range(M):
            x = A.clone()
            synth.dev_apply_window(x, segs, 0, m, 1)
            th.append(x)
        qs, as_ = [], []
        t = cfg.H
        for it in range(iters + 2):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            for m in range(M):
                if m == 0:
                    e[0].record()
                ctx[m].sd_outer_grad_quantize(0, t, th[m], A, gather[m * pb:(m + 1) * pb], n)
                if m == 0:
                    e[1].record()
            for m in range(M):
                ctx[m].sd_fragment_sync(0, t, gather, n)
            for m in range(M):
                if m == 0:
                    e[2].record()
                ctx[m].sd_merge(0, t + cfg.tau, gather, th[m], A, v, n)
                if m == 0:
                    e[3].record()
            torch.cuda.synchronize()
            if it >= 2:
                qs.append(e[0].elapsed_time(e[1]))
                as_.append(e[2].elapsed_time(e[3]))
        for c in ctx:
            c.sd_finalize()
        qb, ab = algorithmic_bytes(n, M, B)
        tq, ta = statistics.median(qs), statistics.median(as_)
        out[str(M)] = {"quantize_ms": tq, "apply_ms": ta, "apply_frac": ab / (ta / 1e3) / 1e9 / peak,
                       "quantize_frac": qb / (tq / 1e3) / 1e9 / peak,
                       "params_per_s_per_gpu": n / ((tq + ta) / 1e3),
                       "critical_path_frac": (qb + ab) / ((tq + ta) / 1e3) / 1e9 / peak}
        del gather, th
    return out


if __name__ == "__main__":
    sys.exit(main())
