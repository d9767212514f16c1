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
    ap.add_argument("--no-extras", "--no-m-sweep", action="store_true",
                    help="skip the N = 1 extras (M-sweep, fused inner steps, offload, 4B and DiLoCo records)")
    ap.add_argument("--no-overlap", action="store_true", help="skip the N > 1 hidden-gather check")
    ap.add_argument("--timeline", default=None,
                    help="N > 1: write a Chrome-trace timeline of one overlap rep per inner-step kind (path.json)")
    ap.add_argument("--serial", action="store_true", help="no send/receive pipelining across fragments")
    ap.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                    help="replay each step as a CUDA graph (auto: single GPU, L2-resident small configs)")
    ap.add_argument("--gather", choices=["auto", "ce", "push", "pull"], default="auto",
                    help="all-gather: NCCL copy engines (ce), fused into the quantize kernel (push) or into "
                         "the merge kernel (pull), or libsd's choice (auto)")
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


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_cores():
    return len(os.sched_getaffinity(0))


def _oracle_rate(wl, B, M, order, segs, n, target_s):
    """or_round (all M replicas) over whole fragments in calendar order until
    ~target_s of CPU time (the last one cut to fit).  -> (elements/s over all
    M replicas, description of the sample)."""
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
    return total_e * M / total_t, f"or_round on {', '.join(used)} (calendar order), all M={M} replicas: " \
                                  f"{total_e} elements in {total_t:.2f} s (n / t = {total_e / total_t:.4g} fragment " \
                                  f"elements per second; value = M n / t, work-normalized)"


def cpu_baseline(wl, B, M, order, segs, n, target_s):
    """The oracle's full round (all M replicas) on the GPU box's host: the
    single-thread build (the oracle proper) and the same source built with
    OpenMP on every core the process may use (bit-identical results,
    tests/test_oracle_omp.py); `value` / `cores` are the N-thread run."""
    import oracle  # test infrastructure, allowed in this leg only

    N = host_cores()
    prev = oracle.set_threads(1)
    v1, s1 = _oracle_rate(wl, B, M, order, segs, n, target_s / 3)
    oracle.set_threads(N)
    vN, sN = _oracle_rate(wl, B, M, order, segs, n, 2 * target_s / 3)
    oracle.set_threads(prev)
    return {"value": vN, "unit": UNIT, "cores": N, "kind": "oracle",
            "sample": f"{sN}; OpenMP build of the oracle on {N} threads, -O2 -ffp-contract=off",
            "value_1thread": v1, "cores_1": 1, "sample_1thread": s1 + ", single thread",
            "cores_N": N, "cpu_model": cpu_model(),
            "note": "the 1-thread and N-thread oracles are bit-identical (tests/test_oracle_omp.py)"}


def ref_layout(wl, B):
    """The workload's fragments from the oracle's own scheduler (no libsd):
    -> (or_config, [(blocks, holds_embed)], calendar sends [(p, t)])."""
    import oracle

    P = wl.layers // wl.fragment_size
    c = oracle.config(L=wl.layers, fs=wl.fragment_size, pattern=1, embed_policy=0, H=wl.H, tau=wl.tau,
                      T=wl.H * 64, alpha=wl.alpha, lr=wl.lr, mu=wl.mu, B=B)
    assert oracle.num_fragments(c) == P
    lay = [(oracle.fragment_blocks(c, p), p == P - 1) for p in range(P)]
    sends = [(e[2], e[0]) for e in oracle.calendar(c) if e[1] == 0]
    return c, lay, sends


# --------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The reference arm of this tier: the CPU oracle (OpenMP build on every
    host core, bit-identical to the single-thread oracle) timed on bounded
    samples of the same workload, the calendar from the oracle's own
    scheduler -- no libsd, no GPU.  Rank 0 only."""
    rank, _, world = dist_env()
    if rank != 0:
        return 0
    import oracle
    import synth
    from synth.workloads import WORKLOADS

    wl = workload_with_overrides(WORKLOADS[args.workload], args)
    B = args.scale_block
    _, lay, sends = ref_layout(wl, B)
    segs = [wl.segments(b, e) for b, e in lay]
    M = world
    N = host_cores()
    oracle.set_threads(N)
    nmin = min(synth.segments_numel(s) for s in segs)
    dt, _ = oracle_sample_rate(wl, B, M, 0, segs[0], min(1 << 20, nmin))
    per_step = min(2.0, 90.0 / max(1, args.steps + args.warmup))
    S = int(min(nmin, max(1 << 16, min(1 << 20, nmin) * per_step / max(dt, 1e-6))))
    S -= S % 1024 if S > 1024 else 0
    events = (sends * (1 + (args.warmup + args.steps) // max(1, len(sends))))[:args.warmup + args.steps]
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
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": N, "kind": "oracle", "cpu_model": cpu_model(),
                         "sample": f"per step: or_round on the first {S} elements of the calendar's fragment, "
                                   f"all M={M} replicas, OpenMP build of the oracle on {N} threads "
                                   f"(bit-identical to the single-thread oracle)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# --------------------------------------------------------------------------- our arm
class Run:
    """One workload's resident state on this GPU (every
    fragment's anchor, momentum and live parameters in HBM), its FragmentSync
    (libsd context + gather buffers) and the step functions over libsd's C ABI."""

    def __init__(self, torch, sd, synth, FragmentSync, wl, B, rank, world, local, dev, gather_mode):
        self.torch, self.sd, self.wl, self.B, self.world, self.dev = torch, sd, wl, B, world, dev
        self.cfg = make_cfg(sd, wl, B)
        cfg = self.cfg
        self.P = P = sd.sd_fragment_count(cfg)
        lay = [sd.sd_fragment_layout(cfg, p) for p in range(P)]
        self.segs = [wl.segments(b, e) for b, _, e in lay]
        self.n = n = [synth.segments_numel(s) for s in self.segs]
        self.A = [synth.dev_init(torch.empty(n[p], device=dev), self.segs[p], p) for p in range(P)]
        self.v = [torch.zeros(n[p], device=dev) for p in range(P)]
        self.theta = []
        for p in range(P):
            th = self.A[p].clone()
            synth.dev_apply_window(th, self.segs[p], p, rank, 1)
            self.theta.append(th)
        self.sync = FragmentSync(cfg, n, rank, world, local, gather_mode=gather_mode)
        self.pending = []
        self.pipelined = False

    def one_step(self, p, t, ev=None):
        """Serialized round of fragment p: quantize, gather, block-receive, apply."""
        ctx, cfg, n = self.sync.ctx, self.cfg, self.n
        if ev is not None:
            ev[0].record()
        ctx.sd_outer_grad_quantize(p, t, self.theta[p], self.A[p], self.sync.slot(p), n[p])     # a1 + a3
        if ev is not None:
            ev[1].record()
        ctx.sd_fragment_sync(p, t, self.sync.gather[p], n[p])                                     # a4
        ctx.sd_fragment_wait(p, t + cfg.tau)                                                      # a5
        if ev is not None:
            ev[2].record()
        ctx.sd_merge(p, t + cfg.tau, self.sync.gather[p], self.theta[p], self.A[p], self.v[p], n[p])  # a6
        if ev is not None:
            ev[3].record()

    def pipe_step(self, p, t, ev=None):
        """Send of fragment p (quantize + async gather), then the receive of the
        fragment sent one step earlier: its gather ran concurrently with this
        quantize (tau >= 1: the receive comes after later compute)."""
        ctx, cfg, n = self.sync.ctx, self.cfg, self.n
        if ev is not None:
            ev[0].record()
        ctx.sd_outer_grad_quantize(p, t, self.theta[p], self.A[p], self.sync.slot(p), n[p])
        if ev is not None:
            ev[1].record()
        ctx.sd_fragment_sync(p, t, self.sync.gather[p], n[p])
        if self.pending:
            pp, tt = self.pending.pop()
            ctx.sd_fragment_wait(pp, tt + cfg.tau)
            if ev is not None:
                ev[2].record()
            ctx.sd_merge(pp, tt + cfg.tau, self.sync.gather[pp], self.theta[pp], self.A[pp], self.v[pp], n[pp])
            if ev is not None:
                ev[3].record()
        elif ev is not None:
            ev[2].record()
            ev[3].record()
        self.pending.append((p, t))

    def drain(self):
        while self.pending:
            pp, tt = self.pending.pop()
            self.sync.ctx.sd_fragment_wait(pp, tt + self.cfg.tau)
            self.sync.ctx.sd_merge(pp, tt + self.cfg.tau, self.sync.gather[pp], self.theta[pp], self.A[pp],
                                   self.v[pp], self.n[pp])

    def timed(self, dist, evs, K, W, fn, flush_buf=None):
        """W untimed steps, then exactly K steps between barrier + synchronize on
        both sides, CUDA events on the compute stream (per step: quantize and
        apply intervals).  -> (ms, per-step events, libsd launches, t0, t1)"""
        torch, sd = self.torch, self.sd
        for p, t in evs[:W]:
            fn(p, t)
        torch.cuda.synchronize()
        if self.world > 1:
            dist.barrier()
        kev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
        sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = sd.sd_kernel_launch_count()
        torch.cuda.synchronize()
        t0 = time.time()
        start.record()
        for i, (p, t) in enumerate(evs[W:W + K]):
            if flush_buf is not None:
                flush_buf.zero_()
                sev[i][0].record()
            fn(p, t, kev[i])
            if flush_buf is not None:
                sev[i][1].record()
        stop.record()
        torch.cuda.synchronize()
        t1 = time.time()
        nl = sd.sd_kernel_launch_count() - l0
        self.drain()
        torch.cuda.synchronize()
        if self.world > 1:
            dist.barrier()
        total = sum(a.elapsed_time(b) for a, b in sev) if flush_buf is not None else start.elapsed_time(stop)
        return total, kev, nl, t0, t1

    def close(self):
        self.sync.close()
        self.A = self.v = self.theta = None


def maxr(torch, dist, dev, x, world):
    if world == 1:
        return x
    t = torch.tensor([x], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def config_record(torch, dist, sd, synth, FragmentSync, wl, B, rank, world, local, dev, K, W, gather_mode, peak,
                  label):
    """One more configuration measured the way the headline is (pipelined when
    tau >= 1 and P > 1, else serialized), as a record of the same JSON line."""
    run = Run(torch, sd, synth, FragmentSync, wl, B, rank, world, local, dev, gather_mode)
    run.pipelined = run.P > 1 and run.cfg.tau > 0
    evs = calendar_sends(sd, run.cfg, W + K)
    ms, kev, nl, _, _ = run.timed(dist, evs, K, W, run.pipe_step if run.pipelined else run.one_step)
    ms = maxr(torch, dist, dev, ms, world)
    st, fb = run.sync.check()
    if st != sd.SD_OK:
        raise SystemExit(f"libsd reported {sd.STATUS_NAMES[st]} in {label} (first bad index {fb})")
    n = run.n
    applied = evs[W - 1:W + K - 1] if run.pipelined else evs[W:W + K]
    elems = sum(n[p] for p, _ in applied)
    q_ms = [e[0].elapsed_time(e[1]) for e in kev]
    a_ms = [e[2].elapsed_time(e[3]) for e in kev]
    qb = sum(algorithmic_bytes(n[p], world, B)[0] for p, _ in evs[W:W + K])
    ab = sum(algorithmic_bytes(n[p], world, B)[1] for p, _ in applied)
    rec = {"label": label, "workload": wl.describe() + f"; M = {world}; E3M0 B={B}",
           "fragments": [int(x) for x in n], "value": elems * world / (ms / 1e3), "unit": UNIT,
           "per_gpu_value": elems / (ms / 1e3), "ms_per_step": ms / K, "steps": K, "warmup": W,
           "schedule": "pipelined across fragments" if run.pipelined else "serialized (tau = 0 or P = 1)",
           "k_quantize_frac": qb / (sum(q_ms) / 1e3) / 1e9 / peak,
           "k_apply_frac": ab / (sum(a_ms) / 1e3) / 1e9 / peak,
           "critical_path_frac": (qb + ab) / ((sum(q_ms) + sum(a_ms)) / 1e3) / 1e9 / peak,
           "gpu_launches": nl}
    run.close()
    del run
    torch.cuda.empty_cache()
    return rec


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
        os.environ.setdefault("SD_LOG_INIT", "1")  # libsd logs its communicator (ranks, LSA team) to stderr
        dist.init_process_group("nccl", device_id=dev)
    wl = workload_with_overrides(WORKLOADS[args.workload], args)
    B = args.scale_block
    M = world
    gmode = {"auto": sd.SD_GATHER_AUTO, "ce": sd.SD_GATHER_COPY_ENGINE, "push": sd.SD_GATHER_PUSH,
             "pull": sd.SD_GATHER_PULL}[args.gather]
    run = Run(torch, sd, synth, FragmentSync, wl, B, rank, world, local, dev, gmode)
    cfg, P, n = run.cfg, run.P, run.n
    theta, A, v, sync = run.theta, run.A, run.v, run.sync
    torch.cuda.synchronize()

    K, W = args.steps, max(1, args.warmup)
    events = calendar_sends(sd, cfg, W + K)
    sampler = ClockSampler(local)

    pipelined = P > 1 and not args.serial and cfg.tau > 0  # tau = 0: the receive is in the send's step
    run.pipelined = pipelined
    step_fn = run.pipe_step if pipelined else run.one_step

    # L2 policy: the 1B/4B state (12 B/param, GBs) streams through HBM; small
    # configs (toy, 35M) would stay L2-resident, so they flush L2 between steps
    # and time only the steps (sum of per-step event intervals).
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = 12 * sum(n) < 4 * l2_bytes
    flush_buf = torch.empty(2 * l2_bytes, dtype=torch.uint8, device=dev) if flush else None

    ms, kev, launches, w0, w1 = run.timed(dist, events, K, W, step_fn, flush_buf)
    remeasured = False
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    if bad & set(sampler.summary(w0, w1).get("reasons", [])):
        # a throttled timed region is not a valid number: take it once more
        more_ev = calendar_sends(sd, cfg, 7 * (W + K))[6 * (W + K):]
        ms, kev, launches, w0, w1 = run.timed(dist, more_ev, K, W, step_fn, flush_buf)
        events = more_ev
        remeasured = True
    ms_eager = None
    # graphs: small L2-resident configs on one GPU (with N > 1, capturing the step with NCCL's all-gather
    # in it hung on B200 -- not used; the fused modes' round ids are host counters baked into the kernels)
    use_graph = (args.graph == "on" and world == 1) or (args.graph == "auto" and flush and world == 1)
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
                run.one_step(p, t)
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
    ms = maxr(torch, dist, dev, ms, world)
    ms_serial = None
    if pipelined and world > 1:
        ser_events = calendar_sends(sd, cfg, 4 * (W + K) + 12)[3 * (W + K) + 12:]
        ms_serial, _, _, _, _ = run.timed(dist, ser_events, K, W, run.one_step)
        ms_serial = maxr(torch, dist, dev, ms_serial, world)
    st, fb = sync.check()
    if st != sd.SD_OK:
        raise SystemExit(f"libsd reported {sd.STATUS_NAMES[st]} (first bad index {fb})")

    applied = events[W - 1:W + K - 1] if pipelined else events[W:W + K]
    elems_eager = sum(n[p] for p, _ in applied)
    if use_graph:
        applied = applied_g
    elems = sum(n[p] for p, _ in applied)                # fragment elements per replica over K steps
    value = elems * world / (ms / 1e3)                   # whole job: all replicas' elements / max time
    qb = sum(algorithmic_bytes(n[p], M, B)[0] for p, _ in events[W:W + K])
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

    # ---- end to end through the C ABI with host buffers (theta; then theta + offloaded A, v)
    e2e = e2e_off = None
    if not args.no_e2e:
        e2e = e2e_run(torch, dist, run, K, W, world, dev, offload=False)
        # PCIe-bound at ~35 ms per 1B step: a bounded number of steps
        e2e_off = e2e_run(torch, dist, run, min(K, 32), W, world, dev, offload=True)
    sampler.stop()
    clocks = sampler.summary(w0, w1)
    clocks["remeasured_after_throttle"] = remeasured

    # ---- gather hidden behind tau synthetic inner steps? (N > 1 only)
    overlap = None
    if world > 1 and cfg.tau > 0 and not args.no_overlap:
        overlap = {}
        for i, kind in enumerate(("adamw", "gemm")):
            base = 5 * (W + K) + 40 * i
            evs = calendar_sends(sd, cfg, base + 40)[base:]
            tl = args.timeline.replace(".json", f"_{kind}.json") if args.timeline else None
            overlap[kind] = overlap_run(torch, dist, sd, synth, sync, cfg, theta, A, v, n, P, rank, world, evs, dev,
                                        kind=kind, timeline=tl,
                                        gather_label=None if args.gather in ("push", "pull") else "copy engines")
        if args.gather in ("auto", "ce") and world <= 32:
            # the same check with the gather fused into the apply (pull): nothing is in flight during
            # the inner steps; the transfer's cost moves into the apply (apply_after_window_ms)
            psync = FragmentSync(cfg, n, rank, world, local, gather_mode=sd.SD_GATHER_PULL)
            for i, kind in enumerate(("adamw", "gemm")):
                base = 7 * (W + K) + 40 * i
                evs = calendar_sends(sd, cfg, base + 40)[base:]
                tl = args.timeline.replace(".json", f"_pull_{kind}.json") if args.timeline else None
                overlap["pull_" + kind] = overlap_run(torch, dist, sd, synth, psync, cfg, theta, A, v, n, P, rank, world,
                                                      evs, dev, kind=kind, timeline=tl, gather_label=None,
                                                      ref=overlap[kind])
            psync.close()

    extras = not args.no_extras and world == 1
    # ---- per-GPU kernel work at M = 1/2/4/8 replicas, emulated on this GPU (1 fragment)
    m_sweep = m_sweep_run(torch, sd, synth, cfg, run.segs[0], n[0], B, dev, peak) if extras else None
    # ---- NEXT-1: the inner AdamW step before a send, separate vs fused with the quantize
    fused = fused_inner_run(torch, sd, sync, cfg, theta[0], A[0], n[0], B, dev, peak) if extras else None
    # ---- SPEC's B = 0 (one scale per fragment): the two-pass quantize on fragment 0
    b0 = b0_quantize_run(torch, sd, synth, run.wl, run.segs[0], n[0], dev, peak) if extras and B != 0 else None
    # ---- NEXT-3: host-offloaded outer state -- transfer cost of one fragment's A, v
    offload = offload_run(torch, sync, A[0], v[0], n, P, dev) if extras and not args.no_e2e else None

    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl, B, M, [p for p, _ in events[:P]], run.segs, n, args.cpu_seconds)

    order = [p for p, _ in events[:P]]
    segs0 = run.segs
    run.close()
    del run, theta, A, v, sync
    torch.cuda.empty_cache()

    # ---- more configurations in the same line: the largest single-GPU config (4B at M = N)
    # and vanilla DiLoCo (Alg. 1: P = 1, tau = 0, the whole model one fragment)
    more = []
    if extras and args.workload in ("1B", "4B"):
        if args.workload == "1B":
            more.append(config_record(torch, dist, sd, synth, FragmentSync, WORKLOADS["4B"], B, rank, world, local, dev,
                                      min(K, 48), W, gmode, peak, "4B (BASELINE configs[3]/[4] shapes) at M = N"))
        import dataclasses
        dl = dataclasses.replace(WORKLOADS[args.workload], fragment_size=WORKLOADS[args.workload].layers, tau=0)
        more.append(config_record(torch, dist, sd, synth, FragmentSync, dl, B, rank, world, local, dev, min(K, 16), W,
                                  gmode, peak, "vanilla DiLoCo (Alg. 1, PAPER.md:39-62): P = 1, tau = 0, one fragment "
                                               "= the whole model, serialized"))

    if rank == 0:
        avg_a = statistics.fmean(a_ms)
        gather_desc = ("none (M = 1: no collective)" if world == 1 else
                       "fused into k_apply: NVLink loads of the peers' payloads; round flags signalled by "
                       "k_quantize's last CTA, waited on in k_apply's prologue"
                       if (args.gather == "pull" or (args.gather == "auto" and cfg.tau == 0 and world in (4, 8))) else
                       "fused into k_quantize: NVLink stores to the peers' symmetric buffers; round flags signalled "
                       "by its last CTA, waited on in k_apply's prologue"
                       if (args.gather == "push" or (args.gather == "auto" and cfg.tau == 0)) else
                       "NCCL in-place all-gather on copy engines (symmetric window, zero CTAs)")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (seeded counter-based generator, synth/; Chinchilla-shaped fragments)",
            "config": dict(workload_config(wl, B, world), fragments=[int(x) for x in n], gather=gather_desc,
                           l2=("state (12 B/param) fits in ~4x L2: L2 flushed (2x L2 written) between steps, "
                               "only the steps are timed" if flush else
                               "inputs > L2 (fragments of %.0f-%.0f MB per fp32 array, cycled); no flush"
                               % (4 * min(n) / 1e6, 4 * max(n) / 1e6))),
            "per_gpu_value": value / world,
            "nccl": ({"ranks": world, "communicator": "libsd's own (ncclCommInitRankConfig, CTA policy zero); "
                                                      "one '[libsd] rank r/N' line per rank on stderr"}
                     if world > 1 else None),
            "schedule": ("serialized step replayed as a CUDA graph (one per fragment of the cycle)" if use_graph else
                         "pipelined: each step sends fragment k (quantize + async all-gather) and receives "
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
            "e2e_offloaded_state": e2e_off,
            "cpu_baseline": cpu,
            "configs": more or None,
            "m_sweep_emulated": m_sweep,
            "overlap": overlap,
            "offload": offload,
            "inner_adamw_fused": fused,
            "quantize_B0": b0,
        }
        print(json.dumps(line))
    del order, segs0
    if world > 1:
        dist.destroy_process_group()
    return 0


def e2e_run(torch, dist, run, K, W, world, dev, offload):
    """The same C-ABI calls end to end with host buffers, timed on the device.
    offload=False: the fragment's live parameters come from pinned host memory
    before and go back after every step (4 B/param each way).  offload=True:
    the outer state is host-resident too (sd_state_prefetch /
    sd_state_writeback on libsd's copy streams): theta, A and v in, theta, A
    and v out (12 B/param each way); the device holds three staging slots.
    Copies of neighbouring fragments overlap the step (H2D of k+1 and D2H of
    k-1 during step k, PCIe full duplex), ordered per fragment by events."""
    sd = run.sd
    cfg, P, n, sync = run.cfg, run.P, run.n, run.sync
    ctx = sync.ctx
    e_events = calendar_sends(sd, cfg, 2 * (W + K) + (9 * (W + K) if offload else 0))[-(W + K):]
    host = [torch.empty(n[p], dtype=torch.float32, pin_memory=True) for p in range(P)]
    for p in range(P):
        host[p].copy_(run.theta[p])
    if offload:
        hA = [run.A[p].cpu().pin_memory() for p in range(P)]
        hv = [run.v[p].cpu().pin_memory() for p in range(P)]
        nmax = max(n)
        sA = [torch.empty(nmax, device=dev) for _ in range(3)]  # staging slots (HBM holds 3 |p|, not 2 x model)
        sv = [torch.empty(nmax, device=dev) for _ in range(3)]
    cs = torch.cuda.current_stream()
    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
    in_ev = [torch.cuda.Event() for _ in range(P)]
    step_ev = [torch.cuda.Event() for _ in range(P)]
    out_ev = [torch.cuda.Event() for _ in range(P)]

    def h2d(i, p):
        with torch.cuda.stream(h2d_s):
            h2d_s.wait_event(out_ev[p])          # the previous D2H of this fragment is done
            run.theta[p].copy_(host[p], non_blocking=True)
            in_ev[p].record(h2d_s)
        if offload:  # A_p, v_p into staging slot i % 3 on libsd's H2D copy stream
            ctx.sd_state_prefetch(p, hA[p], hv[p], sA[i % 3][:n[p]], sv[i % 3][:n[p]], n[p])

    def one(i, p, t):
        a, vv = (sA[i % 3][:n[p]], sv[i % 3][:n[p]]) if offload else (run.A[p], run.v[p])
        ctx.sd_outer_grad_quantize(p, t, run.theta[p], a, sync.slot(p), n[p])
        ctx.sd_fragment_sync(p, t, sync.gather[p], n[p])
        ctx.sd_merge(p, t + cfg.tau, sync.gather[p], run.theta[p], a, vv, n[p])
        if offload:
            ctx.sd_state_writeback(p, a, vv, hA[p], hv[p], n[p])

    def go(evs):
        h2d(0, evs[0][0])
        for i, (p, t) in enumerate(evs):
            if i + 1 < len(evs):
                h2d(i + 1, evs[i + 1][0])
            cs.wait_event(in_ev[p])
            one(i, p, t)
            step_ev[p].record(cs)
            with torch.cuda.stream(d2h_s):
                d2h_s.wait_event(step_ev[p])
                host[p].copy_(run.theta[p], non_blocking=True)
                out_ev[p].record(d2h_s)
        cs.wait_stream(d2h_s)
        if offload:
            ctx.sd_state_sync()

    for e in out_ev:
        e.record(cs)
    go(e_events[:W])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    go(e_events[W:])
    e1.record()
    torch.cuda.synchronize()
    ems = maxr(torch, dist, dev, e0.elapsed_time(e1), world)
    eel = sum(n[p] for p, _ in e_events[W:])
    per = 12 if offload else 4
    out = {"value": eel * world / (ems / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": per * eel // K, "d2h_bytes_per_step": per * eel // K, "ms_per_step": ems / K,
           "link_gbs_each_way": per * eel / (ems / 1e3) / 1e9,
           "path": (("pinned host theta, anchor, momentum -> H2D (sd_state_prefetch for A, v) -> sd_* C-ABI calls "
                     "-> D2H (sd_state_writeback) for every step's fragment; 3 device staging slots for A, v")
                    if offload else
                    "pinned host theta -> H2D -> sd_* C-ABI calls -> D2H for every step's fragment; "
                    "copies of neighbouring fragments overlap (two copy streams)")}
    if not offload:
        out["pcie_probe"] = pcie_probe(host[0], run.theta[0], h2d_s, d2h_s)
    if offload:  # the host store must be what the device would hold: spot check one fragment round trip
        del sA, sv
    del host
    return out


def overlap_run(torch, dist, sd, synth, sync, cfg, theta, A, v, n, P, rank, world, events, dev, reps=15,
                kind="adamw", timeline=None, gather_label="copy engines", ref=None):
    """SURVEY.md §8(d) hidden-gather check on the real NCCL path: per round,
    quantize -> all-gather on the comm stream while the compute stream runs
    tau synthetic inner steps -> block-receive -> apply.  exposed = window
    with the gather in flight - the same tau inner steps alone (paired, per
    rep); hidden <=> exposed <= 5% of the gather measured alone (the survey's
    rule, applied as written).  Two inner-step kinds: "adamw" = an
    AdamW-shaped pass over the whole replica (24 B/param, HBM-bound: the worst
    case for the gather's own HBM traffic) and "gemm" = bf16 cuBLAS matmuls
    (SM-bound).  CUDA events on the compute and comm streams, max over ranks.
    timeline: one rep's events of every rank as a Chrome trace (no nsys here)."""
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

    def maxr_(x):
        t = torch.tensor([x], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    comm = torch.cuda.ExternalStream(sync.ctx.sd_comm_stream(), device=dev)
    it = iter(events)
    alone, gath, over, bytes_in, app, trace = [], [], [], [], [], None
    for r in range(reps + 1):
        e = [Ev() for _ in range(6)]
        ti = [Ev() for _ in range(tau + 1)]      # inner-step boundaries of the overlapped window
        q = [Ev(), Ev()]                         # quantize of the overlapped round
        gd = Ev()                                # gather done (comm stream)
        ap = [Ev(), Ev()]                        # apply of the overlapped round
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
        q[0].record()
        sync.ctx.sd_outer_grad_quantize(p, t, theta[p], A[p], sync.slot(p), n[p])
        q[1].record()
        sync.ctx.sd_fragment_sync(p, t, sync.gather[p], n[p])
        gd.record(comm)
        e[4].record()
        ti[0].record()
        for k in range(tau):
            inner()
            ti[k + 1].record()
        sync.ctx.sd_fragment_wait(p, t + cfg.tau)
        e[5].record()
        ap[0].record()
        sync.ctx.sd_merge(p, t + cfg.tau, sync.gather[p], theta[p], A[p], v[p], n[p])
        ap[1].record()
        torch.cuda.synchronize()
        dist.barrier()
        if r == 0:
            continue
        alone.append(maxr_(e[0].elapsed_time(e[1])))
        gath.append(maxr_(e[2].elapsed_time(e[3])))
        over.append(maxr_(e[4].elapsed_time(e[5])))
        app.append(maxr_(ap[0].elapsed_time(ap[1])))
        bytes_in.append((world - 1) * sync.payload[p])
        if timeline and r == reps // 2:
            z = q[0]
            us = lambda a, b: 1e3 * a.elapsed_time(b)  # noqa: E731
            evs = [{"name": "k_quantize", "ph": "X", "pid": rank, "tid": "compute", "ts": 0.0, "dur": us(z, q[1])}]
            if gather_label:
                evs.append({"name": f"all-gather ({gather_label}, {(world - 1) * sync.payload[p] / 1e6:.0f} MB in)",
                            "ph": "X", "pid": rank, "tid": "comm", "ts": us(z, q[1]), "dur": us(q[1], gd)})
            for k in range(tau):
                evs.append({"name": f"inner step {k + 1} ({kind})", "ph": "X", "pid": rank, "tid": "compute",
                            "ts": us(z, ti[k]), "dur": us(ti[k], ti[k + 1])})
            evs.append({"name": "block-receive + k_apply", "ph": "X", "pid": rank, "tid": "compute",
                        "ts": us(z, ti[tau]), "dur": us(ti[tau], ap[1])})
            trace = evs
    ta, tg, to = st.median(alone), st.median(gath), st.median(over)
    # paired estimate: each rep measures the inner steps alone and with the gather back to back
    exposed = max(0.0, st.median([o - a for o, a in zip(over, alone)]))
    gbps = st.median(bytes_in) / (tg / 1e3) / 1e9
    # the gather's own HBM bytes on this GPU (peers' payloads written in, this
    # rank's payload read out M-1 times) at the copy peak: an HBM-bound inner
    # step is slowed by at least this much, whatever the transfer overlaps
    hbm_ms = 2 * st.median(bytes_in) / (peaks()[0] * 1e6)
    if timeline:
        allt = [None] * world
        dist.all_gather_object(allt, trace)
        if rank == 0:
            os.makedirs(os.path.dirname(os.path.abspath(timeline)), exist_ok=True)
            with open(timeline, "w") as f:
                json.dump({"traceEvents": [x for tr in allt if tr for x in tr], "displayTimeUnit": "ms",
                           "otherData": {"what": f"one overlapped round, {world} ranks, tau = {tau}, inner = {kind}; "
                                                 "CUDA events on the compute and comm streams (ts relative to each "
                                                 "rank's quantize start)"}}, f)
    if ref is not None:
        # pull mode: no transfer is in flight during the inner steps -- the peers' payloads are read by the
        # apply.  Judge the window against the copy-engine transfer of the same bytes (ref run), and report
        # what the transfer costs inside the apply instead.
        tg_ce = ref["gather_alone_ms"]
        return {"tau": tau, "mode": "pull: the apply reads the peers' payloads over NVLink",
                "inner_window_ms": ta, "overlap_window_ms": to, "exposed_ms": exposed,
                "exposed_frac_of_gather": exposed / tg_ce if tg_ce > 0 else None,
                "exposed_frac_of_window": exposed / ta if ta > 0 else None,
                "hidden": exposed <= 0.05 * tg_ce,
                "hidden_rule": "SURVEY.md §8(d): exposed <= 5% of the gather measured alone (the copy-engine "
                               "transfer of the same payloads, from the copy-engine run)",
                "wait_kernel_alone_ms": tg, "apply_after_window_ms": st.median(app),
                "transfer_cost_in_apply_ms": st.median(app) - ref["apply_after_window_ms"],
                "inner_slowdown": to / ta if ta > 0 else None, "reps": reps}
    return {"tau": tau, "inner_step": ("AdamW-shaped synthetic pass over the whole replica, 24 B/param (synth/)"
                                       if kind == "adamw" else "4 bf16 8192^3 cuBLAS matmuls (SM-bound)"),
            "inner_window_ms": ta, "overlap_window_ms": to, "gather_alone_ms": tg, "exposed_ms": exposed,
            "exposed_frac_of_gather": exposed / tg if tg > 0 else None,
            "exposed_frac_of_window": exposed / ta if ta > 0 else None,
            "hidden": exposed <= 0.05 * tg,
            "hidden_rule": "SURVEY.md §8(d): exposed <= 5% of the gather measured alone",
            "gather_hbm_bytes_ms": hbm_ms,
            "exposed_within_gather_hbm_bytes": exposed <= hbm_ms,
            "inner_slowdown": to / ta if ta > 0 else None,
            "apply_after_window_ms": st.median(app),
            "reps": reps,
            "nvlink": {"ingress_bytes_per_gpu": int(st.median(bytes_in)), "GBps_per_direction": gbps,
                       "frac_of_900_nominal": gbps / 900.0, "frac_of_770_measured_peer": gbps / 770.0,
                       "projection_M8_gather_ms": (7 * st.median(bytes_in) / max(1, world - 1)) / (gbps * 1e6)
                       if world < 8 else None,
                       "projection_note": "PROJECTION (not measured): 7 payloads of this size at the ingress rate "
                                          "measured here; gpurun offers at most 4 GPUs"}}


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


def b0_quantize_run(torch, sd, synth, wl, segs, n, dev, peak, reps=12):
    """SPEC.md:231, :266 (B = 0, one fp32 scale per fragment): the exact max
    over the whole fragment must be known before any code, so the quantize
    makes two passes.  Staged (the default, with a workspace): pass 1 reads
    theta and A once and writes a 16-bit summary per element, pass 2 encodes
    from the summaries (last chunk first, L2-resident tail; exact re-reads only
    where a summary straddles a threshold) -- 12.5 B/elem moved at most.
    Re-read (no workspace): pass 2 reads theta and A again (16.5 B/elem).
    Both reported against the 8.5 B/elem the method needs."""
    cfg = sd.sd_config_default(wl.layers, wl.fragment_size, wl.H, tau=wl.tau, scale_block=0)
    ctx = sd.SdContext(cfg, 0, 1, None, dev.index)
    ws = torch.empty(sd.sd_quantize_workspace_bytes(cfg, n), dtype=torch.uint8, device=dev)
    A = synth.dev_init(torch.empty(n, device=dev), segs, 0)
    th = A.clone()
    synth.dev_apply_window(th, segs, 0, 0, 1)
    v = torch.zeros(n, device=dev)
    slot = torch.empty(sd.sd_payload_bytes(cfg, n), dtype=torch.uint8, device=dev)
    t = cfg.H

    def quantize_ms():
        ts = []
        for r in range(reps + 2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ctx.sd_outer_grad_quantize(0, t, th, A, slot, n)
            e1.record()
            ctx.sd_fragment_sync(0, t, slot, n)
            ctx.sd_merge(0, t + cfg.tau, slot, th, A, v, n)
            torch.cuda.synchronize()
            if r >= 2:
                ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    # the inner AdamW step before a send at B = 0: separate (AdamW, then both passes) vs fused
    # (AdamW + block max in one pass, then the encode pass)
    g = torch.randn(n, device=dev) * 1e-3
    m1, m2 = torch.zeros(n, device=dev), torch.zeros(n, device=dev)
    hp = sd.SdAdamW(lr=3e-4, beta1=0.9, beta2=0.99, eps=1e-8, weight_decay=0.1)

    def adamw_ms():
        sep, fus = [], []
        for r in range(reps + 2):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            e[0].record()
            ctx.sd_inner_adamw(r + 1, th, g, m1, m2, hp, n)
            ctx.sd_outer_grad_quantize(0, t, th, A, slot, n)
            e[1].record()
            ctx.sd_fragment_sync(0, t, slot, n)
            ctx.sd_merge(0, t + cfg.tau, slot, th, A, v, n)
            e[2].record()
            ctx.sd_inner_adamw_quantize(0, t, r + 1, th, g, m1, m2, A, slot, hp, n)
            e[3].record()
            ctx.sd_fragment_sync(0, t, slot, n)
            ctx.sd_merge(0, t + cfg.tau, slot, th, A, v, n)
            torch.cuda.synchronize()
            if r >= 2:
                sep.append(e[0].elapsed_time(e[1]))
                fus.append(e[2].elapsed_time(e[3]))
        return statistics.median(sep), statistics.median(fus)

    tq_rr = quantize_ms()
    sep_rr, fus_rr = adamw_ms()
    ctx.sd_set_workspace(ws)
    tq = quantize_ms()
    ts_, tf_ = adamw_ms()
    ctx.sd_finalize()
    alg = 8.5 * n + 4
    return {"fragment_elems": int(n), "quantize_ms": tq, "kernels": "k_absmax<staged> + k_encode_staged (two passes)",
            "frac_algorithmic": alg / (tq / 1e3) / 1e9 / peak,
            "frac_moved": 12.5 * n / (tq / 1e3) / 1e9 / peak,
            "algorithmic_bytes_per_elem": 8.5, "moved_bytes_per_elem_max": 12.5,
            "workspace_bytes": int(ws.numel()),
            "reread": {"quantize_ms": tq_rr, "frac_algorithmic": alg / (tq_rr / 1e3) / 1e9 / peak,
                       "frac_moved": 16.5 * n / (tq_rr / 1e3) / 1e9 / peak, "moved_bytes_per_elem": 16.5,
                       "speedup_of_staged": tq_rr / tq},
            "inner_adamw_before_send": {"separate_ms": ts_, "fused_ms": tf_, "speedup": ts_ / tf_,
                                        "moved_bytes_per_elem_max": {"separate": 28 + 12.5, "fused": 32 + 4.5},
                                        "fused_frac_moved": (36.5 * n) / (tf_ / 1e3) / 1e9 / peak,
                                        "reread": {"separate_ms": sep_rr, "fused_ms": fus_rr,
                                                   "moved_bytes_per_elem": {"separate": 28 + 16.5,
                                                                            "fused": 32 + 8.5}}}}


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
