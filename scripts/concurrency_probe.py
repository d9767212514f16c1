"""Does running the send of fragment k (quantize) and the receive of fragment
k-1 (apply) on two streams at once beat issuing them back to back?  They
touch disjoint data, so a caller may fork them after the inner step and join
before the next one.  1B workload, M = 1, fragments cycled on the calendar
as in bench.py's pipelined step; K steps timed with CUDA events.
  python scripts/concurrency_probe.py [K]"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from synth.workloads import WORKLOADS  # noqa: E402
from paper_2501_18512_b200 import FragmentSync, sd  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 256
wl = WORKLOADS["1B"]
cfg = sd.sd_config_default(wl.layers, wl.fragment_size, wl.H, tau=wl.tau)
P = sd.sd_fragment_count(cfg)
layout = [sd.sd_fragment_layout(cfg, q) for q in range(P)]
segs = [wl.segments(b, e) for b, _, e in layout]
n = [synth.segments_numel(s) for s in segs]
dev = torch.device("cuda", 0)
sync = FragmentSync(cfg, n, 0, 1, 0)
ctx = sync.ctx
A = [synth.dev_init(torch.empty(k, device=dev), s, p) for p, (k, s) in enumerate(zip(n, segs))]
th = []
for p in range(P):
    x = A[p].clone()
    synth.dev_apply_window(x, segs[p], p, 0, 1)
    th.append(x)
v = [torch.zeros(k, device=dev) for k in n]
events, t = [], cfg.H
while len(events) < 6 * (K + 8) + 8:
    s, _ = sd.sd_fragment_schedule(cfg, t)
    events.extend((p, t) for p in s)
    t += 1
main = torch.cuda.current_stream()
s_send, s_recv = torch.cuda.Stream(), torch.cuda.Stream()
fork = [torch.cuda.Event() for _ in range(2)]


def run(evs, concurrent):
    prev = None
    for i, (p, t) in enumerate(evs):
        if concurrent:
            f = fork[i % 2]
            f.record(main)
            s_send.wait_event(f)
            s_recv.wait_event(f)
            ctx.sd_outer_grad_quantize(p, t, th[p], A[p], sync.slot(p), n[p], s_send)
            ctx.sd_fragment_sync(p, t, sync.gather[p], n[p], s_send)
            if prev is not None:
                q, tq = prev
                ctx.sd_merge(q, tq + cfg.tau, sync.gather[q], th[q], A[q], v[q], n[q], s_recv)
            main.wait_stream(s_send)
            main.wait_stream(s_recv)
        else:
            ctx.sd_outer_grad_quantize(p, t, th[p], A[p], sync.slot(p), n[p])
            ctx.sd_fragment_sync(p, t, sync.gather[p], n[p])
            if prev is not None:
                q, tq = prev
                ctx.sd_merge(q, tq + cfg.tau, sync.gather[q], th[q], A[q], v[q], n[q])
        prev = (p, t)
    q, tq = prev
    ctx.sd_merge(q, tq + cfg.tau, sync.gather[q], th[q], A[q], v[q], n[q])


res = {}
base = 0
for rep in range(3):
    for mode in (False, True):
        evs = events[base:base + K + 8]
        base += K + 8
        run(evs[:8], mode)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(evs[8:], mode)
        e1.record()
        torch.cuda.synchronize()
        elems = sum(n[p] for p, _ in evs[8:])
        res.setdefault(mode, []).append(elems / (e0.elapsed_time(e1) / 1e3))
for mode, vals in res.items():
    print(f"{'two streams (fork/join)' if mode else 'one stream (serial)    '}: "
          f"{statistics.median(vals):.4e} params/s  (runs {', '.join('%.4e' % x for x in vals)})")
assert sync.check()[0] == sd.SD_OK
sync.close()
