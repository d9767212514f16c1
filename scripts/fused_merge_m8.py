"""Times sd_inner_adamw_merge (AdamW + decode/mean/Nesterov/merge in one
kernel) for replica 0 of M = 1, 2, 4, 8 emulated replicas on one GPU, 1B
fragment; prints ms and the fraction of the copy peak at 44.5 + 0.5M B/param."""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import synth  # noqa: E402
from gpu_harness import EmulatedReplicas  # noqa: E402
from paper_2501_18512_b200 import sd  # noqa: E402

peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6548.8
segs = synth.fragment_segments(2048, [0, 8, 16], False)
n = synth.segments_numel(segs)
cfg = sd.sd_config_default(24, 3, 100, tau=5)
dev = torch.device("cuda", 0)
A = synth.dev_init(torch.empty(n, device=dev), segs, 0)
hp = sd.SdAdamW(lr=1e-3, beta1=0.9, beta2=0.99, eps=1e-8, weight_decay=0.1)
g = torch.randn(n, device=dev) * 1e-3
m1, m2, v = torch.zeros(n, device=dev), torch.zeros(n, device=dev), torch.zeros(n, device=dev)
for M in (1, 2, 4, 8):
    rep = EmulatedReplicas(cfg, M, n)
    th = []
    for m in range(M):
        x = A.clone()
        synth.dev_apply_window(x, segs, 0, m, 1)
        th.append(x)
    ts = []
    for r in range(6):
        rep.quantize_all(0, 100, th, [A] * M)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rep.ctx[0].sd_inner_adamw_merge(0, 105, r + 1, th[0], g, m1, m2, rep.gather, A, v, hp, n)
        e1.record()
        for m in range(1, M):
            rep.ctx[m].sd_merge(0, 105, rep.gather, th[m], A, v, n)
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    byt = (44.5 + M * (0.5 + 4 / 1024)) * n
    print(f"M={M} fused AdamW+merge {ms:.4f} ms  {byt / (ms * 1e-3) / 1e9:.0f} GB/s  frac {byt / (ms * 1e-3) / 1e9 / peak:.3f}")
    rep.close()
    del th
