"""One 1B-fragment round for M = 2, 4, 8 replicas emulated on one GPU (for ncu
captures of k_apply<M>): quantize all M slots, then the M applies; replica 0's
apply of the second round runs inside an NVTX range "capture", so
`ncu --nvtx --nvtx-include "capture/"` captures exactly one launch per M."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import synth  # noqa: E402
from gpu_harness import EmulatedReplicas  # noqa: E402
from paper_2501_18512_b200 import sd  # noqa: E402

segs = synth.fragment_segments(2048, [0, 8, 16], False)
n = synth.segments_numel(segs)
cfg = sd.sd_config_default(24, 3, 100, tau=5)
dev = torch.device("cuda", 0)
A = synth.dev_init(torch.empty(n, device=dev), segs, 0)
v = torch.zeros(n, device=dev)
for M in (2, 4, 8):
    rep = EmulatedReplicas(cfg, M, n)
    th = []
    for m in range(M):
        x = A.clone()
        synth.dev_apply_window(x, segs, 0, m, 1)
        th.append(x)
    for r in range(2):
        rep.quantize_all(0, 100, th, [A] * M)
        for m in range(M):  # the second round's apply of replica 0 is the one ncu captures (NVTX range)
            if r == 1 and m == 0:
                torch.cuda.nvtx.range_push("capture")
            rep.ctx[m].sd_merge(0, 105, rep.gather, th[m], A, v, n)
            if r == 1 and m == 0:
                torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    rep.close()
    del th
print("emulated_apply: ok")
