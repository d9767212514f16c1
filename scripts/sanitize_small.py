"""Small, fast exercise of every libsd kernel for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per run):
  compute-sanitizer --tool memcheck python scripts/sanitize_small.py
Ragged sizes, every scale-block mode, M = 1 and 3, AdamW and the fused
AdamW + quantize, a poisoned round, an offloaded-state round."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_18512_b200 import sd  # noqa: E402

dev = torch.device("cuda", 0)
rng = np.random.default_rng(0)
hp = sd.SdAdamW(lr=1e-3, beta1=0.9, beta2=0.99, eps=1e-8, weight_decay=0.1)
for n in (1, 5, 1025, 4099):
    for B in (0, 256, 1024, 2048):
        for M in (1, 3):
            cfg = sd.sd_config_default(2, 1, 10, scale_block=B)
            pb = sd.sd_payload_bytes(cfg, n)
            ctx = [sd.SdContext(cfg, m, M, None, 0) for m in range(M)]
            gather = torch.zeros(M * pb, dtype=torch.uint8, device=dev)
            A = [torch.from_numpy((rng.standard_normal(n) * 0.02).astype(np.float32)).to(dev) for _ in range(M)]
            th = [a - 1e-3 for a in A]
            v = [torch.zeros(n, device=dev) for _ in range(M)]
            g = [torch.randn(n, device=dev) * 1e-3 for _ in range(M)]
            m1 = [torch.zeros(n, device=dev) for _ in range(M)]
            m2 = [torch.zeros(n, device=dev) for _ in range(M)]
            for m in range(M):
                if m == 0:
                    ctx[m].sd_inner_adamw_quantize(0, 10, 1, th[m], g[m], m1[m], m2[m], A[m],
                                                   gather[m * pb:(m + 1) * pb], hp, n)
                else:
                    ctx[m].sd_inner_adamw(1, th[m], g[m], m1[m], m2[m], hp, n)
                    ctx[m].sd_outer_grad_quantize(0, 10, th[m], A[m], gather[m * pb:(m + 1) * pb], n)
            for m in range(M):
                ctx[m].sd_fragment_sync(0, 10, gather, n)
            for m in range(M):
                ctx[m].sd_merge(0, 11, gather, th[m], A[m], v[m], n)
            torch.cuda.synchronize()
            for c in ctx:
                assert c.sd_check()[0] == sd.SD_OK
                c.sd_finalize()
# poisoned round and offloaded state
cfg = sd.sd_config_default(2, 1, 10)
n = 3000
ctx = sd.SdContext(cfg, 0, 1, None, 0)
buf = ctx.sd_gather_alloc(n)
A = torch.zeros(n, device=dev)
th = torch.zeros(n, device=dev)
th[17] = float("nan")
v = torch.zeros(n, device=dev)
hA, hv = torch.zeros(n).pin_memory(), torch.zeros(n).pin_memory()
ctx.sd_state_prefetch(0, hA, hv, A, v, n)
ctx.sd_outer_grad_quantize(0, 10, th, A, buf, n)
ctx.sd_fragment_sync(0, 10, buf, n)
ctx.sd_merge(0, 11, buf, th, A, v, n)
ctx.sd_state_writeback(0, A, v, hA, hv, n)
ctx.sd_state_sync()
torch.cuda.synchronize()
assert ctx.sd_check() == (sd.SD_ERR_NONFINITE, 17)
ctx.sd_finalize()
print("sanitize_small: ok")
