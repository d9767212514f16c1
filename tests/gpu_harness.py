"""Harness for the GPU parity tests: drives libsd through its C ABI (the
Python binding) for M replicas emulated on one GPU (one sd_ctx per replica,
id = NULL, every replica quantizing into its slot of one shared gather
buffer -- the single-GPU seam of include/sd.h), and builds edge-case inputs.
No method arithmetic here: inputs, calls, copies."""
from __future__ import annotations

import numpy as np
import torch

from paper_2501_18512_b200 import sd

DEV = torch.device("cuda", 0)


def to_dev(x: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def bits(x) -> np.ndarray:
    if isinstance(x, torch.Tensor):
        x = x.cpu().numpy()
    return np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)


class EmulatedReplicas:
    """M replicas of one fragment on cuda:0, each with its own copy of the
    (replicated) anchor and momentum, as on M separate GPUs."""

    def __init__(self, cfg, M: int, n: int, staged: bool = True):
        """staged: give every replica's ctx its own quantize workspace (the
        two-pass quantize then encodes from 16-bit summaries; as FragmentSync
        does); False: no workspace (the second pass re-reads theta and A)."""
        self.cfg, self.M, self.n = cfg, M, n
        self.pb = sd.sd_payload_bytes(cfg, n)
        self.ctx = [sd.SdContext(cfg, m, M, None, 0) for m in range(M)]
        self.gather = torch.empty(M * self.pb, dtype=torch.uint8, device=DEV)
        ws = sd.sd_quantize_workspace_bytes(cfg, n)
        if staged and ws > 0:
            for c in self.ctx:
                # garbage: nothing may depend on the workspace's previous contents
                c.sd_set_workspace(torch.full((ws,), 0xC5, dtype=torch.uint8, device=DEV))

    def slot(self, m):
        return self.gather[m * self.pb:(m + 1) * self.pb]

    def quantize_all(self, p, t, thetas, anchors):
        for m in range(self.M):
            self.ctx[m].sd_outer_grad_quantize(p, t, thetas[m], anchors[m], self.slot(m), self.n)
        for m in range(self.M):
            self.ctx[m].sd_fragment_sync(p, t, self.gather, self.n)

    def merge_all(self, p, t, thetas, anchors, moms):
        for m in range(self.M):
            self.ctx[m].sd_merge(p, t, self.gather, thetas[m], anchors[m], moms[m], self.n)

    def check_all(self):
        return [c.sd_check() for c in self.ctx]

    def close(self):
        for c in self.ctx:
            c.sd_finalize()


def edge_deltas(n: int, B: int, rng: np.random.Generator) -> np.ndarray:
    """Outer gradients exercising the codec's edges: values
    within +-4 ulps of every threshold, subnormal values and scales, +-0,
    all-zero blocks (scale 0), one element >> the rest, random signs."""
    from decimal import Decimal

    blen = B if B else n
    d = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    nblk = max(1, -(-n // blen))
    for b in range(nblk):
        lo, hi = b * blen, min(n, (b + 1) * blen)
        kind = b % 6
        seg = d[lo:hi]
        if kind == 0:  # near-threshold values of scale s
            s = np.float32(rng.uniform(0.5, 2.0) * 10.0 ** rng.integers(-6, 2))
            seg[0] = s
            for i in range(1, hi - lo):
                j = int(rng.integers(0, 7))
                t = np.float32(float(Decimal(float(s)) * (Decimal(2) ** Decimal(-j - 0.5))))
                tb = int(t.view(np.uint32)) + int(rng.integers(-4, 5))
                seg[i] = np.uint32(tb).view(np.float32) * (1 if rng.random() < 0.5 else -1)
        elif kind == 1:  # subnormal values and scale
            seg[:] = (rng.integers(-(2 ** 22), 2 ** 22, hi - lo).astype(np.int64)).astype(np.float32) * np.float32(2.0 ** -149)
        elif kind == 2:  # scale 0
            seg[:] = 0.0
        elif kind == 3:  # one element far above the rest
            seg[int(rng.integers(0, hi - lo))] = 1e3
        elif kind == 4:  # signed zeros mixed with tiny values
            seg[::3] = 0.0
            seg[1::3] = -0.0
        d[lo:hi] = seg
    return d


def theta_anchor_for(delta: np.ndarray, rng: np.random.Generator, exact: bool):
    """exact: A = 0 (or -0 where delta is -0), theta = -delta, so A - theta
    == delta bit-exactly; else a realistic A with theta = A - delta (rounded)."""
    if exact:
        A = np.where(np.signbit(delta) & (delta == 0), np.float32(-0.0), np.float32(0.0)).astype(np.float32)
        th = np.where(np.signbit(delta) & (delta == 0), np.float32(0.0), -delta).astype(np.float32)
        return A, th
    A = (rng.standard_normal(delta.size) * 0.02).astype(np.float32)
    return A, (A - delta).astype(np.float32)
