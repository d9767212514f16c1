#!/usr/bin/env python
"""Streaming DiLoCo (Alg. 2) end to end on a Chinchilla-shaped
decoder with synthetic tokens.

One replica per GPU (torchrun for N > 1).  The model's forward/backward is
plain PyTorch (the inner loss L3-4 is not the method); everything from the
gradients on is libsd: the AdamW inner step (sd_inner_adamw), the fused
last-inner-step + Delta + E3M0 for the fragment that sends at t
(sd_inner_adamw_quantize), the copy-engine all-gather (sd_fragment_sync),
and, tau steps later, the inner step fused with decode + fp32 mean +
Nesterov + alpha-merge (sd_inner_adamw_merge).
The model's parameters are views into fragment-contiguous fp32 slabs (AMB-18),
so libsd operates on the live weights in place.

  python examples/train_streaming_diloco.py --steps 300
  torchrun --nproc-per-node 2 examples/train_streaming_diloco.py --steps 300
"""
from __future__ import annotations

import argparse
import math
import os
import sys
import time

import torch
import torch.distributed as dist
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2501_18512_b200 import FragmentSync, sd  # noqa: E402

HEAD = 64


def layer_shapes(d):
    """Per-layer tensors in slab order (synth.fragment_segments / AMB-17)."""
    return [("ln1", (d,)), ("wq", (d, d)), ("wk", (d, d)), ("wv", (d, d)), ("wo", (d, d)), ("qn", (HEAD,)),
            ("kn", (HEAD,)), ("ln2", (d,)), ("w1", (4 * d, d)), ("w2", (d, 4 * d))]


class SlabModel:
    """Chinchilla-style decoder (QKNorm, z-loss, tied embedding)
    whose parameters live in fragment slabs."""

    def __init__(self, cfg, d, layers, vocab, dev, seed=0):
        self.d, self.vocab = d, vocab
        P = sd.sd_fragment_count(cfg)
        self.P = P
        self.frag_layers, self.holds_embed = [], []
        for p in range(P):
            blocks, _, emb = sd.sd_fragment_layout(cfg, p)
            self.frag_layers.append(sorted(blocks))
            self.holds_embed.append(emb)
        sizes = []
        for p in range(P):
            n = sum(math.prod(s) for _, s in layer_shapes(d)) * len(self.frag_layers[p])
            if self.holds_embed[p]:
                n += vocab * d + d
            sizes.append(n)
        self.n = sizes
        self.theta = [torch.empty(n, device=dev) for n in sizes]
        self.grad = [torch.zeros(n, device=dev) for n in sizes]
        self.params = []  # (param view, grad slab view)
        self.layer = {}
        gen = torch.Generator(device=dev).manual_seed(seed)
        for p in range(P):
            off = 0

            def take(shape, init):
                nonlocal off
                k = math.prod(shape)
                view = self.theta[p][off:off + k].view(shape)
                if init == "one":
                    view.fill_(1.0)
                else:
                    view.normal_(0.0, 0.02, generator=gen)
                prm = torch.nn.Parameter(view)
                self.params.append((prm, self.grad[p][off:off + k]))
                off += k
                return prm

            for l in self.frag_layers[p]:
                self.layer[l] = {name: take(shape, "one" if name in ("ln1", "ln2", "qn", "kn") else "n")
                                 for name, shape in layer_shapes(d)}
            if self.holds_embed[p]:
                self.emb = take((vocab, d), "n")
                self.lnf = take((d,), "one")
        self.L = len(self.layer)

    def forward(self, x, y):
        d, H = self.d, self.d // HEAD
        h = F.embedding(x, self.emb)
        B, S, _ = h.shape
        for l in range(self.L):
            w = self.layer[l]
            a = F.rms_norm(h, (d,), w["ln1"])
            q = (a @ w["wq"].t()).view(B, S, H, HEAD)
            k = (a @ w["wk"].t()).view(B, S, H, HEAD)
            v = (a @ w["wv"].t()).view(B, S, H, HEAD).transpose(1, 2)
            q = F.rms_norm(q, (HEAD,), w["qn"]).transpose(1, 2)  # QKNorm
            k = F.rms_norm(k, (HEAD,), w["kn"]).transpose(1, 2)
            o = F.scaled_dot_product_attention(q, k, v, is_causal=True).transpose(1, 2).reshape(B, S, d)
            h = h + o @ w["wo"].t()
            a = F.rms_norm(h, (d,), w["ln2"])
            h = h + F.gelu(a @ w["w1"].t()) @ w["w2"].t()
        logits = F.rms_norm(h, (d,), self.lnf) @ self.emb.t()
        lf = logits.float().view(-1, self.vocab)
        loss = F.cross_entropy(lf, y.reshape(-1))
        z = torch.logsumexp(lf, dim=-1)
        return loss + 1e-4 * (z * z).mean(), loss  # z-loss 1e-4

    def collect_grads(self):
        for prm, gslab in self.params:
            if prm.grad is not None:
                gslab.copy_(prm.grad.view(-1))
                prm.grad = None


def synthetic_batch(gen, batch, seq, vocab, perm):
    """Tokens from a fixed random first-order chain (learnable): next = perm[cur]
    with probability 0.9, uniform otherwise.  Each replica has its own stream."""
    x = torch.empty(batch, seq + 1, dtype=torch.long, device=perm.device)
    x[:, 0] = torch.randint(0, vocab, (batch,), generator=gen, device=perm.device)
    noise = torch.randint(0, vocab, (batch, seq), generator=gen, device=perm.device)
    keep = torch.rand(batch, seq, generator=gen, device=perm.device) < 0.9
    for s in range(seq):
        x[:, s + 1] = torch.where(keep[:, s], perm[x[:, s]], noise[:, s])
    return x[:, :-1], x[:, 1:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--d-model", type=int, default=512)
    ap.add_argument("--layers", type=int, default=6)
    ap.add_argument("--fragment-size", type=int, default=2)
    ap.add_argument("--vocab", type=int, default=32000)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--seq", type=int, default=256)
    ap.add_argument("--H", type=int, default=30)
    ap.add_argument("--tau", type=int, default=1)
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--log-every", type=int, default=20)
    ap.add_argument("--amp", action="store_true", help="bf16 autocast for the forward/backward (weights stay fp32)")
    args = ap.parse_args()

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = sd.sd_config_default(args.layers, args.fragment_size, args.H, tau=args.tau, T=args.steps)
    model = SlabModel(cfg, args.d_model, args.layers, args.vocab, dev, seed=0)  # same init on every replica
    sync = FragmentSync(cfg, model.n, rank, world, local)
    P = model.P
    A = [torch.empty_like(t) for t in model.theta]
    vout = [torch.empty_like(t) for t in model.theta]
    m1 = [torch.zeros_like(t) for t in model.theta]
    m2 = [torch.zeros_like(t) for t in model.theta]
    for p in range(P):
        sync.outer_state_init(p, model.theta[p], A[p], vout[p])  # anchor = theta_init, momentum = 0 (AMB-2)
    hp = sd.SdAdamW(lr=args.lr, beta1=0.9, beta2=0.99, eps=1e-8, weight_decay=0.0)
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    perm = torch.randperm(args.vocab, generator=torch.Generator(device=dev).manual_seed(7), device=dev)
    if rank == 0:
        print(f"replicas {world}, params {sum(model.n) / 1e6:.1f}M in {P} fragments {model.n}, "
              f"H={args.H} tau={args.tau}", flush=True)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    outer_ms, t0 = 0.0, time.time()
    for t in range(1, args.steps + 1):
        x, y = synthetic_batch(gen, args.batch, args.seq, args.vocab, perm)
        with torch.autocast("cuda", dtype=torch.bfloat16, enabled=args.amp):
            total, loss = model.forward(x, y)                               # Alg. 2 L3-4
        total.backward()
        model.collect_grads()
        send, recv = sd.sd_fragment_schedule(cfg, t)
        ev[0].record()
        fused_recv = [p for p in recv if p not in send]
        for p in range(P):                                                  # L5, fused with L7 for senders
            if p in send:
                sync.ctx.sd_inner_adamw_quantize(p, t, t, model.theta[p], model.grad[p], m1[p], m2[p], A[p],
                                                 sync.slot(p), hp, model.n[p])
            elif p not in fused_recv:
                sync.ctx.sd_inner_adamw(t, model.theta[p], model.grad[p], m1[p], m2[p], hp, model.n[p])
        for p in send:                                                      # L8: async all-gather
            sync.ctx.sd_fragment_sync(p, t, sync.gather[p], model.n[p])
        for p in recv:                                                      # L10-13 (+ L5 fused)
            if p in fused_recv:
                sync.ctx.sd_inner_adamw_merge(p, t, t, model.theta[p], model.grad[p], m1[p], m2[p], sync.gather[p],
                                              A[p], vout[p], hp, model.n[p])
            else:
                sync.receive(p, t, model.theta[p], A[p], vout[p])
        ev[1].record()
        if t % args.log_every == 0 or t == args.steps:
            torch.cuda.synchronize()
            outer_ms = ev[0].elapsed_time(ev[1])
            lv = loss.detach()
            if world > 1:
                dist.all_reduce(lv, op=dist.ReduceOp.AVG)
            if rank == 0:
                print(f"step {t:5d} loss {lv.item():.4f} (ln V = {math.log(args.vocab):.2f}) "
                      f"libsd optimizer+sync {outer_ms:.2f} ms  sends {send} recvs {recv}  "
                      f"{(time.time() - t0) / t * 1e3:.1f} ms/step", flush=True)
    st, fb = sync.check()
    assert st == sd.SD_OK, (st, fb)
    # after the final flush every replica holds the same anchors
    if world > 1:
        for p in range(P):
            ref = A[p].clone()
            dist.broadcast(ref, src=0)
            assert torch.equal(ref, A[p]), f"anchor of fragment {p} differs across replicas"
    if rank == 0:
        print("done: anchors identical across replicas", flush=True)
    sync.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
