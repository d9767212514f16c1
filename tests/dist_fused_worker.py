"""Worker for tests/test_gpu_multi.py: the fused inner-step calls on real
NCCL ranks, in every gather mode (SD_TEST_GATHER = ce | push | pull).

Per round, on every rank (replica m = rank):
  send step   sd_inner_adamw_quantize  (AdamW + Delta + E3M0 in one kernel;
              in push mode it also stores the payload into the peers)
  in between  sd_inner_adamw           (the tau overlapped inner steps, tau = 1)
  receive     sd_inner_adamw_merge     (AdamW + decode/mean/Nesterov/merge;
              in pull mode it reads the peers' payloads over NVLink)
Gradients are seeded per (rank, step).  After every round rank 0 gathers
every rank's theta, AdamW moments, anchor, momentum and own payload and
checks them bit for bit against the oracle: or_adamw per replica, then
or_round.  Prints OK on success."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2501_18512_b200 import FragmentSync, sd  # noqa: E402

HP = dict(lr=1e-3, beta1=0.9, beta2=0.99, eps=1e-8, weight_decay=0.1)


def grad(m, step, n):
    return (np.random.default_rng(1000 * step + m).standard_normal(n) * 1e-2).astype(np.float32)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    B = 1024
    n = 6 * 1024 + 37
    cfg = sd.sd_config_default(4, 2, 20, tau=1, scale_block=B)  # P = 2 fragments, H = 20
    P = sd.sd_fragment_count(cfg)
    p = 1
    t_p = sd.sd_fragment_layout(cfg, p)[1]
    mode = {"push": sd.SD_GATHER_PUSH, "pull": sd.SD_GATHER_PULL}.get(
        os.environ.get("SD_TEST_GATHER"), sd.SD_GATHER_COPY_ENGINE)
    fsync = FragmentSync(cfg, [n] * P, rank, world, local, gather_mode=mode)
    ctx = fsync.ctx
    hp = sd.SdAdamW(**HP)
    A0 = (np.random.default_rng(7).standard_normal(n) * 0.02).astype(np.float32)
    A = torch.from_numpy(A0).to(dev)
    v = torch.zeros(n, device=dev)
    th = A.clone()
    m1 = torch.zeros(n, device=dev)
    m2 = torch.zeros(n, device=dev)
    pb = fsync.payload[p]
    ok = True
    if rank == 0:
        import oracle

        o_th = [A0.copy() for _ in range(world)]
        o_m1 = [np.zeros(n, np.float32) for _ in range(world)]
        o_m2 = [np.zeros(n, np.float32) for _ in range(world)]
        o_A, o_v = A0.copy(), np.zeros(n, np.float32)

        def o_adamw(m, k, step):
            oracle.adamw(o_th[m], grad(m, step, n), o_m1[m], o_m2[m], k, lr=HP["lr"], b1=HP["beta1"],
                         b2=HP["beta2"], eps=HP["eps"], wd=HP["weight_decay"])
    k = 0
    for r in (1, 2, 3):
        t = r * cfg.H + t_p
        k += 1
        ctx.sd_inner_adamw_quantize(p, t, k, th, torch.from_numpy(grad(rank, t, n)).to(dev), m1, m2, A, fsync.slot(p),
                                    hp, n)
        ctx.sd_fragment_sync(p, t, fsync.gather[p], n)
        k += 1
        ctx.sd_inner_adamw(k, th, torch.from_numpy(grad(rank, t + 1000, n)).to(dev), m1, m2, hp, n)
        k += 1
        assert p in sd.sd_fragment_schedule(cfg, t + cfg.tau)[1]
        ctx.sd_inner_adamw_merge(p, t + cfg.tau, k, th, torch.from_numpy(grad(rank, t + cfg.tau, n)).to(dev), m1, m2,
                                 fsync.gather[p], A, v, hp, n)
        torch.cuda.synchronize()
        own = fsync.payloads(p)[rank * pb:(rank + 1) * pb]
        got = {}
        for name, x in (("payload", own), ("theta", th), ("m1", m1), ("m2", m2), ("A", A), ("v", v)):
            parts = [torch.empty_like(x) for _ in range(world)]
            dist.all_gather(parts, x.contiguous())
            got[name] = [q.cpu().numpy() for q in parts]
        if rank == 0:
            sends = []
            for m in range(world):
                o_adamw(m, k - 2, t)
                sends.append(o_th[m].copy())
                o_adamw(m, k - 1, t + 1000)
                o_adamw(m, k, t + cfg.tau)
            st, g_o = oracle.round_(sends, o_th, o_A, o_v, B=B)
            ok &= st == 0
            for m in range(world):
                ok &= np.array_equal(got["payload"][m], g_o[m * pb:(m + 1) * pb])
                for name, want in (("theta", o_th[m]), ("m1", o_m1[m]), ("m2", o_m2[m]), ("A", o_A), ("v", o_v)):
                    same = np.array_equal(got[name][m].view(np.uint32), want.view(np.uint32))
                    if not same:
                        print(f"round {r} rank {m} {name}: MISMATCH", flush=True)
                    ok &= same
            print(f"round {r}: {'match' if ok else 'MISMATCH'}", flush=True)
    st, fb = fsync.check()
    ok &= st == sd.SD_OK
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    fsync.close()
    dist.destroy_process_group()
    if rank == 0:
        print("OK" if flag.item() == 1 else "FAIL", flush=True)
    return 0 if flag.item() == 1 else 1


if __name__ == "__main__":
    sys.exit(main())
