"""Worker for tests/test_gpu_multi.py: BASELINE.json's full 1B fragment
(n = 151,007,616) on every rank, in bench.py's launch configuration (the
1B config, libsd-allocated gather buffers, the gather mode bench.py uses
by default unless SD_TEST_GATHER names another).  Two rounds; after each,
  - sampled scale blocks (incl. the first and the ragged last) of every
    rank's payload and outer state equal the CPU oracle's, recomputed block
    by block from the same seeded generator (blocks are independent at
    B = 1024);
  - properties that hold at any size, on the whole fragment: A and v are
    bit-identical on every rank (SURVEY §8(b) "anchors identical"), and
    every rank's gathered slot m equals rank m's own payload byte for byte
    (in the pull mode the peers' slots stay in the peers' buffers, so only
    the own slot is local).
Prints OK on success."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from synth.workloads import WORKLOADS  # noqa: E402
from paper_2501_18512_b200 import FragmentSync, sd  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    wl = WORKLOADS["1B"]
    B = 1024
    cfg = sd.sd_config_default(wl.layers, wl.fragment_size, wl.H, tau=wl.tau, scale_block=B)
    P = sd.sd_fragment_count(cfg)
    p = 1
    layout = [sd.sd_fragment_layout(cfg, q) for q in range(P)]
    t_p = layout[p][1]
    segs_all = [wl.segments(blocks, emb) for blocks, _, emb in layout]
    segs = segs_all[p]
    n = synth.segments_numel(segs)
    mode = {"push": sd.SD_GATHER_PUSH, "pull": sd.SD_GATHER_PULL,
            "ce": sd.SD_GATHER_COPY_ENGINE}.get(os.environ.get("SD_TEST_GATHER"), sd.SD_GATHER_AUTO)
    fsync = FragmentSync(cfg, [synth.segments_numel(s) for s in segs_all], rank, world, local, gather_mode=mode)
    A = synth.dev_init(torch.empty(n, device=dev), segs, p)
    v = torch.zeros(n, device=dev)
    th = A.clone()
    ok = True
    nb = -(-n // B)
    rng = np.random.default_rng(7)
    sample = sorted(set([0, nb - 1] + list(rng.integers(0, nb, 24))))
    soff = sd.sd_payload_scales_offset(n)
    pb = fsync.payload[p]
    if rank == 0:
        import oracle

        state = {b: (synth.host_init(segs, p, b * B, min(n, (b + 1) * B)),) for b in sample}
        state = {b: [a[0], np.zeros_like(a[0]), [a[0].copy() for _ in range(world)]] for b, a in state.items()}
    for r in (1, 2):
        t = r * cfg.H + t_p
        assert p in sd.sd_fragment_schedule(cfg, t)[0]
        synth.dev_apply_window(th, segs, p, rank, r)
        fsync.send(p, t, th, A)
        synth.dev_apply_drift(th, segs, p, rank, r)
        fsync.receive(p, t + cfg.tau, th, A, v)
        torch.cuda.synchronize()
        # any-size properties on the whole fragment
        ref = A.clone()
        dist.broadcast(ref, 0)
        ok &= bool(torch.equal(ref.view(torch.int32), A.view(torch.int32)))
        ref.copy_(v)
        dist.broadcast(ref, 0)
        ok &= bool(torch.equal(ref.view(torch.int32), v.view(torch.int32)))
        del ref
        allp = fsync.payloads(p)
        own = allp[rank * pb:(rank + 1) * pb]
        if mode != sd.SD_GATHER_PULL:
            for m in range(world):
                x = own.clone()
                dist.broadcast(x, m)
                ok &= bool(torch.equal(x, allp[m * pb:(m + 1) * pb]))
        # sampled blocks against the oracle: this rank's own codes and scale, A, v, theta
        rows = []
        for b in sample:
            lo, hi = b * B, min(n, (b + 1) * B)
            rows.append(torch.cat([own[lo // 2:(hi + 1) // 2], own[soff + 4 * b: soff + 4 * b + 4]] +
                                  [x[lo:hi].view(torch.uint8) for x in (A, v, th)]).cpu())
        gathered = [None] * world
        dist.all_gather_object(gathered, rows)
        if rank == 0:
            for k, b in enumerate(sample):
                lo, hi = b * B, min(n, (b + 1) * B)
                A0, v0, ths = state[b]
                sends = []
                for m in range(world):
                    synth.host_apply_window(ths[m], segs, p, m, r, i0=lo)
                    sends.append(ths[m].copy())
                    synth.host_apply_drift(ths[m], segs, p, m, r, i0=lo)
                st, g_o = oracle.round_(sends, ths, A0, v0, B=B)
                ok &= st == 0
                pbo, so, nc = oracle.payload_bytes(hi - lo, B), oracle.scales_offset(hi - lo), (hi - lo + 1) // 2
                for m in range(world):
                    got = gathered[m][k].numpy()
                    exp = np.concatenate([g_o[m * pbo: m * pbo + nc], g_o[m * pbo + so: m * pbo + so + 4],
                                          A0.view(np.uint8), v0.view(np.uint8), ths[m].view(np.uint8)])
                    if not np.array_equal(got, exp):
                        ok = False
                        print(f"round {r} block {b} rank {m}: MISMATCH", flush=True)
            print(f"round {r}: {'match' if ok else 'MISMATCH'} ({len(sample)} sampled blocks)", flush=True)
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
