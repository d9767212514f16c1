"""Worker for test_gpu_multi.py::test_fsdp_composition (4 ranks): M = 2 DiLoCo
replicas x G = 2 FSDP shards per replica ("split each slab
into G shards at multiples of B; run G independent M-way all-gathers through
communicators split by shard index").  Rank r = replica r // 2, shard r % 2;
shard group s = {s, s + 2} has its own libsd communicator.  After 3 rounds
rank 0 reassembles every replica's fragment and compares it bit for bit with
the unsharded oracle round (codes are unchanged because no scale block
straddles a shard)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2501_18512_b200 import FragmentSync, sd  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    assert world == 4
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    M, G, B = 2, 2, 1024
    m, s = rank // G, rank % G
    ids = [sd.sd_get_unique_id() if rank < G else None]  # rank s creates shard group s's id
    all_ids = [None] * world
    dist.all_gather_object(all_ids, ids[0])
    uid = all_ids[s]
    segs = synth.fragment_segments(128, [0, 3], with_embed=False)
    n = synth.segments_numel(segs)
    n -= n % (G * B)  # shard boundaries at multiples of B
    ns = n // G
    cfg = sd.sd_config_default(4, 2, 20, tau=2, scale_block=B)
    P = sd.sd_fragment_count(cfg)
    p = 0
    fsync = FragmentSync(cfg, [ns] * P, m, M, local, unique_id=uid)
    full_A = synth.dev_init(torch.empty(n, device=dev), segs, p)
    A = full_A[s * ns:(s + 1) * ns].clone()
    v = torch.zeros(ns, device=dev)
    th_full = full_A.clone()
    ok = True
    if rank == 0:
        import oracle

        A_o = synth.host_init(segs, p, 0, n)
        v_o = np.zeros(n, np.float32)
        th_o = [A_o.copy() for _ in range(M)]
    for r in range(1, 4):
        t = r * cfg.H
        synth.dev_apply_window(th_full, segs, p, m, r)
        th = th_full[s * ns:(s + 1) * ns].clone()
        fsync.send(p, t, th, A)
        merged = th_full.clone()
        synth.dev_apply_drift(merged, segs, p, m, r)
        th_full = merged
        th = th_full[s * ns:(s + 1) * ns].clone()
        fsync.receive(p, t + cfg.tau, th, A, v)
        th_full[s * ns:(s + 1) * ns] = th
        # the other shard of this replica lives on the partner rank: exchange to keep th_full whole
        parts = [torch.empty_like(th) for _ in range(world)]
        dist.all_gather(parts, th)
        th_full = torch.cat([parts[m * G + q] for q in range(G)])
        got = {}
        for name, x in (("A", A), ("v", v)):
            pp = [torch.empty_like(x) for _ in range(world)]
            dist.all_gather(pp, x)
            got[name] = [q.cpu().numpy() for q in pp]
        if rank == 0:
            sends = []
            for mm in range(M):
                synth.host_apply_window(th_o[mm], segs, p, mm, r, i0=0)
                sends.append(th_o[mm].copy())
                synth.host_apply_drift(th_o[mm], segs, p, mm, r)
            st, _ = oracle.round_(sends, th_o, A_o, v_o, B=B)
            assert st == 0
            full_th = [torch.cat([parts[mm * G + q] for q in range(G)]).cpu().numpy() for mm in range(M)]
            for mm in range(M):
                A_full = np.concatenate([got["A"][mm * G + q] for q in range(G)])
                v_full = np.concatenate([got["v"][mm * G + q] for q in range(G)])
                ok &= np.array_equal(A_full.view(np.uint32), A_o.view(np.uint32))
                ok &= np.array_equal(v_full.view(np.uint32), v_o.view(np.uint32))
                ok &= np.array_equal(full_th[mm].view(np.uint32), th_o[mm].view(np.uint32))
            print(f"round {r}: {'match' if ok else 'MISMATCH'}", flush=True)
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    fsync.close()
    dist.destroy_process_group()
    if rank == 0:
        print("OK" if flag.item() == 1 else "FAIL", flush=True)
    return 0 if flag.item() == 1 else 1


if __name__ == "__main__":
    sys.exit(main())
