"""Worker for tests/test_gpu_multi.py (run under torchrun, one rank per GPU).

Each rank is one replica: libsd context with an NCCL communicator (unique id
broadcast through torch.distributed), real in-place all-gather over NVLink.
R rounds of one fragment; after every round rank 0 collects every rank's
gather buffer, anchor, momentum and live parameters and checks them against
the CPU oracle (inputs regenerated on the host from the same seeded
generator): byte-identical payloads, bit-identical outer state on every
rank (SURVEY.md §4 "distributed tests").  Prints OK on success."""
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
    local = int(os.environ.get("LOCAL_RANK", rank))
    B = int(os.environ.get("SD_TEST_B", "1024"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    tiny = os.environ.get("SD_TEST_TINY")  # SD_TEST_TINY=<n>: a flat fragment of n elements (0, 1, 7, ...)
    segs = synth.flat_segments(int(tiny)) if tiny else synth.fragment_segments(96, [0, 4], with_embed=True, vocab=333)
    n = synth.segments_numel(segs)
    # per-replica tau: SD_TEST_TAU_PER_RANK=1 gives rank m tau = 1 + 2m
    tau = 1 + 2 * rank if os.environ.get("SD_TEST_TAU_PER_RANK") == "1" else 3
    cfg = sd.sd_config_default(8, 2, 40, tau=tau, scale_block=B)  # P = 4 fragments, H = 40
    P = sd.sd_fragment_count(cfg)
    p = 2
    _, t_p, _ = sd.sd_fragment_layout(cfg, p)
    mode = {"push": sd.SD_GATHER_PUSH, "pull": sd.SD_GATHER_PULL}.get(
        os.environ.get("SD_TEST_GATHER"), sd.SD_GATHER_COPY_ENGINE)
    # SD_TEST_COMM=1: a communicator even at world = 1 (the one-rank gather paths, runnable on one GPU)
    fsync = FragmentSync(cfg, [n] * P, rank, world, local, gather_mode=mode,
                         communicator=True if os.environ.get("SD_TEST_COMM") == "1" else None)
    if os.environ.get("SD_TEST_TORCH_BUF") == "1":  # caller-owned (non-symmetric) gather buffers
        fsync.gather = [torch.empty(world * pb, dtype=torch.uint8, device=dev) for pb in fsync.payload]
    A = synth.dev_init(torch.empty(n, device=dev), segs, p)
    v = torch.zeros(n, device=dev)
    th = A.clone()
    ok = True
    # SD_TEST_POISON=1: the last rank's theta holds a NaN at index 17 in the last round's send -> every
    # rank skips that round (A, v, theta unchanged) and sd_check reports SD_ERR_NONFINITE at 17 (AMB-10)
    poison = os.environ.get("SD_TEST_POISON") == "1"
    # SD_TEST_OFFLOAD=1: A and v live in pinned host memory (NEXT-3); A, v on the device are staging
    # buffers, scribbled before every prefetch, so the round can only be right if the copies are ordered
    offload = os.environ.get("SD_TEST_OFFLOAD") == "1"
    if offload:
        hA, hv = A.cpu().pin_memory(), v.cpu().pin_memory()
    R = 5

    def same(a, b):  # bit-identical, NaN payloads aside
        nan = np.isnan(a) & np.isnan(b)
        return bool(np.array_equal(a.view(np.uint32)[~nan], b.view(np.uint32)[~nan]) and
                    np.array_equal(np.isnan(a), np.isnan(b)))

    if rank == 0:
        import oracle

        A_o = synth.host_init(segs, p)
        v_o = np.zeros(n, np.float32)
        th_o = [A_o.copy() for _ in range(world)]
    for r in range(1, R + 1):
        bad = poison and r == R
        t = min(r, 3) * cfg.H + t_p  # rounds 4, 5 repeat step t of round 3 (round ids must not rely on t)
        assert p in sd.sd_fragment_schedule(cfg, t)[0]
        synth.dev_apply_window(th, segs, p, rank, r)
        if bad and rank == world - 1:
            th[17] = float("nan")
        if offload:
            A.fill_(float("nan"))
            v.fill_(-1.0)
            fsync.ctx.sd_state_prefetch(p, hA, hv, A, v, n)
        fsync.send(p, t, th, A)
        synth.dev_apply_drift(th, segs, p, rank, r)      # tau overlapped inner steps
        assert p in sd.sd_fragment_schedule(cfg, t + cfg.tau)[1]
        fsync.receive(p, t + cfg.tau, th, A, v)
        if offload:
            fsync.ctx.sd_state_writeback(p, A, v, hA, hv, n)
            fsync.ctx.sd_state_sync()
            torch.cuda.synchronize()
            A.copy_(hA)  # compare what the host store holds
            v.copy_(hv)
        torch.cuda.synchronize()
        got = {}
        pb = fsync.payload[p]
        own = fsync.payloads(p)[rank * pb:(rank + 1) * pb]  # each rank's own slot (valid in every mode)
        for name, x in (("gather", own), ("A", A), ("v", v), ("theta", th)):
            parts = [torch.empty_like(x) for _ in range(world)]
            dist.all_gather(parts, x)
            got[name] = [q.cpu().numpy() for q in parts]
        if rank == 0:
            sends = []
            for m in range(world):
                synth.host_apply_window(th_o[m], segs, p, m, r)
                if bad and m == world - 1:
                    th_o[m][17] = np.nan
                sends.append(th_o[m].copy())
                synth.host_apply_drift(th_o[m], segs, p, m, r)
            st, g_o = oracle.round_(sends, th_o, A_o, v_o, B=B)
            assert st == (1 if bad else 0), st
            if not bad:  # a poisoned slot's codes are unspecified; its trailer names the index
                ok &= np.array_equal(np.concatenate(got["gather"]), g_o)
            for m in range(world):
                ok &= same(got["A"][m], A_o) and same(got["v"][m], v_o) and same(got["theta"][m], th_o[m])
            print(f"round {r}: {'match' if ok else 'MISMATCH'}", flush=True)
    st, fb = fsync.check()
    ok &= (st, fb) == ((sd.SD_ERR_NONFINITE, 17) if poison else (sd.SD_OK, -1))
    if (st, fb) != ((sd.SD_ERR_NONFINITE, 17) if poison else (sd.SD_OK, -1)):
        print(f"rank {rank}: sd_check -> {st}, {fb}", flush=True)
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    fsync.close()
    dist.destroy_process_group()
    if rank == 0:
        print("OK" if flag.item() == 1 else "FAIL", flush=True)
    return 0 if flag.item() == 1 else 1


if __name__ == "__main__":
    sys.exit(main())
