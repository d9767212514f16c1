"""Worker for tests/test_gpu_multi.py: a bounded block-receive (SD_TEST_GATHER
= push | pull, SD_WAIT_TIMEOUT_MS short).  On both ranks rounds 1-2 run
normally, so both buffer halves hold valid payloads of rank 1.  Round 3:
  SD_TEST_SLOW=0: rank 1 never sends (nor merges); rank 0 sends and merges.
  SD_TEST_SLOW=1: rank 1 is slow but alive: it sends and merges round 3
                  only after rank 0's wait has timed out.
Rank 0's block-receive times out, rank 1's stale round-1 payload is not
used, the round is skipped on rank 0 (A, v, theta exactly as before) and
sd_check reports SD_ERR_STATE; the context is then dead (sticky): a later
send fails with SD_ERR_STATE.  With the slow peer, rank 1 also skips the
round (rank 0 told it so), so the anchors stay identical, and is dead too.
Prints OK on success."""
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2501_18512_b200 import FragmentSync, sd  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    n = 5000
    cfg = sd.sd_config_default(4, 2, 20, tau=1)  # P = 2, H = 20
    P = sd.sd_fragment_count(cfg)
    p = 0
    mode = {"push": sd.SD_GATHER_PUSH, "pull": sd.SD_GATHER_PULL}[os.environ["SD_TEST_GATHER"]]
    slow = os.environ.get("SD_TEST_SLOW") == "1"
    fsync = FragmentSync(cfg, [n] * P, rank, world, local, gather_mode=mode)
    g = torch.Generator(device=dev).manual_seed(rank)
    A = torch.randn(n, device=dev, generator=g) * 0.02
    A0 = torch.randn(n, device=dev, generator=torch.Generator(device=dev).manual_seed(99)) * 0.02
    A.copy_(A0)
    v = torch.zeros(n, device=dev)
    th = A0 - 1e-3 * torch.randn(n, device=dev, generator=g)
    ok = True
    for t in (20, 40):  # both buffer halves hold a valid round of rank 1 afterwards
        fsync.send(p, t, th, A)
        fsync.receive(p, t + 1, th, A, v)
        th.sub_(1e-3)
    torch.cuda.synchronize()
    ok &= fsync.check() == (sd.SD_OK, -1)
    dist.barrier()
    t = 60  # same buffer half as round 1: rank 1's stale round-1 payload must not be used

    def skipped_round_then_dead(label):
        good = True
        before = [x.clone() for x in (A, v)]
        fsync.send(p, t, th, A)
        th_before = th.clone()
        fsync.receive(p, t + 1, th, A, v)
        torch.cuda.synchronize()
        try:
            st = fsync.check()[0]
        except sd.SdError as e:  # sd_check raises for statuses other than OK / NONFINITE
            st = e.status
        good &= st == sd.SD_ERR_STATE
        good &= bool(torch.equal(A, before[0]) and torch.equal(v, before[1]) and torch.equal(th, th_before))
        try:  # sticky: the next send is refused
            fsync.send(p, t + 20, th, A)
            good = False
        except sd.SdError as e:
            good &= e.status == sd.SD_ERR_STATE
        print(f"{label}: sd_check -> {st}, state untouched and context dead: {good}", flush=True)
        return good

    if rank == 0 or slow:
        try:
            if rank == 1:  # alive but late: starts round 3 after rank 0's deadline
                time.sleep(3.0 * float(os.environ.get("SD_WAIT_TIMEOUT_MS", "1500")) / 1000.0)
            ok &= skipped_round_then_dead(f"rank {rank}")
        except Exception as e:  # never leave the other rank waiting in the all-reduce below
            print(f"rank {rank}: {e!r}", flush=True)
            ok = False
    if slow:  # the anchors are still identical across the ranks
        ref = A.clone()
        dist.broadcast(ref, src=0)
        ok &= bool(torch.equal(ref, A))
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    fsync.close()
    dist.destroy_process_group()
    if rank == 0:
        print("OK" if flag.item() == 1 else "FAIL", flush=True)
    return 0 if flag.item() == 1 else 1


if __name__ == "__main__":
    sys.exit(main())
