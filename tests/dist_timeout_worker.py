"""Worker for tests/test_gpu_multi.py: a peer that never sends (SD_TEST_GATHER
= push | pull | mc, SD_WAIT_TIMEOUT_MS short).  On both ranks rounds 1-2 run
normally, so both buffer halves hold valid payloads of rank 1; in round 3
rank 1 skips its send (and so its merge), rank 0 sends and merges: its
block-receive times out, rank 1's stale round-1 payload is not used, the
round is skipped on rank 0 (A, v, theta exactly as before the merge) and
sd_check reports SD_ERR_STATE.  Prints OK on success."""
import os
import sys

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
    mode = {"push": sd.SD_GATHER_PUSH, "pull": sd.SD_GATHER_PULL, "mc": sd.SD_GATHER_MULTICAST}[
        os.environ["SD_TEST_GATHER"]]
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
    if rank == 0:
        try:
            before = [x.clone() for x in (A, v)]
            fsync.send(p, t, th, A)
            th_before = th.clone()
            fsync.receive(p, t + 1, th, A, v)
            torch.cuda.synchronize()
            try:
                st = fsync.check()[0]
            except sd.SdError as e:  # sd_check raises for statuses other than OK / NONFINITE
                st = e.status
            ok &= st == sd.SD_ERR_STATE
            ok &= bool(torch.equal(A, before[0]) and torch.equal(v, before[1]) and torch.equal(th, th_before))
            print(f"rank 0: sd_check -> {st}, state untouched: {ok}", flush=True)
        except Exception as e:  # never leave rank 1 waiting in the all-reduce below
            print(f"rank 0: {e!r}", flush=True)
            ok = False
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    fsync.close()
    dist.destroy_process_group()
    if rank == 0:
        print("OK" if flag.item() == 1 else "FAIL", flush=True)
    return 0 if flag.item() == 1 else 1


if __name__ == "__main__":
    sys.exit(main())
