"""Soak worker for tests/test_gpu_multi.py: many pipelined rounds of the full
1B workload (all 8 fragments on the calendar, sends of step k overlapping
the receive of step k-1 as in bench.py) in one gather mode (SD_TEST_GATHER),
then a property that holds at any size and after any number of rounds: the
anchors and momenta of every fragment are bit-identical on every rank, and
no round was skipped.  A race in the payload exchange (a half overwritten
while read, a flag seen before its data) would desynchronize them.
Prints OK on success."""
import os
import sys

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
    rounds = int(os.environ.get("SD_TEST_ROUNDS", "200"))
    wl = WORKLOADS["1B"]
    cfg = sd.sd_config_default(wl.layers, wl.fragment_size, wl.H, tau=wl.tau)
    P = sd.sd_fragment_count(cfg)
    layout = [sd.sd_fragment_layout(cfg, q) for q in range(P)]
    segs = [wl.segments(b, e) for b, _, e in layout]
    n = [synth.segments_numel(s) for s in segs]
    mode = {"push": sd.SD_GATHER_PUSH, "pull": sd.SD_GATHER_PULL,
            "ce": sd.SD_GATHER_COPY_ENGINE}[os.environ["SD_TEST_GATHER"]]
    fsync = FragmentSync(cfg, n, rank, world, local, gather_mode=mode)
    A = [synth.dev_init(torch.empty(k, device=dev), s, p) for p, (k, s) in enumerate(zip(n, segs))]
    v = [torch.zeros(k, device=dev) for k in n]
    th = [a.clone() for a in A]
    events, t = [], cfg.H
    while len(events) < rounds:
        s, _ = sd.sd_fragment_schedule(cfg, t)
        events.extend((p, t) for p in s)
        t += 1
    prev = None
    for i, (p, t) in enumerate(events[:rounds]):
        synth.dev_apply_window(th[p], segs[p], p, rank, i + 1)   # this replica's inner progress
        fsync.send(p, t, th[p], A[p])
        if prev is not None:
            q, tq = prev
            fsync.receive(q, tq + cfg.tau, th[q], A[q], v[q])
        prev = (p, t)
    q, tq = prev
    fsync.receive(q, tq + cfg.tau, th[q], A[q], v[q])
    torch.cuda.synchronize()
    ok = fsync.check() == (sd.SD_OK, -1)
    for p in range(P):
        for x in (A[p], v[p]):
            ref = x.clone()
            dist.broadcast(ref, 0)
            ok &= bool(torch.equal(ref.view(torch.int32), x.view(torch.int32)))
    # every replica contributed: the anchors moved away from the initial parameters
    ok &= any(not torch.equal(A[p], synth.dev_init(torch.empty(n[p], device=dev), segs[p], p)) for p in range(P))
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    fsync.close()
    dist.destroy_process_group()
    if rank == 0:
        print(f"{rounds} rounds: " + ("OK" if flag.item() == 1 else "FAIL"), flush=True)
    return 0 if flag.item() == 1 else 1


if __name__ == "__main__":
    sys.exit(main())
