"""Isolated k_apply timing per gather mode on N ranks (torchrun):
every round quantizes + gathers one 1B fragment, waits for the payloads to
be complete on every rank (sd_fragment_wait + synchronize + barrier), then
times the merge alone with CUDA events.  CE mode: the apply reads M local
slots; PULL mode: M-1 of them over NVLink from the peers' buffers.

  torchrun --nproc-per-node N scripts/pull_apply_probe.py [rounds]
"""
import os
import statistics
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2501_18512_b200 import FragmentSync, sd  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
R = int(sys.argv[1]) if len(sys.argv) > 1 else 12
segs = synth.fragment_segments(2048, [0, 8, 16], False)
n = synth.segments_numel(segs)
cfg = sd.sd_config_default(24, 24, 100, tau=1)
A0 = synth.dev_init(torch.empty(n, device=dev), segs, 0)
out = {}
for name, mode in (("ce", sd.SD_GATHER_COPY_ENGINE), ("pull", sd.SD_GATHER_PULL), ("ce2", sd.SD_GATHER_COPY_ENGINE)):
    fs = FragmentSync(cfg, [n], rank, world, dev.index, gather_mode=mode)
    A, v = A0.clone(), torch.zeros(n, device=dev)
    th = A0.clone()
    q_ms, a_ms = [], []
    for r in range(1, R + 1):
        t = 100 * r
        synth.dev_apply_window(th, segs, 0, rank, r)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        fs.ctx.sd_outer_grad_quantize(0, t, th, A, fs.slot(0), n)
        e1.record()
        fs.ctx.sd_fragment_sync(0, t, fs.gather[0], n)
        fs.ctx.sd_fragment_wait(0, t + 1)
        torch.cuda.synchronize()
        dist.barrier()
        e3 = torch.cuda.Event(enable_timing=True)
        e2.record()
        fs.receive(0, t + 1, th, A, v)
        e3.record()
        torch.cuda.synchronize()
        if r > 2:
            q_ms.append(e0.elapsed_time(e1))
            a_ms.append(e2.elapsed_time(e3))
    st = fs.check()
    assert st[0] == sd.SD_OK, st
    fs.close()
    out[name] = (statistics.median(q_ms), statistics.median(a_ms))
    dist.barrier()
res = [None] * world
dist.all_gather_object(res, out)
if rank == 0:
    for name in out:
        qs = [r[name][0] for r in res]
        as_ = [r[name][1] for r in res]
        print(f"{name:5s} M={world} n={n}: quantize ms {['%.4f' % x for x in qs]}  apply ms {['%.4f' % x for x in as_]}")
dist.destroy_process_group()
