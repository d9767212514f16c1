"""Multi-process host logic on CPU (world_size 2, gloo, 127.0.0.1):
  * every rank's libsd scheduler produces the same calendar and payload sizes;
  * the NCCL unique id broadcast that FragmentSync performs reaches every rank intact;
  * the replica protocol is rank-consistent: each rank quantizes only its own
    replica, the payloads are exchanged (gloo all_gather standing in for the
    NCCL all-gather), each rank applies all M payloads to its own copy of the
    anchor/momentum -> identical outer state on every rank, equal to the
    single-process oracle round (the oracle stands in for the kernels here);
  * bench.py --impl reference under torchrun prints exactly one JSON line (rank 0)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import oracle
    import synth
    from paper_2501_18512_b200 import sd

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    cfg = sd.sd_config_default(24, 3, 100, tau=5, T=1000)
    cal = [sd.sd_fragment_schedule(cfg, t) for t in range(1, 1001)]
    sizes = [sd.sd_payload_bytes(cfg, n) for n in (151007616, 216545664)]
    objs = [None] * world
    dist.all_gather_object(objs, (cal, sizes))
    out["calendar_same"] = all(o == objs[0] for o in objs)
    try:
        uid = [sd.sd_get_unique_id() if rank == 0 else None]
    except sd.SdError:
        uid = [b"x" * 128 if rank == 0 else None]  # no NCCL bootstrap network here: test the broadcast only
    dist.broadcast_object_list(uid, src=0)
    ids = [None] * world
    dist.all_gather_object(ids, uid[0])
    out["uid_same"] = len(uid[0]) == 128 and all(i == ids[0] for i in ids)

    # replica protocol: own quantize -> exchange -> apply on own copies
    segs = synth.fragment_segments(64, [0, 3], with_embed=False)
    n = synth.segments_numel(segs)
    B, p, r = 1024, 1, 1
    A = synth.host_init(segs, p)
    v = np.zeros(n, np.float32)
    th = synth.host_apply_window(A.copy(), segs, p, rank, r)
    pay, _ = oracle.quantize(th, A, B)
    parts = [torch.empty(pay.size, dtype=torch.uint8) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(pay))
    gather = np.concatenate([x.numpy() for x in parts])
    merged = synth.host_apply_drift(th.copy(), segs, p, rank, r)
    st = oracle.apply(gather, world, n, B, A, v, merged)
    states = [None] * world
    dist.all_gather_object(states, (A.tobytes(), v.tobytes()))
    out["outer_state_same"] = st == 0 and all(s == states[0] for s in states)
    if rank == 0:  # equals one process running all replicas
        A1 = synth.host_init(segs, p)
        v1 = np.zeros(n, np.float32)
        sends = [synth.host_apply_window(A1.copy(), segs, p, m, r) for m in range(world)]
        merges = [synth.host_apply_drift(s.copy(), segs, p, m, r) for m, s in enumerate(sends)]
        oracle.round_(sends, merges, A1, v1, B=B)
        out["equals_single_process"] = A1.tobytes() == A.tobytes() and v1.tobytes() == v.tobytes() and \
            merges[0].tobytes() == merged.tobytes()
    dist.destroy_process_group()
    q.put((rank, out))


def test_replica_protocol_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, out in res.items():
        assert all(out.values()), (rank, out)
    assert res[0]["equals_single_process"]


def test_bench_reference_arm_under_torchrun_prints_once():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "2", "--warmup", "1",
           "--workload", "toy"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    assert j["impl"] == "reference" and j["n_gpus"] == 2 and j["value"] > 0
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["cpu_baseline"]["kind"] == "oracle"
