"""Pins of the oracle's fragment schedule (oracle/sd_oracle.c: or_num_fragments,
or_fragment_blocks, or_offset, or_calendar) against the paper's worked
examples (tests/golden/paper_examples.json, each with its citation) and the
calendar invariants of SPEC.md:69-70, :291-292, :317-319."""
import json
import os
import random

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def _cal(**kw):
    return oracle.calendar(oracle.config(**kw))


def test_paper_worked_example_P2_H100():
    g = GOLD["calendar_P2_H100"]
    c = oracle.config(L=g["L"], fs=g["fs"], H=g["H"], tau=g["tau"], T=g["T"])
    assert [oracle.offset(c, p) for p in range(2)] == g["offsets"]
    ev = oracle.calendar(c)
    sends = {}
    for t, kind, p, s in ev:
        if kind == 0:
            sends.setdefault(str(t), []).append(p)
    assert sends == g["sends"]
    # tau = 0: each receive falls on its send step ("receives at same steps")
    assert [(t, p) for t, k, p, s in ev if k == 1] == [(t, p) for t, k, p, s in ev if k == 0]


def test_per_worker_tau_receive_steps():
    g = GOLD["calendar_tau_per_worker"]
    for case in g["cases"]:
        ev = _cal(L=g["L"], fs=g["fs"], H=g["H"], tau=case["tau"], T=g["T"])
        rec = [t for t, k, p, s in ev if k == 1 and s == 100]
        assert rec == [case["receive_of_send_100"]]


def test_partition_examples():
    for case in GOLD["partition"]["cases"]:
        c = oracle.config(L=case["L"], fs=case["fs"], pattern=case["pattern"], H=100)
        assert oracle.num_fragments(c) == case["P"]
        if "fragment0" in case:
            assert oracle.fragment_blocks(c, 0) == case["fragment0"]
        if "fragments" in case:
            assert [oracle.fragment_blocks(c, p) for p in range(case["P"])] == case["fragments"]


def test_offsets_examples():
    for case in GOLD["offsets"]["cases"]:
        c = oracle.config(L=case["L"], fs=case["fs"], H=case["H"])
        assert [oracle.offset(c, p) for p in range(len(case["offsets"]))] == case["offsets"]


def test_offsets_at_the_baseline_configs():
    """S:61 floor(p H / P) where the division is not exact (35M, 1B, 4B: SURVEY §8(a) a1)."""
    for case in GOLD["offsets_configs"]["cases"]:
        c = oracle.config(L=case["L"], fs=case["fs"], H=case["H"])
        assert oracle.num_fragments(c) == len(case["offsets"]), case["name"]
        assert [oracle.offset(c, p) for p in range(len(case["offsets"]))] == case["offsets"], case["name"]


def test_fragment_counts_and_peak_reduction():
    # "8x" peak reduction = L/|p| fragments (AMB-19)
    for case in GOLD["fragment_counts"]["cases"]:
        c = oracle.config(L=case["L"], fs=case["fs"], H=100)
        assert oracle.num_fragments(c) == case["P"] == case["L"] // case["fs"]


def test_sync_every_11_5_2_with_embedding_fragment():
    """at H=100 a fragment syncs every 11, 5, 2 steps with 8/16/36 block
    fragments -> requires the extra embedding fragment (embed_policy 1, AMB-4);
    the SPEC placement (policy 0) gives 12, 6, 2."""
    g = GOLD["sync_every"]
    for case in g["cases"]:
        for policy, expect in ((1, case["every"]), (0, g["H"] // (case["L"] // case["fs"]))):
            c = oracle.config(L=case["L"], fs=case["fs"], H=g["H"], tau=0, T=4 * g["H"], embed_policy=policy)
            sends = sorted({t for t, k, p, s in oracle.calendar(c) if k == 0 and t > g["H"]})
            gaps = [b - a for a, b in zip(sends, sends[1:])]
            assert min(gaps) == expect, (case, policy, gaps[:10])


def _check_invariants(L, fs, pattern, policy, H, tau, T):
    c = oracle.config(L=L, fs=fs, pattern=pattern, embed_policy=policy, H=H, tau=tau, T=T)
    P = oracle.num_fragments(c)
    Pb = L // fs
    # partition property
    blocks = sorted(b for p in range(P) for b in oracle.fragment_blocks(c, p))
    assert blocks == list(range(L))
    offs = [oracle.offset(c, p) for p in range(P)]
    assert all(0 <= o < H for o in offs) and offs == sorted(offs) and len(set(offs)) == P
    ev = oracle.calendar(c)
    sends = [(t, p) for t, k, p, s in ev if k == 0]
    recvs = [(t, p, s) for t, k, p, s in ev if k == 1]
    for p in range(P):
        st = [t for t, q in sends if q == p]
        if st:
            assert st[0] == (H if offs[p] == 0 else H + offs[p])           # first-send rule
            assert all(b - a == H for a, b in zip(st, st[1:]))             # gap property
    per_step = {}
    for t, p in sends:
        per_step[t] = per_step.get(t, 0) + 1
    assert max(per_step.values(), default=0) <= 1                          # H >= P -> one send per step
    # coverage: every H-window after H + max offset sends each fragment exactly once
    for w0 in range(H + max(offs), T - H + 2, max(1, H // 3)):
        got = sorted(p for t, p in sends if w0 <= t < w0 + H)
        assert got == list(range(P))
    # each send received exactly once, at send + tau or flushed at T
    assert sorted((s, p) for t, p, s in recvs) == sorted(sends)
    for t, p, s in recvs:
        assert t == (s + tau if s + tau <= T else T)
    # receive after send within a step when tau = 0 (Alg. 2 order)
    idx = {(k, p, s): i for i, (t, k, p, s) in enumerate(ev)}
    for t, p, s in recvs:
        assert idx[(1, p, s)] > idx[(0, p, s)]
    return c


def test_calendar_invariants_random():
    rng = random.Random(20250130)
    for _ in range(200):
        fs = rng.randint(1, 4)
        L = fs * rng.randint(1, 12)
        policy = rng.randint(0, 1)
        P = L // fs + policy
        H = rng.randint(P, 60)
        tau = rng.randint(0, H - 1)
        T = rng.randint(H, 5 * H)
        _check_invariants(L, fs, rng.randint(0, 1), policy, H, tau, T)


def test_streaming_P1_tau0_is_diloco_calendar():
    # P=1, tau=0 -> send = receive at every multiple of H (Alg. 1)
    ev = _cal(L=4, fs=4, H=30, tau=0, T=200)
    assert [t for t, k, p, s in ev if k == 0] == [30, 60, 90, 120, 150, 180]
    assert [t for t, k, p, s in ev if k == 1] == [30, 60, 90, 120, 150, 180]
