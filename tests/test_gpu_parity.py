"""GPU parity: libsd's CUDA path (through the C ABI) vs the CPU oracle.

Bar: payload bytes (codes, scales, padding, trailer) are
byte-identical; anchor, momentum and live parameters are bit-identical
(0 differing elements is the expectation under the pinned fp32 operation
sequence), with the floored 1e-6 relative check of BASELINE.json's
north_star as the stated tolerance.  Inputs: seeded synthetic data shaped
like the paper's Chinchilla fragments (synth/) plus codec edge cases."""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2501_18512_b200 import sd

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from gpu_harness import DEV, EmulatedReplicas, bits, edge_deltas, theta_anchor_for, to_dev


def floored_rel_err(gpu: np.ndarray, ora: np.ndarray) -> float:
    """max_i |g_i - o_i| / max(|o_i|, 2^-10 max_j |o_j|)"""
    g, o = gpu.astype(np.float64), ora.astype(np.float64)
    if o.size == 0:
        return 0.0
    floor = 2.0 ** -10 * np.max(np.abs(o))
    den = np.maximum(np.abs(o), floor)
    den[den == 0] = 1.0
    return float(np.max(np.abs(g - o) / den))


def assert_same(gpu, ora, what):
    gb, ob = bits(gpu), bits(ora)
    nbad = int(np.count_nonzero(gb != ob))
    assert floored_rel_err(gpu if isinstance(gpu, np.ndarray) else gpu.cpu().numpy(), ora) <= 1e-6, what
    assert nbad == 0, f"{what}: {nbad} elements differ bitwise"


def cfg_for(B, alpha=0.5, lr=0.4, mu=0.9, tau=1):
    return sd.sd_config_default(2, 1, 10, tau=tau, scale_block=B, alpha=alpha, outer_lr=lr, outer_momentum=mu)


# ------------------------------------------------------------------ quantize
@pytest.mark.parametrize("B,staged", [(0, True), (0, False), (256, True), (512, True), (1024, True), (2048, True),
                                      (2048, False), (65536, True), (65536, False)])
@pytest.mark.parametrize("n", [1, 2, 3, 5, 1023, 1024, 1025, 4097, 33 * 1024 + 511, 262144 + 3])
def test_quantize_payload_bytes_match(n, B, staged):
    """staged: the two-pass quantize (B = 0, 2048, 65536) with a workspace
    (encode from 16-bit summaries, exact re-read at straddled thresholds) and
    without one (re-read); the single-pass B's ignore it."""
    rng = np.random.default_rng(n * 7 + B)
    cfg = cfg_for(B)
    for exact in (True, False):
        delta = edge_deltas(n, B, rng)
        A, th = theta_anchor_for(delta, rng, exact)
        rep = EmulatedReplicas(cfg, 1, n, staged=staged)
        rep.slot(0).fill_(0xAB)  # garbage: every byte must be written
        rep.quantize_all(0, 10, [to_dev(th)], [to_dev(A)])
        torch.cuda.synchronize()
        want, poisoned = oracle.quantize(th, A, B)
        got = rep.gather.cpu().numpy()
        assert not poisoned
        diff = np.nonzero(got != want)[0]
        assert diff.size == 0, f"n={n} B={B} exact={exact}: {diff.size} bytes differ, first at {diff[:8]}"
        rep.close()


@pytest.mark.parametrize("B", [0, 4096])
@pytest.mark.parametrize("n", [256 * 1024 + 77, 3 * 1024 * 1024 + 5])
def test_quantize_staged_buckets(n, B):
    """The staged two-pass quantize against the oracle where its 16-bit
    summaries are tested hardest: rows (256 elements) whose maxima sit 0..8
    octaves below the block scale s (so the summary's base moves), every
    value within +-6 ulps of a threshold T_j(s) = s 2^(-j-1/2) that lies
    below its row's max (so most buckets straddle or touch a threshold and
    take the exact re-read), values below 2^-7 of the row max, and -0 / +0."""
    from decimal import Decimal

    rng = np.random.default_rng(n + B)
    blen = B if B else n
    d = np.zeros(n, np.float32)
    for b0 in range(0, n, blen):
        s = np.float32(rng.uniform(0.5, 2.0) * 2.0 ** int(rng.integers(-20, 20)))
        T = [np.float32(float(Decimal(float(s)) * (Decimal(2) ** Decimal(-j - 0.5)))) for j in range(7)]
        for r0 in range(b0, min(n, b0 + blen), 256):
            r1 = min(n, r0 + 256, b0 + blen)
            oct_ = int(rng.integers(0, 9))
            j = rng.integers(min(oct_, 6), 7, r1 - r0)
            tb = np.array([int(T[k].view(np.uint32)) for k in j], np.int64) + rng.integers(-6, 7, r1 - r0)
            vals = tb.astype(np.uint32).view(np.float32) * np.where(rng.random(r1 - r0) < 0.5, 1, -1).astype(np.float32)
            low = rng.random(r1 - r0) < 0.2  # far below the row max
            vals[low] = (s * np.float32(2.0 ** -(oct_ + 8)) * rng.random(int(low.sum()))).astype(np.float32)
            vals[rng.random(r1 - r0) < 0.05] = -0.0
            vals[0] = np.float32(s * np.float32(2.0 ** -oct_))  # the row max
            d[r0:r1] = vals
        d[b0 + int(rng.integers(0, min(blen, n - b0)))] = s  # the block max
    A, th = theta_anchor_for(d, rng, True)
    rep = EmulatedReplicas(cfg_for(B), 1, n, staged=True)
    rep.quantize_all(0, 10, [to_dev(th)], [to_dev(A)])
    torch.cuda.synchronize()
    want, poisoned = oracle.quantize(th, A, B)
    got = rep.gather.cpu().numpy()
    assert not poisoned
    diff = np.nonzero(got != want)[0]
    assert diff.size == 0, f"{diff.size} bytes differ, first at {diff[:8]}"
    rep.close()


def test_quantize_workspace_rules():
    """sd_set_workspace: a 256-byte-misaligned workspace is refused; one
    smaller than sd_quantize_workspace_bytes(n) is not used (the re-reading
    pass runs); detaching works; all give the oracle's payload."""
    n, B = 5 * 1024 + 3, 0
    cfg = cfg_for(B)
    need = sd.sd_quantize_workspace_bytes(cfg, n)
    assert need == 6 * (2048 + 16)
    rng = np.random.default_rng(3)
    delta = edge_deltas(n, B, rng)
    A, th = theta_anchor_for(delta, rng, False)
    want, _ = oracle.quantize(th, A, B)
    big = torch.zeros(need + 512, dtype=torch.uint8, device=DEV)
    for ws, nbytes in ((big[1:], need), (big, need - 1), (big, need), (None, 0)):
        rep = EmulatedReplicas(cfg, 1, n, staged=False)
        if ws is not None and ws.data_ptr() % 256:
            with pytest.raises(sd.SdError) as e:
                rep.ctx[0].sd_set_workspace(ws, nbytes)
            assert e.value.status == sd.SD_ERR_ARG and "aligned" in e.value.msg
        else:
            rep.ctx[0].sd_set_workspace(ws, nbytes)
        rep.quantize_all(0, 10, [to_dev(th)], [to_dev(A)])
        torch.cuda.synchronize()
        assert np.array_equal(rep.gather.cpu().numpy(), want)
        rep.close()


def test_quantize_synthetic_chinchilla_fragment():
    segs = synth.fragment_segments(128, [0, 5], with_embed=True, vocab=1000)
    n = synth.segments_numel(segs)
    A = synth.host_init(segs, 3)
    th = synth.host_apply_window(A.copy(), segs, 3, 1, 1)
    for B in (1024, 0):
        rep = EmulatedReplicas(cfg_for(B), 1, n)
        rep.quantize_all(0, 10, [to_dev(th)], [to_dev(A)])
        torch.cuda.synchronize()
        want, _ = oracle.quantize(th, A, B)
        assert np.array_equal(rep.gather.cpu().numpy(), want)
        rep.close()


# -------------------------------------------------------------- full rounds
@pytest.mark.parametrize("M", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("B", [1024, 256, 0])
def test_rounds_bit_exact(M, B):
    """R = 3 rounds of one fragment on M emulated replicas: payloads, anchor,
    momentum and every replica's merged parameters vs or_round."""
    segs = synth.fragment_segments(64, [0, 2], with_embed=False)
    n = synth.segments_numel(segs) + 123  # ragged: not a multiple of 4 or of B
    segs = np.concatenate([segs, np.array([(n - 123, 123, synth.NORM, 0, 1, 0)], dtype=synth.SEG_DTYPE)])
    p, H, tau = 0, 10, 1
    cfg = cfg_for(B, tau=tau)
    A_o = synth.host_init(segs, p)
    v_o = np.zeros(n, np.float32)
    th_o = [A_o.copy() for _ in range(M)]
    rep = EmulatedReplicas(cfg, M, n)
    A_d = [to_dev(A_o) for _ in range(M)]
    v_d = [torch.zeros(n, dtype=torch.float32, device=DEV) for _ in range(M)]
    th_d = [to_dev(A_o) for _ in range(M)]
    for r in range(1, 4):
        t_send = r * H
        for m in range(M):
            synth.host_apply_window(th_o[m], segs, p, m, r)
            synth.dev_apply_window(th_d[m], segs, p, m, r)
        rep.quantize_all(p, t_send, th_d, A_d)
        sends = [x.copy() for x in th_o]
        for m in range(M):
            synth.host_apply_drift(th_o[m], segs, p, m, r)
            synth.dev_apply_drift(th_d[m], segs, p, m, r)
        rep.merge_all(p, t_send + tau, th_d, A_d, v_d)
        st, g_o = oracle.round_(sends, th_o, A_o, v_o, B=B)
        torch.cuda.synchronize()
        assert st == 0
        assert np.array_equal(rep.gather.cpu().numpy(), g_o), f"round {r}: gather bytes differ"
        for m in range(M):
            assert_same(A_d[m], A_o, f"round {r} anchor (replica {m})")
            assert_same(v_d[m], v_o, f"round {r} momentum (replica {m})")
            assert_same(th_d[m], th_o[m], f"round {r} theta (replica {m})")
    assert all(s == (sd.SD_OK, -1) for s in rep.check_all())
    rep.close()


@pytest.mark.parametrize("alpha,lr,mu", [(0.0, 1.0, 0.0), (1.0, 0.4, 0.9), (0.25, 0.7, 0.5)])
def test_rounds_hyperparameter_edges(alpha, lr, mu):
    rng = np.random.default_rng(int(alpha * 100 + lr * 10))
    n, M = 8192 + 5, 2
    cfg = cfg_for(1024, alpha=alpha, lr=lr, mu=mu)
    A0 = (rng.standard_normal(n) * 0.02).astype(np.float32)
    sends = [(A0 - edge_deltas(n, 1024, rng)).astype(np.float32) for _ in range(M)]
    merges = [(s - np.float32(1e-4)).astype(np.float32) for s in sends]
    rep = EmulatedReplicas(cfg, M, n)
    A_d, v_d = [to_dev(A0) for _ in range(M)], [torch.full((n,), 0.01, device=DEV) for _ in range(M)]
    th_d = [to_dev(s) for s in sends]
    rep.quantize_all(0, 10, th_d, A_d)
    for m in range(M):
        th_d[m].copy_(to_dev(merges[m]))
    rep.merge_all(0, 11, th_d, A_d, v_d)
    A_o, v_o = A0.copy(), np.full(n, 0.01, np.float32)
    mo = [x.copy() for x in merges]
    oracle.round_(sends, mo, A_o, v_o, B=1024, lr=lr, mu=mu, alpha=alpha)
    torch.cuda.synchronize()
    for m in range(M):
        assert_same(A_d[m], A_o, "anchor")
        assert_same(v_d[m], v_o, "momentum")
        assert_same(th_d[m], mo[m], "theta")
    rep.close()


def test_empty_fragment():
    cfg = cfg_for(1024)
    rep = EmulatedReplicas(cfg, 2, 0)
    e = torch.empty(0, device=DEV)
    rep.quantize_all(0, 10, [e, e], [e, e])
    rep.merge_all(0, 11, [e, e], [e, e], [e, e])
    torch.cuda.synchronize()
    want, _ = oracle.quantize(np.zeros(0, np.float32), np.zeros(0, np.float32), 1024)
    assert np.array_equal(rep.gather.cpu().numpy(), np.concatenate([want, want]))
    rep.close()


# ------------------------------------------------------------------- poison
def test_nonfinite_round_skipped_on_every_replica():
    n, M = 5000, 2
    cfg = cfg_for(1024)
    rep = EmulatedReplicas(cfg, M, n)
    A0 = np.ones(n, np.float32)
    th = [np.zeros(n, np.float32) for _ in range(M)]
    th[1][4321] = np.inf
    th[1][2222] = np.nan
    A_d = [to_dev(A0) for _ in range(M)]
    v_d = [torch.zeros(n, device=DEV) for _ in range(M)]
    th_d = [to_dev(x) for x in th]
    rep.quantize_all(0, 10, th_d, A_d)
    rep.merge_all(0, 11, th_d, A_d, v_d)
    torch.cuda.synchronize()
    r, fb = oracle.payload_poisoned(rep.gather.cpu().numpy()[rep.pb:], n, 1024)
    assert r == 1 and fb == 2222
    for m in range(M):
        assert np.array_equal(A_d[m].cpu().numpy(), A0) and not v_d[m].any()
        assert np.array_equal(bits(th_d[m]), bits(th[m]))
    for st in rep.check_all():
        assert st == (sd.SD_ERR_NONFINITE, 2222)
    rep.close()


# -------------------------------------------------------- call-order checks
def test_schedule_and_state_errors():
    n = 4096
    cfg = cfg_for(1024)
    rep = EmulatedReplicas(cfg, 2, n)
    x = torch.zeros(n, device=DEV)
    with pytest.raises(sd.SdError) as e:
        rep.ctx[0].sd_outer_grad_quantize(0, 11, x, x, rep.slot(0), n)  # fragment 0 sends at 10, 20, ...
    assert e.value.status == sd.SD_ERR_SCHEDULE
    with pytest.raises(sd.SdError) as e:
        rep.ctx[0].sd_merge(0, 11, rep.gather, x, x, x, n)  # nothing in flight
    assert e.value.status == sd.SD_ERR_STATE
    rep.ctx[0].sd_outer_grad_quantize(0, 10, x, x, rep.slot(0), n)
    with pytest.raises(sd.SdError) as e:
        rep.ctx[0].sd_outer_grad_quantize(0, 10, x, x, rep.slot(0), n)  # still in flight
    assert e.value.status == sd.SD_ERR_STATE
    with pytest.raises(sd.SdError) as e:
        rep.ctx[1].sd_outer_grad_quantize(1, 15, x, x, rep.slot(0), n)  # fine...
        rep.ctx[1].sd_fragment_sync(1, 15, rep.gather, n)              # ...but slot 0 is not rank 1's
    assert e.value.status == sd.SD_ERR_ARG
    rep.ctx[0].sd_fragment_sync(0, 10, rep.gather, n)
    with pytest.raises(sd.SdError) as e:
        rep.ctx[0].sd_merge(0, 12, rep.gather, x, x, x, n)  # tau = 1: receive at 11
    assert e.value.status == sd.SD_ERR_SCHEDULE
    with pytest.raises(sd.SdError) as e:
        rep.ctx[0].sd_merge(0, 11, rep.gather, x[1:], x, x, n)  # misaligned theta
    assert e.value.status == sd.SD_ERR_ARG
    torch.cuda.synchronize()
    rep.close()


# ---------------------------------------------------------------- toy, e2e
@pytest.mark.parametrize("L,fs,H,tau,T,M,bl", [
    (2, 1, 10, 1, 100, 2, 2 ** 19),      # BASELINE.json configs[0]
    (1, 1, 5, 0, 23, 3, 3000),           # DiLoCo (Alg. 1): P = 1, tau = 0, M = 3
    (6, 2, 12, 0, 50, 2, 4096 + 4),      # tau = 0 with 3 strided fragments, ragged (n = 8200)
    (4, 1, 9, 8, 40, 4, 2048),           # tau = H - 1, flush at T
])
def test_toy_config_alg2_end_to_end(L, fs, H, tau, T, M, bl):
    """Alg. 2 end to end.  configs[0]: M=2, 2^20 fp32 params in 2 fragments,
    H=10, tau=1, T=100; plus the degenerate schedules.  Every step: synthetic
    inner step on each replica, then the calendar's sends and receives
    through libsd; final theta (every replica), anchors and momenta
    bit-identical to or_toy_run."""
    c_or = oracle.config(L=L, fs=fs, H=H, tau=tau, T=T)
    th_o, A_o, v_o, sent_o, st = oracle.toy_run(c_or, M, bl, synth.SEED)
    assert st == 0
    cfg = sd.sd_config_default(L, fs, H, tau=tau, T=T)
    P = sd.sd_fragment_count(cfg)
    n = fs * bl
    reps = [EmulatedReplicas(cfg, M, n) for _ in range(P)]
    A = [[synth.dev_init(torch.empty(n, device=DEV), synth.flat_segments(n), p) for _ in range(M)] for p in range(P)]
    v = [[torch.zeros(n, device=DEV) for _ in range(M)] for p in range(P)]
    th = [torch.cat([A[p][0] for p in range(P)]).clone() for _ in range(M)]  # replica m's full vector
    frag = lambda m, p: th[m][p * n:(p + 1) * n]
    sent = 0
    for t in range(1, T + 1):
        for m in range(M):
            synth.dev_apply_toy(th[m], m, t)
        send, recv = sd.sd_fragment_schedule(cfg, t)
        for p in send:
            reps[p].quantize_all(p, t, [frag(m, p) for m in range(M)], A[p])
            sent += M * reps[p].pb
        for p in recv:
            reps[p].merge_all(p, t, [frag(m, p) for m in range(M)], A[p], v[p])
    torch.cuda.synchronize()
    assert sent == sent_o
    for m in range(M):
        assert_same(th[m], th_o[m], f"theta replica {m}")
    for p in range(P):
        for m in range(M):
            assert_same(A[p][m], A_o[p * n:(p + 1) * n], f"anchor fragment {p}")
            assert_same(v[p][m], v_o[p * n:(p + 1) * n], f"momentum fragment {p}")
    for r in reps:
        r.close()


# ------------------------------------------------- full size, bench layout
@pytest.mark.parametrize("shape", ["1B", "4B_last"])
def test_full_size_sampled_blocks(shape):
    """BASELINE.json full sizes in the bench's launch configuration: the 1B
    fragment (n = 151,007,616, M = 2) and the 4B last fragment (n =
    438,064,512 incl. embedding, M = 4), emulated on one GPU.  The oracle
    recomputes sampled 1024-element scale blocks one by one (each block's
    codes, scale and outputs depend only on that block), inputs regenerated
    on the host from the same counter-based generator."""
    if shape == "1B":
        d, layers, emb, M = 2048, [0, 8, 16], False, 2
    else:
        d, layers, emb, M = 3072, [11, 23, 35], True, 4
    segs = synth.fragment_segments(d, layers, emb)
    n = synth.segments_numel(segs)
    p, r, B = 0, 1, 1024
    cfg = cfg_for(B, tau=1)
    rep = EmulatedReplicas(cfg, M, n)
    A_d = synth.dev_init(torch.empty(n, device=DEV), segs, p)
    Acopies = [A_d] + [A_d.clone() for _ in range(M - 1)]
    v_d = [torch.zeros(n, device=DEV) for _ in range(M)]
    th_d = []
    for m in range(M):
        th = A_d.clone()
        synth.dev_apply_window(th, segs, p, m, r)
        th_d.append(th)
    rep.quantize_all(p, 10, th_d, Acopies)
    for m in range(M):
        synth.dev_apply_drift(th_d[m], segs, p, m, r)
    rep.merge_all(p, 11, th_d, Acopies, v_d)
    torch.cuda.synchronize()
    nb = -(-n // B)
    rng = np.random.default_rng(4)
    blocks = sorted(set([0, nb - 1] + list(rng.integers(0, nb, 48))))
    soff = sd.sd_payload_scales_offset(n)
    gat = rep.gather
    for b in blocks:
        lo, hi = b * B, min(n, (b + 1) * B)
        A0 = synth.host_init(segs, p, lo, hi)
        sends = [synth.host_apply_window(A0.copy(), segs, p, m, r, i0=lo) for m in range(M)]
        merges = [synth.host_apply_drift(s.copy(), segs, p, m, r, i0=lo) for m, s in enumerate(sends)]
        Ao, vo = A0.copy(), np.zeros(hi - lo, np.float32)
        st, g_o = oracle.round_(sends, merges, Ao, vo, B=B)
        assert st == 0
        pb_o = oracle.payload_bytes(hi - lo, B)
        for m in range(M):
            base = m * rep.pb
            got_codes = gat[base + lo // 2: base + (hi + 1) // 2].cpu().numpy()
            assert np.array_equal(got_codes, g_o[m * pb_o: m * pb_o + (hi - lo + 1) // 2]), f"block {b} codes"
            got_s = gat[base + soff + 4 * b: base + soff + 4 * b + 4].cpu().numpy()
            so = oracle.scales_offset(hi - lo)
            assert np.array_equal(got_s, g_o[m * pb_o + so: m * pb_o + so + 4]), f"block {b} scale"
            assert_same(Acopies[m][lo:hi], Ao, f"block {b} anchor")
            assert_same(v_d[m][lo:hi], vo, f"block {b} momentum")
            assert_same(th_d[m][lo:hi], merges[m], f"block {b} theta")
    rep.close()


@pytest.mark.parametrize("adamw", [False, True])
def test_full_size_b0_staged_whole_fragment(adamw):
    """SPEC's B = 0 (one scale per fragment) at the full 1B fragment
    size (n = 151,007,616) in the bench's launch configuration: the staged
    two-pass quantize with its workspace (FragmentSync's), M = 2 emulated.
    One scale depends on the whole fragment, so nothing short of the whole
    round is checked: both payloads byte for byte (76 MB each) and A, v,
    theta element for element against the oracle's full round (OpenMP
    build, bit-identical to the single-thread one).  adamw: the send goes
    through sd_inner_adamw_quantize (AdamW + block max + summaries, then the
    encode pass), against or_adamw then the oracle round."""
    segs = synth.fragment_segments(2048, [0, 8, 16], False)
    n = synth.segments_numel(segs)
    assert n == 151007616
    M, p, r, B = 2, 0, 1, 0
    cfg = cfg_for(B, tau=1)
    rep = EmulatedReplicas(cfg, M, n)
    A_d = synth.dev_init(torch.empty(n, device=DEV), segs, p)
    Acopies = [A_d] + [A_d.clone() for _ in range(M - 1)]
    v_d = [torch.zeros(n, device=DEV) for _ in range(M)]
    th_d = []
    for m in range(M):
        th = A_d.clone()
        synth.dev_apply_window(th, segs, p, m, r)
        th_d.append(th)
    A0 = synth.host_init(segs, p)
    sends = [synth.host_apply_window(A0.copy(), segs, p, m, r) for m in range(M)]
    if adamw:
        hp = sd.SdAdamW(**HP)
        rng = np.random.default_rng(5)
        g = [(rng.standard_normal(n, dtype=np.float32) * np.float32(1e-3)).astype(np.float32) for _ in range(M)]
        m1 = [np.zeros(n, np.float32) for _ in range(M)]
        m2 = [np.zeros(n, np.float32) for _ in range(M)]
        m1_d, m2_d = [to_dev(x) for x in m1], [to_dev(x) for x in m2]
        for m in range(M):
            rep.ctx[m].sd_inner_adamw_quantize(p, 10, 1, th_d[m], to_dev(g[m]), m1_d[m], m2_d[m], Acopies[m],
                                               rep.slot(m), hp, n)
        for m in range(M):
            rep.ctx[m].sd_fragment_sync(p, 10, rep.gather, n)
        for m in range(M):
            oracle.adamw(sends[m], g[m], m1[m], m2[m], 1, lr=HP["lr"], b1=HP["beta1"], b2=HP["beta2"], eps=HP["eps"],
                         wd=HP["weight_decay"])
    else:
        rep.quantize_all(p, 10, th_d, Acopies)
    for m in range(M):
        synth.dev_apply_drift(th_d[m], segs, p, m, r)
    rep.merge_all(p, 11, th_d, Acopies, v_d)
    torch.cuda.synchronize()
    merges = [synth.host_apply_drift(s.copy(), segs, p, m, r) for m, s in enumerate(sends)]
    Ao, vo = A0.copy(), np.zeros(n, np.float32)
    prev = oracle.threads()
    oracle.set_threads(max(1, os.cpu_count() or 1))
    try:
        st, g_o = oracle.round_(sends, merges, Ao, vo, B=B)
    finally:
        oracle.set_threads(prev)
    assert st == 0
    got = rep.gather.cpu().numpy()
    diff = np.nonzero(got != g_o)[0]
    assert diff.size == 0, f"{diff.size} payload bytes differ, first at {diff[:8]}"
    for m in range(M):
        assert_same(Acopies[m], Ao, f"anchor {m}")
        assert_same(v_d[m], vo, f"momentum {m}")
        assert_same(th_d[m], merges[m], f"theta {m}")
    rep.close()


@pytest.mark.parametrize("B", [1024, 4096])
def test_fragment_beyond_2_31_elements(B):
    """Maximum sizes: one fragment of 2.42e9 elements (3 layers at d = 8192;
    every fp32 array > 8 GiB, byte offsets > 2^33), M = 2 emulated, the
    one-pass (B = 1024) and two-pass (B = 4096) quantize.  Sampled
    scale blocks -- including those at element 2^30, 2^31 and the ragged
    tail -- are bit-identical to the oracle: no 32-bit index or offset
    anywhere in the quantize, the slot stride or the apply."""
    segs = synth.fragment_segments(8192, [0, 1, 2], False)
    segs = np.concatenate([segs, np.array([(int(synth.segments_numel(segs)), 333, synth.NORM, 0, 1, 0)],
                                          dtype=segs.dtype)])
    n = synth.segments_numel(segs)
    assert n > 2 ** 31 and n % 8 == 5
    free, _ = torch.cuda.mem_get_info()
    need = 6 * 4 * n + 2 * n
    if free < need + (4 << 30):
        pytest.skip(f"needs {need / 2**30:.0f} GiB of free HBM")
    M, p, r = 2, 0, 1
    cfg = cfg_for(B, tau=1)
    rep = EmulatedReplicas(cfg, M, n)
    A_d = synth.dev_init(torch.empty(n, device=DEV), segs, p)
    Acopies = [A_d, A_d.clone()]
    v_d = [torch.zeros(n, device=DEV) for _ in range(M)]
    th_d = []
    for m in range(M):
        th = A_d.clone()
        synth.dev_apply_window(th, segs, p, m, r)
        th_d.append(th)
    rep.quantize_all(p, 10, th_d, Acopies)
    for m in range(M):
        synth.dev_apply_drift(th_d[m], segs, p, m, r)
    rep.merge_all(p, 11, th_d, Acopies, v_d)
    torch.cuda.synchronize()
    nb = -(-n // B)
    rng = np.random.default_rng(31)
    edges = [2 ** 30 // B - 1, 2 ** 30 // B, 2 ** 31 // B - 1, 2 ** 31 // B]
    blocks = sorted(set([0, nb - 1] + edges + list(rng.integers(0, nb, 16))))
    soff = sd.sd_payload_scales_offset(n)
    gat = rep.gather
    for b in blocks:
        lo, hi = b * B, min(n, (b + 1) * B)
        A0 = synth.host_init(segs, p, lo, hi)
        sends = [synth.host_apply_window(A0.copy(), segs, p, m, r, i0=lo) for m in range(M)]
        merges = [synth.host_apply_drift(x.copy(), segs, p, m, r, i0=lo) for m, x in enumerate(sends)]
        Ao, vo = A0.copy(), np.zeros(hi - lo, np.float32)
        st, g_o = oracle.round_(sends, merges, Ao, vo, B=B)
        assert st == 0
        pb_o = oracle.payload_bytes(hi - lo, B)
        so = oracle.scales_offset(hi - lo)
        for m in range(M):
            base = m * rep.pb
            got_codes = gat[base + lo // 2: base + (hi + 1) // 2].cpu().numpy()
            assert np.array_equal(got_codes, g_o[m * pb_o: m * pb_o + (hi - lo + 1) // 2]), f"block {b} codes"
            got_s = gat[base + soff + 4 * b: base + soff + 4 * b + 4].cpu().numpy()
            assert np.array_equal(got_s, g_o[m * pb_o + so: m * pb_o + so + 4]), f"block {b} scale"
            assert_same(Acopies[m][lo:hi], Ao, f"block {b} anchor")
            assert_same(v_d[m][lo:hi], vo, f"block {b} momentum")
            assert_same(th_d[m][lo:hi], merges[m], f"block {b} theta")
    rep.close()


def test_gather_alloc_single_gpu_and_free_errors():
    """sd_gather_alloc without a communicator: plain device memory, usable by
    the round; freeing a pointer it did not allocate is SD_ERR_ARG."""
    n, M = 3000, 1
    cfg = cfg_for(1024)
    ctx = sd.SdContext(cfg, 0, M, None, 0)
    buf = ctx.sd_gather_alloc(n)
    assert buf.numel() == M * sd.sd_payload_bytes(cfg, n) and buf.data_ptr() % 256 == 0
    A0 = (np.arange(n, dtype=np.float32) * 1e-3).astype(np.float32)
    th = (A0 - np.float32(1e-4)).astype(np.float32)
    A_d, v_d, th_d = to_dev(A0), torch.zeros(n, device=DEV), to_dev(th)
    ctx.sd_outer_grad_quantize(0, 10, th_d, A_d, buf, n)
    ctx.sd_fragment_sync(0, 10, buf, n)
    ctx.sd_merge(0, 11, buf, th_d, A_d, v_d, n)
    torch.cuda.synchronize()
    want, _ = oracle.quantize(th, A0, 1024)
    assert np.array_equal(buf.cpu().numpy(), want)
    with pytest.raises(sd.SdError) as e:
        ctx.sd_gather_free(torch.empty(256, dtype=torch.uint8, device=DEV))
    assert e.value.status == sd.SD_ERR_ARG
    ctx.sd_gather_free(buf)
    ctx.sd_finalize()


def test_per_replica_tau_toy_run():
    """NEXT-4: heterogeneous slack.  Replica m's context
    is created with its own tau_m; all replicas send at the same steps, each
    block-receives and merges tau_m steps later.  Final parameters, anchors and
    momenta of both replicas bit-identical to or_toy_run_taus."""
    M, bl, H, T, taus = 2, 1 << 16, 10, 60, [1, 5]
    c_or = oracle.config(L=2, fs=1, H=H, tau=1, T=T)
    th_o, A_o, v_o, sent_o, st = oracle.toy_run_taus(c_or, M, bl, synth.SEED, taus)
    assert st == 0
    cfgs = [sd.sd_config_default(2, 1, H, tau=taus[m], T=T) for m in range(M)]
    P, n = sd.sd_fragment_count(cfgs[0]), bl
    ctx = [sd.SdContext(cfgs[m], m, M, None, 0) for m in range(M)]
    pb = sd.sd_payload_bytes(cfgs[0], n)
    gather = [torch.empty(M * pb, dtype=torch.uint8, device=DEV) for _ in range(P)]
    A = [[synth.dev_init(torch.empty(n, device=DEV), synth.flat_segments(n), p) for p in range(P)] for _ in range(M)]
    v = [[torch.zeros(n, device=DEV) for _ in range(P)] for _ in range(M)]
    th = [torch.cat(A[0]).clone() for _ in range(M)]
    for t in range(1, T + 1):
        for m in range(M):
            synth.dev_apply_toy(th[m], m, t)
        sends = [sd.sd_fragment_schedule(cfgs[m], t)[0] for m in range(M)]
        assert sends[0] == sends[1]  # same send steps for every replica
        for p in sends[0]:
            for m in range(M):
                ctx[m].sd_outer_grad_quantize(p, t, th[m][p * n:(p + 1) * n], A[m][p], gather[p][m * pb:(m + 1) * pb], n)
            for m in range(M):
                ctx[m].sd_fragment_sync(p, t, gather[p], n)
        for m in range(M):
            for p in sd.sd_fragment_schedule(cfgs[m], t)[1]:
                ctx[m].sd_merge(p, t, gather[p], th[m][p * n:(p + 1) * n], A[m][p], v[m][p], n)
    torch.cuda.synchronize()
    for m in range(M):
        assert_same(th[m], th_o[m], f"theta replica {m}")
        assert_same(torch.cat(A[m]), A_o[m], f"anchor replica {m}")
        assert_same(torch.cat(v[m]), v_o[m], f"momentum replica {m}")
    for c in ctx:
        c.sd_finalize()


def test_offloaded_outer_state_toy_run():
    """NEXT-3: anchors and momenta of all fragments live in
    pinned host memory; HBM holds two staging slots.  Each fragment's state is
    prefetched two steps before its send and written back after its merge.
    Result bit-identical to the resident-state oracle run (or_toy_run)."""
    M, bl, H, tau, T = 2, 1 << 15, 12, 3, 80
    c_or = oracle.config(L=4, fs=1, H=H, tau=tau, T=T)
    th_o, A_o, v_o, _, st = oracle.toy_run(c_or, M, bl, synth.SEED)
    assert st == 0
    cfg = sd.sd_config_default(4, 1, H, tau=tau, T=T)
    P, n = sd.sd_fragment_count(cfg), bl
    ctx = [sd.SdContext(cfg, m, M, None, 0) for m in range(M)]
    pb = sd.sd_payload_bytes(cfg, n)
    gather = [torch.empty(M * pb, dtype=torch.uint8, device=DEV) for _ in range(P)]
    # host store (per replica, as on separate GPUs) and 2 device staging slots per replica
    A_h = [[synth.dev_init(torch.empty(n, device=DEV), synth.flat_segments(n), p).cpu().pin_memory() for p in range(P)]
           for _ in range(M)]
    v_h = [[torch.zeros(n).pin_memory() for _ in range(P)] for _ in range(M)]
    A_s = [[torch.empty(n, device=DEV) for _ in range(2)] for _ in range(M)]
    v_s = [[torch.empty(n, device=DEV) for _ in range(2)] for _ in range(M)]
    th = [torch.cat([A_h[0][p] for p in range(P)]).to(DEV) for _ in range(M)]
    sends = {}
    for t in range(1, T + 3):
        s_ahead, _ = sd.sd_fragment_schedule(cfg, t + 2) if t + 2 <= T else ([], [])
        for p in s_ahead:  # prefetch two steps ahead of the send
            for m in range(M):
                ctx[m].sd_state_prefetch(p, A_h[m][p], v_h[m][p], A_s[m][p % 2], v_s[m][p % 2], n)
        if t > T:
            continue
        for m in range(M):
            synth.dev_apply_toy(th[m], m, t)
        send, recv = sd.sd_fragment_schedule(cfg, t)
        for p in send:
            for m in range(M):
                ctx[m].sd_outer_grad_quantize(p, t, th[m][p * n:(p + 1) * n], A_s[m][p % 2], gather[p][m * pb:(m + 1) * pb], n)
            for m in range(M):
                ctx[m].sd_fragment_sync(p, t, gather[p], n)
        for p in recv:
            for m in range(M):
                ctx[m].sd_merge(p, t, gather[p], th[m][p * n:(p + 1) * n], A_s[m][p % 2], v_s[m][p % 2], n)
                ctx[m].sd_state_writeback(p, A_s[m][p % 2], v_s[m][p % 2], A_h[m][p], v_h[m][p], n)
    for m in range(M):
        ctx[m].sd_state_sync()
    torch.cuda.synchronize()
    for m in range(M):
        assert_same(th[m], th_o[m], f"theta replica {m}")
        assert_same(torch.cat(A_h[m]), A_o, f"host anchor store replica {m}")
        assert_same(torch.cat(v_h[m]), v_o, f"host momentum store replica {m}")
    for c in ctx:
        c.sd_finalize()


# ------------------------------------------------------------ InnerOpt (NEXT-1)
HP = dict(lr=3e-4, beta1=0.9, beta2=0.99, eps=1e-8, weight_decay=0.1)


@pytest.mark.parametrize("n", [1, 7, 1000, 8 * 1024 + 5, 300001])
def test_inner_adamw_bit_exact(n):
    rng = np.random.default_rng(n)
    th = rng.standard_normal(n).astype(np.float32) * 0.02
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    ctx = sd.SdContext(cfg_for(1024), 0, 1, None, 0)
    hp = sd.SdAdamW(**HP)
    th_d, m_d, v_d = to_dev(th), to_dev(m), to_dev(v)
    for k in range(1, 4):
        g = (rng.standard_normal(n) * 1e-3).astype(np.float32)
        g[:: 97] = 0.0
        ctx.sd_inner_adamw(k, th_d, to_dev(g), m_d, v_d, hp, n)
        oracle.adamw(th, g, m, v, k, lr=HP["lr"], b1=HP["beta1"], b2=HP["beta2"], eps=HP["eps"], wd=HP["weight_decay"])
    torch.cuda.synchronize()
    assert_same(th_d, th, "theta")
    assert_same(m_d, m, "m")
    assert_same(v_d, v, "v")
    ctx.sd_finalize()


@pytest.mark.parametrize("B,staged", [(1024, True), (512, True), (256, True), (0, True), (0, False), (4096, True),
                                      (4096, False)])
@pytest.mark.parametrize("n", [1025, 64 * 1024 + 77])
def test_inner_adamw_quantize_fused_bit_exact(n, B, staged):
    """The fused last-inner-step + quantize equals AdamW then or_quantize
    (B = 0 / 4096: AdamW + block max + staged summaries, or no workspace)."""
    rng = np.random.default_rng(n + B)
    A = (rng.standard_normal(n) * 0.02).astype(np.float32)
    th = (A - rng.standard_normal(n).astype(np.float32) * 1e-3).astype(np.float32)
    m = (rng.standard_normal(n) * 1e-4).astype(np.float32)
    v = (rng.random(n) * 1e-7).astype(np.float32)
    g = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    cfg = cfg_for(B)
    rep = EmulatedReplicas(cfg, 1, n, staged=staged)
    hp = sd.SdAdamW(**HP)
    th_d, m_d, v_d = to_dev(th), to_dev(m), to_dev(v)
    rep.ctx[0].sd_inner_adamw_quantize(0, 10, 7, th_d, to_dev(g), m_d, v_d, to_dev(A), rep.slot(0), hp, n)
    torch.cuda.synchronize()
    oracle.adamw(th, g, m, v, 7, lr=HP["lr"], b1=HP["beta1"], b2=HP["beta2"], eps=HP["eps"], wd=HP["weight_decay"])
    want, _ = oracle.quantize(th, A, B)
    assert np.array_equal(rep.gather.cpu().numpy(), want)
    assert_same(th_d, th, "theta")
    assert_same(m_d, m, "m")
    assert_same(v_d, v, "v")
    rep.ctx[0].sd_fragment_sync(0, 10, rep.gather, n)
    rep.close()


@pytest.mark.parametrize("B", [1024, 0, 4096])
def test_inner_adamw_quantize_fused_poison_index(B):
    """Non-finite updated parameters in the fused AdamW + quantize (single pass,
    and for B = 0 / 4096 the AdamW + block-max first pass): the payload records
    the first non-finite Delta's index exactly as or_quantize does."""
    rng = np.random.default_rng(B + 5)
    n = 3 * 4096 + 77
    A = (rng.standard_normal(n) * 0.02).astype(np.float32)
    th = (A - rng.standard_normal(n).astype(np.float32) * 1e-3).astype(np.float32)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    g = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    th[n - 3] = np.nan
    th[9000] = np.inf
    th[5000] = -np.inf
    g[7001] = np.nan
    cfg = cfg_for(B)
    rep = EmulatedReplicas(cfg, 1, n)
    hp = sd.SdAdamW(**HP)
    th_d = to_dev(th)
    rep.ctx[0].sd_inner_adamw_quantize(0, 10, 3, th_d, to_dev(g), to_dev(m), to_dev(v), to_dev(A), rep.slot(0), hp, n)
    torch.cuda.synchronize()
    oracle.adamw(th, g, m, v, 3, lr=HP["lr"], b1=HP["beta1"], b2=HP["beta2"], eps=HP["eps"], wd=HP["weight_decay"])
    want, poisoned = oracle.quantize(th, A, B)
    assert poisoned
    got = rep.gather.cpu().numpy()
    assert oracle.payload_poisoned(got, n, B) == oracle.payload_poisoned(want, n, B) == (1, 5000)
    assert np.array_equal(th_d.cpu().numpy(), th, equal_nan=True)  # NaN payload bits may differ (CPU vs GPU)
    rep.ctx[0].sd_fragment_sync(0, 10, rep.gather, n)
    rep.close()


@pytest.mark.parametrize("B", [0, 256, 1024, 4096])
@pytest.mark.parametrize("n", [1, 9, 1023, 4099, 65536 + 13])
def test_no_writes_outside_buffers(n, B):
    """Guard bands (compute-sanitizer is not available on this pool): every
    array lives between 4 KB canaries; quantize, fused AdamW + quantize and
    apply must leave the canaries intact (no out-of-bounds writes in the
    ragged tails)."""
    G = 1024  # floats of canary on each side
    M = 2
    cfg = cfg_for(B)
    pb = sd.sd_payload_bytes(cfg, n)

    def guarded(x):
        buf = torch.full((n + 2 * G,), 7.25, device=DEV)
        buf[G:G + n] = x
        return buf, buf[G:G + n]

    rng = np.random.default_rng(n + B)
    A_np = (rng.standard_normal(n) * 0.02).astype(np.float32)
    Ab = [guarded(to_dev(A_np)) for _ in range(M)]
    thb = [guarded(to_dev((A_np - 1e-3).astype(np.float32))) for _ in range(M)]
    vb = [guarded(torch.zeros(n, device=DEV)) for _ in range(M)]
    gb = [guarded(torch.randn(n, device=DEV) * 1e-3) for _ in range(M)]
    m1b = [guarded(torch.zeros(n, device=DEV)) for _ in range(M)]
    m2b = [guarded(torch.zeros(n, device=DEV)) for _ in range(M)]
    gbuf = torch.full((M * pb + 4096,), 0x5A, dtype=torch.uint8, device=DEV)
    gather = gbuf[:M * pb]
    ctx = [sd.SdContext(cfg, m, M, None, 0) for m in range(M)]
    hp = sd.SdAdamW(**HP)
    ctx[0].sd_inner_adamw_quantize(0, 10, 1, thb[0][1], gb[0][1], m1b[0][1], m2b[0][1], Ab[0][1], gather[:pb], hp, n)
    ctx[1].sd_outer_grad_quantize(0, 10, thb[1][1], Ab[1][1], gather[pb:2 * pb], n)
    for m in range(M):
        ctx[m].sd_fragment_sync(0, 10, gather, n)
    for m in range(M):
        ctx[m].sd_merge(0, 11, gather, thb[m][1], Ab[m][1], vb[m][1], n)
    torch.cuda.synchronize()
    for bufs in (Ab, thb, vb, gb, m1b, m2b):
        for full, _ in bufs:
            assert torch.all(full[:G] == 7.25) and torch.all(full[G + n:] == 7.25)
    assert torch.all(gbuf[M * pb:] == 0x5A)
    for c in ctx:
        assert c.sd_check()[0] == sd.SD_OK
        c.sd_finalize()


@pytest.mark.parametrize("M", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("poison", [False, True])
def test_inner_adamw_merge_fused_bit_exact(M, poison):
    """The receive step's inner AdamW fused with the merge equals
    or_adamw followed by or_apply (merge skipped, AdamW kept, if poisoned)."""
    n, B = 8 * 1024 + 3, 1024
    rng = np.random.default_rng(M * 10 + poison)
    cfg = cfg_for(B)
    rep = EmulatedReplicas(cfg, M, n)
    A0 = (rng.standard_normal(n) * 0.02).astype(np.float32)
    sends = [(A0 - rng.standard_normal(n).astype(np.float32) * 1e-3).astype(np.float32) for _ in range(M)]
    if poison:
        sends[M - 1][123] = np.inf
    th_live = (A0 - np.float32(5e-4)).astype(np.float32)
    g = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    m1 = (rng.standard_normal(n) * 1e-4).astype(np.float32)
    m2 = (rng.random(n) * 1e-7).astype(np.float32)
    v0 = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    A_d = [to_dev(A0) for _ in range(M)]
    rep.quantize_all(0, 10, [to_dev(x) for x in sends], A_d)
    th_d, m1_d, m2_d, v_d = to_dev(th_live), to_dev(m1), to_dev(m2), to_dev(v0)
    hp = sd.SdAdamW(**HP)
    rep.ctx[0].sd_inner_adamw_merge(0, 11, 5, th_d, to_dev(g), m1_d, m2_d, rep.gather, A_d[0], v_d, hp, n)
    for m in range(1, M):
        rep.ctx[m].sd_merge(0, 11, rep.gather, to_dev(th_live), A_d[m], to_dev(v0), n)
    torch.cuda.synchronize()
    th_o, A_o, v_o = th_live.copy(), A0.copy(), v0.copy()
    oracle.adamw(th_o, g, m1, m2, 5, lr=HP["lr"], b1=HP["beta1"], b2=HP["beta2"], eps=HP["eps"], wd=HP["weight_decay"])
    st = oracle.apply(rep.gather.cpu().numpy(), M, n, B, A_o, v_o, th_o)
    assert st == (1 if poison else 0)
    assert_same(th_d, th_o, "theta")
    assert_same(m1_d, m1, "adam m")
    assert_same(m2_d, m2, "adam v")
    assert_same(A_d[0], A_o, "anchor")
    assert_same(v_d, v_o, "momentum")
    rep.close()


def test_cuda_graph_capture_replay_matches_eager():
    """A step captured as a CUDA graph (libsd's calls are capturable) and
    replayed gives the same bits as issuing it eagerly again."""
    n, M = 20000 + 3, 1
    rng = np.random.default_rng(77)
    A0 = (rng.standard_normal(n) * 0.02).astype(np.float32)
    th0 = (A0 - rng.standard_normal(n).astype(np.float32) * 1e-3).astype(np.float32)
    cfg = cfg_for(1024)
    outs = []
    for mode in ("eager", "graph"):
        ctx = sd.SdContext(cfg, 0, M, None, 0)
        gather = torch.empty(sd.sd_payload_bytes(cfg, n), dtype=torch.uint8, device=DEV)
        A, v, th = to_dev(A0), torch.zeros(n, device=DEV), to_dev(th0)

        def step():
            ctx.sd_outer_grad_quantize(0, 10, th, A, gather, n)
            ctx.sd_fragment_sync(0, 10, gather, n)
            ctx.sd_merge(0, 11, gather, th, A, v, n)

        if mode == "eager":
            for _ in range(3):
                step()
        else:
            step()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step()  # captured (second round) ...
            g.replay()  # ... and executed, then once more
            g.replay()
        torch.cuda.synchronize()
        outs.append([bits(x) for x in (A, v, th)])
        ctx.sd_finalize()
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


def test_many_rounds_wide_dynamic_range():
    """40 rounds, M = 3, every scale block scaled by 2^k with k uniform in
    [-140, 100] (subnormal to huge scales, both encode paths, underflowing
    decodes): payloads and outer state stay bit-identical to the oracle."""
    rng = np.random.default_rng(2025)
    n, M, B = 16 * 1024 + 9, 3, 1024
    cfg = cfg_for(B, alpha=0.25, lr=0.4, mu=0.9)
    rep = EmulatedReplicas(cfg, M, n)
    A_o = (rng.standard_normal(n) * 0.02).astype(np.float32)
    v_o = np.zeros(n, np.float32)
    A_d = [to_dev(A_o) for _ in range(M)]
    v_d = [torch.zeros(n, device=DEV) for _ in range(M)]
    nb = -(-n // B)
    for r in range(40):
        sends, merges = [], []
        for m in range(M):
            d = edge_deltas(n, B, rng).astype(np.float64)
            for b in range(nb):
                d[b * B:(b + 1) * B] *= 2.0 ** int(rng.integers(-140, 101))
            d = np.clip(d, -3e38, 3e38).astype(np.float32)
            th = (A_o - d).astype(np.float32)
            th = np.where(np.isfinite(th), th, A_o).astype(np.float32)
            sends.append(th)
            merges.append((th * np.float32(0.5)).astype(np.float32))
        t = 10 * (r + 1)
        rep.quantize_all(0, t, [to_dev(x) for x in sends], A_d)
        th_d = [to_dev(x) for x in merges]
        rep.merge_all(0, t + 1, th_d, A_d, v_d)
        mo = [x.copy() for x in merges]
        st, g_o = oracle.round_(sends, mo, A_o, v_o, B=B, lr=0.4, mu=0.9, alpha=0.25)
        torch.cuda.synchronize()
        if st != 0:  # a non-finite Delta (huge scale overflow) poisons the round on both sides
            assert all(s[0] == sd.SD_ERR_NONFINITE for s in rep.check_all())
            # or_round leaves A, v (and theta) untouched on poison; so must every replica
            # (rank-consistent skip, DESIGN.md §1 errors; PAPER.md:141 / SPEC.md:232)
            for m in range(M):
                assert_same(A_d[m], A_o, f"round {r} anchor (poisoned round)")
                assert_same(v_d[m], v_o, f"round {r} momentum (poisoned round)")
                assert_same(th_d[m], mo[m], f"round {r} theta (poisoned round)")
            continue
        assert np.array_equal(rep.gather.cpu().numpy(), g_o), f"round {r}: payload bytes differ"
        for m in range(M):
            assert_same(A_d[m], A_o, f"round {r} anchor")
            assert_same(v_d[m], v_o, f"round {r} momentum")
            assert_same(th_d[m], mo[m], f"round {r} theta")
    rep.close()


@pytest.mark.parametrize("n", [1, 7, 1024, 300001])
@pytest.mark.parametrize("inplace", [False, True])
def test_outer_state_init_matches_oracle(n, inplace):
    """sd_outer_state_init: A = theta
    bit for bit (including -0 and NaN payloads), v = +0; the caller's
    garbage in A and v is overwritten; A may alias theta."""
    rng = np.random.default_rng(n)
    raw = rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
    raw[: min(n, 3)] = [0x80000000, 0x7fc00001, 0x00000001][: min(n, 3)]
    theta = raw.view(np.float32)
    A_o, v_o = oracle.outer_state_init(theta)
    cfg = cfg_for(1024)
    ctx = sd.SdContext(cfg, 0, 1, None, 0)
    th = to_dev(theta)
    A = th if inplace else to_dev(rng.standard_normal(n).astype(np.float32))
    v = to_dev(np.full(n, np.nan, np.float32))
    ctx.sd_outer_state_init(th, A, v, n)
    torch.cuda.synchronize()
    assert np.array_equal(bits(A), bits(A_o)) and np.array_equal(bits(v), bits(v_o))
    assert np.array_equal(bits(th), raw)
    ctx.sd_finalize()
