"""Pins of the oracle's receive side and whole rounds (or_decode_mean,
or_nesterov, or_merge, or_apply, or_round, or_toy_run) against:
  * SPEC examples (golden/paper_examples.json): Nesterov -0.76 / 1.084,
    merge (2,2)/(0,4) -> (1,3), on-grid exact mean, {x, -x} -> 0;
  * the library routine torch.optim.SGD(nesterov=True) (operand-scaled
    tolerance: torch's CPU kernels may contract into FMA; momentum bitwise);
  * textbook reductions: FedAvg (lr=1, mu=0, alpha=0 -> parameter average,
    P:13), M=1 identity, H=1 data-parallel averaging, and
    Streaming with P=1, tau=0 == DiLoCo (Alg. 1);
  * invariants: alpha=1 leaves theta unchanged while momentum advances
    (P:137); momentum advances once per round regardless of M.
On-grid data: A = k 2^-20, Delta in {0, +-2^-8 2^-j},
+-2^-8 present in every block, theta = A - Delta (exact)."""
import json
import os

import numpy as np
import pytest
import torch

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def on_grid(rng, n, B):
    A = (rng.integers(-(2 ** 21) + 1, 2 ** 21, n) * 2.0 ** -20).astype(np.float32)
    mags = np.concatenate([[0.0], 2.0 ** -8 * 2.0 ** -np.arange(7)])
    D = (rng.choice(mags, n) * rng.choice([-1.0, 1.0], n)).astype(np.float32)
    blen = B if B else n
    D[::blen] = 2.0 ** -8  # every block holds the max -> scale 2^-8
    th = (A - D).astype(np.float32)
    assert np.array_equal((A - th).astype(np.float32), D)
    return A, D, th


def bits(x):
    return np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)


def test_nesterov_spec_examples():
    g = GOLD["nesterov"]
    A = np.array([5.0], np.float32)
    v = np.zeros(1, np.float32)
    one = np.ones(1, np.float32)
    oracle.nesterov(A, v, one, g["lr"], g["mu"])
    assert v[0] == 1.0
    assert abs((5.0 - A[0]) - g["first_update"]) <= 4 * np.spacing(np.float32(5.0))
    A2 = A.copy()
    oracle.nesterov(A2, v, one, g["lr"], g["mu"])
    assert abs((A[0] - A2[0]) - g["second_update"]) <= 4 * np.spacing(np.float32(5.0))
    # mu = 0 is plain SGD exactly
    A3, v3 = np.array([1.25], np.float32), np.array([7.0], np.float32)
    gg = np.array([0.375], np.float32)
    oracle.nesterov(A3, v3, gg, 0.5, 0.0)
    assert A3[0] == np.float32(1.25) - np.float32(0.5) * np.float32(0.375) and v3[0] == gg[0]


def test_nesterov_vs_torch_sgd():
    rng = np.random.default_rng(11)
    n = 100000
    A = rng.standard_normal(n).astype(np.float32)
    v = (rng.standard_normal(n) * 0.1).astype(np.float32)
    for step in range(3):
        g = (rng.standard_normal(n) * 0.05).astype(np.float32)
        p = torch.nn.Parameter(torch.from_numpy(A.copy()))
        opt = torch.optim.SGD([p], lr=0.4, momentum=0.9, nesterov=True, dampening=0.0)
        opt.state[p]["momentum_buffer"] = torch.from_numpy(v.copy())
        p.grad = torch.from_numpy(g.copy())
        opt.step()
        oracle.nesterov(A, v, g, 0.4, 0.9)
        assert np.array_equal(bits(opt.state[p]["momentum_buffer"].numpy()), bits(v))
        ref = p.detach().numpy()
        scale = np.maximum.reduce([np.abs(ref), 0.4 * np.abs(g), 0.4 * 0.9 * np.abs(v)])
        assert np.all(np.abs(ref - A) <= 16 * 2.0 ** -24 * scale)
        A = ref.copy()  # continue from the library's state


def test_merge_spec_examples():
    g = GOLD["merge"]
    th = np.array(g["theta"], np.float32)
    oracle.merge(th, np.array(g["tilde"], np.float32), g["alpha"])
    assert th.tolist() == g["merged"]
    th = np.array([1.5, -2.0], np.float32)
    oracle.merge(th, np.array([9.0, 9.0], np.float32), 1.0)  # alpha = 1: no communication
    assert th.tolist() == [1.5, -2.0]
    oracle.merge(th, np.array([9.0, -3.0], np.float32), 0.0)  # alpha = 0: theta = tilde
    assert th.tolist() == [9.0, -3.0]


@pytest.mark.parametrize("M", [1, 2, 4, 8])
def test_mean_exact_on_grid(M):
    rng = np.random.default_rng(M)
    n, B = 3000, 1024
    A = np.zeros(n, np.float32)
    Ds, slots = [], []
    for m in range(M):
        _, D, _ = on_grid(rng, n, B)
        Ds.append(D)
        pay, _ = oracle.quantize(np.zeros(n, np.float32), D, B)  # Delta = D - 0
        slots.append(pay)
    g = oracle.decode_mean(np.concatenate(slots), M, n, B)
    assert np.array_equal(g.astype(np.float64), np.mean(np.stack(Ds).astype(np.float64), axis=0))
    if M == 2:  # {x, -x} -> 0
        p1, _ = oracle.quantize(np.zeros(n, np.float32), Ds[0], B)
        p2, _ = oracle.quantize(np.zeros(n, np.float32), -Ds[0], B)
        assert not oracle.decode_mean(np.concatenate([p1, p2]), 2, n, B).any()


@pytest.mark.parametrize("M", [1, 2, 4, 8])
def test_fedavg_reduction(M):
    """lr = 1, mu = 0, alpha = 0: the anchor becomes the plain parameter
    average (1/M) sum_m theta_m (FedAvg), bit-exact on grid."""
    rng = np.random.default_rng(100 + M)
    n, B = 4096 + 333, 1024
    A, _, _ = on_grid(rng, n, B)
    thetas = []
    for m in range(M):
        _, D, _ = on_grid(rng, n, B)
        thetas.append((A - D).astype(np.float32))
    merges = [t.copy() for t in thetas]
    Aw, v = A.copy(), np.zeros(n, np.float32)
    st, _ = oracle.round_(thetas, merges, Aw, v, B=B, lr=1.0, mu=0.0, alpha=0.0)
    assert st == 0
    avg = np.mean(np.stack(thetas).astype(np.float64), axis=0)
    assert np.array_equal(Aw.astype(np.float64), avg)
    for mth in merges:
        assert np.array_equal(bits(mth), bits(Aw))


def test_m1_identity():
    rng = np.random.default_rng(5)
    n = 2048 + 17
    A, D, th = on_grid(rng, n, 1024)
    drift = (th - np.float32(2.0 ** -10)).astype(np.float32)
    merged = [drift.copy()]
    Aw, v = A.copy(), np.zeros(n, np.float32)
    st, _ = oracle.round_([th], merged, Aw, v, B=1024, lr=1.0, mu=0.0, alpha=0.0)
    assert st == 0 and np.array_equal(bits(merged[0]), bits(th)) and np.array_equal(bits(Aw), bits(th))


def test_h1_data_parallel_averaging():
    """P = 1, H = 1, tau = 0, lr = 1, mu = 0, alpha = 0: every step equals
    data-parallel averaging of the replicas' updates: the
    reference averages the per-replica updates (what an AVG all-reduce of
    the gradients computes) and applies them to one shared copy."""
    rng = np.random.default_rng(9)
    n, M, B = 1500, 4, 1024
    A0, _, _ = on_grid(rng, n, B)
    theta = [A0.copy() for _ in range(M)]
    A, v = A0.copy(), np.zeros(n, np.float32)
    dp = A0.astype(np.float64)
    for t in range(5):
        ups = [on_grid(rng, n, B)[1] for _ in range(M)]
        sends = [(theta[m] - ups[m]).astype(np.float32) for m in range(M)]   # inner step
        merges = [s.copy() for s in sends]
        st, _ = oracle.round_(sends, merges, A, v, B=B, lr=1.0, mu=0.0, alpha=0.0)
        assert st == 0
        theta = merges
        dp = dp - np.mean(np.stack(ups).astype(np.float64), axis=0)
        for m in range(M):
            assert np.array_equal(theta[m].astype(np.float64), dp)
    # with the standard outer optimizer: torch SGD(nesterov) on the averaged
    # update, one step at a time from the same on-grid anchor and momentum
    v2 = np.zeros(n, np.float32)
    for t in range(4):
        A2, _, _ = on_grid(rng, n, B)
        ups = [on_grid(rng, n, B)[1] for _ in range(M)]
        sends = [(A2 - u).astype(np.float32) for u in ups]
        p = torch.nn.Parameter(torch.from_numpy(A2.copy()))
        opt = torch.optim.SGD([p], lr=0.4, momentum=0.9, nesterov=True)
        if t > 0:
            opt.state[p]["momentum_buffer"] = torch.from_numpy(v2.copy())
        p.grad = torch.from_numpy(np.mean(np.stack(ups).astype(np.float64), axis=0).astype(np.float32))
        opt.step()
        st, _ = oracle.round_(sends, [s.copy() for s in sends], A2, v2, B=B, lr=0.4, mu=0.9, alpha=0.0)
        assert st == 0
        ref = p.detach().numpy()
        assert np.array_equal(bits(opt.state[p]["momentum_buffer"].numpy()), bits(v2))
        scale = np.maximum.reduce([np.abs(ref), 0.4 * np.abs(p.grad.numpy()), 0.36 * np.abs(v2)])
        assert np.all(np.abs(ref - A2) <= 16 * 2.0 ** -24 * scale)


def test_alpha1_keeps_theta_momentum_advances():
    rng = np.random.default_rng(21)
    n = 1100
    A, D, th = on_grid(rng, n, 1024)
    m0 = (th - np.float32(2.0 ** -12)).astype(np.float32)
    merged = [m0.copy()]
    Aw, v = A.copy(), np.zeros(n, np.float32)
    oracle.round_([th], merged, Aw, v, B=1024, alpha=1.0)
    assert np.array_equal(bits(merged[0]), bits(m0)) and v.any() and not np.array_equal(Aw, A)


def test_momentum_single_advance_regardless_of_M():
    """Identical replicas: the mean equals each replica's decoded Delta, so
    A, v after one round are the same for M = 1 and M = 4."""
    rng = np.random.default_rng(4)
    n = 2500
    A, D, th = on_grid(rng, n, 1024)
    out = []
    for M in (1, 4):
        Aw, v = A.copy(), np.zeros(n, np.float32)
        oracle.round_([th] * M, [th.copy() for _ in range(M)], Aw, v, B=1024)
        out.append((bits(Aw).copy(), bits(v).copy()))
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])


def test_poisoned_round_is_skipped():
    n = 2000
    A = np.ones(n, np.float32)
    th = [np.zeros(n, np.float32), np.zeros(n, np.float32)]
    th[1][777] = np.nan
    merged = [x.copy() for x in th]
    Aw, v = A.copy(), np.zeros(n, np.float32)
    st, g = oracle.round_(th, merged, Aw, v)
    assert st == 1 and np.array_equal(Aw, A) and not v.any()


def test_toy_run_streaming_P1_tau0_equals_diloco():
    """Streaming with P = 1, tau = 0 is Alg. 1 (DiLoCo).  The reference
    loop below is Alg. 1 written with the oracle's per-round
    primitives: every H steps quantize, mean, Nesterov, merge with alpha = 0."""
    import synth

    M, bl, H, T = 2, 3000, 5, 23
    c = oracle.config(L=1, fs=1, H=H, tau=0, T=T, alpha=0.0)
    theta, A, v, sent, st = oracle.toy_run(c, M, bl, synth.SEED)
    assert st == 0
    n = bl
    A2 = synth.host_init(synth.flat_segments(n), 0)
    v2 = np.zeros(n, np.float32)
    th2 = [A2.copy() for _ in range(M)]
    for t in range(1, T + 1):
        for m in range(M):
            synth.host_apply_toy(th2[m], m, t)
        if t % H == 0:
            st2, _ = oracle.round_(th2, th2, A2, v2, B=1024, alpha=0.0)
            assert st2 == 0
    for m in range(M):
        assert np.array_equal(bits(theta[m]), bits(th2[m]))
    assert np.array_equal(bits(A), bits(A2)) and np.array_equal(bits(v), bits(v2))
    assert sent == (T // H) * M * oracle.payload_bytes(n, 1024)  # byte accounting


def test_toy_config_runs_and_keeps_outer_state_shared():
    """The toy config of BASELINE.json (M=2, 2^20 params, 2 fragments, H=10,
    tau=1) runs end to end; byte total = sends x M x payload."""
    c = oracle.config(L=2, fs=1, H=10, tau=1, T=100)
    theta, A, v, sent, st = oracle.toy_run(c, 2, 2 ** 19, 250118512)
    assert st == 0 and np.all(np.isfinite(theta)) and v.any()
    sends = sum(1 for e in oracle.calendar(c) if e[1] == 0)
    assert sent == sends * 2 * oracle.payload_bytes(2 ** 19, 1024)


def test_per_replica_tau_equal_taus_reduce_to_toy_run():
    """NEXT-4: with tau_m = tau for every replica the
    per-replica run is the plain Alg. 2 run bit for bit."""
    c = oracle.config(L=2, fs=1, H=8, tau=2, T=41)
    th1, A1, v1, b1, s1 = oracle.toy_run(c, 2, 3000, 7)
    th2, A2, v2, b2, s2 = oracle.toy_run_taus(c, 2, 3000, 7, [2, 2])
    assert s1 == s2 == 0 and b1 == b2
    assert np.array_equal(bits(th1), bits(th2))
    for m in range(2):
        assert np.array_equal(bits(A2[m]), bits(A1)) and np.array_equal(bits(v2[m]), bits(v1))


def test_per_replica_tau_slack_keeps_outer_state_replicated():
    """tau_1 = 1, tau_2 = 5: both replicas send at the same
    step and receive at their own; the outer state each holds is the same
    after every completed round (flush at T), while the live parameters differ
    from the equal-tau run (the slower replica merges later)."""
    c = oracle.config(L=2, fs=1, H=10, tau=1, T=60)
    th, A, v, b, st = oracle.toy_run_taus(c, 2, 2048, 11, [1, 5])
    assert st == 0
    assert np.array_equal(bits(A[0]), bits(A[1])) and np.array_equal(bits(v[0]), bits(v[1]))
    th_eq, A_eq, _, _, _ = oracle.toy_run(c, 2, 2048, 11)
    assert not np.array_equal(bits(th[1]), bits(th_eq[1]))


# --------------------------------------------------------------- InnerOpt (NEXT-1)
def test_adamw_spec_examples():
    """SPEC.md:177-179 adamw_step examples."""
    th = np.array([0.3, -1.25], np.float32)
    m, v = np.zeros(2, np.float32), np.zeros(2, np.float32)
    oracle.adamw(th, np.zeros(2, np.float32), m, v, 1, lr=0.1, wd=0.0)       # g = 0 -> unchanged
    assert th.tolist() == [np.float32(0.3), -1.25]
    th = np.zeros(1, np.float32)
    m, v = np.zeros(1, np.float32), np.zeros(1, np.float32)
    oracle.adamw(th, np.array([0.5], np.float32), m, v, 1, lr=0.1, wd=0.0)   # first step -> ~ -lr
    assert abs(th[0] + 0.1) < 1e-6
    th = np.ones(1, np.float32)
    m, v = np.zeros(1, np.float32), np.zeros(1, np.float32)
    oracle.adamw(th, np.zeros(1, np.float32), m, v, 1, lr=0.1, wd=0.1)      # decoupled decay only -> 0.99
    assert th[0] == np.float32(0.99)


def test_adamw_vs_torch():
    """torch.optim.AdamW (betas, eps, decoupled weight decay) over 5 steps from
    the same state; torch computes exp_avg by lerp and may contract, so the
    comparison is operand-scaled (moments and parameters)."""
    rng = np.random.default_rng(2)
    n = 50000
    th = rng.standard_normal(n).astype(np.float32)
    m, v = np.zeros(n, np.float32), np.zeros(n, np.float32)
    p = torch.nn.Parameter(torch.from_numpy(th.copy()))
    opt = torch.optim.AdamW([p], lr=1e-3, betas=(0.9, 0.99), eps=1e-8, weight_decay=0.1)
    for k in range(1, 6):
        g = (rng.standard_normal(n) * 0.01).astype(np.float32)
        p.grad = torch.from_numpy(g.copy())
        opt.step()
        oracle.adamw(th, g, m, v, k, lr=1e-3, b1=0.9, b2=0.99, eps=1e-8, wd=0.1)
        st = opt.state[p]
        assert np.allclose(st["exp_avg"].numpy(), m, rtol=1e-5, atol=1e-9)
        assert np.allclose(st["exp_avg_sq"].numpy(), v, rtol=1e-5, atol=1e-12)
        assert np.max(np.abs(p.detach().numpy() - th)) <= 1e-6 * max(1.0, float(np.max(np.abs(th))))


@pytest.mark.parametrize("M", [1, 2, 4])
def test_apply_single_replica_fedavg_and_poison(M):
    """or_apply (one replica's receive side on a given gather buffer):
    lr = 1, mu = 0, alpha = 0.5 on grid -> the anchor is the plain average
    of the M senders' parameters (FedAvg) and theta = (theta + A) / 2
    (P:137), bit-exact; the momentum is the mean outer gradient
    (v = 0 + g).  A poisoned slot leaves A, v, theta untouched and
    returns nonzero."""
    rng = np.random.default_rng(300 + M)
    n, B = 2048 + 77, 1024
    A, _, _ = on_grid(rng, n, B)
    sends = [(A - on_grid(rng, n, B)[1]).astype(np.float32) for _ in range(M)]
    pb = oracle.payload_bytes(n, B)
    gather = np.concatenate([oracle.quantize(s, A, B)[0] for s in sends])
    assert gather.size == M * pb
    theta = (A + np.float32(2.0 ** -10)).astype(np.float32)
    Aw, v, th = A.copy(), np.zeros(n, np.float32), theta.copy()
    st = oracle.apply(gather, M, n, B, Aw, v, th, lr=1.0, mu=0.0, alpha=0.5)
    assert st == 0
    avg = np.mean(np.stack(sends).astype(np.float64), axis=0)
    assert np.array_equal(Aw.astype(np.float64), avg)
    assert np.array_equal(v.astype(np.float64), A.astype(np.float64) - avg)
    assert np.array_equal(th.astype(np.float64), 0.5 * theta.astype(np.float64) + 0.5 * avg)
    bad = [s.copy() for s in sends]
    bad[-1][n // 2] = np.nan
    gather = np.concatenate([oracle.quantize(s, A, B)[0] for s in bad])
    Aw, v, th = A.copy(), np.zeros(n, np.float32), theta.copy()
    assert oracle.apply(gather, M, n, B, Aw, v, th) != 0
    assert np.array_equal(bits(Aw), bits(A)) and not v.any() and np.array_equal(bits(th), bits(theta))


# ------------------------------------------- scale addressing: per slot, per block
# Every pin above draws its outer gradients with `on_grid`, which puts the
# same scale 2^-8 in every block of every replica: a decoder reading slot 0's
# scale (or block 0's) for all (m, b) would still pass them.  The pins below
# give every (slot m, block b) its own power-of-two scale
#     s_{m,b} = 2^-(8 + m + 3b)
# and decode with exact rationals, independently of or_quantize:
#     q = LUT[c] * s,  LUT[e] = 2^(e-7), LUT[8|e] = -2^(e-7), LUT[0] = LUT[8] = +0
#     (SPEC.md:245, :264), summed over m and divided by M (
#     SPEC.md:385).
# With M <= 8 and b <= 3 every partial sum spans < 24 bits, so the fp32 fold is
# exact and must equal the rational mean bit for bit.
from fractions import Fraction  # noqa: E402


def _scale(m, b):
    return 2.0 ** -(8 + m + 3 * b)


def _lut(c):
    e = c & 7
    if e == 0:
        return Fraction(0)
    v = Fraction(2) ** (e - 7)
    return -v if c & 8 else v


def _hand_payload(codes, scales, n, B):
    """Payload bytes built from the layout definition (S:272 nibble order,
    DESIGN.md §5 layout), not by or_quantize."""
    pay = np.zeros(oracle.payload_bytes(n, B), np.uint8)
    c = np.zeros(2 * ((n + 1) // 2), np.uint8)
    c[:n] = codes
    pay[:(n + 1) // 2] = c[0::2] | (c[1::2] << 4)
    so = oracle.scales_offset(n)
    nb = len(scales)
    pay[so:so + 4 * nb] = np.asarray(scales, np.float32).view(np.uint8)
    to = so + -(-4 * nb // 16) * 16
    pay[to:to + 4] = np.frombuffer(np.uint32(0x31304453).tobytes(), np.uint8)
    pay[to + 4:to + 8] = np.frombuffer(np.uint32(nb).tobytes(), np.uint8)
    pay[to + 8:to + 16] = 0xFF
    return pay


def _rational_mean(codes, n, B, M):
    blen = B if B else n
    out = []
    for i in range(n):
        b = i // blen
        S = sum(_lut(int(codes[m][i])) * Fraction(_scale(m, b)) for m in range(M))
        out.append(S / M)
    return out


@pytest.mark.parametrize("M", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("B,n", [(256, 4 * 256 - 37), (256, 3 * 256), (0, 700)])
def test_decode_mean_distinct_scale_per_slot_and_block(M, B, n):
    rng = np.random.default_rng(7000 + 10 * M + B)
    nb = oracle.num_scale_blocks(n, B)
    codes = [rng.integers(0, 16, n).astype(np.uint8) for _ in range(M)]
    gather = np.concatenate([_hand_payload(codes[m], [_scale(m, b) for b in range(nb)], n, B) for m in range(M)])
    g = oracle.decode_mean(gather, M, n, B)
    ref = _rational_mean(codes, n, B, M)
    if M == 3:  # S/3 rounds: compare with the correctly rounded quotient of the exact (fp32) sum
        ref = [float(np.float32(float(r * 3)) / np.float32(3)) for r in ref]
        assert np.array_equal(g.astype(np.float64), np.array(ref))
    else:
        assert all(Fraction(float(x)) == r for x, r in zip(g, ref))
    assert g.any()


@pytest.mark.parametrize("M", [1, 2, 4])
def test_round_and_apply_distinct_scale_per_slot_and_block(M):
    """or_round (quantize + mean + Nesterov + merge) and or_apply on inputs
    whose outer gradients have scale s_{m,b} in block b of replica m:
    with lr = 1, mu = 0, alpha = 0 (FedAvg) the new anchor is
    A - (1/M) sum_m Delta_m exactly, v = the mean, theta = A'."""
    rng = np.random.default_rng(800 + M)
    B, n = 256, 3 * 256 - 11
    nb = oracle.num_scale_blocks(n, B)
    # A on a 2^-25 grid with |A| < 2^-2; Delta_{m,i} in {0, +-s_{m,b} 2^-j}:
    # theta = A - Delta and A - mean are exact in fp32 (<= 24 significant bits)
    A = (rng.integers(-(2 ** 23) + 1, 2 ** 23, n) * 2.0 ** -25).astype(np.float32)
    D = []
    for m in range(M):
        d = np.zeros(n)
        for b in range(nb):
            lo, hi = b * B, min(n, (b + 1) * B)
            j = rng.integers(-1, 7, hi - lo)
            v = np.where(j < 0, 0.0, _scale(m, b) * 2.0 ** -np.maximum(j, 0)) * rng.choice([-1.0, 1.0], hi - lo)
            v[0] = -_scale(m, b) if b % 2 else _scale(m, b)  # the block's max |Delta| is exactly s_{m,b}
            d[lo:hi] = v
        D.append(d.astype(np.float32))
    thetas = [(A - d).astype(np.float32) for d in D]
    for th, d in zip(thetas, D):
        assert np.array_equal((A - th).astype(np.float32), d)
    mean = [sum(Fraction(float(D[m][i])) for m in range(M)) / M for i in range(n)]
    want_A = [Fraction(float(a)) - g for a, g in zip(A, mean)]

    # scales in the payloads are the distinct s_{m,b}
    pays = [oracle.quantize(th, A, B)[0] for th in thetas]
    so = oracle.scales_offset(n)
    for m in range(M):
        assert pays[m][so:so + 4 * nb].view(np.float32).tolist() == [_scale(m, b) for b in range(nb)]

    merges = [t.copy() for t in thetas]
    Aw, v = A.copy(), np.zeros(n, np.float32)
    st, _ = oracle.round_(thetas, merges, Aw, v, B=B, lr=1.0, mu=0.0, alpha=0.0)
    assert st == 0
    assert all(Fraction(float(x)) == w for x, w in zip(Aw, want_A))
    assert all(Fraction(float(x)) == g for x, g in zip(v, mean))
    for mth in merges:
        assert np.array_equal(bits(mth), bits(Aw))

    Aw2, v2, th2 = A.copy(), np.zeros(n, np.float32), thetas[0].copy()
    assert oracle.apply(np.concatenate(pays), M, n, B, Aw2, v2, th2, lr=1.0, mu=0.0, alpha=0.0) == 0
    assert np.array_equal(bits(Aw2), bits(Aw)) and np.array_equal(bits(v2), bits(v))
    assert np.array_equal(bits(th2), bits(Aw))


def test_outer_state_init_is_bit_copy_and_zero():
    """A_p <- theta_init, v_p <- 0:
    the anchor is the parameters' bit pattern (including -0 and NaN
    payloads), the momentum is +0 everywhere."""
    rng = np.random.default_rng(3)
    raw = rng.integers(0, 2 ** 32, 4099, dtype=np.uint64).astype(np.uint32)
    raw[:4] = [0x80000000, 0x7fc00001, 0xff800000, 0x00000001]
    theta = raw.view(np.float32)
    A, v = oracle.outer_state_init(theta)
    assert np.array_equal(A.view(np.uint32), raw)
    assert not v.view(np.uint32).any()
