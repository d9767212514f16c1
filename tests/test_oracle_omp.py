"""Determinism under parallelism (SPEC.md:437, :614 acceptance 12; SURVEY.md
§8(c)-c3 "the single-thread oracle equals the N-thread oracle"): the same
oracle source built with OpenMP (liboracle_omp.so) on N threads produces
payloads, anchors, momenta and parameters bit-identical to the
single-threaded build (liboracle.so), on the paper-shaped synthetic inputs
and on the codec's edge cases, including ragged sizes, B = 0 (one scale per
fragment: the max and the encode split inside the block), poisoned rounds
(the first non-finite index is a min over threads) and the toy Alg. 2 run."""
import os

import numpy as np
import pytest

import oracle
import synth

NT = max(2, min(16, len(os.sched_getaffinity(0))))


def both(fn):
    """fn() under the 1-thread build, then under NT threads."""
    prev = oracle.set_threads(1)
    try:
        a = fn()
        oracle.set_threads(NT)
        b = fn()
    finally:
        oracle.set_threads(prev)
    return a, b


def _bits(x):
    return np.ascontiguousarray(x).view(np.uint8)


def _round_inputs(n, M, seed, poison=None):
    segs = synth.flat_segments(n)
    A = synth.host_init(segs, 0, 0, n)
    thetas = [synth.host_apply_window(A.copy(), segs, 0, m, 1) for m in range(M)]
    if poison is not None:
        m, i = poison
        thetas[m][i] = np.inf
    rng = np.random.default_rng(seed)
    merges = [(t - np.float32(2.0 ** -12) * rng.standard_normal(n).astype(np.float32)).astype(np.float32)
              for t in thetas]
    return A, thetas, merges


@pytest.mark.parametrize("B", [1024, 256, 0, 65536])
@pytest.mark.parametrize("M", [1, 2, 3, 8])
def test_round_n_threads_equals_one_thread(M, B):
    n = 3 * (1 << 18) + 12345  # 0.8M elements: several OpenMP chunks, a ragged last block
    A0, thetas, merges0 = _round_inputs(n, M, 10 * M + B)

    def run():
        A, v = A0.copy(), np.zeros(n, np.float32)
        out = []
        for r in range(2):  # two rounds: the second starts from nonzero momentum
            mg = [x.copy() for x in merges0]
            st, g = oracle.round_(thetas, mg, A, v, B=B)
            out.append((st, g.copy(), A.copy(), v.copy(), [x.copy() for x in mg]))
        return out

    one, many = both(run)
    for (s1, g1, A1, v1, m1), (s2, g2, A2, v2, m2) in zip(one, many):
        assert s1 == s2 == 0
        assert np.array_equal(g1, g2)
        assert np.array_equal(_bits(A1), _bits(A2)) and np.array_equal(_bits(v1), _bits(v2))
        for x, y in zip(m1, m2):
            assert np.array_equal(_bits(x), _bits(y))


@pytest.mark.parametrize("B", [1024, 0])
def test_poisoned_first_index_n_threads(B):
    n = 1 << 20
    bad = [n - 5, 700001, 3]  # several non-finite values: the payload records the smallest index

    def run():
        A, thetas, merges = _round_inputs(n, 2, 4, poison=(1, bad[0]))
        thetas[1][bad[1]] = np.nan
        thetas[1][bad[2]] = -np.inf
        pay, poisoned = oracle.quantize(thetas[1], A, B)
        return poisoned, oracle.payload_poisoned(pay, n, B)

    (p1, (r1, f1)), (p2, (r2, f2)) = both(run)
    assert p1 and p2 and r1 == r2 == 1 and f1 == f2 == min(bad)


def test_codec_edges_n_threads():
    """Threshold-adjacent, subnormal, +-0 and all-zero blocks (SURVEY.md §8(d) edge sets)."""
    rng = np.random.default_rng(77)
    n = (1 << 19) + 3
    s = np.float32(1.5)
    thr = s * 2.0 ** (-np.arange(7) - 0.5)
    d = rng.choice(thr, n) * (1 + rng.integers(-4, 5, n) * 2.0 ** -23) * rng.choice([-1, 1], n)
    d[::97] = 0.0
    d[5::101] = -0.0
    d[7::89] = 1e-41
    d[: 4096] = 0.0
    d = d.astype(np.float32)
    d[4096] = s
    A = np.zeros(n, np.float32)
    th = (A - d).astype(np.float32)
    for B in (1024, 0):
        a, b = both(lambda: oracle.quantize(th, A, B)[0])
        assert np.array_equal(a, b)


def test_adamw_and_toy_run_n_threads():
    rng = np.random.default_rng(5)
    n = 600001
    th0 = rng.standard_normal(n).astype(np.float32)
    g = (rng.standard_normal(n) * 1e-2).astype(np.float32)

    def adam():
        th, m, v = th0.copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)
        for k in (1, 2, 3):
            oracle.adamw(th, g, m, v, k, lr=1e-3, wd=0.1)
        return th, m, v

    a, b = both(adam)
    for x, y in zip(a, b):
        assert np.array_equal(_bits(x), _bits(y))
    c = oracle.config(L=2, fs=1, H=10, tau=1, T=40)
    a, b = both(lambda: oracle.toy_run(c, 2, 1 << 17, synth.SEED))
    for x, y in zip(a[:3], b[:3]):
        assert np.array_equal(_bits(x), _bits(y))
    assert a[3:] == b[3:]
