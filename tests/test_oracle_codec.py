"""Pins of the oracle's E3M0 codec and payload (or_e3m0_code, or_e3m0_decode,
or_block_scale, or_quantize, or_payload_bytes) against:
  * the SPEC/paper examples (golden/paper_examples.json),
  * the closed-form code table,
  * an exact-logarithm brute force (Python Decimal, 60 digits): SPEC's own
    wording "round-to-nearest of log2(|x|/scale) to {-6..0}, zero below
    2^-6.5" evaluated directly, independent of the oracle's squared
    thresholds,
  * an exhaustive sweep of every fp32 within 2^18 ulps of each threshold
    (and of every fp32 <= s for subnormal scales) against an independent
    integer-mantissa encoder (numpy int64),
  * invariants: the (sqrt2 - 1) relative error bound, monotonicity
    (S:260), exact maximum, idempotence, exact wire size."""
import json
import os
import random
import struct
from decimal import Decimal, getcontext

import numpy as np

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))
getcontext().prec = 60
LN2 = Decimal(2).ln()


def f32(x):
    return struct.unpack("<f", struct.pack("<f", x))[0]


def log_rule_code(x: float, s: float) -> int:
    """SPEC S:231 read literally: nearest integer k of log2(|x|/s) in {-6..0},
    zero code below 2^-6.5 s; e = 7 + k; sign bit from x."""
    if s == 0.0 or x == 0.0:
        return 0
    r = Decimal(abs(x)) / Decimal(s)  # Decimal(float) is exact
    lg = r.ln() / LN2
    if lg < Decimal(-6.5):
        return 0
    k = int((lg + Decimal("0.5")).to_integral_value(rounding="ROUND_FLOOR"))  # no ties exist (AMB-9)
    k = max(-6, min(0, k))
    e = 7 + k
    return (8 if np.signbit(x) else 0) | e


def int_mantissa_codes(x: np.ndarray, s: float) -> np.ndarray:
    """Independent encoder: x = mx 2^ex, s = ms 2^es with integer mantissas;
    e = #{j : mx^2 2^(2(ex-es)+2j+1) >= ms^2}, all in exact int64 shifts."""
    xb = x.astype(np.float32).view(np.uint32).astype(np.int64)
    sb = int(np.float32(s).view(np.uint32))
    def split(b):
        ebits = (b >> 23) & 0xFF
        mant = b & 0x7FFFFF
        m = np.where(ebits > 0, mant | 0x800000, mant)
        e = np.where(ebits > 0, ebits - 150, -149)
        return m, e
    mx, ex = split(xb & 0x7FFFFFFF)
    ms, es = split(np.array([sb & 0x7FFFFFFF], dtype=np.int64))
    ms, es = int(ms[0]), int(es[0])
    mx2 = mx * mx
    ms2 = ms * ms
    e = np.zeros(x.shape, dtype=np.int64)
    for j in range(7):
        D = 2 * (ex - es) + 2 * j + 1
        pos = D >= 0
        Dp = np.clip(D, 0, 62)
        need = np.where(Dp >= 48, 1, (ms2 + (np.int64(1) << Dp) - 1) >> Dp)   # ceil(ms2 / 2^D)
        cond_pos = mx2 >= need
        Dn = np.clip(-D, 0, 62)
        cond_neg = np.where(Dn >= 48, False, (mx2 >> Dn) >= ms2)               # floor(mx2 / 2^-D) >= ms2
        e += np.where(pos, cond_pos, cond_neg)
    if s == 0.0:
        e[:] = 0
    sign = (xb >> 31) & 1
    return np.where(e > 0, (sign << 3) | e, 0).astype(np.uint8)


def oracle_codes(values: np.ndarray) -> tuple:
    """or_quantize with B = 0 on anchor = values, theta = 0: Delta = values
    exactly, scale = max|values|; returns (codes unpacked, scale)."""
    values = np.ascontiguousarray(values, dtype=np.float32)
    n = values.size
    payload, poisoned = oracle.quantize(np.zeros(n, np.float32), values, B=0)
    assert not poisoned
    packed = payload[: (n + 1) // 2]
    codes = np.empty(2 * packed.size, dtype=np.uint8)
    codes[0::2] = packed & 15
    codes[1::2] = packed >> 4
    s = float(payload[oracle.scales_offset(n): oracle.scales_offset(n) + 4].view(np.float32)[0])
    return codes[:n], s


# ----------------------------------------------------------------- examples
def test_code_table_closed_form():
    for s in (1.0, 2.0, 0.75, 2.0 ** -140):
        for c in range(16):
            e = c & 7
            want = 0.0 if e == 0 else (-1.0 if c & 8 else 1.0) * 2.0 ** (e - 7) * s
            got = oracle.e3m0_decode(c, s)
            assert got == f32(want), (c, s)
            if e == 0:
                assert not np.signbit(got)  # both e=0 codes decode to +0


def test_spec_examples():
    g = GOLD["e3m0_examples"]
    xs = g["roundtrip_exact_at_scale_1"]
    for x in xs:
        c = oracle.e3m0_code(x, 1.0)
        assert oracle.e3m0_decode(c, 1.0) == x
    for ex in g["nearest_in_log2"]:
        assert oracle.e3m0_decode(oracle.e3m0_code(ex["x"], ex["scale"]), ex["scale"]) == ex["decoded"]
    for ex in g["decode"]:
        assert oracle.e3m0_decode(ex["code"], ex["scale"]) == ex["value"]
    codes, s = oracle_codes(np.zeros(37, np.float32))  # all zeros -> scale 0, zero codes
    assert s == 0.0 and not codes.any()


def test_scale_is_exact_absmax():
    rng = np.random.default_rng(1)
    d = (rng.standard_normal(999) * 1e-3).astype(np.float32)
    d[123] = -0.25
    assert oracle.block_scale(d) == 0.25
    assert oracle.block_scale(np.array([-0.0, 0.0], np.float32)) == 0.0


# ------------------------------------------------------------ brute force
def _near_threshold_samples(rng, s, count):
    out = []
    for _ in range(count):
        j = rng.randrange(7)
        t = float(Decimal(s) * (Decimal(2) ** Decimal(-j - 0.5)).normalize())
        x = np.float32(t)
        steps = rng.randint(-4, 4)
        xb = int(np.float32(x).view(np.uint32)) + steps
        out.append(float(np.uint32(xb).view(np.float32)) * rng.choice((-1, 1)))
    return out


def test_exact_log2_brute_force():
    rng = random.Random(7)
    scales = [1.0, 1.5, 3.0e-3, 2.0 ** -126, 2.0 ** -140, 12345.678]
    for s in scales:
        s = f32(s)
        xs = _near_threshold_samples(rng, s, 250)
        xs += [f32(s * rng.uniform(-1, 1) ** 3) for _ in range(250)]
        xs += [s, -s, 0.0, -0.0]
        for x in xs:
            if abs(x) > s:
                continue
            assert oracle.e3m0_code(x, s) == log_rule_code(x, s), (x, s)


def test_exhaustive_against_integer_mantissa_encoder():
    """Every fp32 within 2^18 ulps of each of the 7 thresholds s 2^(-j-1/2)
    (where the code changes), for three scales, plus every fp32 in [0, s]
    for subnormal / smallest-normal scales."""
    for s in (1.0, 1.5, 0.3):
        s = f32(s)
        for j in range(7):
            t = np.float32(float(Decimal(s) * (Decimal(2) ** Decimal(-j - 0.5))))
            c = int(t.view(np.uint32))
            xs = np.arange(c - (1 << 18), c + (1 << 18), dtype=np.uint32).view(np.float32)
            vals = np.concatenate([[np.float32(s)], xs])
            vals[1::2] *= -1  # exercise the sign bit on half of them
            got, sc = oracle_codes(vals)
            assert sc == s
            want = int_mantissa_codes(vals, s)
            bad = np.nonzero(got != want)[0]
            assert bad.size == 0, (s, j, vals[bad[:5]], got[bad[:5]], want[bad[:5]])
    # tiny (subnormal) scales: every fp32 in [0, s]
    for sbits in (1, 7, 0x3FFF, 0x7FFFFF, 0x00800000, 0x00800123):
        s = float(np.uint32(sbits).view(np.float32))
        xs = np.arange(0, sbits + 1, dtype=np.uint32).view(np.float32)
        vals = np.concatenate([[np.float32(s)], xs])
        got, sc = oracle_codes(vals)
        assert sc == np.float32(s)
        assert np.array_equal(got, int_mantissa_codes(vals, s)), s


def test_invariants_error_bound_monotone_idempotent():
    rng = np.random.default_rng(3)
    s = np.float32(0.0421)
    x = (rng.uniform(-1, 1, 200000) * s).astype(np.float32)
    x[0] = s
    codes, sc = oracle_codes(x)
    assert sc == s
    dec = np.array([oracle.e3m0_decode(int(c), float(sc)) for c in codes[:20000]], dtype=np.float64)
    xx = x[:20000].astype(np.float64)
    inband = np.abs(xx) >= 2.0 ** -6 * float(s)
    rel = np.abs(dec - xx)[inband] / np.abs(xx)[inband]
    assert rel.max() <= np.sqrt(2.0) - 1.0 + 1e-12
    assert dec[0] == float(s)                                                  # the max is exact
    order = np.argsort(np.abs(xx), kind="stable")                              # S:260 monotone
    mags = np.where(codes[:20000] & 7, codes[:20000] & 7, 0)[order]
    assert np.all(np.diff(mags.astype(int)) >= 0)
    assert np.all((codes[:20000][xx < 0] & 8) | ((codes[:20000][xx < 0] & 7) == 0))
    # idempotence: decode(encode(decode(b))) = decode(b)
    again, sc2 = oracle_codes(dec.astype(np.float32))
    assert sc2 == sc and np.array_equal(again, codes[:20000])


# ------------------------------------------------------------------ payload
def test_payload_layout_and_wire_size():
    rng = np.random.default_rng(5)
    for n, B in ((1, 1024), (2, 1024), (1023, 256), (4097, 1024), (5000, 0), (65536 + 3, 2048), (0, 1024)):
        pb = oracle.payload_bytes(n, B)
        nb = oracle.num_scale_blocks(n, B)
        assert nb == (0 if n == 0 else (1 if B == 0 else -(-n // B)))
        soff = oracle.scales_offset(n)
        assert soff == -(-((n + 1) // 2) // 256) * 256 and pb % 256 == 0
        # exact wire size: ceil(n/2) code bytes + 4 nb scale bytes + 16 trailer, padded
        assert pb == soff + -(-(-(-4 * nb // 16) * 16 + 16) // 256) * 256
        A = rng.standard_normal(n).astype(np.float32)
        th = (A - rng.standard_normal(n).astype(np.float32) * 1e-3).astype(np.float32)
        pay, poisoned = oracle.quantize(th, A, B)
        assert not poisoned and pay.size == pb
        toff = soff + -(-4 * nb // 16) * 16
        assert pay[toff:toff + 4].view(np.uint32)[0] == 0x31304453
        assert pay[toff + 4:toff + 8].view(np.uint32)[0] == nb
        assert pay[toff + 8:toff + 16].view(np.uint64)[0] == np.uint64(2 ** 64 - 1)
        # zero padding everywhere outside codes / scales / trailer
        assert not pay[(n + 1) // 2:soff].any()
        assert not pay[soff + 4 * nb:toff].any() and not pay[toff + 16:].any()
        if n % 2 == 1:
            assert pay[(n - 1) // 2] >> 4 == 0  # odd tail: high nibble 0
        # nibble order: element 2k in the low nibble of byte k
        d = (A - th).astype(np.float32)
        blen = B if B else max(n, 1)
        for i in rng.integers(0, max(n, 1), size=min(n, 50)):
            s = float(pay[soff + 4 * (i // blen): soff + 4 * (i // blen) + 4].view(np.float32)[0])
            c = (pay[i // 2] >> (4 * (i % 2))) & 15
            assert c == oracle.e3m0_code(float(d[i]), s)


def test_nonfinite_poisons_with_first_index():
    A = np.zeros(3000, np.float32)
    th = np.zeros(3000, np.float32)
    th[2500] = np.inf
    th[1700] = np.nan
    pay, poisoned = oracle.quantize(th, A, 1024)
    assert poisoned
    r, fb = oracle.payload_poisoned(pay, 3000, 1024)
    assert r == 1 and fb == 1700
