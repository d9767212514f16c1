"""Mutation check of the oracle's pins: plausible one-line mistakes in
oracle/sd_oracle.c (a dropped term, a wrong sign or index, a transposed
operand, the wrong scale slot or block) are compiled into a throwaway
library and the CPU pin tests (tests/test_oracle_*.py, -m "not gpu") are run
against it; each mutant must make at least one pin fail.  The oracle source
in the repo is never modified; the mutant is loaded in-process in place of
liboracle.so while the pin functions run.  (two scale-addressing mutants
of or_decode_mean passed every pin before the distinct-scale pins.)"""
import itertools
import os
import subprocess
import sys
import tempfile

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "sd_oracle.c")

MUTANTS = {
    # or_decode_mean: slot 0's scale for every replica m
    "scale_slot0": ("memcpy(&s, slot + soff + 4 * (size_t)(i / blen), 4);",
                    "memcpy(&s, gather + soff + 4 * (size_t)(i / blen), 4);"),
    # or_decode_mean: block 0's scale for every element
    "scale_block0": ("memcpy(&s, slot + soff + 4 * (size_t)(i / blen), 4);", "memcpy(&s, slot + soff, 4);"),
    # or_decode_mean: last replica overwrites instead of accumulating (dropped term)
    "dropped_sum_term": ("S = (m == 0) ? q : S + q;", "S = q;"),
    # or_decode_mean: missing 1/M
    "missing_mean_div": ("g[i] = S / (float)M;", "g[i] = S;"),
    # or_nesterov: wrong sign of the anchor update
    "nesterov_sign": ("A[i] = A[i] - lr * (g[i] + mu * v[i]);", "A[i] = A[i] + lr * (g[i] + mu * v[i]);"),
    # or_nesterov: look-ahead term dropped (heavy-ball instead of Nesterov)
    "nesterov_no_lookahead": ("A[i] = A[i] - lr * (g[i] + mu * v[i]);", "A[i] = A[i] - lr * (mu * v[i]);"),
    # or_merge: alpha and 1 - alpha transposed
    "merge_transposed": ("theta[i] = alpha * theta[i] + beta * A[i];", "theta[i] = beta * theta[i] + alpha * A[i];"),
    # or_quantize: Delta = theta - A (transposed operands)
    "delta_sign": ("delta[i] = anchor[i] - theta[i];", "delta[i] = theta[i] - anchor[i];"),
    # or_quantize: nibble order swapped
    "nibble_order": ("payload[k] = (uint8_t)(c0 | (c1 << 4));", "payload[k] = (uint8_t)(c1 | (c0 << 4));"),
    # or_e3m0_decode: wrong table index
    "decode_index": ("return LUT[code & 15] * s;", "return LUT[code & 7] * s;"),
    # encoder: thresholds at the grid points instead of the log2 midpoints
    "threshold_exponent": ("if (d2 >= ldexp(s2, -2 * j - 1)) ++e;", "if (d2 >= ldexp(s2, -2 * j)) ++e;"),
    # encoder: code 8 (sign with e = 0) emitted for small negative values
    "sign_on_zero_code": ("  if (e == 0) return 0; /* encoders emit s=0 with e=0 (S:264) */\n", ""),
    # block scale: the first element instead of the max
    "scale_first_element": ("    if (a > s) s = a;", "    if (i == 0) s = a;"),
    # calendar: offsets rounded up instead of floor(p H / P)
    "offset_rounding": ("return (int32_t)(((int64_t)p * c->H) / P);", "return (int32_t)(((int64_t)p * c->H + P - 1) / P);"),
    # calendar: receive one step after send + tau
    "receive_one_late": ("if (pending[p] + c->tau == t || t == c->T) {", "if (pending[p] + c->tau + 1 == t || t == c->T) {"),
    # calendar: no flush of in-flight fragments at T
    "no_flush": ("if (pending[p] + c->tau == t || t == c->T) {", "if (pending[p] + c->tau == t) {"),
    # calendar: first send before a full window (t >= H dropped)
    "first_send_before_H": ("if (t >= c->H && (t - tp) % c->H == 0) {", "if ((t - tp) % c->H == 0) {"),
    # partition: sequential and strided patterns swapped
    "pattern_swapped": ("out[k] = c->pattern == 0 ? p * c->fs + k : p + k * Pb;",
                        "out[k] = c->pattern != 0 ? p * c->fs + k : p + k * Pb;"),
}


def _pin_calls(module):
    """Every test function of a pin module with its parametrize marks
    expanded (cartesian product), in file order."""
    out = []
    for name, fn in vars(module).items():
        if not (name.startswith("test_") and callable(fn)):
            continue
        grids = [[{}]]
        for mark in getattr(fn, "pytestmark", []):
            if mark.name != "parametrize":
                continue
            names, values = mark.args[0], mark.args[1]
            names = [x.strip() for x in names.split(",")] if isinstance(names, str) else list(names)
            grids.append([dict(zip(names, v if len(names) > 1 else (v,))) for v in values])
        for combo in itertools.product(*grids):
            kw = {}
            for d in combo:
                kw.update(d)
            out.append((name, fn, kw))
    return out


def _caught(so):
    """Runs the pins against the library at `so`; returns the first failing pin or None."""
    import test_oracle_codec
    import test_oracle_outer
    import test_oracle_schedule

    saved = dict(oracle._libs)
    oracle._libs["liboracle.so"] = oracle._load_path(so)
    prev = oracle.set_threads(1)
    try:
        for mod in (test_oracle_outer, test_oracle_codec, test_oracle_schedule):
            for name, fn, kw in _pin_calls(mod):
                try:
                    fn(**kw)
                except Exception as e:  # noqa: BLE001 - any failing pin catches the mutant
                    return f"{mod.__name__}::{name}{kw}: {type(e).__name__}"
        return None
    finally:
        oracle._libs.clear()
        oracle._libs.update(saved)
        oracle.set_threads(prev)


@pytest.mark.parametrize("name", sorted(MUTANTS))
def test_mutant_is_caught_by_a_pin(name):
    old, new = MUTANTS[name]
    orig = open(SRC).read()
    assert orig.count(old) == 1, f"mutant {name}: anchor text not found exactly once in sd_oracle.c"
    src = orig.replace(old, new)
    with tempfile.TemporaryDirectory() as tmp:
        # compiled from a hidden sibling file: the source includes "../synth/synth.h"
        mpath = os.path.join(ROOT, "oracle", f".mutant_{name}_{os.getpid()}.c")
        try:
            with open(mpath, "w") as f:
                f.write(src)
            so = os.path.join(tmp, f"liboracle_{name}.so")
            subprocess.run(["gcc", "-std=c99", "-O2", "-fno-fast-math", "-ffp-contract=off", "-w", "-shared", "-fPIC",
                            "-o", so, mpath, os.path.join(ROOT, "synth", "synth_cpu.c"), "-lm"],
                           check=True, capture_output=True)
        finally:
            os.remove(mpath)
        hit = _caught(so)
        assert hit is not None, f"mutant {name} survived every CPU pin"
        print(f"mutant {name}: caught by {hit}")


def test_unmutated_oracle_passes_the_same_harness():
    """Control: the harness itself reports no failure on the real oracle."""
    assert _caught(os.path.join(ROOT, "oracle", "liboracle.so")) is None
