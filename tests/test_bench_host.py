"""Host logic of bench.py: the algorithmic-byte model and
the calendar order it cycles through (libsd's scheduler == the oracle's
brute-force scan), plus the workload shapes it names."""
import bench
import oracle
import synth
from synth.workloads import WORKLOADS
from paper_2501_18512_b200 import sd


def test_algorithmic_bytes_per_element():
    n = 1 << 20
    q, a = bench.algorithmic_bytes(n, 1, 1024)
    assert abs(q / n - 8.50390625) < 1e-12          # 8 + 0.5 + 4/1024
    assert abs(a / n - 24.50390625) < 1e-12
    for M in (2, 4, 8):
        assert abs(bench.algorithmic_bytes(n, M, 1024)[1] / n - (24 + M * 0.50390625)) < 1e-12
    q0, a0 = bench.algorithmic_bytes(n, 2, 0)       # B = 0: one scale
    assert q0 == 8 * n + n / 2 + 4 and a0 == 24 * n + 2 * (n / 2 + 4)


def test_calendar_sends_match_oracle_scan():
    wl = WORKLOADS["1B"]
    cfg = bench.make_cfg(sd, wl, 1024)
    got = bench.calendar_sends(sd, cfg, 40)
    c = oracle.config(L=wl.layers, fs=wl.fragment_size, H=wl.H, tau=wl.tau, T=10_000)
    want = [(p, t) for t, kind, p, s in oracle.calendar(c) if kind == 0][:40]
    assert got == want
    assert [p for p, _ in got[:8]] == list(range(8))          # strided offsets 0,12,25,...
    assert [t for _, t in got[:8]] == [100, 112, 125, 137, 150, 162, 175, 187]


def test_workload_fragment_sizes():
    for name, sizes in (("1B", (151007616, 216545664)), ("4B", (339757440, 438064512)),
                        ("35M", (6293760, 22678272))):
        wl = WORKLOADS[name]
        cfg = bench.make_cfg(sd, wl, 1024)
        P = sd.sd_fragment_count(cfg)
        n = [synth.segments_numel(wl.segments(b, e)) for b, _, e in (sd.sd_fragment_layout(cfg, p) for p in range(P))]
        assert n[0] == sizes[0] and n[-1] == sizes[1] and sum(n) in (1273598976, 4175396352, 35265792)


def test_overrides():
    import argparse

    args = argparse.Namespace(tau=0, fragment_size=6)
    wl = bench.workload_with_overrides(WORKLOADS["1B"], args)
    assert wl.tau == 0 and wl.fragment_size == 6 and WORKLOADS["1B"].tau == 5


def test_reference_arm_uses_only_the_oracle():
    """`bench.py --impl reference` takes its calendar and fragment layout from
    the oracle's own scheduler (identical to libsd's) and never loads libsd."""
    import subprocess
    import sys

    wl = WORKLOADS["1B"]
    _, lay, sends = bench.ref_layout(wl, 1024)
    cfg = bench.make_cfg(sd, wl, 1024)
    assert sends[:40] == bench.calendar_sends(sd, cfg, 40)
    for p, (blocks, emb) in enumerate(lay):
        b, t_p, e = sd.sd_fragment_layout(cfg, p)
        assert list(b) == blocks and bool(e) == emb
    code = ("import sys, bench, argparse; bench.run_reference(argparse.Namespace(workload='toy', scale_block=1024, tau=None, "
            "fragment_size=None, steps=1, warmup=1, gpus=1)); "
            "import os; maps = open('/proc/self/maps').read(); "
            "assert 'libsd.so' not in maps and 'paper_2501_18512_b200' not in sys.modules, 'libsd loaded'")
    r = subprocess.run([sys.executable, "-c", code], cwd=bench.ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert '"impl": "reference"' in r.stdout
