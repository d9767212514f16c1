"""Host-side checks of the product library, no GPU needed:
  * libsd.so loads and exports every function include/sd.h declares;
  * the closed-form scheduler (sd_fragment_schedule / sd_fragment_layout) is
    integer-identical to the oracle's brute-force calendar scan over ~200
    random valid configs (acceptance 7);
  * payload sizes/offsets agree with the oracle's;
  * config validation rejects bad configs before any work, naming the
    offending values."""
import os
import random
import re

import pytest

import oracle
from paper_2501_18512_b200 import sd

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    import ctypes

    L = ctypes.CDLL(sd.LIB_PATH)
    header = open(os.path.join(ROOT, "include", "sd.h")).read()
    declared = set(re.findall(r"^\s*(?:sd_status|size_t|int64_t|uint64_t|const char\*)\s+(sd_\w+)\(", header, re.M))
    assert declared == set(sd.EXPORTS), declared ^ set(sd.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name


def test_library_is_sm100a_and_links_nccl():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", sd.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    ldd = subprocess.run(["ldd", sd.LIB_PATH], capture_output=True, text=True).stdout
    assert "libnccl.so.2" in ldd


def _both(L, fs, pattern, policy, H, tau, T):
    c_or = oracle.config(L=L, fs=fs, pattern=pattern, embed_policy=policy, H=H, tau=tau, T=T)
    c_sd = sd.sd_config_default(L, fs, H, pattern=pattern, embed_policy=policy, tau=tau, T=T)
    return c_or, c_sd


def test_schedule_matches_oracle_bruteforce_random_configs():
    rng = random.Random(250118512)
    for trial in range(200):
        fs = rng.randint(1, 4)
        L = fs * rng.randint(1, 12)
        policy = rng.randint(0, 1)
        P = L // fs + policy
        H = rng.randint(P, 50)
        tau = rng.randint(0, H - 1)
        T = rng.randint(1, 4 * H)
        c_or, c_sd = _both(L, fs, rng.randint(0, 1), policy, H, tau, T)
        assert sd.sd_fragment_count(c_sd) == oracle.num_fragments(c_or)
        for p in range(P):
            blocks, tp, _ = sd.sd_fragment_layout(c_sd, p)
            assert blocks == oracle.fragment_blocks(c_or, p) and tp == oracle.offset(c_or, p)
        want = {}
        for t, kind, p, s in oracle.calendar(c_or):
            want.setdefault(t, ([], []))[kind].append(p)
        for t in range(1, T + 3):
            got = sd.sd_fragment_schedule(c_sd, t)
            exp = want.get(t, ([], []))
            assert (got[0], got[1]) == (exp[0], exp[1]), (trial, t, got, exp)


def test_embedding_placement():
    c = sd.sd_config_default(24, 3, 100)
    assert [sd.sd_fragment_layout(c, p)[2] for p in range(8)] == [False] * 7 + [True]
    c = sd.sd_config_default(24, 3, 100, embed_policy=1)
    assert sd.sd_fragment_count(c) == 9
    assert sd.sd_fragment_layout(c, 8) == ([], 88, True)


def test_payload_sizes_match_oracle():
    for n in (0, 1, 2, 255, 256, 1023, 1025, 4096, 5197, 151007616, 438064512):
        for B in (0, 256, 512, 1024, 2048, 1 << 20):
            c = sd.sd_config_default(2, 1, 10, scale_block=B)
            assert sd.sd_payload_bytes(c, n) == oracle.payload_bytes(n, B)
            assert sd.sd_payload_scales_offset(n) == oracle.scales_offset(n)
            assert sd.sd_num_scale_blocks(c, n) == oracle.num_scale_blocks(n, B)


@pytest.mark.parametrize(
    "kw,needle",
    [
        (dict(num_blocks=24, fragment_size=5), "fragment_size 5 does not divide num_blocks 24"),
        (dict(H=4), "H 4 must be >= 1 and >= the number of fragments P 8"),
        (dict(tau=100), "tau 100 violates 0 <= tau < H (H = 100)"),
        (dict(alpha=1.5), "alpha 1.5 is not in [0, 1]"),
        (dict(outer_momentum=1.0), "outer_momentum 1 is not in [0, 1)"),
        (dict(scale_block=1000), "scale_block 1000 is neither 0 nor a power of two"),
        (dict(pattern=3), "pattern 3"),
        (dict(abi_version=7), "abi_version 7"),
    ],
)
def test_config_validation_names_values(kw, needle):
    c = sd.sd_config_default(24, 3, 100)
    for k, v in kw.items():
        setattr(c, k, v)
    st, msg = sd.sd_config_validate(c)
    assert st == sd.SD_ERR_CONFIG and needle in msg, msg
    with pytest.raises(sd.SdError):
        sd.sd_fragment_schedule(c, 100)


def test_schedule_rejects_step_zero():
    c = sd.sd_config_default(24, 3, 100)
    with pytest.raises(sd.SdError, match="must be >= 1"):
        sd.sd_fragment_schedule(c, 0)


def test_quantize_workspace_bytes():
    """Scratch only for the two-pass quantize (B = 0 or B > 1024): 2 bytes of
    summary per element plus one 16-byte row-max record per 1024-element chunk."""
    for B in (256, 512, 1024):
        assert sd.sd_quantize_workspace_bytes(sd.sd_config_default(2, 1, 10, scale_block=B), 10 ** 6) == 0
    for B in (0, 2048, 1 << 20):
        c = sd.sd_config_default(2, 1, 10, scale_block=B)
        assert sd.sd_quantize_workspace_bytes(c, 0) == 0
        assert sd.sd_quantize_workspace_bytes(c, 1) == 2064
        assert sd.sd_quantize_workspace_bytes(c, 1024) == 2064
        assert sd.sd_quantize_workspace_bytes(c, 1025) == 2 * 2064
        assert sd.sd_quantize_workspace_bytes(c, 151007616) == 147469 * 2064
    assert sd.sd_quantize_workspace_bytes(sd.sd_config_default(2, 1, 10, scale_block=3000), 4096) == 0  # invalid B
