"""ctypes view of the CPU oracle (oracle/sd_oracle.c).

Two builds of the same C source: liboracle.so (single thread, the oracle
proper) and liboracle_omp.so (OpenMP, selected by set_threads(n > 1)).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product
package paper_2501_18512_b200/.  See sd_oracle.h for the parity status of
each function and DESIGN.md §2 for the readings of the paper it follows.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))


class OrConfig(ctypes.Structure):
    _fields_ = [
        ("L", ctypes.c_int32), ("fs", ctypes.c_int32), ("pattern", ctypes.c_int32),
        ("embed_policy", ctypes.c_int32), ("H", ctypes.c_int32), ("tau", ctypes.c_int32),
        ("T", ctypes.c_int64), ("alpha", ctypes.c_float), ("lr", ctypes.c_float),
        ("mu", ctypes.c_float), ("B", ctypes.c_int32),
    ]


class OrEvent(ctypes.Structure):
    _fields_ = [("t", ctypes.c_int64), ("kind", ctypes.c_int32), ("p", ctypes.c_int32), ("send_step", ctypes.c_int64)]


_libs = {}
_active = "liboracle.so"
_threads = 1


def _load(name):
    return _load_path(os.path.join(_HERE, name))


def _load_path(path):
    if not os.path.exists(path):
        raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
    L = ctypes.CDLL(path)
    P, I64, I32, F = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_float
    C = ctypes.POINTER(OrConfig)
    sig = {
        "or_num_fragments": ([C], I32),
        "or_fragment_blocks": ([C, I32, P], I32),
        "or_offset": ([C, I32], I32),
        "or_calendar": ([C, P, I64], I64),
        "or_block_scale": ([P, I64], F),
        "or_e3m0_code": ([F, F], ctypes.c_uint8),
        "or_e3m0_decode": ([ctypes.c_uint8, F], F),
        "or_num_scale_blocks": ([I64, I32], I64),
        "or_payload_bytes": ([I64, I32], ctypes.c_size_t),
        "or_scales_offset": ([I64], ctypes.c_size_t),
        "or_quantize": ([P, P, I64, I32, P], ctypes.c_int),
        "or_payload_poisoned": ([P, I64, I32, ctypes.POINTER(ctypes.c_uint64)], ctypes.c_int),
        "or_decode_mean": ([P, I32, I64, I32, P], None),
        "or_nesterov": ([P, P, P, I64, F, F], None),
        "or_merge": ([P, P, I64, F], None),
        "or_outer_state_init": ([P, P, P, I64], None),
        "or_apply": ([P, I32, I64, I32, F, F, F, P, P, P], ctypes.c_int),
        "or_round": ([I32, I64, I32, F, F, F, P, P, P, P, P], ctypes.c_int),
        "or_toy_run": ([C, I32, I64, ctypes.c_uint64, P, P, P, ctypes.POINTER(I64)], ctypes.c_int),
        "or_adamw": ([P, P, P, P, I64, I64, F, F, F, F, F], None),
        "or_toy_run_taus": ([C, I32, I64, ctypes.c_uint64, P, P, P, P, ctypes.POINTER(I64)], ctypes.c_int),
    }
    for fname, (args, res) in sig.items():
        fn = getattr(L, fname)
        fn.argtypes = args
        fn.restype = res
    return L


def lib():
    if _active not in _libs:
        _libs[_active] = _load(_active)
    return _libs[_active]


def set_threads(n: int) -> int:
    """n == 1: the single-threaded build (liboracle.so, the oracle proper);
    n > 1: the same source built with OpenMP (liboracle_omp.so) on n threads.
    Both produce bit-identical results (tests/test_oracle_omp.py).  Returns
    the previous thread count."""
    global _active, _threads
    prev = _threads
    if n <= 1:
        _active, _threads = "liboracle.so", 1
    else:
        _active, _threads = "liboracle_omp.so", int(n)
        lib()
        ctypes.CDLL("libgomp.so.1").omp_set_num_threads(ctypes.c_int(int(n)))
    return prev


def threads() -> int:
    return _threads


def _p(a: np.ndarray):
    assert a.flags.c_contiguous, "oracle arrays must be contiguous"
    return a.ctypes.data


def config(L=2, fs=1, pattern=1, embed_policy=0, H=10, tau=1, T=100, alpha=0.5, lr=0.4, mu=0.9, B=1024) -> OrConfig:
    return OrConfig(L, fs, pattern, embed_policy, H, tau, T, alpha, lr, mu, B)


# ---- schedule ----------------------------------------------------------------
def num_fragments(c: OrConfig) -> int:
    return lib().or_num_fragments(ctypes.byref(c))


def fragment_blocks(c: OrConfig, p: int):
    out = np.zeros(max(c.fs, 1), dtype=np.int32)
    k = lib().or_fragment_blocks(ctypes.byref(c), p, _p(out))
    return [int(x) for x in out[:k]]


def offset(c: OrConfig, p: int) -> int:
    return lib().or_offset(ctypes.byref(c), p)


def calendar(c: OrConfig):
    """[(t, kind, p, send_step)], kind 0 = send, 1 = receive."""
    n = lib().or_calendar(ctypes.byref(c), None, 0)
    ev = (OrEvent * max(n, 1))()
    lib().or_calendar(ctypes.byref(c), ev, n)
    return [(e.t, e.kind, e.p, e.send_step) for e in ev[:n]]


# ---- codec -------------------------------------------------------------------
def e3m0_code(d: float, s: float) -> int:
    return lib().or_e3m0_code(d, s)


def e3m0_decode(code: int, s: float) -> float:
    return lib().or_e3m0_decode(code, s)


def block_scale(d: np.ndarray) -> float:
    d = np.ascontiguousarray(d, dtype=np.float32)
    return lib().or_block_scale(_p(d), d.size)


def num_scale_blocks(n: int, B: int) -> int:
    return lib().or_num_scale_blocks(n, B)


def payload_bytes(n: int, B: int) -> int:
    return lib().or_payload_bytes(n, B)


def scales_offset(n: int) -> int:
    return lib().or_scales_offset(n)


def quantize(theta: np.ndarray, anchor: np.ndarray, B: int):
    """-> (payload bytes as np.uint8, poisoned flag)"""
    theta = np.ascontiguousarray(theta, dtype=np.float32)
    anchor = np.ascontiguousarray(anchor, dtype=np.float32)
    n = theta.size
    out = np.empty(payload_bytes(n, B), dtype=np.uint8)
    r = lib().or_quantize(_p(theta), _p(anchor), n, B, _p(out))
    return out, bool(r)


def payload_poisoned(payload: np.ndarray, n: int, B: int):
    fb = ctypes.c_uint64(0)
    r = lib().or_payload_poisoned(_p(payload), n, B, ctypes.byref(fb))
    return r, fb.value


def decode_mean(gather: np.ndarray, M: int, n: int, B: int) -> np.ndarray:
    g = np.empty(n, dtype=np.float32)
    lib().or_decode_mean(_p(gather), M, n, B, _p(g))
    return g


def nesterov(A, v, g, lr=0.4, mu=0.9):
    """in place on float32 arrays A, v"""
    lib().or_nesterov(_p(A), _p(v), _p(g), A.size, lr, mu)


def merge(theta, A, alpha=0.5):
    lib().or_merge(_p(theta), _p(A), theta.size, alpha)


def outer_state_init(theta):
    """-> (A, v): A_p <- theta_init (bit copy), v_p <- 0."""
    theta = np.ascontiguousarray(theta, dtype=np.float32)
    A = np.empty_like(theta)
    v = np.empty_like(theta)
    lib().or_outer_state_init(_p(theta), _p(A), _p(v), theta.size)
    return A, v


def apply(gather, M, n, B, A, v, theta, lr=0.4, mu=0.9, alpha=0.5) -> int:
    return lib().or_apply(_p(gather), M, n, B, lr, mu, alpha, _p(A), _p(v), _p(theta))


def round_(theta_send, theta_merge, A, v, B=1024, lr=0.4, mu=0.9, alpha=0.5):
    """One fragment round on all replicas; theta_merge (list), A, v updated in place.
    Returns (status, gather buffer)."""
    M = len(theta_send)
    n = A.size
    gather = np.empty(M * payload_bytes(n, B), dtype=np.uint8)
    ps = (ctypes.c_void_p * M)(*[_p(x) for x in theta_send])
    pm = (ctypes.c_void_p * M)(*[_p(x) for x in theta_merge])
    r = lib().or_round(M, n, B, lr, mu, alpha, ps, pm, _p(A), _p(v), _p(gather))
    return r, gather


def toy_run(c: OrConfig, M: int, block_len: int, seed: int):
    """-> (theta [M, P*n], A [P*n], v [P*n], bytes_sent, status)"""
    P = num_fragments(c)
    n = c.fs * block_len
    theta = np.empty((M, P * n), dtype=np.float32)
    A = np.empty(P * n, dtype=np.float32)
    v = np.empty(P * n, dtype=np.float32)
    bs = ctypes.c_int64(0)
    r = lib().or_toy_run(ctypes.byref(c), M, block_len, seed, _p(theta), _p(A), _p(v), ctypes.byref(bs))
    return theta, A, v, bs.value, r


def toy_run_taus(c: OrConfig, M: int, block_len: int, seed: int, taus):
    """Per-replica tau_m -> (theta [M, P*n], A [M, P*n], v [M, P*n], bytes, status)"""
    P = num_fragments(c)
    n = c.fs * block_len
    theta = np.empty((M, P * n), dtype=np.float32)
    A = np.empty((M, P * n), dtype=np.float32)
    v = np.empty((M, P * n), dtype=np.float32)
    t = np.ascontiguousarray(taus, dtype=np.int32)
    bs = ctypes.c_int64(0)
    r = lib().or_toy_run_taus(ctypes.byref(c), M, block_len, seed, _p(t), _p(theta), _p(A), _p(v), ctypes.byref(bs))
    return theta, A, v, bs.value, r


def adamw(theta, g, m, v, k, lr=1e-3, b1=0.9, b2=0.99, eps=1e-8, wd=0.0):
    """One AdamW step in place on float32 arrays theta, m, v."""
    lib().or_adamw(_p(theta), _p(g), _p(m), _p(v), theta.size, k, lr, b1, b2, eps, wd)
