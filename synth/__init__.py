"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

Holds none of the method's arithmetic (see synth.h).  Host generation goes
through ``libsynth_cpu.so`` (numpy arrays), device generation through
``libsynth_cuda.so`` (raw device pointers from torch tensors).  Both are
built from the same ``synth.h``, so a value is a pure function of
(seed, purpose, fragment, replica, round/step, element index).

Fragment shapes follow SURVEY.md §8(d) / AMB-17: Chinchilla-style layers of
width d_model with FFN width 4*d_model, head dim 64, vocabulary 32,000
(Table 2 read as "Hidden dim" = FFN width).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SEED = 250118512

SEG_DTYPE = np.dtype(
    [("start", "<i8"), ("len", "<i8"), ("kind", "<i4"), ("first_block", "<i4"), ("row", "<i4"), ("pad_", "<i4")]
)
MATRIX, NORM, EMBED = 0, 1, 2
VOCAB = 32000
HEAD_DIM = 64


def layer_numel(d: int) -> int:
    """ln1[d], Wq/Wk/Wv/Wo [d x d], q_norm/k_norm [64], ln2[d], W1 [d x 4d], W2 [4d x d]."""
    return 12 * d * d + 2 * d + 2 * HEAD_DIM


def fragment_segments(d_model: int, layers, with_embed: bool, vocab: int = VOCAB) -> np.ndarray:
    """Segment table of one fragment-contiguous slab: the fragment's layers in
    ascending order, then (if it holds the non-block parameters) the tied
    embedding [vocab x d] and the final norm [d]."""
    segs = []
    pos = 0

    def add(n, kind, first=0, row=1):
        nonlocal pos
        segs.append((pos, n, kind, first, row, 0))
        pos += n

    d = d_model
    for layer in sorted(layers):
        f = 1 if layer == 0 else 0
        add(d, NORM, f)                     # ln1
        add(4 * d * d, MATRIX, f)           # Wq Wk Wv Wo
        add(2 * HEAD_DIM, NORM, f)          # q_norm, k_norm (QKNorm)
        add(d, NORM, f)                     # ln2
        add(8 * d * d, MATRIX, f)           # W1, W2
    if with_embed:
        add(vocab * d, EMBED, 0, d)         # tied embedding
        add(d, NORM, 0)                     # final norm
    return np.array(segs, dtype=SEG_DTYPE)


def flat_segments(n: int) -> np.ndarray:
    """A flat vector (toy config): one matrix-kind segment."""
    return np.array([(0, n, MATRIX, 0, 1, 0)], dtype=SEG_DTYPE)


def segments_numel(segs: np.ndarray) -> int:
    return int(segs["start"][-1] + segs["len"][-1]) if len(segs) else 0


# --------------------------------------------------------------------------- host
_cpu = None


def _lib_cpu():
    global _cpu
    if _cpu is None:
        path = os.path.join(_HERE, "libsynth_cpu.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        P, I64, I32, U64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64
        lib.synth_fill_init.argtypes = [P, P, ctypes.c_int, U64, I32, I64, I64]
        lib.synth_apply_window.argtypes = [P, P, ctypes.c_int, U64, I32, I32, I32, I64, I64]
        lib.synth_apply_drift.argtypes = [P, P, ctypes.c_int, U64, I32, I32, I32, I64, I64]
        lib.synth_apply_toy.argtypes = [P, U64, I32, I64, I64, I64]
        lib.synth_fill_U.argtypes = [P, U64, I64, I64]
        lib.synth_key.argtypes = [U64, U64, U64, U64, U64]
        lib.synth_key.restype = U64
        lib.synth_H.argtypes = [U64]
        lib.synth_H.restype = U64
        _cpu = lib
    return _cpu


def _ptr(a: np.ndarray):
    assert a.flags.c_contiguous
    return a.ctypes.data


def host_init(segs, p, i0=0, i1=None, seed=SEED) -> np.ndarray:
    i1 = segments_numel(segs) if i1 is None else i1
    out = np.empty(i1 - i0, dtype=np.float32)
    _lib_cpu().synth_fill_init(_ptr(out), _ptr(segs), len(segs), seed, p, i0, i1)
    return out


def host_apply_window(x, segs, p, m, r, i0=0, seed=SEED):
    _lib_cpu().synth_apply_window(_ptr(x), _ptr(segs), len(segs), seed, p, m, r, i0, i0 + x.size)
    return x


def host_apply_drift(x, segs, p, m, r, i0=0, seed=SEED):
    _lib_cpu().synth_apply_drift(_ptr(x), _ptr(segs), len(segs), seed, p, m, r, i0, i0 + x.size)
    return x


def host_apply_toy(x, m, t, i0=0, seed=SEED):
    _lib_cpu().synth_apply_toy(_ptr(x), seed, m, t, i0, i0 + x.size)
    return x


def host_U(key, i0, i1) -> np.ndarray:
    out = np.empty(i1 - i0, dtype=np.float32)
    _lib_cpu().synth_fill_U(_ptr(out), key, i0, i1)
    return out


def key(purpose, p, m, r, seed=SEED) -> int:
    return int(_lib_cpu().synth_key(seed, purpose, p, m, r))


def H(x) -> int:
    return int(_lib_cpu().synth_H(x))


# --------------------------------------------------------------------------- device
_cuda = None


def _lib_cuda():
    global _cuda
    if _cuda is None:
        path = os.path.join(_HERE, "libsynth_cuda.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        P, I64, I32, U64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64
        lib.synth_cuda_fill_init.argtypes = [P, P, ctypes.c_int, U64, I32, I64, I64, P]
        lib.synth_cuda_apply_window.argtypes = [P, P, ctypes.c_int, U64, I32, I32, I32, I64, I64, P]
        lib.synth_cuda_apply_drift.argtypes = [P, P, ctypes.c_int, U64, I32, I32, I32, I64, I64, P]
        lib.synth_cuda_apply_toy.argtypes = [P, U64, I32, I64, I64, I64, P]
        lib.synth_cuda_inner_adamw.argtypes = [P, P, P, I64, U64, I32, I64, P]
        lib.synth_cuda_inner_adamw.restype = ctypes.c_int
        for f in ("synth_cuda_fill_init", "synth_cuda_apply_window", "synth_cuda_apply_drift", "synth_cuda_apply_toy"):
            getattr(lib, f).restype = ctypes.c_int
        _cuda = lib
    return _cuda


def _chk(rc):
    if rc != 0:
        raise RuntimeError(f"synth CUDA launch failed: cudaError {rc}")


def _stream(stream):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def dev_init(x, segs, p, i0=0, seed=SEED, stream=None):
    """x: contiguous float32 CUDA tensor holding elements [i0, i0 + x.numel())."""
    _chk(_lib_cuda().synth_cuda_fill_init(x.data_ptr(), _ptr(segs), len(segs), seed, p, i0, i0 + x.numel(), _stream(stream)))
    return x


def dev_apply_window(x, segs, p, m, r, i0=0, seed=SEED, stream=None):
    _chk(_lib_cuda().synth_cuda_apply_window(x.data_ptr(), _ptr(segs), len(segs), seed, p, m, r, i0, i0 + x.numel(), _stream(stream)))
    return x


def dev_apply_drift(x, segs, p, m, r, i0=0, seed=SEED, stream=None):
    _chk(_lib_cuda().synth_cuda_apply_drift(x.data_ptr(), _ptr(segs), len(segs), seed, p, m, r, i0, i0 + x.numel(), _stream(stream)))
    return x


def dev_apply_toy(x, m, t, i0=0, seed=SEED, stream=None):
    _chk(_lib_cuda().synth_cuda_apply_toy(x.data_ptr(), seed, m, t, i0, i0 + x.numel(), _stream(stream)))
    return x


def dev_inner_adamw(theta, m1, m2, m, t, seed=SEED, stream=None):
    """AdamW-shaped synthetic inner step over theta (harness overlap load)."""
    _chk(_lib_cuda().synth_cuda_inner_adamw(theta.data_ptr(), m1.data_ptr(), m2.data_ptr(), theta.numel(), seed, m, t,
                                             _stream(stream)))
