"""Thin ctypes binding of libsd (include/sd.h), same names as the C ABI.

Argument marshalling only: every step of the method runs in libsd's CUDA
kernels (csrc/sd_kernels.cu) and NCCL.  There is no CPU fallback: if the
shared library or a CUDA device is missing, the calls raise.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SD_LIBSD") or os.path.join(_HERE, "libsd.so")  # override: experiments only

SD_ABI_VERSION = 1
SD_UNIQUE_ID_BYTES = 128
SD_PAYLOAD_MAGIC = 0x31304453
SD_GATHER_COPY_ENGINE, SD_GATHER_PUSH, SD_GATHER_AUTO, SD_GATHER_PULL = 0, 1, 2, 3

SD_OK, SD_ERR_ARG, SD_ERR_CONFIG, SD_ERR_SCHEDULE, SD_ERR_STATE, SD_ERR_NONFINITE, SD_ERR_CUDA, SD_ERR_NCCL = range(8)
STATUS_NAMES = {
    0: "SD_OK", 1: "SD_ERR_ARG", 2: "SD_ERR_CONFIG", 3: "SD_ERR_SCHEDULE", 4: "SD_ERR_STATE",
    5: "SD_ERR_NONFINITE", 6: "SD_ERR_CUDA", 7: "SD_ERR_NCCL",
}

# every symbol include/sd.h declares (tests check the library exports all of them)
EXPORTS = (
    "sd_config_default", "sd_config_validate", "sd_fragment_count", "sd_fragment_layout",
    "sd_fragment_schedule", "sd_num_scale_blocks", "sd_payload_bytes", "sd_payload_scales_offset",
    "sd_payload_trailer_offset", "sd_get_unique_id", "sd_init", "sd_gather_alloc", "sd_gather_free", "sd_set_gather_mode",
    "sd_gather_payloads",
    "sd_quantize_workspace_bytes", "sd_set_workspace", "sd_outer_state_init", "sd_state_prefetch", "sd_state_writeback", "sd_state_sync", "sd_comm_stream",
    "sd_inner_adamw", "sd_inner_adamw_quantize", "sd_inner_adamw_merge", "sd_outer_grad_quantize", "sd_fragment_sync", "sd_fragment_wait", "sd_merge", "sd_check", "sd_last_error",
    "sd_finalize", "sd_kernel_launch_count",
)


class SdConfig(ctypes.Structure):
    _fields_ = [
        ("abi_version", ctypes.c_uint32), ("num_blocks", ctypes.c_int32), ("fragment_size", ctypes.c_int32),
        ("pattern", ctypes.c_int32), ("embed_policy", ctypes.c_int32), ("H", ctypes.c_int32),
        ("tau", ctypes.c_int32), ("T", ctypes.c_int64), ("alpha", ctypes.c_float), ("outer_lr", ctypes.c_float),
        ("outer_momentum", ctypes.c_float), ("scale_block", ctypes.c_int32),
    ]


class SdAdamW(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_float), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float), ("eps", ctypes.c_float),
                ("weight_decay", ctypes.c_float)]


class SdError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.msg = msg


_lib = None


def lib():
    """Loads libsd.so (in-tree build); raises if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() (no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P, I32, I64, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
        C = ctypes.POINTER(SdConfig)
        pI32, pI64 = ctypes.POINTER(I32), ctypes.POINTER(I64)
        sig = {
            "sd_config_default": ([C, I32, I32, I32], I32),
            "sd_config_validate": ([C, ctypes.c_char_p, SZ], I32),
            "sd_fragment_count": ([C, pI32], I32),
            "sd_fragment_layout": ([C, I32, pI32, I32, pI32, pI32, pI32], I32),
            "sd_fragment_schedule": ([C, I64, pI32, pI32, pI32, pI32, I32], I32),
            "sd_num_scale_blocks": ([C, I64], I64),
            "sd_payload_bytes": ([C, I64], SZ),
            "sd_payload_scales_offset": ([I64], SZ),
            "sd_payload_trailer_offset": ([C, I64], SZ),
            "sd_get_unique_id": ([P], I32),
            "sd_init": ([ctypes.POINTER(P), C, I32, I32, P, I32], I32),
            "sd_gather_alloc": ([P, I64, ctypes.POINTER(P)], I32),
            "sd_gather_free": ([P, P], I32),
            "sd_set_gather_mode": ([P, I32], I32),
            "sd_gather_payloads": ([P, I32, P, ctypes.POINTER(P)], I32),
            "sd_quantize_workspace_bytes": ([C, I64], SZ),
            "sd_set_workspace": ([P, P, SZ], I32),
            "sd_outer_state_init": ([P, P, P, P, I64, P], I32),
            "sd_state_prefetch": ([P, I32, P, P, P, P, I64, P], I32),
            "sd_state_writeback": ([P, I32, P, P, P, P, I64, P], I32),
            "sd_state_sync": ([P, P], I32),
            "sd_comm_stream": ([P, ctypes.POINTER(P)], I32),
            "sd_outer_grad_quantize": ([P, I32, I64, P, P, I64, P, P], I32),
            "sd_inner_adamw": ([P, I64, P, P, P, P, I64, ctypes.POINTER(SdAdamW), P], I32),
            "sd_inner_adamw_quantize": ([P, I32, I64, I64, P, P, P, P, P, I64, P, ctypes.POINTER(SdAdamW), P], I32),
            "sd_fragment_sync": ([P, I32, I64, P, I64, P], I32),
            "sd_fragment_wait": ([P, I32, I64, P], I32),
            "sd_merge": ([P, I32, I64, P, P, P, P, I64, P], I32),
            "sd_inner_adamw_merge": ([P, I32, I64, I64, P, P, P, P, P, P, P, I64, ctypes.POINTER(SdAdamW), P], I32),
            "sd_check": ([P, pI64], I32),
            "sd_last_error": ([P], ctypes.c_char_p),
            "sd_finalize": ([P], I32),
            "sd_kernel_launch_count": ([], ctypes.c_uint64),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def _err(ctx=None) -> str:
    m = lib().sd_last_error(ctx)
    return m.decode() if m else ""


def _check(st: int, ctx=None):
    if st != SD_OK:
        raise SdError(st, _err(ctx))


# ---- host-only -------------------------------------------------------------
def sd_config_default(num_blocks: int, fragment_size: int, H: int, **overrides) -> SdConfig:
    c = SdConfig()
    _check(lib().sd_config_default(ctypes.byref(c), num_blocks, fragment_size, H))
    for k, v in overrides.items():
        if not hasattr(c, k):
            raise AttributeError(f"sd_config has no field {k}")
        setattr(c, k, v)
    return c


def sd_config_validate(cfg: SdConfig):
    """-> (status, message)"""
    buf = ctypes.create_string_buffer(512)
    st = lib().sd_config_validate(ctypes.byref(cfg), buf, 512)
    return st, buf.value.decode()


def sd_fragment_count(cfg: SdConfig) -> int:
    P = ctypes.c_int32(0)
    _check(lib().sd_fragment_count(ctypes.byref(cfg), ctypes.byref(P)))
    return P.value


def sd_fragment_layout(cfg: SdConfig, p: int):
    """-> (blocks list, t_p, holds_embed)"""
    cap = max(cfg.fragment_size, 1)
    blocks = (ctypes.c_int32 * cap)()
    nb, tp, he = ctypes.c_int32(0), ctypes.c_int32(0), ctypes.c_int32(0)
    _check(lib().sd_fragment_layout(ctypes.byref(cfg), p, blocks, cap, ctypes.byref(nb), ctypes.byref(tp), ctypes.byref(he)))
    return [blocks[i] for i in range(nb.value)], tp.value, bool(he.value)


def sd_fragment_schedule(cfg: SdConfig, t: int):
    """-> (send list, receive list) at step t"""
    cap = sd_fragment_count(cfg)
    s, r = (ctypes.c_int32 * cap)(), (ctypes.c_int32 * cap)()
    ns, nr = ctypes.c_int32(0), ctypes.c_int32(0)
    _check(lib().sd_fragment_schedule(ctypes.byref(cfg), t, s, ctypes.byref(ns), r, ctypes.byref(nr), cap))
    return [s[i] for i in range(ns.value)], [r[i] for i in range(nr.value)]


def sd_num_scale_blocks(cfg: SdConfig, n: int) -> int:
    return lib().sd_num_scale_blocks(ctypes.byref(cfg), n)


def sd_payload_bytes(cfg: SdConfig, n: int) -> int:
    b = lib().sd_payload_bytes(ctypes.byref(cfg), n)
    if b == 0:
        raise SdError(SD_ERR_CONFIG, _err())
    return b


def sd_payload_scales_offset(n: int) -> int:
    return lib().sd_payload_scales_offset(n)


def sd_payload_trailer_offset(cfg: SdConfig, n: int) -> int:
    return lib().sd_payload_trailer_offset(ctypes.byref(cfg), n)


def sd_quantize_workspace_bytes(cfg: SdConfig, n: int) -> int:
    return lib().sd_quantize_workspace_bytes(ctypes.byref(cfg), n)


def sd_kernel_launch_count() -> int:
    return lib().sd_kernel_launch_count()


# ---- device ----------------------------------------------------------------
def sd_get_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * SD_UNIQUE_ID_BYTES)()
    _check(lib().sd_get_unique_id(buf))
    return bytes(buf)


def _ptr(t):
    """device pointer of a torch tensor (or an int address)"""
    return ctypes.c_void_p(t if isinstance(t, int) else t.data_ptr())


def _stream(stream):
    if stream is None:
        import torch

        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream if isinstance(stream, int) else stream.cuda_stream)


class _CudaBytes:
    """__cuda_array_interface__ view of raw device memory (libsd-owned)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3,
                                         "strides": None}


def _device_bytes(ptr: int, nbytes: int, device: int):
    import torch

    with torch.cuda.device(device):
        return torch.as_tensor(_CudaBytes(ptr, nbytes), device=torch.device("cuda", device))


class SdContext:
    """One replica's libsd context (sd_init ... sd_finalize)."""

    def __init__(self, cfg: SdConfig, rank: int, M: int, unique_id: bytes | None, device: int):
        self.cfg = cfg
        self.rank, self.M, self.device = rank, M, device
        h = ctypes.c_void_p()
        idbuf = None
        if unique_id is not None:
            idbuf = (ctypes.c_uint8 * SD_UNIQUE_ID_BYTES).from_buffer_copy(unique_id)
        _check(lib().sd_init(ctypes.byref(h), ctypes.byref(cfg), rank, M, idbuf, device))
        self.h = h

    def _c(self, st):
        _check(st, self.h)

    def sd_gather_alloc(self, n: int, device=None):
        """-> uint8 torch tensor view (M payloads) of a libsd-owned gather buffer"""
        ptr = ctypes.c_void_p()
        self._c(lib().sd_gather_alloc(self.h, n, ctypes.byref(ptr)))
        nbytes = self.M * sd_payload_bytes(self.cfg, n)
        return _device_bytes(ptr.value, nbytes, self.device if device is None else device)

    def sd_set_gather_mode(self, mode: int):
        self._c(lib().sd_set_gather_mode(self.h, mode))

    def sd_gather_payloads(self, p, buf, n):
        """-> uint8 view of the M payloads of fragment p's most recent round"""
        out = ctypes.c_void_p()
        self._c(lib().sd_gather_payloads(self.h, p, _ptr(buf), ctypes.byref(out)))
        return _device_bytes(out.value, self.M * sd_payload_bytes(self.cfg, n), self.device)

    def sd_gather_free(self, buf):
        self._c(lib().sd_gather_free(self.h, _ptr(buf)))

    def sd_state_prefetch(self, p, anchor_host, momentum_host, anchor, momentum, n=None, stream=None):
        n = anchor.numel() if n is None else n
        self._c(lib().sd_state_prefetch(self.h, p, _ptr(anchor_host), _ptr(momentum_host), _ptr(anchor),
                                        _ptr(momentum), n, _stream(stream)))

    def sd_state_writeback(self, p, anchor, momentum, anchor_host, momentum_host, n=None, stream=None):
        n = anchor.numel() if n is None else n
        self._c(lib().sd_state_writeback(self.h, p, _ptr(anchor), _ptr(momentum), _ptr(anchor_host),
                                         _ptr(momentum_host), n, _stream(stream)))

    def sd_state_sync(self, stream=None):
        self._c(lib().sd_state_sync(self.h, _stream(stream)))

    def sd_comm_stream(self) -> int:
        """cudaStream_t handle (int) of the ctx's comm stream, for tracing (torch.cuda.ExternalStream)."""
        out = ctypes.c_void_p(0)
        self._c(lib().sd_comm_stream(self.h, ctypes.byref(out)))
        return out.value or 0

    def sd_set_workspace(self, ws, nbytes=None):
        """ws: a device tensor (or None to detach); the ctx keeps a reference while attached"""
        if ws is None:
            self._ws = None
            self._c(lib().sd_set_workspace(self.h, None, 0))
            return
        nbytes = ws.numel() * ws.element_size() if nbytes is None else nbytes
        self._c(lib().sd_set_workspace(self.h, _ptr(ws), nbytes))
        self._ws = ws

    def sd_outer_state_init(self, theta, anchor, momentum, n=None, stream=None):
        n = theta.numel() if n is None else n
        self._c(lib().sd_outer_state_init(self.h, _ptr(theta), _ptr(anchor), _ptr(momentum), n, _stream(stream)))

    def sd_outer_grad_quantize(self, p, t, theta, anchor, slot_out, n=None, stream=None):
        n = theta.numel() if n is None else n
        self._c(lib().sd_outer_grad_quantize(self.h, p, t, _ptr(theta), _ptr(anchor), n, _ptr(slot_out), _stream(stream)))

    def sd_inner_adamw(self, k, theta, grad, m, v, hp: SdAdamW, n=None, stream=None):
        n = theta.numel() if n is None else n
        self._c(lib().sd_inner_adamw(self.h, k, _ptr(theta), _ptr(grad), _ptr(m), _ptr(v), n, ctypes.byref(hp),
                                     _stream(stream)))

    def sd_inner_adamw_quantize(self, p, t, k, theta, grad, m, v, anchor, slot_out, hp: SdAdamW, n=None, stream=None):
        n = theta.numel() if n is None else n
        self._c(lib().sd_inner_adamw_quantize(self.h, p, t, k, _ptr(theta), _ptr(grad), _ptr(m), _ptr(v),
                                              _ptr(anchor), n, _ptr(slot_out), ctypes.byref(hp), _stream(stream)))

    def sd_fragment_sync(self, p, t, gather_buf, n, stream=None):
        self._c(lib().sd_fragment_sync(self.h, p, t, _ptr(gather_buf), n, _stream(stream)))

    def sd_fragment_wait(self, p, t, stream=None):
        self._c(lib().sd_fragment_wait(self.h, p, t, _stream(stream)))

    def sd_merge(self, p, t, gather_buf, theta, anchor, momentum, n=None, stream=None):
        n = theta.numel() if n is None else n
        self._c(lib().sd_merge(self.h, p, t, _ptr(gather_buf), _ptr(theta), _ptr(anchor), _ptr(momentum), n, _stream(stream)))

    def sd_inner_adamw_merge(self, p, t, k, theta, grad, m, v, gather_buf, anchor, momentum, hp: SdAdamW, n=None,
                             stream=None):
        n = theta.numel() if n is None else n
        self._c(lib().sd_inner_adamw_merge(self.h, p, t, k, _ptr(theta), _ptr(grad), _ptr(m), _ptr(v),
                                           _ptr(gather_buf), _ptr(anchor), _ptr(momentum), n, ctypes.byref(hp),
                                           _stream(stream)))

    def sd_check(self):
        """-> (status, first_bad_index); does not raise on SD_ERR_NONFINITE"""
        fb = ctypes.c_int64(-1)
        st = lib().sd_check(self.h, ctypes.byref(fb))
        if st not in (SD_OK, SD_ERR_NONFINITE):
            _check(st, self.h)
        return st, fb.value

    def sd_last_error(self) -> str:
        return _err(self.h)

    def sd_finalize(self):
        if self.h:
            lib().sd_finalize(self.h)
            self.h = None

    def __del__(self):
        try:
            self.sd_finalize()
        except Exception:
            pass
