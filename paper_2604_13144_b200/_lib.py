"""ctypes binding of ``libtepai_b200.so`` (the C ABI declared in
``include/tepai_b200.h``).  There is no CPU fallback: every engine entry point
raises if the library is missing or no CUDA device can be bound."""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

LIB_NAME = "libtepai_b200.so"
LIB_PATH = os.environ.get("TB_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

EXPORTED = (
    "tb_version", "tb_create", "tb_destroy", "tb_last_error", "tb_num_sms", "tb_num_ctas", "tb_take_status", "tb_debug_profile",
    "tb_run_stream",
    "tb_expectation", "tb_expectation_batch", "tb_svd", "tb_svd_trunc", "tb_run_ensemble", "tb_run_ensemble_device", "tb_step", "tb_step_device",
)

_c_i64p = ctypes.POINTER(ctypes.c_int64)
_c_dp = ctypes.POINTER(ctypes.c_double)


class EnsembleDesc(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int32), ("cap", ctypes.c_int32), ("chi_cut", ctypes.c_int32), ("pi_local", ctypes.c_int32),
        ("svalue_floor", ctypes.c_double),
        ("n_samples", ctypes.c_int32), ("n_ckpt", ctypes.c_int32), ("n_obs", ctypes.c_int32),
        ("n_angles", ctypes.c_int32),
        ("gates", ctypes.c_void_p), ("gate_offsets", ctypes.c_void_p), ("ckpt_gate_end", ctypes.c_void_p),
        ("ckpt_sign", ctypes.c_void_p), ("angle_cs", ctypes.c_void_p), ("ckpt_weight", ctypes.c_void_p),
        ("obs_sites", ctypes.c_void_p), ("init_vecs", ctypes.c_void_p),
        ("init_mps", ctypes.c_void_p), ("init_dims", ctypes.c_void_p), ("init_center", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


class EnsembleOut(ctypes.Structure):
    _fields_ = [
        ("values", ctypes.c_void_p), ("discarded", ctypes.c_void_p), ("ledger", ctypes.c_void_p),
        ("sum_v", ctypes.c_void_p), ("sum_v2", ctypes.c_void_p), ("flops", ctypes.c_void_p),
        ("kernel_ms", ctypes.c_void_p), ("excluded", ctypes.c_void_p), ("states", ctypes.c_void_p),
        ("state_dims", ctypes.c_void_p), ("state_center", ctypes.c_void_p), ("sample_ms", ctypes.c_void_p),
    ]


class StepDesc(ctypes.Structure):
    _fields_ = [("base", EnsembleDesc), ("reset", ctypes.c_void_p), ("sum_row", ctypes.c_void_p),
                ("order", ctypes.c_void_p)]


_lock = threading.Lock()
_lib = None
_ctxs: dict[int, ctypes.c_void_p] = {}


def load() -> ctypes.CDLL:
    """Load the in-tree shared library (raises if it has not been built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_NAME} is not built (run __graft_entry__.build()); no CPU fallback exists")
        lib = ctypes.CDLL(LIB_PATH)
        vp, i64, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double
        lib.tb_version.restype = ctypes.c_int
        lib.tb_create.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
        lib.tb_destroy.argtypes = [vp]
        lib.tb_destroy.restype = None
        lib.tb_last_error.argtypes = [vp]
        lib.tb_last_error.restype = ctypes.c_char_p
        lib.tb_num_sms.argtypes = [vp]
        lib.tb_num_ctas.argtypes = [vp, i64]
        lib.tb_debug_profile.argtypes = [vp, vp]
        lib.tb_take_status.argtypes = [vp, vp]
        lib.tb_run_stream.argtypes = [vp, vp, i64, i64, vp, i64, vp, vp, vp, vp, vp, vp, i64, i64, dbl, vp, vp]
        lib.tb_expectation.argtypes = [vp, vp, i64, i64, vp, vp, vp]
        lib.tb_expectation_batch.argtypes = [vp, vp, i64, i64, i64, vp, vp, i64, vp]
        lib.tb_svd.argtypes = [vp, vp, i64, i64, i64, vp, vp, vp]
        if hasattr(lib, "tb_svd_trunc"):  # absent in pre-r01b builds (A/B timing of old libraries)
            lib.tb_svd_trunc.argtypes = [vp, vp, i64, i64, i64, i64, vp, vp, vp]
        lib.tb_run_ensemble.argtypes = [vp, ctypes.POINTER(EnsembleDesc), ctypes.POINTER(EnsembleOut)]
        lib.tb_run_ensemble_device.argtypes = [vp, ctypes.POINTER(EnsembleDesc), ctypes.POINTER(EnsembleOut), vp]
        lib.tb_step.argtypes = [vp, ctypes.POINTER(StepDesc), ctypes.POINTER(EnsembleOut), i64]
        lib.tb_step_device.argtypes = [vp, ctypes.POINTER(StepDesc), ctypes.POINTER(EnsembleOut), vp]
        _lib = lib
        return lib


def context(device: int = 0) -> ctypes.c_void_p:
    """Per-(process, device) engine context, created on first use."""
    lib = load()
    with _lock:
        ctx = _ctxs.get(device)
        if ctx is None:
            ctx = ctypes.c_void_p()
            rc = lib.tb_create(int(device), ctypes.byref(ctx))
            if rc != 0 or not ctx.value:
                raise RuntimeError(f"tb_create(device={device}) failed ({rc}): no usable CUDA device for the B200 engine")
            _ctxs[device] = ctx
        return ctx


class PrivateContext:
    """An engine context owned by one object (a ``SlotPipeline``): its slot
    pool is never touched by any other engine call.  Destroyed with its owner."""

    def __init__(self, device: int = 0):
        lib = load()
        self.ctx = ctypes.c_void_p()
        rc = lib.tb_create(int(device), ctypes.byref(self.ctx))
        if rc != 0 or not self.ctx.value:
            raise RuntimeError(f"tb_create(device={device}) failed ({rc}): no usable CUDA device for the B200 engine")

    def close(self) -> None:
        if self.ctx is not None and self.ctx.value:
            load().tb_destroy(self.ctx)
        self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def take_status(ctx) -> int:
    """Read and clear the sticky device status word (see tb_take_status)."""
    st = ctypes.c_int32(0)
    check(load().tb_take_status(ctx, ctypes.byref(st)), ctx)
    return int(st.value)


def check(rc: int, ctx) -> None:
    if rc == 0:
        return
    msg = load().tb_last_error(ctx).decode(errors="replace")
    if rc == -1:
        raise ValueError(msg)
    raise RuntimeError(f"tepai_b200 error {rc}: {msg}")


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a is not None else None


def debug_profile(device: int = 0, ctx=None) -> np.ndarray:
    """Phase cycle counters of the last ensemble launch (see tb_debug_profile;
    collected only when TB_PROFILE=1 was set before the context was created)."""
    out = np.zeros(64, np.uint64)
    ctx = ctx if ctx is not None else context(device)
    check(load().tb_debug_profile(ctx, out.ctypes.data), ctx)
    return out
