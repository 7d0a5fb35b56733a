"""ctypes binding of the C-ABI (include/astra_b200.h) -> libastra_b200.so.

There is no fallback: if the library is missing or no CUDA device is present
the calls raise. Signatures mirror the header one to one.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import raise_for_status

HERE = os.path.dirname(os.path.abspath(__file__))
# (ASTRA_LIB_VARIANT=x loads libastra_b200_x.so: in-tree A/B builds for experiments)
LIB_PATH = os.path.join(HERE, "libastra_b200" + (f"_{os.environ['ASTRA_LIB_VARIANT']}" if os.environ.get("ASTRA_LIB_VARIANT") else "") + ".so")

_lib = None
_lock = threading.Lock()

p, i32, i64, u32, u64, f32, f64, sz = C.c_void_p, C.c_int, C.c_int64, C.c_uint32, C.c_uint64, C.c_float, C.c_double, C.c_size_t

_SIGS = {
    "astra_version": ([], C.c_char_p),
    "astra_last_error": ([], C.c_char_p),
    "astra_device_info": ([p, p, p], i32),
    "astra_launch_count": ([], u64),
    "astra_kernel_timing_enable": ([i32], None),
    "astra_kernel_timing": ([C.c_char_p, p, p], i32),
    "astra_set_refresh_sm_budget": ([i32], None),
    "astra_set_step_deterministic": ([i32], None),
    "astra_f32_to_bf16": ([p, p, i64, p], i32),
    "astra_refresh_workspace_size": ([i64, i64, i32, i32, i32], sz),
    "astra_refresh_topk": ([p, p, i64, i32, p, p, p, i64, i64, p, p, i32, i32, p, p, p, p, sz, p], i32),
    "astra_quantize_e4m3": ([p, i32, i64, p, p, p], i32),
    "astra_refresh_flagged": ([p, sz, i64, i64, i32, i32, i32, p, p], i32),
    "astra_merge_workspace_size": ([i64, i32], sz),
    "astra_topk_merge": ([p, i64, i32, i32, i32, p, p, p, p, sz, p], i32),
    "astra_sample_slates": ([u64, u32, u32, p, i32, p, p, p, i32, i32, p, p, i32, i32, i32, i64, i32, i32, p, p, p, p, p], i32),
    "astra_importance_split": ([p, p, i64, i32, i32, p, p, p, p], i32),
    "astra_step_workspace_size": ([i32, i32, i32, i64], sz),
    "astra_slate_step": ([p, p, p, p, p, i64, p, i64, p, i32, i32, i32, p, i32, p, p, i32, i64, i64, f64, f64, f64, f64, f64,
                          i64, p, p, p, p, p, p, sz, p], i32),
    "astra_apply_updates": ([p, i32, i64, i32, p, p, i64, f32, f32, p, p], i32),
    "astra_dense_workspace_size": ([i32], sz),
    "astra_dense_bce": ([p, i32, i32, i64, p, p, p, p, p, sz, p], i32),
    "astra_dense_sgd": ([p, p, i64, f32, f32, p], i32),
    "astra_rerank_candidates": ([p, i64, i32, p, i32, p, i32, i64, i32, p, p, p, p], i32),
    "astra_refresh_plan_j": ([i64, i64, i32, i32], i32),
    "astra_refresh_sharded_stage": ([i32, p, p, i64, i32, p, i64, i64, p, p, i32, p, p, p, p, p, p, sz, p], i32),
    "astra_gemm_f32_workspace_size": ([i64, i64, i64], sz),
    "astra_gemm_f32": ([p, i32, p, i32, i64, i64, i64, p, p, sz, p], i32),
    "astra_stream_sync": ([p], i32),
}

EXPORTED = tuple(_SIGS)


def load():
    """Load (and type) the library once; raises if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"{LIB_PATH} is not built: run `python -m paper_2409_20156_b200.build`")
            lib = C.CDLL(LIB_PATH)
            for name, (args, ret) in _SIGS.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = ret
            _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc:
        raise_for_status(rc, load().astra_last_error().decode(errors="replace"))


def launch_count() -> int:
    return int(load().astra_launch_count())


def kernel_timing_enable(on: bool = True) -> None:
    load().astra_kernel_timing_enable(1 if on else 0)


def set_refresh_sm_budget(n_sms: int) -> None:
    """Cap the SMs the refresh GEMM occupies (0 = all)."""
    load().astra_set_refresh_sm_budget(int(n_sms))


def set_step_deterministic(on: bool) -> None:
    """True: the bitwise run-to-run deterministic two-kernel step schedule;
    False (default): the single label-major pass (grad_emb summed with fp32
    reductions in arrival order)."""
    load().astra_set_step_deterministic(1 if on else 0)


def kernel_timing(name: str):
    """(total_ms, launches) of the named kernel since the last read (syncs its events)."""
    ms, n = C.c_double(0.0), C.c_int64(0)
    check(load().astra_kernel_timing(name.encode(), C.byref(ms), C.byref(n)))
    return ms.value, n.value
