"""ctypes binding of include/wavetune_gemm.h: the B200 validation GEMM family.

bf16 tcgen05 GEMMs (C = A @ B^T, A [M, K], B [N, K], C [M, N]) that the
WaveTune decision path chooses between.  torch tensors are plumbing for device
memory and streams only; every launch is one of lib/libwtgemm.so's kernels.
Importing fails loudly if the library is missing.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .capi import WtError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libwtgemm.so")
SWIZZLES = (1, 2, 4, 8)

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `make -C paper_2604_10187_b200` (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        i32p = C.POINTER(C.c_int32)
        L.wt_gemm_family_size.restype = C.c_int
        L.wt_gemm_config.argtypes = [C.c_int] + [C.POINTER(C.c_int)] * 4
        L.wt_gemm_run.argtypes = [C.c_int] * 5 + [C.c_void_p] * 4
        L.wt_gemm_time.argtypes = [C.c_int] * 5 + [C.c_void_p] * 3 + [C.c_int, C.c_int, C.POINTER(C.c_double)]
        L.wt_gemm_measure_batch.argtypes = [C.c_int] + [i32p] * 5 + [C.c_int, C.c_int, C.c_uint64,
                                                                      C.POINTER(C.c_double)]
        L.wt_gemm_fill_uniform.argtypes = [C.c_void_p, C.c_size_t, C.c_uint64, C.c_void_p]
        for f in ("wt_gemm_config", "wt_gemm_run", "wt_gemm_time", "wt_gemm_measure_batch", "wt_gemm_fill_uniform"):
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def _check(rc, what):
    if rc != 0:
        raise WtError(rc, what)


def family():
    """[(bm, bn, bk, stages)] per compiled instantiation (index = cfg id)."""
    L = lib()
    out = []
    for c in range(L.wt_gemm_family_size()):
        v = [C.c_int() for _ in range(4)]
        _check(L.wt_gemm_config(c, *[C.byref(x) for x in v]), "wt_gemm_config")
        out.append(tuple(x.value for x in v))
    return out


def _stream():
    import torch

    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _operands(a, b, c=None):
    import torch

    if a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16 or not (a.is_cuda and b.is_cuda):
        raise ValueError("A and B must be bf16 CUDA tensors")
    if a.dim() != 2 or b.dim() != 2 or a.shape[1] != b.shape[1]:
        raise ValueError("expected A [M, K] and B [N, K]")
    a, b = a.contiguous(), b.contiguous()
    M, K = a.shape
    N = b.shape[0]
    if c is None:
        c = torch.empty(M, N, dtype=torch.bfloat16, device=a.device)
    return a, b, c, M, N, K


def matmul(a, b, cfg, swizzle=1, out=None):
    """C = a @ b.T with family instantiation `cfg` on torch's current stream."""
    a, b, c, M, N, K = _operands(a, b, out)
    _check(lib().wt_gemm_run(cfg, swizzle, M, N, K, a.data_ptr(), b.data_ptr(), c.data_ptr(), _stream()),
           f"wt_gemm_run(cfg={cfg}, swizzle={swizzle}, {M}x{N}x{K})")
    return c


def time_us(a, b, cfg, swizzle=1, warmup=3, reps=10, out=None):
    """Mean device time (us) of one launch on the caller's operands."""
    a, b, c, M, N, K = _operands(a, b, out)
    us = C.c_double()
    _check(lib().wt_gemm_time(cfg, swizzle, M, N, K, a.data_ptr(), b.data_ptr(), c.data_ptr(), warmup, reps,
                              C.byref(us)), "wt_gemm_time")
    return us.value


def measure_batch(cfg, swizzle, M, N, K, warmup=3, reps=10, seed=0):
    """Batched MeasurementBackend::measure on library-owned operands; -1 where
    the instantiation cannot run the shape."""
    arrs = [np.ascontiguousarray(x, dtype=np.int32) for x in (cfg, swizzle, M, N, K)]
    n = len(arrs[0])
    out = np.empty(n, dtype=np.float64)
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))
    _check(lib().wt_gemm_measure_batch(n, *[p(a) for a in arrs], warmup, reps, seed,
                                       out.ctypes.data_as(C.POINTER(C.c_double))), "wt_gemm_measure_batch")
    return out
