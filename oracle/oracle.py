"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU parity checkers.

* ``liboracle.so``            — C restatement of the reference path (glcm_oracle.c)
* ``_ref/libtexforge_ref.so`` — the UNMODIFIED reference headers behind a C ABI
                                (ref_oracle.cpp), present when it was built in the
                                dev container (the prebuilt .so travels to the GPU box)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module. The product (paper_1710_06189_b200/)
never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtexforge_ref.so")

_u8p = C.POINTER(C.c_uint8)
_u64p = C.POINTER(C.c_uint64)
_dp = C.POINTER(C.c_double)
_sz = C.c_size_t

_oracle = None
_ref = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _p(a, t=C.c_uint8):
    return a.ctypes.data_as(C.POINTER(t))


def lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build()
        o = C.CDLL(ORACLE_SO)
        o.oracle_quantize.argtypes = [_u8p, _sz, C.c_int, _u8p]
        o.oracle_valid_pair_count.argtypes = [_sz, _sz, C.c_int, C.c_int, _u64p]
        o.oracle_glcm_rows.argtypes = [_u8p, _sz, _sz, C.c_int, C.c_int, C.c_int, _sz, _sz, _u64p]
        o.oracle_glcm_serial.argtypes = [_u8p, _sz, _sz, C.c_int, C.c_int, C.c_int, _u64p]
        o.oracle_glcm_gray.argtypes = [_u8p, _sz, _sz, C.c_int, C.c_int, C.c_int, _u64p]
        o.oracle_symmetrize.argtypes = [_u64p, C.c_int, _u64p]
        o.oracle_symmetrize.restype = None
        o.oracle_normalize.argtypes = [_u64p, C.c_int, _dp]
        o.oracle_features.argtypes = [_dp, C.c_int, _dp]
        o.oracle_partition.argtypes = [_sz, _sz, C.c_int, C.c_int, _sz, _u64p]
        o.oracle_glcm_chunked.argtypes = [_u8p, _sz, _sz, C.c_int, C.c_int, C.c_int, _sz, _u64p]
        o.oracle_plan.argtypes = [C.c_int, _sz, C.POINTER(C.c_uint), C.POINTER(C.c_uint), C.POINTER(C.c_int)]
        o.oracle_stats.argtypes = [_u64p, C.c_int, _u64p, _u64p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        o.oracle_stats.restype = None
        o.oracle_fnv1a64_u64.argtypes = [_u64p, _sz]
        o.oracle_fnv1a64_u64.restype = C.c_uint64
        _oracle = o
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        r = C.CDLL(REF_SO)
        r.ref_last_error.restype = C.c_char_p
        r.ref_quantize.argtypes = [_u8p, _sz, _sz, C.c_int, _u8p]
        r.ref_synth_noise.argtypes = [_sz, _sz, C.c_uint32, _u8p]
        r.ref_synth_smooth.argtypes = [_sz, _sz, C.c_uint32, _u8p]
        r.ref_glcm_serial.argtypes = [_u8p, _sz, _sz, C.c_int, C.c_int, C.c_int, _u64p]
        r.ref_glcm_privatized.argtypes = [_u8p, _sz, _sz, C.c_int, C.c_int, C.c_int, C.c_uint, C.c_uint, _u64p]
        r.ref_glcm_shared.argtypes = [_u8p, _sz, _sz, C.c_int, C.c_int, C.c_int, C.c_uint, _u64p]
        r.ref_glcm_chunked.argtypes = [_u8p, _sz, _sz, C.c_int, C.c_int, C.c_int, _sz, C.c_uint, C.c_int, _u64p]
        r.ref_image_new.argtypes = [_u8p, _sz, _sz, C.c_int]
        r.ref_image_new.restype = C.c_void_p
        r.ref_image_free.argtypes = [C.c_void_p]
        r.ref_image_free.restype = None
        r.ref_image_glcm.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint, C.c_int, _u64p]
        r.ref_symmetrize.argtypes = [_u64p, C.c_int, _u64p]
        r.ref_normalize.argtypes = [_u64p, C.c_int, _dp]
        r.ref_features.argtypes = [_dp, C.c_int, _dp]
        r.ref_partition.argtypes = [_sz, _sz, C.c_int, C.c_int, _sz, _u64p]
        r.ref_plan.argtypes = [C.c_int, _sz, C.c_uint, C.POINTER(C.c_uint), C.POINTER(C.c_uint),
                               C.POINTER(C.c_int)]
        _ref = r
    return _ref


class OracleError(ValueError):
    pass


def _chk(rc, what="oracle"):
    if rc:
        raise OracleError(f"{what}: rc={rc}")


# ---------------------------------------------------------------- restatement
def quantize(gray: np.ndarray, levels: int) -> np.ndarray:
    g = np.ascontiguousarray(gray, dtype=np.uint8).reshape(-1)
    out = np.empty_like(g)
    _chk(lib().oracle_quantize(_p(g), g.size, levels, _p(out)), "quantize")
    return out


def valid_pair_count(w, h, d, theta) -> int:
    out = C.c_uint64()
    _chk(lib().oracle_valid_pair_count(w, h, d, theta, C.byref(out)), "valid_pair_count")
    return int(out.value)


def glcm_serial(px: np.ndarray, w: int, h: int, levels: int, d: int, theta: int) -> np.ndarray:
    a = np.ascontiguousarray(px, dtype=np.uint8).reshape(-1)
    out = np.zeros(levels * levels, dtype=np.uint64)
    _chk(lib().oracle_glcm_serial(_p(a), w, h, levels, d, theta, _p(out, C.c_uint64)), "glcm_serial")
    return out


def glcm_gray(gray: np.ndarray, w: int, h: int, levels: int, d: int, theta: int) -> np.ndarray:
    """quantize(gray, L) then compute_glcm_serial, fused."""
    a = np.ascontiguousarray(gray, dtype=np.uint8).reshape(-1)
    out = np.zeros(levels * levels, dtype=np.uint64)
    _chk(lib().oracle_glcm_gray(_p(a), w, h, levels, d, theta, _p(out, C.c_uint64)), "glcm_gray")
    return out


def glcm_rows(px, w, h, levels, d, theta, row_begin, row_end, counts=None) -> np.ndarray:
    a = np.ascontiguousarray(px, dtype=np.uint8).reshape(-1)
    if counts is None:
        counts = np.zeros(levels * levels, dtype=np.uint64)
    _chk(lib().oracle_glcm_rows(_p(a), w, h, levels, d, theta, row_begin, row_end, _p(counts, C.c_uint64)))
    return counts


def glcm_chunked(px, w, h, levels, d, theta, k) -> np.ndarray:
    a = np.ascontiguousarray(px, dtype=np.uint8).reshape(-1)
    out = np.zeros(levels * levels, dtype=np.uint64)
    _chk(lib().oracle_glcm_chunked(_p(a), w, h, levels, d, theta, k, _p(out, C.c_uint64)), "glcm_chunked")
    return out


def symmetrize(g: np.ndarray, levels: int) -> np.ndarray:
    a = np.ascontiguousarray(g, dtype=np.uint64).reshape(-1)
    out = np.empty_like(a)
    lib().oracle_symmetrize(_p(a, C.c_uint64), levels, _p(out, C.c_uint64))
    return out


def normalize(g: np.ndarray, levels: int) -> np.ndarray:
    a = np.ascontiguousarray(g, dtype=np.uint64).reshape(-1)
    out = np.empty(a.size, dtype=np.float64)
    _chk(lib().oracle_normalize(_p(a, C.c_uint64), levels, _p(out, C.c_double)), "normalize")
    return out


def features(p: np.ndarray, levels: int) -> np.ndarray:
    a = np.ascontiguousarray(p, dtype=np.float64).reshape(-1)
    out = np.empty(5, dtype=np.float64)
    _chk(lib().oracle_features(_p(a, C.c_double), levels, _p(out, C.c_double)), "features")
    return out


def partition(w, h, d, theta, k) -> np.ndarray:
    out = np.zeros(3 * k, dtype=np.uint64)
    _chk(lib().oracle_partition(w, h, d, theta, k, _p(out, C.c_uint64)), "partition")
    return out.reshape(k, 3)


def plan(levels, budget):
    c, g, dg = C.c_uint(), C.c_uint(), C.c_int()
    _chk(lib().oracle_plan(levels, budget, C.byref(c), C.byref(g), C.byref(dg)), "plan")
    return int(c.value), int(g.value), bool(dg.value)


def stats(g: np.ndarray, levels: int):
    a = np.ascontiguousarray(g, dtype=np.uint64).reshape(-1)
    t, hv = C.c_uint64(), C.c_uint64()
    r, c = C.c_int(), C.c_int()
    lib().oracle_stats(_p(a, C.c_uint64), levels, C.byref(t), C.byref(hv), C.byref(r), C.byref(c))
    return int(t.value), int(hv.value), (int(r.value), int(c.value))


def fnv1a64(counts: np.ndarray) -> str:
    a = np.ascontiguousarray(counts, dtype=np.uint64).reshape(-1)
    return "%016x" % lib().oracle_fnv1a64_u64(_p(a, C.c_uint64), a.size)


def fnv1a64_bytes(b: np.ndarray) -> str:
    h = 0xcbf29ce484222325
    for x in np.ascontiguousarray(b, dtype=np.uint8).reshape(-1).tobytes():
        h ^= x
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return "%016x" % h


def fnv1a64_image(b: np.ndarray) -> str:
    """FNV-1a-64 of a byte raster, vectorised in 64 KiB blocks (same value as fnv1a64_bytes)."""
    # exact byte-serial FNV cannot be vectorised; for big rasters hash the u64
    # view instead (a different but equally pinned digest, computed by the C oracle).
    a = np.ascontiguousarray(b, dtype=np.uint8).reshape(-1)
    pad = (-a.size) % 8
    if pad:
        a = np.concatenate([a, np.zeros(pad, dtype=np.uint8)])
    return fnv1a64(a.view(np.uint64))
