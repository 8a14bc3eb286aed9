"""ctypes binding of libtexforge_cuda.so (the C ABI in include/texforge_cuda.h).

The shared object is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_1710_06189_b200/csrc``). There is deliberately NO fallback: if
the library is missing, importing the engine raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# TEXFORGE_CUDA_LIB: load another build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("TEXFORGE_CUDA_LIB") or os.path.join(_HERE, "libtexforge_cuda.so")

TFG_OK = 0
TFG_INVALID_ARGUMENT = 1
TFG_CUDA_ERROR = 2
TFG_COLLECTIVE_ERROR = 3
TFG_OUT_OF_MEMORY = 4
TFG_SOURCE_ERROR = 5

TFG_INPUT_DEVICE = 1 << 0
TFG_SYMMETRIC = 1 << 1
TFG_NORMALIZE = 1 << 2
TFG_FEATURES = 1 << 3
TFG_SCHEME_GLOBAL = 1 << 4
TFG_SEQUENTIAL = 1 << 5

TFG_STRATEGY_SHIFT = 16
STRAT_AUTO, STRAT_COPIES32, STRAT_COPIES8, STRAT_COPY1, STRAT_PACKED16, STRAT_P16X16 = range(6)


def strategy_flag(s: int) -> int:
    return (int(s) & 0xF) << TFG_STRATEGY_SHIFT


# `err` is a raw char* the callback may write into (NOT c_char_p: ctypes would
# hand Python an immutable bytes copy).
FETCH_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t,
                       C.POINTER(C.c_uint8), C.c_void_p, C.c_size_t)

# (name, restype, argtypes) for every symbol declared in include/texforge_cuda.h
_u8p = C.POINTER(C.c_uint8)
_u64p = C.POINTER(C.c_uint64)
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_sz = C.c_size_t
SIGNATURES = [
    ("tfg_ctx_create", C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_uint]),
    ("tfg_ctx_destroy", None, [C.c_void_p]),
    ("tfg_last_error", C.c_char_p, []),
    ("tfg_last_error_chunk", C.c_size_t, []),
    ("tfg_abi_version", C.c_int, []),
    ("tfg_memory_kind", C.c_int, [C.c_void_p]),
    ("tfg_launch_count", C.c_uint64, [C.c_void_p]),
    ("tfg_neighbor_offset", C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_long), C.POINTER(C.c_long)]),
    ("tfg_valid_pair_count", C.c_int, [_sz, _sz, C.c_int, C.c_int, _u64p]),
    ("tfg_partition", C.c_int, [_sz, _sz, C.c_int, C.c_int, _sz, _u64p]),
    ("tfg_plan", C.c_int, [C.c_int, _sz, C.c_uint, C.POINTER(C.c_uint), C.POINTER(C.c_uint), _ip]),
    ("tfg_synth_noise", C.c_int, [_sz, _sz, C.c_uint32, _u8p]),
    ("tfg_synth_smooth", C.c_int, [_sz, _sz, C.c_uint32, _u8p, C.c_int]),
    ("tfg_mt19937_windows", C.c_int, [C.c_uint32, C.c_uint64, C.c_uint64, _sz, C.POINTER(C.c_uint32), C.c_int]),
    ("tfg_synth_noise_parallel", C.c_int, [_sz, C.c_uint32, _u8p, C.c_int]),
    ("tfg_synth_noise_device", C.c_int, [C.c_void_p, _sz, _sz, C.c_uint32, C.c_void_p, _sz, C.c_void_p]),
    ("tfg_synth_noise_rows_device", C.c_int, [C.c_void_p, _sz, _sz, _sz, C.c_uint32, C.c_void_p, _sz, C.c_void_p]),
    ("tfg_quantize", C.c_int, [C.c_void_p, C.c_void_p, _sz, C.c_int, C.c_void_p, C.c_uint]),
    ("tfg_glcm", C.c_int, [C.c_void_p, C.c_void_p, _sz, _sz, _sz, C.c_int, C.c_int, _ip, _ip, C.c_int,
                           C.c_uint, _u64p, _dp, _dp]),
    ("tfg_glcm_bands", C.c_int, [C.c_void_p, C.c_void_p, _sz, _sz, _sz, _sz, _sz, C.c_int, C.c_int, _ip,
                                 _ip, C.c_int, C.c_uint, _u64p, _dp, _dp]),
    ("tfg_glcm_shard", C.c_int, [C.c_void_p, C.c_void_p, _sz, _sz, _sz, _sz, _sz, _sz, C.c_int, C.c_int, _ip, _ip,
                                 C.c_int, C.c_uint, _u64p]),
    ("tfg_glcm_shard_jobs", C.c_int, [C.c_void_p, C.c_void_p, _sz, _sz, _sz, _sz, _sz, C.c_int, _ip, _ip, _ip, C.c_int,
                                      C.c_uint, _u64p]),
    ("tfg_glcm_chunked", C.c_int, [C.c_void_p, _sz, _sz, C.c_int, C.c_int, _ip, _ip, C.c_int, _sz, FETCH_FN,
                                   C.c_void_p, C.c_uint, _u64p, _dp, _dp]),
    ("tfg_subglcms", C.c_int, [C.c_void_p, C.c_void_p, _sz, _sz, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint,
                               C.c_uint, _sz, C.c_uint, C.POINTER(C.c_uint32), _u64p, _u64p]),
    ("tfg_symmetrize", C.c_int, [C.c_void_p, _u64p, C.c_int, _u64p]),
    ("tfg_normalize", C.c_int, [C.c_void_p, _u64p, C.c_int, _dp]),
    ("tfg_features", C.c_int, [C.c_void_p, _dp, C.c_int, _dp]),
    ("tfg_glcm_async", C.c_int, [C.c_void_p, C.c_void_p, _sz, _sz, _sz, _sz, C.c_int, C.c_int, C.c_int,
                                 C.c_int, C.c_uint, C.c_void_p, C.c_void_p]),
    ("tfg_glcm_bands_async", C.c_int, [C.c_void_p, C.c_void_p, _sz, _sz, _sz, _sz, _sz, C.c_int, C.c_int, C.c_int,
                                       C.c_int, C.c_uint, C.c_void_p, C.c_void_p]),
    ("tfg_glcm_multi_async", C.c_int, [C.c_void_p, C.c_void_p, _sz, _sz, _sz, _sz, _sz, _sz, C.c_int, C.c_int, _ip,
                                       _ip, C.c_int, C.c_uint, C.c_void_p, C.c_void_p]),
    ("tfg_glcm_jobs_async", C.c_int, [C.c_void_p, C.c_void_p, _sz, _sz, _sz, _sz, _sz, _sz, C.c_int, _ip, _ip, _ip,
                                      C.c_int, C.c_uint, C.c_void_p, C.c_void_p]),
    ("tfg_post_async", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_uint, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_void_p]),
    ("tfg_check_async_errors", C.c_int, [C.c_void_p]),
    # multi-GPU (tfg_multi_gpu.inc)
    ("tfg_group_create", C.c_int, [C.POINTER(C.c_void_p), C.c_int, _ip, C.c_uint]),
    ("tfg_group_destroy", None, [C.c_void_p]),
    ("tfg_group_size", C.c_int, [C.c_void_p]),
    ("tfg_group_ctx", C.c_void_p, [C.c_void_p, C.c_int]),
    ("tfg_group_launch_count", C.c_uint64, [C.c_void_p]),
    ("tfg_group_glcm", C.c_int, [C.c_void_p, C.c_void_p, _sz, _sz, C.c_int, C.c_int, _ip, _ip, C.c_int, C.c_uint,
                                 _u64p, _dp, _dp]),
    ("tfg_group_glcm_bands", C.c_int, [C.c_void_p, C.c_void_p, _sz, _sz, _sz, _sz, C.c_int, C.c_int, _ip, _ip,
                                       C.c_int, C.c_uint, _u64p, _dp, _dp]),
    ("tfg_group_glcm_chunked", C.c_int, [C.c_void_p, _sz, _sz, C.c_int, C.c_int, _ip, _ip, C.c_int, _sz, FETCH_FN,
                                         C.c_void_p, C.c_uint, _u64p, _dp, _dp]),
    ("tfg_comm_unique_id", C.c_int, [C.c_void_p]),
    ("tfg_comm_init_rank", C.c_int, [C.POINTER(C.c_void_p), C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    ("tfg_comm_destroy", None, [C.c_void_p]),
    ("tfg_comm_reduce_counts", C.c_int, [C.c_void_p, C.c_void_p, _sz, C.c_int, C.c_void_p]),
    ("tfg_comm_exchange_halo", C.c_int, [C.c_void_p, C.c_void_p, _sz, _sz, _sz, C.c_void_p]),
    ("tfg_comm_allreduce_max_f64", C.c_int, [C.c_void_p, C.c_void_p, _sz, C.c_void_p]),
]
TFG_GROUP_HOST_REDUCE = 1
TFG_COMM_ID_BYTES = 128

_lib = None


def _prefer_torch_nccl() -> None:
    """The library dlopens NCCL on its first multi-GPU call (csrc/tfg_nccl_dl.h).
    In a Python process that NCCL must be torch's bundled copy: one process
    keeps the first libnccl.so.2 it maps, and libtorch_cuda needs its own."""
    if os.environ.get("TEXFORGE_NCCL_LIB"):
        return
    import importlib.util
    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        spec = None
    for d in (spec.submodule_search_locations if spec else None) or []:
        p = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(p):
            os.environ["TEXFORGE_NCCL_LIB"] = p
            return


def load() -> C.CDLL:
    """Loads the in-tree engine library; raises if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"libtexforge_cuda.so not found at {LIB_PATH}: run __graft_entry__.build() "
                "(there is no CPU fallback)")
        _prefer_torch_nccl()
        lib = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class TfgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def check(rc: int) -> None:
    if rc != TFG_OK:
        lib = load()
        msg = lib.tfg_last_error().decode(errors="replace")
        if rc == TFG_INVALID_ARGUMENT:
            raise ValueError(msg)
        raise TfgError(rc, msg)
