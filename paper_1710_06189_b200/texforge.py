"""Python mirror of the reference's ``texforge`` API, backed by the B200 engine.

Names, argument meaning and error behaviour follow the reference's C++ headers
(R/ = /root/reference/proj/include/texforge/): ``std::invalid_argument``
becomes ``ValueError`` with the same message text, ``PipelineError`` keeps its
``chunk_index``.  Every GLCM-producing call runs on the GPU through
libtexforge_cuda.so (include/texforge_cuda.h); there is no CPU fallback.

Small host-side pieces that the reference also keeps on the host and that are
O(L^2) or O(K) (ContentionStats from a finished GLCM, merge of per-chunk
matrices, the row partition arithmetic) are computed here or in the C library.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib as L

kDefaultScratchBudget = 49152  # parallel.hpp:16


# --------------------------------------------------------------------------- types
class Angle(enum.IntEnum):
    """glcm.hpp:15"""
    deg0 = 0
    deg45 = 45
    deg90 = 90
    deg135 = 135


def angle_from_degrees(deg: int) -> Angle:
    """glcm.hpp:17-25"""
    try:
        return Angle(int(deg))
    except ValueError:
        raise ValueError("angle must be one of 0, 45, 90, 135") from None


def to_degrees(a: Angle) -> int:
    return int(a)


@dataclass
class GlcmParams:
    """glcm.hpp:29-33"""
    distance: int = 1
    angle: Angle = Angle.deg0
    levels: int = 8


@dataclass(eq=False)
class GrayImage:
    """image.hpp:13-28 — 8-bit row-major raster."""
    width: int
    height: int
    pixels: np.ndarray

    def __post_init__(self):
        self.pixels = np.ascontiguousarray(np.asarray(self.pixels, dtype=np.uint8).reshape(-1))
        if self.width == 0 or self.height == 0:
            raise ValueError("GrayImage: dimensions must be positive")
        if self.pixels.size != self.width * self.height:
            raise ValueError("GrayImage: pixel count does not match dimensions")

    def at(self, row: int, col: int) -> int:
        return int(self.pixels[row * self.width + col])


@dataclass(eq=False)
class QuantizedImage:
    """image.hpp:31-52 — gray levels in [0, levels)."""
    width: int
    height: int
    levels: int
    pixels: np.ndarray

    def __post_init__(self):
        self.pixels = np.ascontiguousarray(np.asarray(self.pixels, dtype=np.uint8).reshape(-1))
        if self.width == 0 or self.height == 0:
            raise ValueError("QuantizedImage: dimensions must be positive")
        if self.levels < 2 or self.levels > 256:
            raise ValueError("QuantizedImage: levels must be in [2, 256]")
        if self.pixels.size != self.width * self.height:
            raise ValueError("QuantizedImage: pixel count does not match dimensions")
        if self.levels < 256 and self.pixels.size and int(self.pixels.max()) >= self.levels:
            raise ValueError("QuantizedImage: pixel value exceeds gray level")

    def at(self, row: int, col: int) -> int:
        return int(self.pixels[row * self.width + col])


class Glcm:
    """glcm.hpp:37-60 — L x L u64 counts, row = reference gray, col = anchor gray."""

    def __init__(self, levels: int, counts=None):
        if levels < 2 or levels > 256:
            raise ValueError("Glcm: levels must be in [2, 256]")
        self.levels = int(levels)
        if counts is None:
            self.counts = np.zeros(levels * levels, dtype=np.uint64)
        else:
            c = np.asarray(counts, dtype=np.uint64).reshape(-1).copy()
            if c.size != levels * levels:
                raise ValueError("Glcm: counts length must be levels^2")
            self.counts = c

    def at(self, row: int, col: int) -> int:
        return int(self.counts[row * self.levels + col])

    def set(self, row: int, col: int, v: int) -> None:
        self.counts[row * self.levels + col] = v

    def total(self) -> int:
        return int(self.counts.sum(dtype=np.uint64))

    def matrix(self) -> np.ndarray:
        return self.counts.reshape(self.levels, self.levels)

    def __eq__(self, other) -> bool:
        return (isinstance(other, Glcm) and self.levels == other.levels
                and np.array_equal(self.counts, other.counts))

    def __repr__(self) -> str:
        return f"Glcm(levels={self.levels}, total={self.total()})"


@dataclass
class GlcmProbabilities:
    """glcm.hpp:159-164"""
    levels: int
    values: np.ndarray

    def at(self, row: int, col: int) -> float:
        return float(self.values[row * self.levels + col])


@dataclass
class FeatureVector:
    """features.hpp:11-17"""
    energy: float = 0.0
    contrast: float = 0.0
    homogeneity: float = 0.0
    entropy: float = 0.0
    correlation: float = 0.0

    def as_array(self) -> np.ndarray:
        return np.array([self.energy, self.contrast, self.homogeneity, self.entropy, self.correlation])


@dataclass
class PixelOffset:
    row: int = 0
    col: int = 0


@dataclass
class ExecutionPlan:
    """parallel.hpp:20-27 (host-side Eq. 4-6 plan, kept unchanged)."""
    worker_count: int = 1
    group_size: int = 512
    copies: int = 1
    scratch_budget: int = kDefaultScratchBudget
    groups_per_unit: int = 2
    degraded: bool = False


@dataclass
class ContentionStats:
    """parallel.hpp:29-35"""
    total_votes: int = 0
    hottest_cell_votes: int = 0
    hottest_cell_index: Tuple[int, int] = (0, 0)
    per_copy_hottest: List[int] = field(default_factory=list)
    concentration: float = 0.0


@dataclass
class ChunkSpec:
    """pipeline.hpp:33-43"""
    index: int = 0
    owned_row_start: int = 0
    owned_row_end: int = 0
    buffer_row_end: int = 0
    chunk_count: int = 1

    def owned_rows(self) -> int:
        return self.owned_row_end - self.owned_row_start

    def buffer_rows(self) -> int:
        return self.buffer_row_end - self.owned_row_start


class PipelineError(RuntimeError):
    """pipeline.hpp:25-29"""

    def __init__(self, index: int, what: str):
        super().__init__(what if what.startswith(f"chunk {index}:") else f"chunk {index}: {what}")
        self.chunk_index = index


class ChunkExecution(enum.Enum):
    """pipeline.hpp:205-208"""
    pipelined = 0
    sequential = 1


class ChunkSource:
    """pipeline.hpp:77-84 — fetch(spec, out) fills `out` (a uint8 array of
    exactly buffer_rows()*width bytes, pinned host memory) with the quantised
    rows [owned_row_start, buffer_row_end)."""

    def width(self) -> int: raise NotImplementedError
    def height(self) -> int: raise NotImplementedError
    def levels(self) -> int: raise NotImplementedError
    def fetch(self, spec: ChunkSpec, out: np.ndarray) -> None: raise NotImplementedError


class MemoryChunkSource(ChunkSource):
    """pipeline.hpp:86-101"""

    def __init__(self, img: QuantizedImage):
        self._img = img

    def width(self): return self._img.width
    def height(self): return self._img.height
    def levels(self): return self._img.levels

    def fetch(self, spec: ChunkSpec, out: np.ndarray) -> None:
        b = spec.owned_row_start * self._img.width
        e = spec.buffer_row_end * self._img.width
        out[:] = self._img.pixels[b:e]


# --------------------------------------------------------------------------- engine
def _out_buffer(out: Optional[np.ndarray], n: int) -> np.ndarray:
    if out is None:
        return np.zeros(n, dtype=np.uint64)
    if out.dtype != np.uint64 or out.size != n or not out.flags.c_contiguous:
        raise ValueError(f"out must be a contiguous uint64 array of {n} elements")
    return out.reshape(-1)


def _ptr(a: np.ndarray, t=C.c_uint8):
    return a.ctypes.data_as(C.POINTER(t))


class Engine:
    """One CUDA context of the engine (device buffers, streams, pinned ring)."""

    def __init__(self, device: int = 0):
        self._lib = L.load()
        h = C.c_void_p()
        L.check(self._lib.tfg_ctx_create(C.byref(h), int(device), 0))
        self.handle = h
        self.device = device

    def close(self):
        if getattr(self, "handle", None) and self.handle.value:
            self._lib.tfg_ctx_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(self._lib.tfg_launch_count(self.handle))

    def synth_noise_device(self, width: int, height: int, seed: int, out=None, pitch: int = 0, stream=None):
        """image.hpp:109-116 generated on the device (bit-identical to
        synth_noise). Returns a CUDA uint8 tensor of height*pitch bytes
        (pitch = width unless given), or fills `out` (a CUDA tensor)."""
        import torch
        pitch = int(pitch or width)
        if out is None:
            out = torch.empty(height * pitch, dtype=torch.uint8, device=f"cuda:{self.device}")
        if not out.is_cuda or out.numel() < height * pitch:
            raise ValueError("synth_noise_device: out must be a CUDA tensor of >= height*pitch bytes")
        s = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        L.check(self._lib.tfg_synth_noise_device(self.handle, int(width), int(height), seed & 0xFFFFFFFF,
                                                 C.c_void_p(out.data_ptr()), pitch, C.c_void_p(s)))
        return out

    def synth_noise_rows_device(self, width: int, row0: int, rows: int, seed: int, out=None, pitch: int = 0,
                                stream=None):
        """Rows [row0, row0+rows) of synth_noise(width, *, seed) generated on the
        device (the generator jumps to output row0*width): one GPU's shard of a
        row-partitioned image. Returns a CUDA uint8 tensor of rows*pitch bytes."""
        import torch
        pitch = int(pitch or width)
        if out is None:
            out = torch.empty(rows * pitch, dtype=torch.uint8, device=f"cuda:{self.device}")
        if not out.is_cuda or out.numel() < rows * pitch:
            raise ValueError("synth_noise_rows_device: out must be a CUDA tensor of >= rows*pitch bytes")
        s = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        L.check(self._lib.tfg_synth_noise_rows_device(self.handle, int(width), int(row0), int(rows),
                                                      seed & 0xFFFFFFFF, C.c_void_p(out.data_ptr()), pitch,
                                                      C.c_void_p(s)))
        return out

    # -- raw, multi-(d, theta) entry point -------------------------------------
    def glcm(self, pixels: np.ndarray, width: int, height: int, levels: int, dts: Sequence[Tuple[int, int]],
             pixel_levels: int = 256, flags: int = 0, n_bands: int = 1,
             want_probs: bool = False, want_features: bool = False, out: Optional[np.ndarray] = None):
        """counts[n_bands, n_dt, L, L] (+ probs, features) of host pixels. `out`
        (u64, n_bands*n_dt*L*L) receives the counts; pinned memory gets them by
        DMA with no staging copy."""
        px = np.ascontiguousarray(pixels, dtype=np.uint8).reshape(-1)
        if px.size != width * height * n_bands:
            raise ValueError("glcm: pixel count does not match dimensions")
        n_dt = len(dts)
        d = (C.c_int * n_dt)(*[int(x[0]) for x in dts])
        a = (C.c_int * n_dt)(*[int(x[1]) for x in dts])
        cells = levels * levels
        counts = _out_buffer(out, n_bands * n_dt * cells)
        probs = np.zeros(n_bands * n_dt * cells, dtype=np.float64) if (want_probs or want_features) else None
        feats = np.zeros(n_bands * n_dt * 5, dtype=np.float64) if want_features else None
        if want_probs or want_features:
            flags |= L.TFG_NORMALIZE
        if want_features:
            flags |= L.TFG_FEATURES
        rc = self._lib.tfg_glcm_bands(
            self.handle, px.ctypes.data_as(C.c_void_p), width, height, width, width * height, n_bands,
            pixel_levels, levels, d, a, n_dt, flags, _ptr(counts, C.c_uint64),
            _ptr(probs, C.c_double) if probs is not None else None,
            _ptr(feats, C.c_double) if feats is not None else None)
        L.check(rc)
        counts = counts.reshape(n_bands, n_dt, levels, levels)
        out = [counts]
        if want_probs:
            out.append(probs.reshape(n_bands, n_dt, levels, levels))
        if want_features:
            out.append(feats.reshape(n_bands, n_dt, 5))
        return out[0] if len(out) == 1 else tuple(out)

    def shard(self, pixels, width: int, buffer_rows: int, owned_rows: int, levels: int,
              dts: Sequence[Tuple[int, int]], pixel_levels: int = 256, device: bool = False,
              n_bands: int = 1, band_stride: int = 0, out: Optional[np.ndarray] = None) -> np.ndarray:
        """Partial counts [n_bands, n_dt, L, L] of row shards (tfg_glcm_shard):
        anchors in rows [0, owned_rows) of a buffer of `buffer_rows` rows vote;
        the rest is the next shard's halo. n_bands buffers of that shape sit
        `band_stride` bytes apart (default: dense). `pixels` is host memory
        (numpy) or, with device=True, a device address (int) of a
        16-byte-aligned dense buffer."""
        n_dt = len(dts)
        d = (C.c_int * n_dt)(*[int(x[0]) for x in dts])
        a = (C.c_int * n_dt)(*[int(x[1]) for x in dts])
        counts = _out_buffer(out, n_bands * n_dt * levels * levels)
        stride = band_stride or width * buffer_rows
        if device:
            ptr, flags = C.c_void_p(int(pixels)), L.TFG_INPUT_DEVICE
        else:
            px = np.ascontiguousarray(pixels, dtype=np.uint8).reshape(-1)
            if px.size < stride * (n_bands - 1) + width * buffer_rows:
                raise ValueError("glcm: pixel count does not match dimensions")
            ptr, flags = px.ctypes.data_as(C.c_void_p), 0
        L.check(self._lib.tfg_glcm_shard(self.handle, ptr, width, buffer_rows, owned_rows, width, stride, n_bands,
                                         pixel_levels, levels, d, a, n_dt, flags, _ptr(counts, C.c_uint64)))
        return counts.reshape(n_bands, n_dt, levels, levels)

    def shard_jobs(self, pixels: np.ndarray, width: int, buffer_rows: int, owned_rows: int,
                   jobs: Sequence[Tuple[int, int, int]], pixel_levels: int = 256, n_bands: int = 1,
                   band_stride: int = 0, out: Optional[np.ndarray] = None) -> list:
        """tfg_glcm_shard_jobs: per-job (L, d, theta) counts of a HOST row shard /
        band batch, each band copied up once for all its jobs. Returns, per
        job, counts[n_bands, L, L] (views into one [band][job] buffer)."""
        n = len(jobs)
        lv = (C.c_int * n)(*[int(j[0]) for j in jobs])
        d = (C.c_int * n)(*[int(j[1]) for j in jobs])
        a = (C.c_int * n)(*[int(j[2]) for j in jobs])
        band_words = sum(int(j[0]) ** 2 for j in jobs)
        counts = _out_buffer(out, n_bands * band_words)
        stride = band_stride or width * buffer_rows
        px = np.ascontiguousarray(pixels, dtype=np.uint8).reshape(-1)
        if px.size < stride * (n_bands - 1) + width * buffer_rows:
            raise ValueError("glcm: pixel count does not match dimensions")
        L.check(self._lib.tfg_glcm_shard_jobs(self.handle, px.ctypes.data_as(C.c_void_p), width, buffer_rows,
                                              owned_rows, stride, n_bands, pixel_levels, lv, d, a, n, 0,
                                              _ptr(counts, C.c_uint64)))
        per_band = counts.reshape(n_bands, band_words)
        res, off = [], 0
        for j in jobs:
            c = int(j[0]) ** 2
            res.append(per_band[:, off:off + c].reshape(n_bands, int(j[0]), int(j[0])))
            off += c
        return res

    def chunked(self, source: ChunkSource, dts: Sequence[Tuple[int, int]], chunk_count: int,
                pixel_levels: int, levels: int, flags: int = 0) -> np.ndarray:
        width, height = source.width(), source.height()
        n_dt = len(dts)
        d = (C.c_int * n_dt)(*[int(x[0]) for x in dts])
        a = (C.c_int * n_dt)(*[int(x[1]) for x in dts])
        counts = np.zeros(n_dt * levels * levels, dtype=np.uint64)
        err_box: dict = {}
        cb = _fetch_callback(source, chunk_count, width, err_box)
        rc = self._lib.tfg_glcm_chunked(self.handle, width, height, pixel_levels, levels, d, a, n_dt,
                                        int(chunk_count), cb, None, flags, _ptr(counts, C.c_uint64), None, None)
        _raise_source(self._lib, rc, err_box)
        return counts.reshape(n_dt, levels, levels)

    def quantize(self, gray: np.ndarray, levels: int) -> np.ndarray:
        g = np.ascontiguousarray(gray, dtype=np.uint8).reshape(-1)
        out = np.empty_like(g)
        L.check(self._lib.tfg_quantize(self.handle, g.ctypes.data_as(C.c_void_p), g.size, int(levels),
                                       out.ctypes.data_as(C.c_void_p), 0))
        return out

    def symmetrize(self, counts: np.ndarray, levels: int) -> np.ndarray:
        c = np.ascontiguousarray(counts, dtype=np.uint64).reshape(-1)
        out = np.empty_like(c)
        L.check(self._lib.tfg_symmetrize(self.handle, _ptr(c, C.c_uint64), int(levels), _ptr(out, C.c_uint64)))
        return out

    def normalize(self, counts: np.ndarray, levels: int) -> np.ndarray:
        c = np.ascontiguousarray(counts, dtype=np.uint64).reshape(-1)
        out = np.empty(c.size, dtype=np.float64)
        L.check(self._lib.tfg_normalize(self.handle, _ptr(c, C.c_uint64), int(levels), _ptr(out, C.c_double)))
        return out

    def features(self, probs: np.ndarray, levels: int) -> np.ndarray:
        p = np.ascontiguousarray(probs, dtype=np.float64).reshape(-1)
        out = np.empty(5, dtype=np.float64)
        L.check(self._lib.tfg_features(self.handle, _ptr(p, C.c_double), int(levels), _ptr(out, C.c_double)))
        return out


def _fetch_callback(source: "ChunkSource", chunk_count: int, width: int, err_box: dict):
    """A tfg_fetch_fn over ChunkSource.fetch (pipeline.hpp:77-84); the first
    exception is kept in err_box["exc"] and aborts the pipeline."""
    def _fetch(user, idx, start, owned_end, buf_end, dst, err, err_len):
        try:
            spec = ChunkSpec(int(idx), int(start), int(owned_end), int(buf_end), int(chunk_count))
            out = np.ctypeslib.as_array(dst, shape=(int(buf_end - start) * width,))
            source.fetch(spec, out)
            return 0
        except BaseException as e:  # noqa: BLE001 — any source failure aborts the pipeline
            err_box.setdefault("exc", e)
            msg = str(e).encode()[: max(0, int(err_len) - 1)] + b"\0"
            if err:
                C.memmove(err, msg, len(msg))
            return 1
    return L.FETCH_FN(_fetch)


def _raise_source(lib, rc: int, err_box: dict) -> None:
    if rc == L.TFG_SOURCE_ERROR:
        idx = int(lib.tfg_last_error_chunk())
        exc = err_box.get("exc")
        if isinstance(exc, PipelineError):
            raise exc
        raise PipelineError(idx, lib.tfg_last_error().decode(errors="replace"))
    L.check(rc)


class Group:
    """Several GPUs of one process behind one NCCL communicator
    (tfg_group_*): row-partitioned images with a d-row halo
    and one ncclReduce, band batches sharded with no collective, Scheme 3 with
    chunks spread over the GPUs. host_reduce=True lets contexts share a GPU
    (the sum then goes through host memory; NCCL refuses two ranks on one GPU)."""

    def __init__(self, n_gpus: int, devices: Optional[Sequence[int]] = None, host_reduce: bool = False):
        self._lib = L.load()
        h = C.c_void_p()
        devs = (C.c_int * n_gpus)(*devices) if devices is not None else None
        L.check(self._lib.tfg_group_create(C.byref(h), int(n_gpus), devs,
                                           L.TFG_GROUP_HOST_REDUCE if host_reduce else 0))
        self.handle = h
        self.size = n_gpus

    def close(self):
        if getattr(self, "handle", None) and self.handle.value:
            self._lib.tfg_group_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(self._lib.tfg_group_launch_count(self.handle))

    def _dts(self, dts):
        n = len(dts)
        return n, (C.c_int * n)(*[int(x[0]) for x in dts]), (C.c_int * n)(*[int(x[1]) for x in dts])

    def glcm(self, pixels: np.ndarray, width: int, height: int, levels: int, dts: Sequence[Tuple[int, int]],
             pixel_levels: int = 256, flags: int = 0, n_bands: int = 1) -> np.ndarray:
        """counts[n_bands, n_dt, L, L]: one image row-partitioned over the
        group (n_bands == 1) or a band batch sharded over it."""
        px = np.ascontiguousarray(pixels, dtype=np.uint8).reshape(-1)
        if px.size != width * height * n_bands:
            raise ValueError("glcm: pixel count does not match dimensions")
        n_dt, d, a = self._dts(dts)
        counts = np.zeros(n_bands * n_dt * levels * levels, dtype=np.uint64)
        if n_bands == 1:
            rc = self._lib.tfg_group_glcm(self.handle, px.ctypes.data_as(C.c_void_p), width, height, pixel_levels,
                                          levels, d, a, n_dt, flags, _ptr(counts, C.c_uint64), None, None)
        else:
            rc = self._lib.tfg_group_glcm_bands(self.handle, px.ctypes.data_as(C.c_void_p), width, height,
                                                width * height, n_bands, pixel_levels, levels, d, a, n_dt, flags,
                                                _ptr(counts, C.c_uint64), None, None)
        L.check(rc)
        return counts.reshape(n_bands, n_dt, levels, levels)

    def chunked(self, source: "ChunkSource", dts: Sequence[Tuple[int, int]], chunk_count: int,
                pixel_levels: int, levels: int, flags: int = 0) -> np.ndarray:
        width, height = source.width(), source.height()
        n_dt, d, a = self._dts(dts)
        counts = np.zeros(n_dt * levels * levels, dtype=np.uint64)
        err_box: dict = {}
        cb = _fetch_callback(source, chunk_count, width, err_box)
        rc = self._lib.tfg_group_glcm_chunked(self.handle, width, height, pixel_levels, levels, d, a, n_dt,
                                              int(chunk_count), cb, None, flags, _ptr(counts, C.c_uint64), None,
                                              None)
        _raise_source(self._lib, rc, err_box)
        return counts.reshape(n_dt, levels, levels)


class Comm:
    """One rank's NCCL communicator (tfg_comm_*): one process per GPU, the
    ncclUniqueId shipped by the caller (e.g. torch.distributed)."""

    def __init__(self, engine: Engine, nranks: int, rank: int, uid: bytes):
        self._lib = L.load()
        if len(uid) != L.TFG_COMM_ID_BYTES:
            raise ValueError("Comm: the unique id must be TFG_COMM_ID_BYTES bytes")
        buf = C.create_string_buffer(uid, L.TFG_COMM_ID_BYTES)
        h = C.c_void_p()
        L.check(self._lib.tfg_comm_init_rank(C.byref(h), engine.handle, int(nranks), int(rank), buf))
        self.handle, self.engine, self.nranks, self.rank = h, engine, nranks, rank

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(L.TFG_COMM_ID_BYTES)
        L.check(L.load().tfg_comm_unique_id(buf))
        return buf.raw

    def close(self):
        if getattr(self, "handle", None) and self.handle.value:
            self._lib.tfg_comm_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reduce_counts(self, d_counts_ptr: int, n: int, root: int = 0, stream: int = 0) -> None:
        L.check(self._lib.tfg_comm_reduce_counts(self.handle, C.c_void_p(d_counts_ptr), int(n), int(root),
                                                 C.c_void_p(stream)))

    def exchange_halo(self, d_slab_ptr: int, pitch: int, owned_rows: int, halo: int, stream: int = 0) -> None:
        L.check(self._lib.tfg_comm_exchange_halo(self.handle, C.c_void_p(d_slab_ptr), int(pitch), int(owned_rows),
                                                 int(halo), C.c_void_p(stream)))

    def allreduce_max_f64(self, d_ptr: int, n: int, stream: int = 0) -> None:
        L.check(self._lib.tfg_comm_allreduce_max_f64(self.handle, C.c_void_p(d_ptr), int(n), C.c_void_p(stream)))


_engine: Optional[Engine] = None
_engine_lock = threading.Lock()


def default_engine() -> Engine:
    global _engine
    with _engine_lock:
        if _engine is None:
            _engine = Engine(0)
        return _engine


# --------------------------------------------------------------------------- geometry
def neighbor_offset(p: GlcmParams) -> PixelOffset:
    """glcm.hpp:71-80"""
    dr, dc = C.c_long(), C.c_long()
    L.check(L.load().tfg_neighbor_offset(int(p.distance), int(p.angle), C.byref(dr), C.byref(dc)))
    return PixelOffset(dr.value, dc.value)


def valid_pair_count(width: int, height: int, p: GlcmParams) -> int:
    """glcm.hpp:83-94"""
    out = C.c_uint64()
    L.check(L.load().tfg_valid_pair_count(int(width), int(height), int(p.distance), int(p.angle), C.byref(out)))
    return int(out.value)


def plan(levels: int, scratch_budget: int = kDefaultScratchBudget, worker_count: Optional[int] = None
         ) -> ExecutionPlan:
    """parallel.hpp:39-66 — unchanged host plan (pinned by the reference tests)."""
    import os
    if worker_count is None:
        worker_count = os.cpu_count() or 1
    if worker_count == 0:
        worker_count = 1
    cp, gpu, deg = C.c_uint(), C.c_uint(), C.c_int()
    L.check(L.load().tfg_plan(int(levels), int(scratch_budget), int(worker_count), C.byref(cp), C.byref(gpu),
                              C.byref(deg)))
    return ExecutionPlan(worker_count=int(worker_count), group_size=512, copies=int(cp.value),
                         scratch_budget=int(scratch_budget), groups_per_unit=int(gpu.value), degraded=bool(deg.value))


def partition(width: int, height: int, p: GlcmParams, chunk_count: int) -> List[ChunkSpec]:
    """pipeline.hpp:48-73"""
    if chunk_count < 1 or chunk_count > height:
        # same order of checks as the reference: geometry first
        if p.distance < 1 or p.distance >= width or p.distance >= height:
            raise ValueError("partition: degenerate geometry (d must be in [1, min(width, height)))")
        raise ValueError("partition: chunk count must be in [1, height]")
    specs = np.zeros(3 * int(chunk_count), dtype=np.uint64)
    L.check(L.load().tfg_partition(int(width), int(height), int(p.distance), int(p.angle), int(chunk_count),
                                   _ptr(specs, C.c_uint64)))
    return [ChunkSpec(i, int(specs[3 * i]), int(specs[3 * i + 1]), int(specs[3 * i + 2]), int(chunk_count))
            for i in range(int(chunk_count))]


# --------------------------------------------------------------------------- inputs
def synth_noise(width: int, height: int, seed: int) -> GrayImage:
    """image.hpp:109-116 (bit-identical)."""
    if width < 2 or height < 2:
        raise ValueError("synth_noise: dimensions must be >= 2")
    out = np.empty(width * height, dtype=np.uint8)
    L.check(L.load().tfg_synth_noise(width, height, seed & 0xFFFFFFFF, _ptr(out)))
    return GrayImage(width, height, out)


def mt19937_windows(seed: int, first: int, stride: int, count: int) -> np.ndarray:
    """Generator windows of std::mt19937(seed) at outputs first + s*stride
    (tfg_mt19937_windows; host jump-ahead), shape (count, 624) uint32."""
    out = np.empty((count, 624), dtype=np.uint32)
    L.check(L.load().tfg_mt19937_windows(seed & 0xFFFFFFFF, int(first), int(stride), int(count),
                                         out.ctypes.data_as(C.POINTER(C.c_uint32)), 0))
    return out


def synth_smooth(width: int, height: int, seed: int, threads: int = 0) -> GrayImage:
    """image.hpp:76-106 (bit-identical; rows generated in parallel)."""
    if width < 2 or height < 2:
        raise ValueError("synth_smooth: dimensions must be >= 2")
    out = np.empty(width * height, dtype=np.uint8)
    L.check(L.load().tfg_synth_smooth(width, height, seed & 0xFFFFFFFF, _ptr(out), int(threads)))
    return GrayImage(width, height, out)


def quantize(img: GrayImage, levels: int) -> QuantizedImage:
    """image.hpp:55-62 — on the device."""
    if levels < 2 or levels > 256:
        raise ValueError("quantize: levels must be in [2, 256]")
    q = default_engine().quantize(img.pixels, levels)
    return QuantizedImage(img.width, img.height, levels, q)


# --------------------------------------------------------------------------- GLCM
def _check_inputs(img: QuantizedImage, p: GlcmParams) -> None:
    """glcm.hpp:98-104"""
    if img.levels != p.levels:
        raise ValueError("glcm: image levels do not match params levels")
    if p.distance < 1 or p.distance >= img.width or p.distance >= img.height:
        raise ValueError("glcm: degenerate geometry (d must be in [1, min(width, height)))")


def _device_glcm(img: QuantizedImage, p: GlcmParams, flags: int = 0) -> Glcm:
    _check_inputs(img, p)
    counts = default_engine().glcm(img.pixels, img.width, img.height, p.levels,
                                   [(p.distance, int(p.angle))], pixel_levels=p.levels, flags=flags)
    return Glcm(p.levels, counts.reshape(-1))


def stats_from_counts(g: Glcm) -> ContentionStats:
    """parallel.hpp:91-102 (host, O(L^2) on the finished matrix)."""
    c = g.counts
    best = int(np.argmax(c))  # first maximum = lowest flat index on ties
    total = g.total()
    hot = int(c[best])
    return ContentionStats(total_votes=total, hottest_cell_votes=hot,
                           hottest_cell_index=(best // g.levels, best % g.levels),
                           concentration=(hot / total) if total else 0.0)


def compute_glcm_serial(img: QuantizedImage, p: GlcmParams) -> Glcm:
    """glcm.hpp:144-147 — identical counts, computed by the device engine."""
    return _device_glcm(img, p)


def compute_glcm_shared(img: QuantizedImage, p: GlcmParams, plan_: ExecutionPlan) -> Tuple[Glcm, ContentionStats]:
    """parallel.hpp:143-152 — Scheme 1: one global atomic per pixel pair."""
    g = _device_glcm(img, p, L.TFG_SCHEME_GLOBAL)
    return g, stats_from_counts(g)


def _resolve_group_count(requested: int, plan_: ExecutionPlan, width: int, rows: int) -> int:
    """parallel.hpp:166-181: 0 -> groups_per_unit * worker_count, raised so no
    group can exceed 2^32 votes, clamped to [1, rows]."""
    g = int(requested)
    if g == 0:
        g = (plan_.groups_per_unit or 2) * plan_.worker_count
        floor_groups = -(-(rows * width) // (1 << 32))
        g = max(g, floor_groups)
    return max(1, min(g, rows))


def _subglcms(img: QuantizedImage, p: GlcmParams, plan_: ExecutionPlan, group_count: int, want_subs: bool):
    _check_inputs(img, p)
    if plan_.copies < 1:
        raise ValueError("privatized: plan.copies must be >= 1")
    groups = _resolve_group_count(group_count, plan_, img.width, img.height)
    cells = p.levels * p.levels
    n_subs = groups * plan_.copies
    subs = np.zeros(n_subs * cells, dtype=np.uint32) if want_subs else None
    counts = np.zeros(cells, dtype=np.uint64)
    hottest = np.zeros(n_subs, dtype=np.uint64)
    eng = default_engine()
    px = np.ascontiguousarray(img.pixels, dtype=np.uint8).reshape(-1)
    L.check(eng._lib.tfg_subglcms(eng.handle, px.ctypes.data_as(C.c_void_p), img.width, img.height, img.levels,
                                  p.levels, p.distance, int(p.angle), plan_.group_size, plan_.copies, groups, 0,
                                  subs.ctypes.data_as(C.POINTER(C.c_uint32)) if want_subs else None,
                                  _ptr(counts, C.c_uint64), _ptr(hottest, C.c_uint64)))
    return subs, counts, hottest, n_subs


def compute_subglcms(img: QuantizedImage, p: GlcmParams, plan_: ExecutionPlan,
                     group_count: int = 0) -> List[np.ndarray]:
    """parallel.hpp:218-225 — the raw (group, copy) sub-GLCMs, group-major, with
    the reference's exact lane -> copy routing (glcm_subglcm_kernel)."""
    subs, _, _, n_subs = _subglcms(img, p, plan_, group_count, True)
    cells = p.levels * p.levels
    return [subs[i * cells:(i + 1) * cells] for i in range(n_subs)]


def compute_glcm_privatized(img: QuantizedImage, p: GlcmParams, plan_: ExecutionPlan,
                            group_count: int = 0) -> Tuple[Glcm, ContentionStats]:
    """parallel.hpp:240-254 — Scheme 2: counts from the privatised vote kernel,
    per_copy_hottest from the reference-routed sub-GLCMs."""
    _, counts, hottest, _ = _subglcms(img, p, plan_, group_count, False)
    g = Glcm(p.levels, counts)
    st = stats_from_counts(g)
    st.per_copy_hottest = [int(x) for x in hottest]
    return g, st


def contention_profile(img: QuantizedImage, p: GlcmParams) -> ContentionStats:
    """parallel.hpp:258-260"""
    return stats_from_counts(compute_glcm_serial(img, p))


def reduce_subglcms(subs: Sequence[Sequence[int]], levels: int) -> Glcm:
    """parallel.hpp:228-237 — elementwise u64 sum (order-independent)."""
    out = Glcm(levels)
    for s in subs:
        a = np.asarray(s, dtype=np.uint64).reshape(-1)
        if a.size != levels * levels:
            raise ValueError("reduce_subglcms: sub-GLCM length mismatch")
        out.counts += a
    return out


def merge_chunk_glcms(parts: Sequence[Glcm]) -> Glcm:
    """pipeline.hpp:231-240"""
    if not parts:
        raise ValueError("merge_chunk_glcms: no parts")
    out = Glcm(parts[0].levels)
    for g in parts:
        if g.levels != out.levels:
            raise ValueError("merge_chunk_glcms: level mismatch")
        out.counts += g.counts
    return out


def compute_glcm_chunked(source: ChunkSource, p: GlcmParams, plan_: ExecutionPlan, chunk_count: int,
                         mode: ChunkExecution = ChunkExecution.pipelined) -> Glcm:
    """pipeline.hpp:246-337 — Scheme 3 on CUDA streams (pinned ring, H2D on a
    copy stream overlapped with voting on the exec stream)."""
    if source.levels() != p.levels:
        raise ValueError("glcm: image levels do not match params levels")
    partition(source.width(), source.height(), p, chunk_count)  # same validation + messages
    flags = L.TFG_SEQUENTIAL if mode == ChunkExecution.sequential else 0
    counts = default_engine().chunked(source, [(p.distance, int(p.angle))], chunk_count,
                                      pixel_levels=p.levels, levels=p.levels, flags=flags)
    return Glcm(p.levels, counts.reshape(-1))


def symmetrize(g: Glcm) -> Glcm:
    """glcm.hpp:150-156"""
    return Glcm(g.levels, default_engine().symmetrize(g.counts, g.levels))


def normalize(g: Glcm) -> GlcmProbabilities:
    """glcm.hpp:167-177 (bit-exact)."""
    return GlcmProbabilities(g.levels, default_engine().normalize(g.counts, g.levels))


def extract_features(p: GlcmProbabilities) -> FeatureVector:
    """features.hpp:37-69"""
    f = default_engine().features(p.values, p.levels)
    return FeatureVector(*[float(x) for x in f])
