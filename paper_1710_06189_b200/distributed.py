"""Multi-GPU GLCM: row shards with a d-row halo + one reduce, and band sharding.

One process per GPU (torchrun), ``torch.distributed`` as the plumbing:

* one huge image (BASELINE configs 3/5): ``partition(W, H, p, G)``
  (R/include/texforge/pipeline.hpp:48-73) gives rank g the owned rows
  [owned_row_start, owned_row_end) plus the halo rows up to buffer_row_end;
  the rank votes only its owned anchors (``tfg_glcm_async`` with
  row_end = owned rows) into an L*L u64 partial, and the partials are summed
  with ONE reduce (NCCL over NVLink on B200; integer sums are exact and
  order-independent, like merge_chunk_glcms, pipeline.hpp:231-240);
* multispectral band batches (config 4): bands are independent units, rank g
  owns a contiguous block of bands; no collective on the data path (an
  optional gather brings the per-band GLCMs to rank 0).

The per-shard compute is a callable so the host logic is testable on CPU with
``gloo`` (tests/test_dist_gloo.py injects the oracle there); the product
wires in the CUDA engine (``engine_shard_compute``).
"""
from __future__ import annotations

from typing import Callable, List, Sequence, Tuple

import numpy as np

from .texforge import Angle, ChunkSpec, GlcmParams, partition

ShardCompute = Callable[[ChunkSpec, Sequence[Tuple[int, int]]], np.ndarray]


def halo_params(dts: Sequence[Tuple[int, int]], levels: int) -> GlcmParams:
    """The (d, theta) whose partition() halo covers every requested pair."""
    dmax = max(d for d, _ in dts)
    any_down = any(a != 0 for _, a in dts)
    return GlcmParams(dmax, Angle.deg90 if any_down else Angle.deg0, levels)


def shard_rows(width: int, height: int, dts: Sequence[Tuple[int, int]], levels: int, world: int,
               rank: int) -> ChunkSpec:
    """Rank `rank`'s rows: owned range + halo (partition semantics)."""
    specs = partition(width, height, halo_params(dts, levels), world)
    return specs[rank]


def bands_for_rank(n_bands: int, world: int, rank: int) -> range:
    """Contiguous block of bands (first n_bands % world ranks get one more)."""
    base, extra = divmod(n_bands, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def reduce_partials(partial: np.ndarray, dst: int = 0, all_ranks: bool = False):
    """Sums u64 partial GLCMs across ranks with one collective.

    Accepts a numpy u64 array (CPU / gloo) or a torch int64 CUDA tensor
    (NCCL). u64 counts travel as int64 bit patterns: two's-complement addition
    is the same ring as u64 addition, so the sum is exact."""
    import torch
    import torch.distributed as dist

    if isinstance(partial, np.ndarray):
        t = torch.from_numpy(partial.astype(np.uint64).view(np.int64).copy())
    else:
        t = partial
    if all_ranks:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    else:
        dist.reduce(t, dst=dst, op=dist.ReduceOp.SUM)
    if isinstance(partial, np.ndarray):
        return t.numpy().view(np.uint64)
    return t


def glcm_row_sharded(width: int, height: int, levels: int, dts: Sequence[Tuple[int, int]],
                     compute: ShardCompute, world: int, rank: int, all_ranks: bool = True) -> np.ndarray:
    """Row-partitioned GLCMs of one image across `world` ranks.

    `compute(spec, dts)` returns this rank's u64 partial counts [n_dt, L*L] for
    the anchors it owns. Returns the full counts on rank 0 (all ranks if
    all_ranks)."""
    spec = shard_rows(width, height, dts, levels, world, rank)
    part = compute(spec, dts)
    if isinstance(part, np.ndarray):
        part = np.ascontiguousarray(part, dtype=np.uint64).reshape(len(dts), levels * levels)
        if world == 1:
            return part
        return reduce_partials(part.reshape(-1), all_ranks=all_ranks).reshape(len(dts), levels * levels)
    if world > 1:  # torch CUDA tensor: one NCCL collective over NVLink
        reduce_partials(part.view(-1), all_ranks=all_ranks)
    return part


def engine_shard_compute(engine, device_image, width: int, height: int, pitch: int, levels: int,
                         pixel_levels: int = 256, stream=None):
    """ShardCompute backed by the CUDA engine: `device_image` is a torch uint8
    CUDA tensor holding this rank's rows [owned_row_start, buffer_row_end) (or
    the whole image); returns a torch int64 CUDA tensor [n_dt, L*L]."""
    import ctypes as C

    import torch

    from . import _lib as L

    lib = L.load()

    def compute(spec: ChunkSpec, dts):
        acc = torch.zeros((len(dts), levels * levels), dtype=torch.int64, device=device_image.device)
        base_row = 0 if device_image.shape[0] == spec.buffer_rows() else spec.owned_row_start
        ptr = device_image.data_ptr() + base_row * pitch
        s = stream or torch.cuda.current_stream()
        for t, (d, a) in enumerate(dts):
            L.check(lib.tfg_glcm_async(engine.handle, C.c_void_p(ptr), width, spec.buffer_rows(), pitch,
                                       spec.owned_rows(), pixel_levels, levels, d, a, 0,
                                       C.c_void_p(acc[t].data_ptr()), C.c_void_p(s.cuda_stream)))
        return acc

    return compute


def halo_rows(dts: Sequence[Tuple[int, int]]) -> int:
    """Rows of halo a shard needs below its owned rows (pipeline.hpp:60-61:
    d for the downward angles, none at 0 degrees)."""
    return max([d for d, a in dts if a != 0], default=0)


def exchange_halo(slab, owned_rows: int, width: int, halo: int, world: int, rank: int):
    """Completes each rank's read-only halo with one point-to-point exchange.

    `slab` is a uint8 tensor of (owned_rows + halo) * width bytes whose first
    owned_rows rows are this rank's rows of the global image (rank-major row
    blocks). Rank r sends its first `halo` rows to rank r-1 and receives rank
    r+1's first `halo` rows into its halo (NCCL over NVLink for CUDA tensors,
    gloo for CPU tensors). The last rank owns the image's last rows and needs
    no halo. Returns the number of valid buffer rows on this rank."""
    import torch.distributed as dist

    if halo == 0 or world == 1:
        return owned_rows
    # gloo moves CPU tensors only: stage a CUDA slab through host memory
    # (test mode: several ranks sharing one GPU); NCCL moves it in place.
    stage = slab.is_cuda and dist.get_backend() != "nccl"
    ops = []
    if rank > 0:
        send = slab[: halo * width].contiguous()
        ops.append(dist.P2POp(dist.isend, send.cpu() if stage else send, rank - 1))
    recv = None
    if rank + 1 < world:
        dst = slab[owned_rows * width:(owned_rows + halo) * width]
        recv = dst.cpu() if stage else dst
        ops.append(dist.P2POp(dist.irecv, recv, rank + 1))
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    if stage and recv is not None:
        dst.copy_(recv)
    return owned_rows + (halo if rank + 1 < world else 0)


def reduce_sum_(t, dst: int = 0) -> None:
    """In-place SUM reduce of `t` to rank `dst` (NCCL on the CUDA tensor;
    staged through host memory under gloo)."""
    import torch.distributed as dist

    if t.is_cuda and dist.get_backend() != "nccl":
        c = t.cpu()
        dist.reduce(c, dst=dst, op=dist.ReduceOp.SUM)
        if dist.get_rank() == dst:
            t.copy_(c)
        return
    dist.reduce(t, dst=dst, op=dist.ReduceOp.SUM)


def all_reduce_max_(t) -> None:
    """In-place MAX all-reduce (timing: the slowest rank defines the step)."""
    import torch.distributed as dist

    if t.is_cuda and dist.get_backend() != "nccl":
        c = t.cpu()
        dist.all_reduce(c, op=dist.ReduceOp.MAX)
        t.copy_(c)
        return
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
