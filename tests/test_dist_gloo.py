"""The N>1 host path on CPU: world_size-2 gloo processes run the product's
row-shard + halo + reduce logic (paper_1710_06189_b200/distributed.py) with
the oracle injected as the per-shard compute, and band sharding."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ANGLES = (0, 45, 90, 135)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, results):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_1710_06189_b200 import distributed as D
    from paper_1710_06189_b200 import texforge as tf

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        for (w, h, L) in [(97, 61, 16), (64, 40, 256), (33, 17, 8)]:
            img = tf.synth_noise(w, h, 3).pixels
            q = O.quantize(img, L)
            dts = [(1, a) for a in ANGLES] + [(3, 45), (2, 135)]

            def compute(spec, dts_):
                buf = q[spec.owned_row_start * w: spec.buffer_row_end * w]
                part = np.zeros((len(dts_), L * L), np.uint64)
                for t, (d, a) in enumerate(dts_):
                    O.glcm_rows(buf, w, spec.buffer_rows(), L, d, a, 0, spec.owned_rows(), part[t])
                return part

            got = D.glcm_row_sharded(w, h, L, dts, compute, world, rank)
            want = np.stack([O.glcm_serial(q, w, h, L, d, a) for d, a in dts])
            out[(w, h, L)] = bool(np.array_equal(got, want))
        # halo exchange: each rank starts with ONLY its own row block (the
        # multi-GPU bench layout), receives the next block's first rows over
        # the collective backend, votes its owned anchors, one reduce
        import torch
        w, L, blk = 45, 16, 23
        dts = [(1, 0), (2, 45), (3, 90), (1, 135)]
        halo = D.halo_rows(dts)
        whole = O.quantize(tf.synth_noise(w, blk * world, 5).pixels, L)
        slab = torch.zeros((blk + halo) * w, dtype=torch.uint8)
        slab[: blk * w] = torch.from_numpy(whole[rank * blk * w:(rank + 1) * blk * w].copy())
        rows = D.exchange_halo(slab, blk, w, halo, world, rank)
        buf = slab.numpy()
        part = np.zeros((len(dts), L * L), np.uint64)
        for t, (d, a) in enumerate(dts):
            O.glcm_rows(buf, w, rows, L, d, a, 0, blk, part[t])
        got = D.reduce_partials(part.reshape(-1), all_ranks=True).reshape(len(dts), L * L)
        want = np.stack([O.glcm_serial(whole, w, blk * world, L, d, a) for d, a in dts])
        out["halo_exchange"] = bool(np.array_equal(got, want)) and rows == blk + (halo if rank + 1 < world else 0)
        # bands: contiguous blocks, every band exactly once
        owned = list(D.bands_for_rank(11, world, rank))
        gathered = [None] * world
        dist.all_gather_object(gathered, owned)
        out["bands"] = sorted(b for g in gathered for b in g) == list(range(11))
        results[rank] = out
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_row_shards_with_halo_reduce_to_whole(world):
    ctx = mp.get_context("spawn")
    manager = ctx.Manager()
    results = manager.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, results)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    assert len(results) == world
    for r in range(world):
        assert all(results[r].values()), results[r]


def test_shard_geometry_single_process():
    from paper_1710_06189_b200 import distributed as D
    s0 = D.shard_rows(1000, 1000, [(1, 0), (4, 45)], 8, 4, 0)
    assert (s0.owned_row_start, s0.owned_row_end, s0.buffer_row_end) == (0, 250, 254)
    s3 = D.shard_rows(1000, 1000, [(1, 0), (4, 45)], 8, 4, 3)
    assert (s3.owned_row_start, s3.owned_row_end, s3.buffer_row_end) == (750, 1000, 1000)
    assert D.shard_rows(1000, 1000, [(2, 0)], 8, 4, 1).buffer_row_end == 500  # 0 deg: no halo
    assert [len(D.bands_for_rank(256, 8, r)) for r in range(8)] == [32] * 8
