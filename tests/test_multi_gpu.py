"""Multi-GPU entry points of the C ABI (tfg_group_*, tfg_comm_*).

gpurun grants one GPU, so:
  * Group(1) runs with a REAL NCCL communicator (ncclCommInitAll over one
    device) and the real ncclReduce;
  * Group(G>1, host_reduce=True) puts G contexts on the one GPU and checks the
    partition() row split + d-row halo + reduce logic (the sum goes through
    host memory because NCCL refuses two ranks on one GPU);
  * Comm runs ncclCommInitRank with one rank (reduce, halo, max all-reduce).
Every result is compared bit for bit with the C oracle (pinned to the
reference's own outputs, tests/golden)."""
import numpy as np
import pytest

from oracle import oracle as O

ANGLES = (0, 45, 90, 135)


def want(img, w, h, L, dts, pixel_levels=256):
    q = img if pixel_levels == L else O.quantize(img, L)
    return np.stack([O.glcm_serial(q, w, h, L, d, a) for d, a in dts]).reshape(len(dts), L, L)


@pytest.mark.gpu
@pytest.mark.parametrize("L", [32, 64, 256])
def test_group_one_gpu_real_nccl(L):
    from paper_1710_06189_b200 import texforge as tf
    g = tf.Group(1)
    w, h = 1000, 700
    img = tf.synth_noise(w, h, 5).pixels
    dts = [(1, a) for a in ANGLES] + [(3, 45), (2, 135)]
    n0 = g.launches
    got = g.glcm(img, w, h, L, dts)[0]
    assert np.array_equal(got, want(img, w, h, L, dts))
    assert g.launches > n0


@pytest.mark.gpu
@pytest.mark.parametrize("G,L,kind", [(2, 32, "noise"), (3, 256, "smooth"), (4, 64, "noise"), (3, 16, "smooth")])
def test_group_row_partition_and_halo(G, L, kind):
    from paper_1710_06189_b200 import texforge as tf
    g = tf.Group(G, host_reduce=True)
    w, h = 777, 613
    img = (tf.synth_noise if kind == "noise" else tf.synth_smooth)(w, h, 2).pixels
    dts = [(1, a) for a in ANGLES] + [(5, 90), (4, 135), (7, 45), (3, 0)]
    got = g.glcm(img, w, h, L, dts)[0]
    assert np.array_equal(got, want(img, w, h, L, dts))


@pytest.mark.gpu
def test_group_fewer_rows_than_gpus_and_quantised_input():
    from paper_1710_06189_b200 import texforge as tf
    g = tf.Group(4, host_reduce=True)
    w, h, L = 40, 9, 8  # 9 rows over 4 GPUs at d=3: the partition shrinks to 2 shards
    q = O.quantize(tf.synth_noise(w, h, 7).pixels, L)
    dts = [(3, 90), (1, 45), (2, 0)]
    got = g.glcm(q, w, h, L, dts, pixel_levels=L)[0]
    assert np.array_equal(got, want(q, w, h, L, dts, pixel_levels=L))
    bad = q.copy()
    bad[-1] = L  # a value >= levels on the last shard (image.hpp:46-48)
    with pytest.raises(ValueError, match="exceeds gray level"):
        g.glcm(bad, w, h, L, dts, pixel_levels=L)


@pytest.mark.gpu
def test_group_band_shards():
    from paper_1710_06189_b200 import texforge as tf
    g = tf.Group(3, host_reduce=True)
    w, h, L, nb = 300, 200, 32, 7
    bands = np.concatenate([tf.synth_noise(w, h, b + 1).pixels for b in range(nb)])
    dts = [(1, a) for a in ANGLES]
    got = g.glcm(bands, w, h, L, dts, n_bands=nb)
    for b in range(nb):
        assert np.array_equal(got[b], want(bands[b * w * h:(b + 1) * w * h], w, h, L, dts)), b


@pytest.mark.gpu
@pytest.mark.parametrize("G", [1, 3])
def test_group_chunked_and_failure_index(G):
    from paper_1710_06189_b200 import texforge as tf
    g = tf.Group(G, host_reduce=G > 1)
    w, h, L = 257, 301, 64
    gray = tf.synth_smooth(w, h, 3).pixels
    q = O.quantize(gray, L)
    img = tf.QuantizedImage(w, h, L, q)
    dts = [(2, 45), (1, 90)]
    got = g.chunked(tf.MemoryChunkSource(img), dts, 7, L, L)
    assert np.array_equal(got, want(q, w, h, L, dts, pixel_levels=L))

    class Failing(tf.MemoryChunkSource):
        def fetch(self, spec, out):
            if spec.index == 5:
                raise RuntimeError("disk gone")
            return super().fetch(spec, out)

    with pytest.raises(tf.PipelineError) as e:
        g.chunked(Failing(img), dts, 7, L, L)
    assert e.value.chunk_index == 5


@pytest.mark.gpu
def test_comm_single_rank_nccl():
    import torch
    from paper_1710_06189_b200 import texforge as tf
    eng = tf.Engine(0)
    c = tf.Comm(eng, 1, 0, tf.Comm.unique_id())
    s = torch.cuda.current_stream().cuda_stream
    counts = torch.arange(4096, dtype=torch.int64, device="cuda")
    c.reduce_counts(counts.data_ptr(), counts.numel(), 0, s)
    slab = torch.arange(64 * 10, dtype=torch.int64, device="cuda").to(torch.uint8)
    before = slab.clone()
    c.exchange_halo(slab.data_ptr(), 64, 8, 2, s)  # one rank: nothing to exchange
    vals = torch.tensor([1.5, -2.0], dtype=torch.float64, device="cuda")
    c.allreduce_max_f64(vals.data_ptr(), 2, s)
    torch.cuda.synchronize()
    assert torch.equal(counts.cpu(), torch.arange(4096, dtype=torch.int64))
    assert torch.equal(slab, before)
    assert vals.cpu().tolist() == [1.5, -2.0]
    c.close()
