"""Small engine workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): every vote layout, the PACKED16 drain path (constant
image), the cooperative in-kernel reduce with the shared tail pool, band
batches, the split-K reduce (more bands than SM slots), the multi-(d, theta)
fork, async calls from two streams sharing the context's scratch, and the
post-processing kernels. Each result is checked against the C oracle.

  compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_1710_06189_b200 import _lib as L  # noqa: E402
from paper_1710_06189_b200 import texforge as tf  # noqa: E402


def main():
    import torch
    eng = tf.Engine(0)
    w, h = 1500, 160  # >= 66 segments per row: main (unmasked) + edge passes
    noise = tf.synth_noise(w, h, 3).pixels
    smooth = tf.synth_smooth(w, h, 3).pixels
    const = np.full(w * h, 200, np.uint8)
    dts = [(1, 0), (2, 45), (3, 90), (1, 135)]
    n = 0
    for img in (noise, smooth, const):
        for levels, strats in ((8, (1, 2, 3, 4)), (32, (1, 3)), (64, (2,)), (128, (3,)), (256, (4,))):
            for s in strats:
                got = eng.glcm(img, w, h, levels, dts, flags=L.strategy_flag(s))
                for t, (d, a) in enumerate(dts):
                    assert np.array_equal(got[0, t].reshape(-1), O.glcm_gray(img, w, h, levels, d, a)), (levels, s)
                n += 1
    # bands: 3 bands (cooperative) and 400 bands (> SM slots: split-K reduce kernel)
    for nb, levels in ((3, 256), (400, 256), (5, 32)):
        bw, bh = 256, 40
        bands = np.concatenate([tf.synth_noise(bw, bh, b + 1).pixels for b in range(nb)])
        got = eng.glcm(bands, bw, bh, levels, [(1, 45)], n_bands=nb)
        for b in (0, nb // 2, nb - 1):
            assert np.array_equal(got[b, 0].reshape(-1),
                                  O.glcm_gray(bands[b * bw * bh:(b + 1) * bw * bh], bw, bh, levels, 1, 45))
        n += 1
    # async from two streams sharing the context's partials + counters (L > 64)
    pitch = (w + 15) // 16 * 16  # device entry points need a 16-byte row pitch
    padded = np.zeros((h, pitch), np.uint8)
    padded[:, :w] = noise.reshape(h, w)
    dev = torch.from_numpy(padded).cuda()
    outs = [torch.zeros(256 * 256, dtype=torch.int64, device="cuda") for _ in range(2)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for rep in range(3):
        for i, st in enumerate(streams):
            L.check(eng._lib.tfg_glcm_async(eng.handle, C.c_void_p(dev.data_ptr()), w, h, pitch, h, 256, 256, 1 + i,
                                            45 * i, 0, C.c_void_p(outs[i].data_ptr()), C.c_void_p(st.cuda_stream)))
    torch.cuda.synchronize()
    for i in range(2):
        want = O.glcm_gray(noise, w, h, 256, 1 + i, 45 * i) * np.uint64(3)
        assert np.array_equal(outs[i].cpu().numpy().view(np.uint64), want), i
    # post-processing
    g = eng.glcm(noise, w, h, 32, [(1, 0)], want_probs=True, want_features=True)
    n += 1
    print(f"sanitize workload ok: {n} engine calls, {eng.launches} kernel launches")
    del dev, outs, streams
    eng.close()  # frees every device / pinned buffer, so the leak check sees only real leaks
    torch.cuda.synchronize()
    # torch's caching allocator keeps its blocks until empty_cache(); without
    # this the leak check reports torch's own cached 2 MB block
    import gc
    gc.collect()
    torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
