"""Where c2's end-to-end step time goes (tfg_glcm_shard_jobs from one pinned
host buffer of two 4096^2 images, 8 (L, d, theta) each): wall-time
distribution of the call vs a plain pinned H2D of the same bytes and vs the
call with no rows to vote (memset + counts back + sync only).
python tools/e2e_c2_diag.py"""
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1710_06189_b200 import texforge as tf  # noqa: E402


def dist(fn, n=60):
    for _ in range(5):
        fn()
    t = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        t.append((time.perf_counter() - t0) * 1e3)
    t.sort()
    return {"min_ms": t[0], "median_ms": statistics.median(t), "p90_ms": t[int(0.9 * len(t))], "max_ms": t[-1]}


def main():
    w = 4096
    eng = tf.Engine(0)
    imgs = [tf.synth_noise(w, w, 1).pixels, tf.synth_smooth(w, w, 1).pixels]
    allk = torch.from_numpy(np.concatenate(imgs)).pin_memory()
    jobs = [(L, 1, a) for L in (16, 32) for a in (0, 45, 90, 135)]
    out = torch.zeros(2 * sum(j[0] ** 2 for j in jobs), dtype=torch.int64).pin_memory().numpy().view(np.uint64)
    px = allk.numpy()
    res = {}
    mode = sys.argv[1] if len(sys.argv) > 1 else ""
    if "graph" in mode:  # the bench's device-resident leg first: one step captured and replayed
        import ctypes as C
        from paper_1710_06189_b200 import _lib as Lb
        lib = Lb.load()
        dev = allk.cuda()
        acc = torch.zeros(2 * sum(j[0] ** 2 for j in jobs), dtype=torch.int64, device="cuda")
        n = len(jobs)
        ll = (C.c_int * n)(*[j[0] for j in jobs])
        dd = (C.c_int * n)(*[j[1] for j in jobs])
        aa = (C.c_int * n)(*[j[2] for j in jobs])
        st = torch.cuda.Stream()

        def step():
            Lb.check(lib.tfg_glcm_jobs_async(eng.handle, C.c_void_p(dev.data_ptr()), w, w, w, w * w, 2, w, 256, ll, dd,
                                             aa, n, 0, C.c_void_p(acc.data_ptr()), C.c_void_p(st.cuda_stream)))
        with torch.cuda.stream(st):
            step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            step()
        for _ in range(20):
            g.replay()
        torch.cuda.synchronize()
    if "engine2" in mode:
        eng2 = tf.Engine(0)
        eng2.synth_noise_device(w, 64, 1)
        torch.cuda.synchronize()
    res["shard_jobs"] = dist(lambda: eng.shard_jobs(px, w, w, w, jobs, n_bands=2, band_stride=w * w, out=out))
    res["shard_jobs_no_rows"] = dist(lambda: eng.shard_jobs(px, w, w, 0, jobs, n_bands=2, band_stride=w * w, out=out))
    def with_sync():
        eng.shard_jobs(px, w, w, w, jobs, n_bands=2, band_stride=w * w, out=out)
        torch.cuda.synchronize()
    res["shard_jobs_then_device_sync"] = dist(with_sync)
    out_np = np.zeros(out.size, dtype=np.uint64)
    res["shard_jobs_pageable_out"] = dist(lambda: eng.shard_jobs(px, w, w, w, jobs, n_bands=2, band_stride=w * w,
                                                                 out=out_np))
    res["shard_2band_L16_4dt"] = dist(lambda: eng.shard(px, w, w, w, 16, [(1, a) for a in (0, 45, 90, 135)],
                                                         n_bands=2, band_stride=w * w, out=out[: 8 * 256]))
    res["shard_2band_L16_4dt_pageable_out"] = dist(lambda: eng.shard(px, w, w, w, 16, [(1, a) for a in (0, 45, 90, 135)],
                                                                      n_bands=2, band_stride=w * w,
                                                                      out=out_np[: 8 * 256]))
    one = allk[: w * w].numpy()
    res["shard_jobs_1band"] = dist(lambda: eng.shard_jobs(one, w, w, w, jobs, n_bands=1, out=out[: out.size // 2]))
    res["shard_jobs_1band_1job"] = dist(lambda: eng.shard_jobs(one, w, w, w, jobs[:1], n_bands=1,
                                                               out=out[: 16 * 16]))
    res["shard_1band_L16_4dt"] = dist(lambda: eng.shard(one, w, w, w, 16, [(1, a) for a in (0, 45, 90, 135)],
                                                         n_bands=1, out=out[: 4 * 256]))
    probe = torch.empty(allk.numel(), dtype=torch.uint8, device="cuda")

    def h2d():
        probe.copy_(allk, non_blocking=True)
        torch.cuda.synchronize()
    res["torch_h2d_32MiB"] = dist(h2d)
    half = allk[: w * w]

    def h2d_two():
        probe[: w * w].copy_(half, non_blocking=True)
        probe[w * w:].copy_(allk[w * w:], non_blocking=True)
        torch.cuda.synchronize()
    res["torch_h2d_2x16MiB"] = dist(h2d_two)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
