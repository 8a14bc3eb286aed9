"""Does an H2D copy overlap the vote kernels? Times (a) a 256 MiB pinned H2D
alone, (b) 12 vote launches alone, (c) both on separate streams, for L=256
(cooperative launch) and L=32 (plain launch)."""
import ctypes as C
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1710_06189_b200 import _lib as L  # noqa: E402
from paper_1710_06189_b200 import texforge as tf  # noqa: E402


def main():
    n = 16384
    eng = tf.Engine(0)
    lib = L.load()
    img = torch.from_numpy(tf.synth_noise(n, n, 1).pixels)
    pinned = img.pin_memory()
    dev = img.cuda()
    dst = torch.empty_like(dev)
    acc = torch.zeros(256 * 256, dtype=torch.int64, device="cuda")
    s_copy, s_exec = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    dts = [(d, a) for d in (1, 2, 4) for a in (0, 45, 90, 135)]

    def votes(levels, s):
        for d, a in dts:
            L.check(lib.tfg_glcm_async(eng.handle, C.c_void_p(dev.data_ptr()), n, n, n, n, 256, levels, d, a, 0,
                                       C.c_void_p(acc.data_ptr()), C.c_void_p(s.cuda_stream)))

    def timed(fn):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t) * 1e3

    for levels in (256, 32):
        for _ in range(2):
            copy_ms = timed(lambda: dst.copy_(pinned, non_blocking=True))
            vote_ms = timed(lambda: votes(levels, s_exec))

            def both():
                with torch.cuda.stream(s_copy):
                    dst.copy_(pinned, non_blocking=True)
                votes(levels, s_exec)
            both_ms = timed(both)
        out[f"L{levels}"] = {"copy_ms": copy_ms, "votes_ms": vote_ms, "both_ms": both_ms}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
