"""Per-launch fixed cost of the vote kernel: K back-to-back launches of a tiny
image captured in one CUDA graph (no host gaps), vs the same for a full image.
python tools/launch_overhead.py [--levels 256] [--rows 16] [--k 50]"""
import argparse
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1710_06189_b200 import _lib as L  # noqa: E402
from paper_1710_06189_b200 import texforge as tf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--levels", type=int, default=256)
    ap.add_argument("--width", type=int, default=16384)
    ap.add_argument("--rows", default="8,64,512,4096,16384")
    ap.add_argument("--k", type=int, default=24)
    a = ap.parse_args()
    eng = tf.Engine(0)
    lib = L.load()
    res = {}
    for rows in [int(x) for x in a.rows.split(",")]:
        img = torch.from_numpy(tf.synth_noise(a.width, rows, 1).pixels).cuda()
        acc = torch.zeros(a.levels * a.levels, dtype=torch.int64, device="cuda")
        s = torch.cuda.Stream()
        def launches():
            for i in range(a.k):
                L.check(lib.tfg_glcm_async(eng.handle, C.c_void_p(img.data_ptr()), a.width, rows, a.width, rows, 256,
                                           a.levels, 1, 0, 0, C.c_void_p(acc.data_ptr()), C.c_void_p(s.cuda_stream)))
        with torch.cuda.stream(s):
            launches()  # warm-up (kernel attributes, scratch)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            launches()
        torch.cuda.synchronize()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        per = e0.elapsed_time(e1) / 5 / a.k * 1000
        res[rows] = {"us_per_launch": per, "pairs_per_launch": a.width * rows}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
