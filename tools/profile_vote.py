"""Launches the hot-path vote kernels for ncu / quick timing.

  python tools/profile_vote.py [--size 16384] [--levels 256] [--kinds noise,smooth]
                               [--dts 1:0,1:45] [--reps 3] [--strategy 0] [--time]

With --time prints per-(input, d, theta) CUDA-event times and the achieved
GB/s against the algorithmic bytes (image once + u64 GLCM)."""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1710_06189_b200 import _lib as L  # noqa: E402
from paper_1710_06189_b200 import texforge as tf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=16384)
    ap.add_argument("--levels", type=int, default=256)
    ap.add_argument("--kinds", default="noise,smooth")
    ap.add_argument("--dts", default="1:0")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--strategy", type=int, default=0)
    ap.add_argument("--time", action="store_true")
    ap.add_argument("--multi", action="store_true", help="one tfg_glcm_multi_async call for all --dts")
    ap.add_argument("--scheme1", action="store_true", help="K0: one global atomic per pair (Scheme 1 ablation)")
    a = ap.parse_args()
    xflags = L.TFG_SCHEME_GLOBAL if a.scheme1 else 0
    n, levels = a.size, a.levels
    eng = tf.Engine(0)
    lib = L.load()
    dts = [tuple(int(x) for x in t.split(":")) for t in a.dts.split(",")]
    acc = torch.zeros(levels * levels, dtype=torch.int64, device="cuda")
    res = {}
    for kind in a.kinds.split(","):
        img = (tf.synth_noise if kind == "noise" else tf.synth_smooth)(n, n, 1).pixels
        dev = torch.from_numpy(img).cuda()
        if a.multi:
            nd = len(dts)
            dd = (C.c_int * nd)(*[x[0] for x in dts])
            aa = (C.c_int * nd)(*[x[1] for x in dts])
            accm = torch.zeros(nd * levels * levels, dtype=torch.int64, device="cuda")
            times = []
            for r in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                L.check(lib.tfg_glcm_multi_async(eng.handle, C.c_void_p(dev.data_ptr()), n, n, n, n * n, 1, n, 256,
                                                 levels, dd, aa, len(dts), L.strategy_flag(a.strategy) | xflags,
                                                 C.c_void_p(accm.data_ptr()), None))
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
            t = sorted(times)[len(times) // 2]
            res[f"{kind} multi{nd}"] = {"ms": t, "GBps": nd * (n * n + levels * levels * 8) / (t / 1e3) / 1e9}
            continue
        for d, th in dts:
            times = []
            for r in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                L.check(lib.tfg_glcm_async(eng.handle, C.c_void_p(dev.data_ptr()), n, n, n, n, 256, levels, d, th,
                                           L.strategy_flag(a.strategy) | xflags, C.c_void_p(acc.data_ptr()), None))
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
            t = sorted(times)[len(times) // 2]
            res[f"{kind} d{d} t{th}"] = {"ms": t, "GBps": (n * n + levels * levels * 8) / (t / 1e3) / 1e9}
    if a.time:
        print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
