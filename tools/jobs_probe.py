"""Where a multi-job launch loses time: each (d, theta) alone (tfg_glcm_async)
vs the same set as one multi-job launch (tfg_glcm_jobs_async), on a resident
16384^2 image. max(single) vs the jobs launch shows the row imbalance behind
the shared grid barrier; identical jobs isolate the kernel's own cost.
python tools/jobs_probe.py [--levels 256] [--kind noise|smooth]"""
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
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--kinds", default="noise,smooth")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    eng = tf.Engine(0)
    lib = L.load()
    n, lv = a.n, a.levels
    s = torch.cuda.Stream()
    out = {}
    c3 = [(d, t) for d in (1, 2, 4) for t in (0, 45, 90, 135)]
    sets = {"c3_first8": c3[:8], "c3_last4": c3[8:], "same8_d1_0": [(1, 0)] * 8, "same8_d2_45": [(2, 45)] * 8,
            "same4_d1_0": [(1, 0)] * 4, "c3_d1": c3[:4], "c3_d2": c3[4:8]}
    for kind in a.kinds.split(","):
        gen = tf.synth_noise if kind == "noise" else tf.synth_smooth
        img = torch.from_numpy(gen(n, n, 1).pixels).cuda()
        acc = torch.zeros(8 * lv * lv, dtype=torch.int64, device="cuda")

        def timed(fn):
            with torch.cuda.stream(s):
                for _ in range(2):
                    fn()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(a.reps):
                    fn()
                e1.record(s)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / a.reps * 1000.0

        single = {}
        for (d, t) in sorted(set(c3)):
            single[f"{d},{t}"] = timed(lambda: L.check(lib.tfg_glcm_async(
                eng.handle, C.c_void_p(img.data_ptr()), n, n, n, n, 256, lv, d, t, 0, C.c_void_p(acc.data_ptr()),
                C.c_void_p(s.cuda_stream))))
        res = {"single_us": single}
        for name, jobs in sets.items():
            k = len(jobs)
            lvs = (C.c_int * k)(*([lv] * k))
            dd = (C.c_int * k)(*[j[0] for j in jobs])
            aa = (C.c_int * k)(*[j[1] for j in jobs])
            us = timed(lambda: L.check(lib.tfg_glcm_jobs_async(
                eng.handle, C.c_void_p(img.data_ptr()), n, n, n, n * n, 1, n, 256, lvs, dd, aa, k, 0,
                C.c_void_p(acc.data_ptr()), C.c_void_p(s.cuda_stream))))
            singles = [single[f"{d},{t}"] for d, t in jobs]
            res[name] = {"jobs_us": us, "sum_single_us": sum(singles), "max_single_us": max(singles),
                         "jobs_per_job_us": us / k}
        out[kind] = res
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
