"""End-to-end (host-resident) timing diagnostics of tfg_glcm.

Prints, for the 16384^2 L=256 noise image and 12 (d, theta): where the host
buffer lives (tfg_memory_kind), wall time of one tfg_glcm call from pinned
and from pageable memory, and a plain pinned H2D for reference."""
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1710_06189_b200 import _lib as L  # noqa: E402
from paper_1710_06189_b200 import texforge as tf  # noqa: E402


def main():
    n, levels = 16384, 256
    dts = [(d, a) for d in (1, 2, 4) for a in (0, 45, 90, 135)]
    eng = tf.Engine(0)
    lib = L.load()
    img = tf.synth_noise(n, n, 1).pixels
    pinned = torch.from_numpy(img).pin_memory()
    out = {"kind_pinned": lib.tfg_memory_kind(C.c_void_p(pinned.data_ptr())),
           "kind_numpy": lib.tfg_memory_kind(img.ctypes.data_as(C.c_void_p))}
    for name, arr in (("pinned", pinned.numpy()), ("pageable", img)):
        for dsel in (dts[:1], dts):
            eng.glcm(arr, n, n, levels, dsel)
            ts = []
            for _ in range(3):
                t = time.perf_counter()
                eng.glcm(arr, n, n, levels, dsel)
                ts.append(time.perf_counter() - t)
            out[f"{name}_{len(dsel)}dt_ms"] = min(ts) * 1e3
    dev = torch.empty(n * n, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    t = time.perf_counter()
    dev.copy_(pinned)
    torch.cuda.synchronize()
    out["h2d_pinned_ms"] = (time.perf_counter() - t) * 1e3
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
