"""Golden pins for the large / multi-GPU configs, produced by the REFERENCE ITSELF.

Same recipe as make_golden.py (oracle/_ref/libtexforge_ref.so = the unmodified
reference headers, R/include/texforge/*.hpp): the reference's synth_noise /
synth_smooth (image.hpp:76-116), quantize (image.hpp:55-62) and
compute_glcm_privatized (parallel.hpp:240-254; its counts equal
compute_glcm_serial's, glcm.hpp:144-147, which the small cases pin) on all
host threads. Writes golden_large.json:

  c5      — synth_noise(65536, 65536, 1), L=64, d=1, 4 theta (BASELINE config 5;
            the image bench.py --workload c5 row-partitions over N GPUs, so the
            same hashes pin every N);
  c3_smooth_d — synth_smooth(16384, 16384, 1), L=256, d in {2, 4}, 4 theta
            (Appendix A stops at d=1 for smooth);
  c3_blocks — the weak-scaling c3 image of N 16384-row blocks, block b =
            synth_<kind>(16384, 16384, 1 + b) stacked top to bottom
            (bench.py rows-weak layout), N in {2, 4, 8}, L=256, d in {1, 2, 4}, 4 theta,
            noise and smooth: the bit-exact gate of bench.py at N > 1.

Run in the dev container (needs /root/reference; ~10-20 min on 8 cores):
    python tests/golden/make_golden_large.py [c5] [c3_smooth_d] [c3_blocks]
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(HERE, "golden_large.json")
ANGLES = (0, 45, 90, 135)
THREADS = os.cpu_count() or 1


def p8(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def synth(kind, w, h, seed):
    out = np.empty(w * h, dtype=np.uint8)
    fn = O.ref().ref_synth_noise if kind == "noise" else O.ref().ref_synth_smooth
    assert fn(w, h, seed, p8(out)) == 0
    return out


def quantize(gray, w, h, levels):
    out = np.empty(w * h, dtype=np.uint8)
    assert O.ref().ref_quantize(p8(gray), w, h, levels, p8(out)) == 0
    return out


def glcm(q, w, h, levels, d, theta):
    """compute_glcm_privatized on a persistent QuantizedImage (all host threads)."""
    out = np.zeros(levels * levels, dtype=np.uint64)
    hd = O.ref().ref_image_new(p8(q), w, h, levels)
    assert hd, O.ref().ref_last_error()
    try:
        rc = O.ref().ref_image_glcm(hd, d, theta, THREADS, 1, out.ctypes.data_as(C.POINTER(C.c_uint64)))
        assert rc == 0, O.ref().ref_last_error()
    finally:
        O.ref().ref_image_free(hd)
    return out


def rec(g, levels, **kw):
    total, hv, (r, c) = O.stats(g, levels)
    return dict(kw, levels=levels, total=total, hottest=[r, c], hottest_votes=hv, fnv=O.fnv1a64(g))


def load():
    if os.path.exists(OUT):
        with open(OUT) as f:
            return json.load(f)
    return {}


def save(d):
    with open(OUT, "w") as f:
        json.dump(d, f, indent=1)


def c5(db):
    w = h = 65536
    t = time.time()
    gray = synth("noise", w, h, 1)
    print(f"c5 synth {time.time() - t:.0f}s", flush=True)
    q = quantize(gray, w, h, 64)
    del gray
    out = []
    for th in ANGLES:
        t = time.time()
        g = glcm(q, w, h, 64, 1, th)
        out.append(rec(g, 64, kind="noise", width=w, height=h, seed=1, d=1, theta=th))
        print(f"c5 theta={th} {out[-1]['fnv']} {time.time() - t:.0f}s", flush=True)
    db["c5"] = out


def c3_smooth_d(db):
    n = 16384
    q = quantize(synth("smooth", n, n, 1), n, n, 256)
    out = []
    for d in (2, 4):
        for th in ANGLES:
            g = glcm(q, n, n, 256, d, th)
            out.append(rec(g, 256, kind="smooth", width=n, height=n, seed=1, d=d, theta=th))
            print(f"c3 smooth d={d} theta={th} {out[-1]['fnv']}", flush=True)
    db["c3_smooth_d"] = out


def c3_blocks(db):
    n = 16384
    out = []
    for kind in ("noise", "smooth"):
        blocks = [synth(kind, n, n, 1 + b) for b in range(8)]
        for nb in (2, 4, 8):
            img = np.concatenate(blocks[:nb])
            for d in (1, 2, 4):
                for th in ANGLES:
                    t = time.time()
                    g = glcm(img, n, nb * n, 256, d, th)
                    out.append(rec(g, 256, kind=kind, width=n, height=nb * n, blocks=nb, block_rows=n, seed0=1,
                                   d=d, theta=th))
                    print(f"c3 blocks {kind} N={nb} d={d} theta={th} {out[-1]['fnv']} {time.time() - t:.0f}s",
                          flush=True)
            del img
        del blocks
    db["c3_blocks"] = out


if __name__ == "__main__":
    if not os.path.isdir("/root/reference/proj/include"):
        sys.exit("needs /root/reference (dev container only)")
    O.build()
    parts = sys.argv[1:] or ["c3_smooth_d", "c5", "c3_blocks"]
    for part in parts:
        db = load()
        {"c5": c5, "c3_smooth_d": c3_smooth_d, "c3_blocks": c3_blocks}[part](db)
        save(db)
