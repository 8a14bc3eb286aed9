"""Generates the golden fixtures by running the REFERENCE ITSELF.

Builds oracle/_ref/libtexforge_ref.so from the unmodified headers under
/root/reference/proj/include (oracle/Makefile) and records its outputs:

  golden_hashes.json — FNV-1a-64 digests of synth images and of the GLCM counts
                       for the BASELINE configs (extended),
                       plus total / hottest cell per config.
  small_cases.npz    — full GLCMs (and their inputs) for ~500 small random cases:
                       odd sizes, every theta, d up to min(W,H)-1, L in
                       {2..256 incl. non powers of two}, gray and pre-quantised
                       inputs; normalize() bits and extract_features() values.

Run in the dev container (needs /root/reference):  python tests/golden/make_golden.py
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
ANGLES = (0, 45, 90, 135)


def p8(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def p64(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def pd(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def ref_synth(kind, w, h, seed):
    out = np.empty(w * h, dtype=np.uint8)
    fn = O.ref().ref_synth_noise if kind == "noise" else O.ref().ref_synth_smooth
    assert fn(w, h, seed, p8(out)) == 0
    return out


def ref_quantize(gray, w, h, levels):
    out = np.empty(w * h, dtype=np.uint8)
    assert O.ref().ref_quantize(p8(gray), w, h, levels, p8(out)) == 0
    return out


def ref_glcm(q, w, h, levels, d, theta):
    out = np.zeros(levels * levels, dtype=np.uint64)
    rc = O.ref().ref_glcm_serial(p8(q), w, h, levels, d, theta, p64(out))
    assert rc == 0, O.ref().ref_last_error()
    return out


def stats(g, levels):
    best = int(np.argmax(g))
    return int(g.sum(dtype=np.uint64)), [best // levels, best % levels], int(g[best])


def hashes():
    recs = {"synth": [], "glcm": []}
    # synth digests (u64-view FNV, oracle.fnv1a64_image)
    for kind in ("noise", "smooth"):
        for (w, h, s) in [(64, 64, 1), (513, 77, 3), (4096, 4096, 1), (16384, 16384, 1), (2048, 2048, 2)]:
            t = time.time()
            img = ref_synth(kind, w, h, s)
            recs["synth"].append({"kind": kind, "w": w, "h": h, "seed": s, "fnv_u64view": O.fnv1a64_image(img)})
            print(f"synth {kind} {w}x{h} s{s} {time.time()-t:.1f}s", flush=True)
    configs = []
    configs.append(("noise", 512, 1, 8, [1], [0]))
    for kind in ("noise", "smooth"):
        for L in (16, 32):
            configs.append((kind, 4096, 1, L, [1], list(ANGLES)))
    configs.append(("noise", 16384, 1, 256, [1, 2, 4], list(ANGLES)))
    configs.append(("smooth", 16384, 1, 256, [1], list(ANGLES)))
    # C4 sample: bands b -> synth_noise(2048, 2048, b+1), L=32; + smooth variant
    for b in range(4):
        configs.append(("noise", 2048, b + 1, 32, [1], list(ANGLES)))
    configs.append(("smooth", 2048, 1, 32, [1], list(ANGLES)))
    # other L on the big image (N = 8..256 target)
    for L in (8, 16, 32, 64):
        configs.append(("noise", 16384, 1, L, [1], [0]))
        configs.append(("smooth", 16384, 1, L, [1], [0, 45]))
    cache = {}
    for kind, n, seed, L, ds, thetas in configs:
        key = (kind, n, seed)
        if key not in cache:
            cache.clear()
            cache[key] = ref_synth(kind, n, n, seed)
        q = ref_quantize(cache[key], n, n, L)
        for d in ds:
            for th in thetas:
                t = time.time()
                g = ref_glcm(q, n, n, L, d, th)
                total, hot, hv = stats(g, L)
                recs["glcm"].append({"kind": kind, "size": n, "seed": seed, "levels": L, "d": d, "theta": th,
                                     "total": total, "hottest": hot, "hottest_votes": hv, "fnv": O.fnv1a64(g)})
                print(f"glcm {kind} {n} s{seed} L{L} d{d} t{th} {recs['glcm'][-1]['fnv']} {time.time()-t:.1f}s",
                      flush=True)
    with open(os.path.join(OUT, "golden_hashes.json"), "w") as f:
        json.dump(recs, f, indent=1)


def small_cases():
    rng = np.random.default_rng(20171017)
    imgs, meta, counts, probs, feats = [], [], [], [], []
    levels_pool = [2, 3, 4, 5, 7, 8, 13, 16, 31, 32, 33, 64, 100, 101, 128, 200, 255, 256]
    for i in range(520):
        w = int(rng.integers(2, 48))
        h = int(rng.integers(2, 40))
        if i % 13 == 0:
            w = int(rng.integers(2, 5))
        L = int(levels_pool[i % len(levels_pool)])
        d = int(rng.integers(1, min(w, h)))
        th = ANGLES[i % 4]
        gray_input = (i % 3) != 0
        if gray_input:
            gray = rng.integers(0, 256, size=w * h, dtype=np.uint8)
            if i % 7 == 0:  # smooth-ish ramp
                gray = ((np.arange(w * h) // max(1, w // 3)) % 256).astype(np.uint8)
            q = ref_quantize(gray, w, h, L)
            px, pl = gray, 256
        else:
            q = rng.integers(0, L, size=w * h, dtype=np.uint8) if i % 5 else np.full(w * h, L - 1, np.uint8)
            px, pl = q, L
        g = ref_glcm(q, w, h, L, d, th)
        pr = np.zeros(L * L)
        ft = np.full(5, np.nan)
        if g.sum() > 0:
            assert O.ref().ref_normalize(p64(g), L, pd(pr)) == 0
            if O.ref().ref_features(pd(pr), L, pd(ft)) != 0:
                ft[:] = np.nan
        imgs.append(px)
        meta.append([w, h, L, d, th, pl])
        counts.append(g)
        probs.append(pr)
        feats.append(ft)
    off_i = np.cumsum([0] + [x.size for x in imgs])
    off_c = np.cumsum([0] + [x.size for x in counts])
    np.savez_compressed(os.path.join(OUT, "small_cases.npz"),
                        meta=np.array(meta, dtype=np.int64), pixels=np.concatenate(imgs), pix_off=off_i,
                        counts=np.concatenate(counts), cnt_off=off_c, probs=np.concatenate(probs),
                        feats=np.array(feats))
    print("small cases:", len(meta))


if __name__ == "__main__":
    if not os.path.isdir("/root/reference/proj/include"):
        sys.exit("needs /root/reference (dev container only)")
    O.build()
    small_cases()
    if "--small-only" not in sys.argv:
        hashes()
