"""Pins the oracle (oracle/glcm_oracle.c) before it is trusted as the checker:
against the reference's own known-answer tests (cited per test) and against
golden vectors produced by the reference itself (tests/golden/make_golden.py).
CPU only."""
import itertools

import numpy as np
import pytest

from oracle import oracle as O

ANGLES = (0, 45, 90, 135)


def brute_force(img, w, h, levels, d, theta):
    """Independent predicate scan, R/tests/oracle.hpp:19-48 (numpy restatement)."""
    dr, dc = {0: (0, d), 45: (d, -d), 90: (d, 0), 135: (d, d)}[theta]
    a = img.reshape(h, w).astype(np.int64)
    out = np.zeros((levels, levels), dtype=np.uint64)
    for r in range(h):
        for c in range(w):
            r2, c2 = r + dr, c + dc
            if 0 <= r2 < h and 0 <= c2 < w:
                out[a[r2, c2], a[r, c]] += 1
    return out.reshape(-1)


def test_valid_pair_count_closed_forms():  # R/tests/test_glcm.cpp:28-35
    assert O.valid_pair_count(4, 4, 1, 0) == 12
    assert O.valid_pair_count(4, 4, 1, 45) == 9
    assert O.valid_pair_count(1024, 1024, 4, 135) == 1040400
    assert O.valid_pair_count(7, 5, 1, 90) == 28
    with pytest.raises(O.OracleError):
        O.valid_pair_count(4, 4, 4, 0)
    with pytest.raises(O.OracleError):
        O.valid_pair_count(8, 3, 3, 90)


def test_constant_image_and_hand_2x2():  # test_glcm.cpp:37-51
    g = O.glcm_serial(np.full(16, 3, np.uint8), 4, 4, 8, 1, 0)
    assert g[3 * 8 + 3] == 12 and g.sum() == 12
    g = O.glcm_serial(np.array([0, 1, 1, 0], np.uint8), 2, 2, 2, 1, 0)
    assert g[1 * 2 + 0] == 1 and g[0 * 2 + 1] == 1 and g.sum() == 2


def test_rejects_bad_inputs():  # test_glcm.cpp:53-57
    img = np.zeros(16, np.uint8)
    with pytest.raises(O.OracleError):
        O.glcm_serial(img, 4, 4, 8, 4, 0)
    with pytest.raises(O.OracleError):
        O.glcm_serial(np.full(16, 9, np.uint8), 4, 4, 8, 1, 0)  # value >= L


def test_conservation():  # test_glcm.cpp:59-72
    rng = np.random.default_rng(7)
    for _ in range(40):
        w, h = int(rng.integers(2, 14)), int(rng.integers(2, 14))
        L = int(rng.integers(2, 9))
        d = int(rng.integers(1, min(w, h)))
        img = rng.integers(0, L, w * h, dtype=np.uint8)
        for a in ANGLES:
            assert O.glcm_serial(img, w, h, L, d, a).sum() == O.valid_pair_count(w, h, d, a)


def test_permutation_law():  # test_glcm.cpp:87-105
    rng = np.random.default_rng(13)
    L = 5
    img = rng.integers(0, L, 9 * 7, dtype=np.uint8)
    perm = rng.permutation(L).astype(np.uint8)
    for a in ANGLES:
        before = O.glcm_serial(img, 9, 7, L, 2, a).reshape(L, L)
        after = O.glcm_serial(perm[img], 9, 7, L, 2, a).reshape(L, L)
        assert np.array_equal(after[np.ix_(perm, perm)], before)


def test_predicate_scan_exhaustive():  # acceptance.cpp:126-177 (criterion 2)
    for L in (2, 3, 4):
        for code in range(L ** 4):
            px = np.array([(code // L ** k) % L for k in range(4)], np.uint8)
            for a in ANGLES:
                assert np.array_equal(O.glcm_serial(px, 2, 2, L, 1, a), brute_force(px, 2, 2, L, 1, a))
    for code in range(64):
        px = np.array([(code >> b) & 1 for b in range(6)], np.uint8)
        for a in ANGLES:
            assert np.array_equal(O.glcm_serial(px, 3, 2, 2, 1, a), brute_force(px, 3, 2, 2, 1, a))
    rng = np.random.default_rng(424242)
    for _ in range(150):
        w, h, L = int(rng.integers(2, 9)), int(rng.integers(2, 9)), int(rng.integers(2, 5))
        px = rng.integers(0, L, w * h, dtype=np.uint8)
        for d in range(1, min(w, h)):
            for a in ANGLES:
                assert np.array_equal(O.glcm_serial(px, w, h, L, d, a), brute_force(px, w, h, L, d, a))


def test_symmetrize_normalize_kats():  # test_glcm.cpp:123-151
    g = np.array([3, 0, 1, 2], np.uint64)
    assert list(O.symmetrize(g, 2)) == [6, 1, 1, 4]
    assert list(O.symmetrize(np.array([2, 5, 5, 1], np.uint64), 2)) == [4, 10, 10, 2]
    p = O.normalize(g, 2)
    assert p[0] == pytest.approx(0.5) and p[1] == 0.0
    assert p[2] == pytest.approx(1 / 6) and p[3] == pytest.approx(1 / 3)
    single = np.zeros(16, np.uint64)
    single[2 * 4 + 1] = 77
    assert O.normalize(single, 4)[9] == 1.0
    with pytest.raises(O.OracleError):
        O.normalize(np.zeros(4, np.uint64), 2)


def test_features_kats():  # test_features.cpp:22-91, acceptance criterion 9
    f = O.features(np.full(16, 1 / 16), 4)
    assert f[0] == pytest.approx(1 / 16, rel=1e-12) and f[3] == pytest.approx(4.0, rel=1e-12)
    pm = np.zeros(9)
    pm[4] = 1.0
    assert list(O.features(pm, 3)) == [1.0, 0.0, 1.0, 0.0, 0.0]
    f = O.features(np.array([0.5, 0, 0, 0.5]), 2)
    assert f[1] == 0.0 and f[4] == pytest.approx(1.0, rel=1e-12)
    with pytest.raises(O.OracleError):
        O.features(np.array([0.5, 0.5, 0.5, 0.5]), 2)


def test_quantize_kats():  # test_image.cpp:73-91
    assert list(O.quantize(np.array([255, 0, 32], np.uint8), 8)) == [7, 0, 1]
    ramp = np.arange(256, dtype=np.uint8)
    for L in (2, 8, 32, 101, 256):
        q = O.quantize(ramp, L)
        assert np.all(np.diff(q.astype(int)) >= 0) and q[-1] == L - 1
    assert np.array_equal(O.quantize(ramp, 256), ramp)


def test_partition_kats():  # test_pipeline.cpp:45-107
    s = O.partition(1024, 1024, 1, 90, 4)
    assert [list(r) for r in s] == [[0, 256, 257], [256, 512, 513], [512, 768, 769], [768, 1024, 1024]]
    assert [list(r) for r in O.partition(64, 64, 3, 135, 1)] == [[0, 64, 64]]
    s = O.partition(16, 10, 1, 90, 3)
    assert [int(r[1] - r[0]) for r in s] == [4, 3, 3]
    for bad in [(8, 8, 1, 90, 0), (8, 8, 1, 90, 9), (8, 8, 4, 90, 2), (8, 8, 8, 90, 1)]:
        with pytest.raises(O.OracleError):
            O.partition(*bad)


def test_plan_kats():  # test_parallel.cpp:22-56
    assert O.plan(32, 49152) == (6, 2, False)
    assert O.plan(8, 49152) == (8, 2, False)
    assert O.plan(256, 49152) == (1, 1, True)


def test_chunked_equals_serial():  # test_pipeline.cpp:109-125
    rng = np.random.default_rng(41)
    img = rng.integers(0, 8, 37 * 29, dtype=np.uint8)
    for a, d in itertools.product(ANGLES, (1, 4)):
        want = O.glcm_serial(img, 37, 29, 8, d, a)
        for k in (1, 2, 3, 5):
            if 29 // k <= d and k > 1:
                continue
            assert np.array_equal(O.glcm_chunked(img, 37, 29, 8, d, a, k), want)


def test_stats_tie_break():  # test_parallel.cpp:184-198
    g = O.glcm_serial(np.array([0, 1, 1, 0], np.uint8), 2, 2, 2, 1, 0)
    assert O.stats(g, 2) == (2, 1, (0, 1))


def test_golden_small_cases(small_cases):
    """Every small case recorded from the reference: counts, normalize bits, features."""
    for c in small_cases:
        if c["pixel_levels"] == 256:
            got = O.glcm_gray(c["pixels"], c["w"], c["h"], c["L"], c["d"], c["theta"])
        else:
            got = O.glcm_serial(c["pixels"], c["w"], c["h"], c["L"], c["d"], c["theta"])
        assert np.array_equal(got, c["counts"]), c
        if got.sum():
            p = O.normalize(got, c["L"])
            assert np.array_equal(p.view(np.uint64), c["probs"].view(np.uint64))
            if not np.isnan(c["feats"]).any():
                assert np.array_equal(O.features(p, c["L"]), c["feats"])  # same op order: exact


def test_golden_hashes_c1_c2(golden_hashes):
    from paper_1710_06189_b200 import texforge as tf
    recs = [r for r in golden_hashes["glcm"] if r["size"] in (512, 4096)]
    cache = {}
    for r in recs:
        key = (r["kind"], r["size"], r["seed"])
        if key not in cache:
            cache.clear()
            cache[key] = (tf.synth_noise if r["kind"] == "noise" else tf.synth_smooth)(r["size"], r["size"],
                                                                                       r["seed"]).pixels
        g = O.glcm_gray(cache[key], r["size"], r["size"], r["levels"], r["d"], r["theta"])
        assert O.fnv1a64(g) == r["fnv"], r
        assert list(O.stats(g, r["levels"])) == [r["total"], r["hottest_votes"], tuple(r["hottest"])]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_oracle_matches_reference_library():
    """Random cases: restatement == the reference headers (serial, privatized, shared, chunked)."""
    import ctypes as C
    r = O.ref()
    rng = np.random.default_rng(99)
    p8 = lambda a: a.ctypes.data_as(C.POINTER(C.c_uint8))  # noqa: E731
    p64 = lambda a: a.ctypes.data_as(C.POINTER(C.c_uint64))  # noqa: E731
    for _ in range(60):
        w, h = int(rng.integers(3, 60)), int(rng.integers(3, 50))
        L = int(rng.integers(2, 40))
        d = int(rng.integers(1, min(w, h)))
        a = ANGLES[int(rng.integers(0, 4))]
        img = rng.integers(0, L, w * h, dtype=np.uint8)
        want = O.glcm_serial(img, w, h, L, d, a)
        for fn, extra in ((r.ref_glcm_serial, ()), (r.ref_glcm_privatized, (3, 4)), (r.ref_glcm_shared, (3,))):
            out = np.zeros(L * L, np.uint64)
            assert fn(p8(img), w, h, L, d, a, *extra, p64(out)) == 0
            assert np.array_equal(out, want)
        k = int(rng.integers(1, 4))
        if h // k > d or k == 1:
            out = np.zeros(L * L, np.uint64)
            assert r.ref_glcm_chunked(p8(img), w, h, L, d, a, k, 2, 0, p64(out)) == 0
            assert np.array_equal(out, want)
            assert np.array_equal(O.glcm_chunked(img, w, h, L, d, a, k), want)


def test_product_synth_bit_identical(golden_hashes):
    """The engine's host input generators reproduce the reference's synth_* bytes."""
    from paper_1710_06189_b200 import texforge as tf
    for r in golden_hashes["synth"]:
        if r["kind"] == "smooth" and r["w"] * r["h"] > 4096 * 4096:
            continue  # noise is generated on every host thread (mt19937 jump-ahead): 16384^2 in ~0.3 s
        img = (tf.synth_noise if r["kind"] == "noise" else tf.synth_smooth)(r["w"], r["h"], r["seed"]).pixels
        assert O.fnv1a64_image(img) == r["fnv_u64view"], r
