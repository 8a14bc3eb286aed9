"""Parity of the CUDA path (through the C ABI) with the oracle and with golden
vectors produced by the reference itself. Integer GLCMs: bit-exact.
normalize(): bit-exact. Haralick features: |diff| <= 1e-10 * max(1, |ref|)."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O
from paper_1710_06189_b200 import _lib as L
from paper_1710_06189_b200 import texforge as tf

pytestmark = pytest.mark.gpu
ANGLES = (0, 45, 90, 135)
FEAT_TOL = 1e-10


def _strategies_for(levels):
    """Every vote layout that supports `levels` (tfg_kernels.cuh, enum Strat)."""
    s = [L.STRAT_PACKED16]
    if levels <= 128:
        s.append(L.STRAT_COPY1)
    if levels <= 64:
        s.append(L.STRAT_COPIES8)
        s.append(L.STRAT_P16X16)
    if levels <= 32:
        s.append(L.STRAT_COPIES32)
    return s


def test_golden_small_cases_auto(engine, small_cases):
    for c in small_cases:
        got = engine.glcm(c["pixels"], c["w"], c["h"], c["L"], [(c["d"], c["theta"])],
                          pixel_levels=c["pixel_levels"])
        assert np.array_equal(got.reshape(-1), c["counts"]), c


def test_golden_small_cases_every_strategy(engine, small_cases):
    for c in small_cases[::3]:
        for s in _strategies_for(c["L"]):
            got = engine.glcm(c["pixels"], c["w"], c["h"], c["L"], [(c["d"], c["theta"])],
                              pixel_levels=c["pixel_levels"], flags=L.strategy_flag(s))
            assert np.array_equal(got.reshape(-1), c["counts"]), (s, c["w"], c["h"], c["L"], c["d"], c["theta"])


def test_scheme1_global_atomics_matches(engine, small_cases):
    for c in small_cases[::5]:
        got = engine.glcm(c["pixels"], c["w"], c["h"], c["L"], [(c["d"], c["theta"])],
                          pixel_levels=c["pixel_levels"], flags=L.TFG_SCHEME_GLOBAL)
        assert np.array_equal(got.reshape(-1), c["counts"])


@pytest.mark.parametrize("levels", [2, 5, 8, 16, 32, 64, 101, 128, 181, 256])
def test_random_shapes_vs_oracle(engine, levels):
    rng = np.random.default_rng(levels)
    for trial in range(12):
        w = int(rng.integers(17, 700))
        h = int(rng.integers(2, 90))
        gray = rng.integers(0, 256, size=w * h, dtype=np.uint8)
        ds = sorted(d for d in {1, 2, 4, int(rng.integers(1, min(w, h))), min(w, h) - 1} if d < min(w, h))
        dts = [(d, a) for d in ds for a in ANGLES]
        got = engine.glcm(gray, w, h, levels, dts)
        for t, (d, a) in enumerate(dts):
            want = O.glcm_gray(gray, w, h, levels, d, a)
            assert np.array_equal(got[0, t].reshape(-1), want), (w, h, levels, d, a)


def test_large_distance_every_word_shift(engine):
    # dcol = 16q + 4k + s for every k, s (template KSEL 0..4 and funnel shift)
    rng = np.random.default_rng(7)
    w, h = 333, 61
    gray = rng.integers(0, 256, size=w * h, dtype=np.uint8)
    dts = [(d, a) for d in range(1, 60) for a in (0, 45, 135)]
    got = engine.glcm(gray, w, h, 16, dts)
    for t, (d, a) in enumerate(dts):
        assert np.array_equal(got[0, t].reshape(-1), O.glcm_gray(gray, w, h, 16, d, a)), (d, a)


@pytest.mark.parametrize("levels", [8, 64, 256])
def test_constant_image_all_votes_one_cell(engine, levels):
    # 4096^2 constant: every CTA sees > 2^15 votes on ONE cell (PACKED16 spill path,
    # the run-length shortcut, and the hot-cell case of every strategy).
    w = h = 2048
    v = levels - 1
    img = np.full(w * h, v, dtype=np.uint8)
    for s in _strategies_for(levels):
        for a in ANGLES:
            got = engine.glcm(img, w, h, levels, [(1, a)], pixel_levels=levels, flags=L.strategy_flag(s))
            total = O.valid_pair_count(w, h, 1, a)
            want = np.zeros(levels * levels, dtype=np.uint64)
            want[v * levels + v] = total
            assert np.array_equal(got.reshape(-1), want), (s, a)


def test_two_tone_spill_both_halves(engine):
    # cells (255,0), (0,255), (128,128), (200,3) in both u16 halves with heavy counts
    w, h = 4096, 1024
    rng = np.random.default_rng(3)
    base = np.where(rng.random(w * h) < 0.5, 0, 255).astype(np.uint8)
    base[: w * 300] = 128
    base[w * 600: w * 700] = np.where(np.arange(w * 100) % 7 == 0, 200, 3)
    for s in _strategies_for(256):
        got = engine.glcm(base, w, h, 256, [(d, a) for d in (1, 3) for a in ANGLES], pixel_levels=256,
                          flags=L.strategy_flag(s))
        for t, (d, a) in enumerate([(d, a) for d in (1, 3) for a in ANGLES]):
            assert np.array_equal(got[0, t].reshape(-1), O.glcm_serial(base, w, h, 256, d, a)), (s, d, a)


def test_quantize_kernel(engine):
    rng = np.random.default_rng(1)
    g = rng.integers(0, 256, size=1_000_003, dtype=np.uint8)
    for levels in (2, 8, 32, 101, 255, 256):
        assert np.array_equal(engine.quantize(g, levels), O.quantize(g, levels))


def _hash_cases(golden_hashes, size, kinds=("noise", "smooth")):
    return [r for r in golden_hashes["glcm"] if r["size"] == size and r["kind"] in kinds]


def _check_hashes(engine, recs):
    by_img = {}
    for r in recs:
        by_img.setdefault((r["kind"], r["size"], r["seed"], r["levels"]), []).append(r)
    for (kind, n, seed, levels), rs in by_img.items():
        img = (tf.synth_noise if kind == "noise" else tf.synth_smooth)(n, n, seed).pixels
        dts = [(r["d"], r["theta"]) for r in rs]
        got = engine.glcm(img, n, n, levels, dts)
        for t, r in enumerate(rs):
            g = got[0, t].reshape(-1)
            assert O.fnv1a64(g) == r["fnv"], r
            assert int(g.sum()) == r["total"]
            best = int(np.argmax(g))
            assert [best // levels, best % levels] == r["hottest"] and int(g[best]) == r["hottest_votes"]


def test_appendix_a_c1_c2(engine, golden_hashes):
    _check_hashes(engine, _hash_cases(golden_hashes, 512) + _hash_cases(golden_hashes, 4096))


@pytest.mark.slow
def test_appendix_a_c3_and_bands(engine, golden_hashes):
    _check_hashes(engine, _hash_cases(golden_hashes, 16384) + _hash_cases(golden_hashes, 2048))


def test_bands_batch(engine):
    w, h, nb = 301, 97, 6
    imgs = [tf.synth_noise(w, h, b + 1).pixels for b in range(nb)]
    dts = [(1, a) for a in ANGLES] + [(3, 45)]
    got = engine.glcm(np.concatenate(imgs), w, h, 32, dts, n_bands=nb)
    for b in range(nb):
        for t, (d, a) in enumerate(dts):
            assert np.array_equal(got[b, t].reshape(-1), O.glcm_gray(imgs[b], w, h, 32, d, a)), (b, d, a)


def test_host_stream_pipeline_large(engine):
    # > 32 MiB host image -> the K-chunk copy/compute pipeline (auto K > 1)
    w, h = 8192, 6000
    img = tf.synth_noise(w, h, 5).pixels
    dts = [(1, 0), (2, 45), (4, 90), (1, 135)]
    got = engine.glcm(img, w, h, 64, dts)
    for t, (d, a) in enumerate(dts):
        assert np.array_equal(got[0, t].reshape(-1), O.glcm_gray(img, w, h, 64, d, a))


@pytest.mark.parametrize("mode", [tf.ChunkExecution.pipelined, tf.ChunkExecution.sequential])
def test_chunked_equals_serial_every_k(engine, mode):
    # mirrors R/tests/test_pipeline.cpp:109-125
    q = tf.QuantizedImage(37, 29, 8, O.quantize(np.random.default_rng(41).integers(0, 256, 37 * 29,
                                                                                   dtype=np.uint8), 8))
    for a in ANGLES:
        for d in (1, 4):
            p = tf.GlcmParams(d, tf.Angle(a), 8)
            want = O.glcm_serial(q.pixels, 37, 29, 8, d, a)
            for k in (1, 2, 3, 5):
                if 29 // k <= d and k > 1:
                    continue
                g = tf.compute_glcm_chunked(tf.MemoryChunkSource(q), p, tf.plan(8, 49152, 2), k, mode)
                assert np.array_equal(g.counts, want), (a, d, k)


def test_chunked_failure_carries_index(engine):
    q = tf.QuantizedImage(32, 32, 8, np.random.default_rng(53).integers(0, 8, 1024, dtype=np.uint8))

    class Failing(tf.MemoryChunkSource):
        def fetch(self, spec, out):
            if spec.index == 3:
                raise RuntimeError("simulated source failure")
            super().fetch(spec, out)

    with pytest.raises(tf.PipelineError) as ei:
        tf.compute_glcm_chunked(Failing(q), tf.GlcmParams(1, tf.Angle.deg90, 8), tf.plan(8), 8)
    assert ei.value.chunk_index == 3
    assert "chunk 3" in str(ei.value)
    # the engine stays usable after an aborted pipeline
    g = tf.compute_glcm_chunked(tf.MemoryChunkSource(q), tf.GlcmParams(1, tf.Angle.deg90, 8), tf.plan(8), 8)
    assert np.array_equal(g.counts, O.glcm_serial(q.pixels, 32, 32, 8, 1, 90))


def test_normalize_bit_exact_and_features(engine, small_cases):
    n = 0
    for c in small_cases:
        g = c["counts"]
        if g.sum() == 0:
            continue
        p = engine.normalize(g, c["L"])
        assert np.array_equal(p.view(np.uint64), c["probs"].view(np.uint64)), c  # bit-exact
        if not np.isnan(c["feats"]).any():
            f = engine.features(p, c["L"])
            assert np.all(np.abs(f - c["feats"]) <= FEAT_TOL * np.maximum(1.0, np.abs(c["feats"]))), (f, c["feats"])
            n += 1
    assert n > 100


def test_symmetrize_and_fused_post(engine):
    rng = np.random.default_rng(11)
    w, h = 211, 123
    gray = rng.integers(0, 256, size=w * h, dtype=np.uint8)
    dts = [(1, a) for a in ANGLES]
    counts, probs, feats = engine.glcm(gray, w, h, 16, dts, flags=L.TFG_SYMMETRIC, want_probs=True,
                                       want_features=True)
    for t, (d, a) in enumerate(dts):
        sym = O.symmetrize(O.glcm_gray(gray, w, h, 16, d, a), 16)
        assert np.array_equal(counts[0, t].reshape(-1), sym)
        pr = O.normalize(sym, 16)
        assert np.array_equal(probs[0, t].reshape(-1).view(np.uint64), pr.view(np.uint64))
        ft = O.features(pr, 16)
        assert np.all(np.abs(feats[0, t] - ft) <= FEAT_TOL * np.maximum(1.0, np.abs(ft)))


def test_reference_error_behaviour(engine):
    img = tf.QuantizedImage(4, 4, 8, np.zeros(16, np.uint8))
    with pytest.raises(ValueError, match="levels do not match"):
        tf.compute_glcm_serial(img, tf.GlcmParams(1, tf.Angle.deg0, 16))
    with pytest.raises(ValueError, match="degenerate geometry"):
        tf.compute_glcm_serial(img, tf.GlcmParams(4, tf.Angle.deg0, 8))
    with pytest.raises(ValueError, match="all-zero"):
        tf.normalize(tf.Glcm(2))
    with pytest.raises(ValueError, match="not normalized"):
        tf.extract_features(tf.GlcmProbabilities(2, np.array([0.5, 0.5, 0.5, 0.5])))
    # raw C ABI: a pre-quantised raster holding a value >= L is rejected
    bad = np.zeros(64 * 64, np.uint8)
    bad[64 * 63 + 63] = 9  # bottom-right corner: not an anchor at 45 degrees
    with pytest.raises(ValueError, match="exceeds gray level"):
        engine.glcm(bad, 64, 64, 8, [(1, 45)], pixel_levels=8)
    with pytest.raises(ValueError, match="levels do not match"):
        engine.glcm(bad, 64, 64, 8, [(1, 45)], pixel_levels=16)
    with pytest.raises(ValueError, match="angle"):
        engine.glcm(bad, 64, 64, 8, [(1, 30)])


def test_async_device_shards_sum_to_whole(engine):
    torch = pytest.importorskip("torch")
    w, h, levels = 1000, 777, 32
    gray = tf.synth_noise(w, h, 9).pixels
    pitch = 1008
    dev = torch.zeros((h, pitch), dtype=torch.uint8, device="cuda")
    dev[:, :w] = torch.from_numpy(gray.reshape(h, w)).cuda()
    lib = L.load()
    stream = torch.cuda.current_stream().cuda_stream
    for d, a in [(1, 0), (2, 45), (3, 90), (1, 135)]:
        acc = torch.zeros(levels * levels, dtype=torch.int64, device="cuda")
        specs = tf.partition(w, h, tf.GlcmParams(d, tf.Angle(a), levels), 4)
        for s in specs:  # each shard: its rows + halo, votes only its owned anchors
            base = dev[s.owned_row_start:s.buffer_row_end]
            L.check(lib.tfg_glcm_async(engine.handle, C.c_void_p(base.data_ptr()), w, s.buffer_rows(), pitch,
                                       s.owned_rows(), 256, levels, d, a, 0, C.c_void_p(acc.data_ptr()),
                                       C.c_void_p(stream)))
        torch.cuda.synchronize()
        got = acc.cpu().numpy().view(np.uint64)
        assert np.array_equal(got, O.glcm_gray(gray, w, h, levels, d, a)), (d, a)
    L.check(lib.tfg_check_async_errors(engine.handle))


def _oracle_rows(gray, w, rows, levels, d, a, owned):
    q = O.quantize(gray, levels)
    return O.glcm_rows(q, w, rows, levels, d, a, 0, owned)


def test_shard_bands_host_pipeline(engine):
    # row shards of two images through one continuous host pipeline: owned
    # rows vote, the halo rows below them are read-only (tfg_glcm_shard)
    w, rows, owned = 2048, 9000, 8997
    imgs = [tf.synth_noise(w, rows, 11).pixels, tf.synth_smooth(w, rows, 12).pixels]
    dts = [(1, 0), (3, 45), (2, 90), (1, 135)]
    got = engine.shard(np.concatenate(imgs), w, rows, owned, 256, dts, n_bands=2)
    for b in range(2):
        for t, (d, a) in enumerate(dts):
            assert np.array_equal(got[b, t].reshape(-1), _oracle_rows(imgs[b], w, rows, 256, d, a, owned)), (b, d, a)


def test_shard_device_input(engine):
    import torch
    w, rows, owned = 1040, 700, 650
    gray = tf.synth_noise(w, rows, 13).pixels
    dev = torch.from_numpy(gray).cuda()
    dts = [(1, 0), (4, 135)]
    for levels in (32, 256):
        got = engine.shard(dev.data_ptr(), w, rows, owned, levels, dts, device=True)
        for t, (d, a) in enumerate(dts):
            assert np.array_equal(got[0, t].reshape(-1), _oracle_rows(gray, w, rows, levels, d, a, owned))


def test_pinned_host_input(engine):
    import torch
    w, h = 4096, 3000
    gray = tf.synth_smooth(w, h, 3).pixels
    pinned = torch.from_numpy(gray).pin_memory()
    assert engine._lib.tfg_memory_kind(C.c_void_p(pinned.data_ptr())) == 1
    dts = [(1, 0), (2, 90)]
    got = engine.glcm(pinned.numpy(), w, h, 256, dts)
    for t, (d, a) in enumerate(dts):
        assert np.array_equal(got[0, t].reshape(-1), O.glcm_gray(gray, w, h, 256, d, a))


@pytest.mark.parametrize("levels,nb", [(256, 2), (256, 300), (100, 300)])
def test_partials_reduce_paths(engine, levels, nb):
    # L > 64 keeps per-CTA partials: a co-resident grid reduces them in-kernel
    # behind a grid barrier (cooperative launch); 300 bands exceed one CTA per
    # SM and take the separate reduce kernels
    w, h = 160, 40
    imgs = [tf.synth_noise(w, h, 100 + b).pixels for b in range(nb)]
    got = engine.glcm(np.concatenate(imgs), w, h, levels, [(1, 45)], n_bands=nb)
    for b in range(0, nb, max(1, nb // 7)):
        assert np.array_equal(got[b, 0].reshape(-1), O.glcm_gray(imgs[b], w, h, levels, 1, 45)), b


@pytest.mark.parametrize("w", [1024, 1040, 1041, 1056, 1057, 1071, 2047, 3001])
def test_two_pass_split_boundaries(engine, w):
    # widths around the main/edge split (nch >= 66 -> interior double batches
    # with row wraps; nch < 66 -> everything in the edge pass), odd widths,
    # heights that leave < 64 leftover interior items per CTA
    h = 67
    gray = tf.synth_noise(w, h, w).pixels
    dts = [(1, 0), (3, 45), (2, 90), (5, 135), (17, 0), (16, 45)]
    for levels in (32, 256):
        got = engine.glcm(gray, w, h, levels, dts)
        for t, (d, a) in enumerate(dts):
            assert np.array_equal(got[0, t].reshape(-1), O.glcm_gray(gray, w, h, levels, d, a)), (w, levels, d, a)


def _subglcms_numpy(q, w, h, L, d, a, group_size, copies, groups):
    """parallel.hpp:160-212 restated in numpy: stripe_rows(h, groups), stripe
    pixel k -> lane (k - stripe_begin*w) % group_size -> copy lane % copies."""
    dr, dc = {0: (0, d), 45: (d, -d), 90: (d, 0), 135: (d, d)}[a]
    img = q.reshape(h, w).astype(np.int64)
    base, extra = divmod(h, groups)
    subs = np.zeros((groups, copies, L * L), np.uint32)
    row = 0
    c0, c1 = (d if dc < 0 else 0), (w - d if dc > 0 else w)
    for g in range(groups):
        end = row + base + (1 if g < extra else 0)
        for r in range(row, min(end, h - dr)):
            cols = np.arange(c0, c1)
            anchor = img[r, cols]
            ref = img[r + dr, cols + dc]
            lane = ((r - row) * w + cols) % group_size
            np.add.at(subs[g], (lane % copies, ref * L + anchor), 1)
        row = end
    return subs.reshape(groups * copies, L * L)


@pytest.mark.parametrize("copies,groups", [(1, 1), (3, 4), (8, 7)])
def test_python_subglcms_and_per_copy_hottest(copies, groups):
    w, h, L = 97, 53, 16
    q = O.quantize(tf.synth_noise(w, h, 21).pixels, L)
    img = tf.QuantizedImage(w, h, L, q)
    p = tf.GlcmParams(2, tf.Angle.deg135, L)
    plan = tf.plan(L, tf.kDefaultScratchBudget, 3)
    plan.copies = copies
    got = tf.compute_subglcms(img, p, plan, groups)
    want = _subglcms_numpy(q, w, h, L, 2, 135, plan.group_size, copies, groups)
    assert len(got) == groups * copies
    for i in range(len(got)):
        assert np.array_equal(got[i], want[i]), i
    g, st = tf.compute_glcm_privatized(img, p, plan, groups)
    assert np.array_equal(g.counts, want.sum(axis=0).astype(np.uint64))
    assert st.per_copy_hottest == [int(x) for x in want.max(axis=1)]


@pytest.mark.parametrize("L,groups,d,a,kind", [(256, 1, 1, 0, "noise"), (256, 7, 2, 45, "smooth"),
                                                (181, 32, 3, 135, "noise"), (256, 40, 1, 90, "smooth"),
                                                (200, 5, 4, 90, "noise")])
def test_privatized_one_copy_stripe_path(L, groups, d, a, kind):
    # plan.copies == 1 with sub-GLCMs over the shared-memory budget (the
    # reference's own plan at L >= 157): stripes voted as bands of one launch,
    # sum + per-stripe maxima on the device; exact vs the numpy restatement
    w, h = 333, 211
    gray = (tf.synth_noise if kind == "noise" else tf.synth_smooth)(w, h, 9).pixels
    q = O.quantize(gray, L)
    img = tf.QuantizedImage(w, h, L, q)
    p = tf.GlcmParams(d, tf.angle_from_degrees(a), L)
    plan = tf.plan(L, tf.kDefaultScratchBudget, 4)
    assert plan.copies == 1
    want = _subglcms_numpy(q, w, h, L, d, a, plan.group_size, 1, groups)
    g, st = tf.compute_glcm_privatized(img, p, plan, groups)
    assert np.array_equal(g.counts, want.sum(axis=0).astype(np.uint64))
    assert st.per_copy_hottest == [int(x) for x in want.max(axis=1)]
    subs = tf.compute_subglcms(img, p, plan, groups)
    for i in range(groups):
        assert np.array_equal(subs[i], want[i]), i


@pytest.mark.parametrize("levels", [16, 64, 256])
def test_multi_async_all_dts_bands_row_end(engine, levels):
    # tfg_glcm_multi_async: every (d, theta) in one call; L <= 64 forks the
    # launches over the context's aux streams, L > 64 stays ordered
    import torch
    w, h, nb, row_end = 1200, 300, 3, 280
    imgs = [tf.synth_smooth(w, h, 40 + b).pixels if b % 2 else tf.synth_noise(w, h, 40 + b).pixels
            for b in range(nb)]
    pitch = 1216  # 16-byte aligned pitch > width
    buf = np.zeros((nb, h, pitch), np.uint8)
    for b in range(nb):
        buf[b, :, :w] = imgs[b].reshape(h, w)
    dev = torch.from_numpy(buf).cuda()
    dts = [(1, 0), (2, 45), (3, 90), (4, 135), (7, 0)]
    cells = levels * levels
    out = torch.zeros(len(dts) * nb * cells, dtype=torch.int64, device="cuda")
    d = (C.c_int * len(dts))(*[x[0] for x in dts])
    a = (C.c_int * len(dts))(*[x[1] for x in dts])
    s = torch.cuda.current_stream()
    L.check(engine._lib.tfg_glcm_multi_async(engine.handle, C.c_void_p(dev.data_ptr()), w, h, pitch, pitch * h, nb,
                                             row_end, 256, levels, d, a, len(dts), 0, C.c_void_p(out.data_ptr()),
                                             C.c_void_p(s.cuda_stream)))
    got = out.cpu().numpy().view(np.uint64).reshape(len(dts), nb, cells)
    for t, (dd, aa) in enumerate(dts):
        for b in range(nb):
            assert np.array_equal(got[t, b], _oracle_rows(imgs[b], w, h, levels, dd, aa, row_end)), (t, b)


@pytest.mark.parametrize("pattern", ["constant", "alternating", "stripes"])
def test_packed16_drains_exact(engine, pattern):
    # > 2^15 votes per CTA on single cells (8192^2 / 148 CTAs ~ 450K votes
    # each): the PACKED16 drain path runs many times, through the run-length
    # votes (constant), through plain votes with both u16 halves (alternating:
    # no 16-pixel item is uniform), and with a hot cell per half (stripes)
    w = h = 8192
    if pattern == "constant":
        img = np.full(w * h, 200, np.uint8)
    elif pattern == "alternating":
        img = np.tile(np.array([10, 250], np.uint8), w * h // 2)
    else:
        row = np.where((np.arange(w) // 3) % 2 == 0, 7, 131).astype(np.uint8)
        img = np.tile(row, h)
    for d, a in [(1, 0), (1, 90), (2, 45), (3, 135)]:
        got = engine.glcm(img, w, h, 256, [(d, a)])
        assert np.array_equal(got.reshape(-1), O.glcm_serial(img, w, h, 256, d, a)), (pattern, d, a)


_POOL_SCRIPT = r"""
import numpy as np
from oracle import oracle as O
from paper_1710_06189_b200 import texforge as tf
eng = tf.Engine(0)
dts = [(1, 0), (3, 45), (2, 90), (1, 135)]
for w, h, nb, levels in [(4096, 777, 1, 256), (3001, 301, 3, 256), (2048, 513, 2, 128), (1100, 2000, 1, 100)]:
    imgs = [tf.synth_noise(w, h, 7 * w + b).pixels for b in range(nb)]
    got = eng.glcm(np.concatenate(imgs), w, h, levels, dts, n_bands=nb)
    for b in range(nb):
        for t, (d, a) in enumerate(dts):
            ref = O.glcm_gray(imgs[b], w, h, levels, d, a)
            assert np.array_equal(got[b, t].reshape(-1), ref), (w, h, nb, levels, b, d, a)
print("POOL-OK")
"""


@pytest.mark.parametrize("pct", [0, 3, 90])
def test_shared_tail_pool_fractions(pct):
    # cooperative launches (L*L > 4096, co-resident grid) hand the last
    # TEXFORGE_POOL_PCT % of each band's interior items to a shared pool; the
    # counts must not depend on how much work goes through it (read once per
    # process, hence the subprocess)
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TEXFORGE_POOL_PCT=str(pct), PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", _POOL_SCRIPT], cwd=root, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "POOL-OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("levels,prequant", [(256, False), (64, False), (32, True)])
def test_pinned_counts_early_band_d2h(engine, levels, prequant):
    # several bands through the host pipeline into a PINNED counts buffer: the
    # counts of band b go down (aux stream) while later bands still upload
    import torch
    w, h, nb = 2048, 2500, 3
    imgs = [(tf.synth_noise if b % 2 == 0 else tf.synth_smooth)(w, h, 40 + b).pixels for b in range(nb)]
    if prequant:
        imgs = [((im.astype(np.uint32) * levels) >> 8).astype(np.uint8) for im in imgs]
    dts = [(1, 0), (3, 45), (2, 90), (1, 135)]
    cells = levels * levels
    for pinned_in in (True, False):
        src = np.concatenate(imgs)
        if pinned_in:
            src = torch.from_numpy(src).pin_memory().numpy()
        out = torch.zeros(nb * len(dts) * cells, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
        got = engine.glcm(src, w, h, levels, dts, pixel_levels=levels if prequant else 256, n_bands=nb, out=out)
        for b in range(nb):
            for t, (d, a) in enumerate(dts):
                want = (O.glcm_serial(imgs[b], w, h, levels, d, a) if prequant
                        else O.glcm_gray(imgs[b], w, h, levels, d, a))
                assert np.array_equal(got[b, t].reshape(-1), want), (pinned_in, b, d, a)


@pytest.mark.parametrize("levels,prequant", [(8, False), (37, False), (20, True), (64, False)])
@pytest.mark.parametrize("w", [1031, 2048])
def test_jobs_launch_every_window(engine, levels, prequant, w):
    # glcm_vote_jobs_kernel: up to 8 (d, theta) of one image in ONE launch,
    # the reference-window variant picked per CTA (every KSEL: d < 16 at
    # 0 deg, aligned 16/32 deg-0 windows, 45/135 word shifts, 90 deg); 9
    # pairs exceed kMaxJobs and take the per-(d, theta) launches
    # (tfg_glcm_multi_async: test_multi_async_all_dts_bands_row_end).
    h = 203
    gray = tf.synth_noise(w, h, 7).pixels
    px = O.quantize(gray, levels) if prequant else gray
    src_levels = levels if prequant else 256
    sets = [[(1, 0), (5, 0), (16, 0), (32, 0), (1, 45), (6, 45), (3, 90), (2, 135)],
            [(1, 0), (2, 0), (3, 0), (4, 0), (1, 45), (1, 90), (1, 135), (9, 135), (12, 90)]]
    for dts in sets:
        got = engine.glcm(px, w, h, levels, dts, pixel_levels=src_levels)
        for t, (d, a) in enumerate(dts):
            want = O.glcm_gray(gray, w, h, levels, d, a)
            assert np.array_equal(got[0, t].reshape(-1), want), (dts, d, a)


@pytest.mark.parametrize("levels,prequant,nb", [(100, False, 1), (256, False, 1), (200, True, 2), (256, False, 3)])
def test_jobs_cooperative_partials(engine, levels, prequant, nb):
    # L > 64 (COPY1 / PACKED16, per-CTA partials): the (d, theta) of one image
    # or band batch that share a reference-window group go out as ONE
    # cooperative launch; each (job, band) row keeps its own partials, pool
    # counter and reduce slices behind the shared grid barrier. 12 pairs, 7
    # KSELs (0 deg d=1,2 | 0 deg d=7 | 90 deg | 45 deg d=1,2 | 45 deg d=7 |
    # 135 deg d=1,2 | 135 deg d=7): COPY1 7 launches (glcm_vote_jobs1_kernel,
    # one KSEL each); PACKED16 4 (glcm_vote_jobs2_kernel, KSEL pairs, + KSEL 4).
    import torch
    w, h = 1296, 260  # pitch % 16 == 0 (the async ABI's alignment rule)
    imgs = [(tf.synth_noise if b % 2 == 0 else tf.synth_smooth)(w, h, 90 + b).pixels for b in range(nb)]
    px = [O.quantize(g, levels) if prequant else g for g in imgs]
    dts = [(d, a) for d in (1, 2, 7) for a in (0, 45, 90, 135)]
    dev = torch.from_numpy(np.concatenate(px)).cuda()
    n = len(dts)
    lv = (C.c_int * n)(*([levels] * n))
    dd = (C.c_int * n)(*[d for d, _ in dts])
    aa = (C.c_int * n)(*[a for _, a in dts])
    out = torch.zeros(n * nb * levels * levels, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    for rep in range(2):  # the second launch reuses the re-armed counters and scratch
        out.zero_()
        before = engine.launches
        L.check(engine._lib.tfg_glcm_jobs_async(engine.handle, C.c_void_p(dev.data_ptr()), w, h, w, w * h, nb, h,
                                                levels if prequant else 256, lv, dd, aa, n, 0,
                                                C.c_void_p(out.data_ptr()), C.c_void_p(s.cuda_stream)))
        # + the range check of a pre-quantised image (launch_validate)
        assert engine.launches - before == (7 if levels <= 128 else 4) + int(prequant)
        got = out.cpu().numpy().view(np.uint64).reshape(n, nb, -1)
        for t, (d, a) in enumerate(dts):
            for b in range(nb):
                want = O.glcm_gray(imgs[b], w, h, levels, d, a)
                assert np.array_equal(got[t, b], want), (rep, levels, d, a, b)


@pytest.mark.parametrize("levels", [256, 120])
def test_jobs_ksel_pair_7_8(engine, levels):
    # 0 deg with 8 <= d < 16: KSEL 7 (d % 16 in 8..11) and 8 (12..15), the
    # {7, 8} pair of glcm_vote_jobs2_kernel (PACKED16: one launch) and two
    # one-KSEL launches for COPY1
    import torch
    w, h = 1024, 96
    img = tf.synth_smooth(w, h, 7).pixels
    dev = torch.from_numpy(img).cuda()
    dts = [(8, 0), (9, 0), (12, 0), (13, 0), (15, 0)]
    n = len(dts)
    lv = (C.c_int * n)(*([levels] * n))
    dd = (C.c_int * n)(*[d for d, _ in dts])
    aa = (C.c_int * n)(*[a for _, a in dts])
    out = torch.zeros(n * levels * levels, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    before = engine.launches
    L.check(engine._lib.tfg_glcm_jobs_async(engine.handle, C.c_void_p(dev.data_ptr()), w, h, w, w * h, 1, h, 256,
                                            lv, dd, aa, n, 0, C.c_void_p(out.data_ptr()), C.c_void_p(s.cuda_stream)))
    assert engine.launches - before == (1 if levels > 128 else 2)
    got = out.cpu().numpy().view(np.uint64).reshape(n, -1)
    for t, (d, a) in enumerate(dts):
        assert np.array_equal(got[t], O.glcm_gray(img, w, h, levels, d, a)), (levels, d)


def test_jobs_cooperative_rows_exceed_one_wave(engine):
    # 20 bands x 8 jobs of one KSEL (90 deg) = 160 (job, band) rows > 148 SM
    # slots: the cooperative launch needs every row co-resident, so
    # launch_job_set shrinks the launch to 7 jobs (140 rows) and the 8th job
    # takes its own launch — 2 launches, every GLCM exact.
    import torch
    w, h, nb = 304, 40, 20
    imgs = [(tf.synth_noise if b % 3 else tf.synth_smooth)(w, h, 120 + b).pixels for b in range(nb)]
    dev = torch.from_numpy(np.concatenate(imgs)).cuda()
    dts = [(d, 90) for d in range(1, 9)]
    n = len(dts)
    lv = (C.c_int * n)(*([256] * n))
    dd = (C.c_int * n)(*[d for d, _ in dts])
    aa = (C.c_int * n)(*[a for _, a in dts])
    out = torch.zeros(n * nb * 65536, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    before = engine.launches
    L.check(engine._lib.tfg_glcm_jobs_async(engine.handle, C.c_void_p(dev.data_ptr()), w, h, w, w * h, nb, h, 256,
                                            lv, dd, aa, n, 0, C.c_void_p(out.data_ptr()), C.c_void_p(s.cuda_stream)))
    assert engine.launches - before == 2
    got = out.cpu().numpy().view(np.uint64).reshape(n, nb, -1)
    for t, (d, a) in enumerate(dts):
        for b in range(nb):
            assert np.array_equal(got[t, b], O.glcm_gray(imgs[b], w, h, 256, d, a)), (d, b)


@pytest.mark.parametrize("nb", [1, 3])
def test_jobs_async_mixed_levels(engine, nb):
    # tfg_glcm_jobs_async: per-job (L, d, theta) of one device image / band
    # batch; runs sharing a kernel instantiation (L=16 and 32: COPIES32) go
    # out as one launch, L=64 (COPIES8) and L=256 (PACKED16) on their own
    import torch
    w, h = 700, 130
    imgs = [tf.synth_noise(w, h, 60 + b).pixels if b % 2 == 0 else tf.synth_smooth(w, h, 60 + b).pixels
            for b in range(nb)]
    pitch = 704
    buf = np.zeros((nb, h, pitch), np.uint8)
    for b in range(nb):
        buf[b, :, :w] = imgs[b].reshape(h, w)
    dev = torch.from_numpy(buf).cuda()
    jobs = [(16, 1, 0), (16, 2, 45), (32, 1, 90), (32, 3, 135), (32, 1, 0), (64, 1, 45), (256, 2, 90), (16, 4, 0),
            (32, 2, 0), (16, 1, 135)]
    n = len(jobs)
    lv = (C.c_int * n)(*[j[0] for j in jobs])
    dd = (C.c_int * n)(*[j[1] for j in jobs])
    aa = (C.c_int * n)(*[j[2] for j in jobs])
    total = sum(nb * j[0] * j[0] for j in jobs)
    out = torch.zeros(total, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    L.check(engine._lib.tfg_glcm_jobs_async(engine.handle, C.c_void_p(dev.data_ptr()), w, h, pitch, pitch * h, nb, h,
                                            256, lv, dd, aa, n, 0, C.c_void_p(out.data_ptr()),
                                            C.c_void_p(s.cuda_stream)))
    got = out.cpu().numpy().view(np.uint64)
    off = 0
    for (levels, d, a) in jobs:
        cells = levels * levels
        for b in range(nb):
            want = O.glcm_gray(imgs[b], w, h, levels, d, a)
            assert np.array_equal(got[off + b * cells: off + (b + 1) * cells], want), (levels, d, a, b)
        off += nb * cells


@pytest.mark.parametrize("pinned", [False, True])
def test_shard_jobs_one_upload_many_levels(engine, pinned):
    # tfg_glcm_shard_jobs: host bands copied up once; every (L, d, theta) job
    # votes from that copy; owned rows + halo like tfg_glcm_shard
    import torch
    w, rows, owned, nb = 1500, 700, 690, 2
    imgs = [tf.synth_noise(w, rows, 71).pixels, tf.synth_smooth(w, rows, 72).pixels]
    host = np.concatenate(imgs)
    if pinned:
        t = torch.from_numpy(host).pin_memory()
        host = t.numpy()
    jobs = [(16, 1, 0), (16, 1, 45), (32, 1, 90), (32, 2, 135), (64, 1, 0), (256, 3, 45), (8, 4, 90)]
    got = engine.shard_jobs(host, w, rows, owned, jobs, n_bands=nb)
    for t, (levels, d, a) in enumerate(jobs):
        for b in range(nb):
            want = _oracle_rows(imgs[b], w, rows, levels, d, a, owned)
            assert np.array_equal(got[t][b].reshape(-1), want), (levels, d, a, b)


@pytest.mark.parametrize("pattern", ["constant", "alternating", "stripes"])
def test_p16x16_drains_exact(engine, pattern):
    # S_P16X16: 16 copies of u16 fields; > 2^15 votes per copy per CTA on
    # single cells (8192 x 16384 at L=64: ~900K votes per CTA, ~57K per copy
    # on a constant image: the drain path runs; forced strategy)
    w, h = 8192, 16384
    if pattern == "constant":
        img = np.full(w * h, 200, np.uint8)
    elif pattern == "alternating":
        img = np.tile(np.array([10, 250], np.uint8), w * h // 2)
    else:
        row = np.where((np.arange(w) // 3) % 2 == 0, 7, 131).astype(np.uint8)
        img = np.tile(row, h)
    for d, a in [(1, 0), (1, 90), (2, 45), (3, 135)]:
        got = engine.glcm(img, w, h, 64, [(d, a)], flags=L.strategy_flag(L.STRAT_P16X16))
        assert np.array_equal(got.reshape(-1), O.glcm_gray(img, w, h, 64, d, a)), (pattern, d, a)
