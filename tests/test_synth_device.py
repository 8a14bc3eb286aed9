"""Device synth_noise: std::mt19937 jump-ahead on the
host (tfg_mt19937_windows) and segment-parallel generation on the device,
bit-identical to the reference's sequential generator (image.hpp:109-116)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1710_06189_b200 import texforge as tf


def _outputs_from_window(w, n):
    """A generator whose state array is window w (624 words) emits these n
    outputs after one twist (std::mt19937's twist + temper, restated)."""
    mt = [int(v) for v in w]
    out = []
    while len(out) < n:
        for i in range(624):
            y = (mt[i] & 0x80000000) | (mt[(i + 1) % 624] & 0x7FFFFFFF)
            mt[i] = mt[(i + 397) % 624] ^ (y >> 1) ^ (0x9908B0DF if y & 1 else 0)
        for i in range(624):
            y = mt[i]
            y ^= y >> 11
            y ^= (y << 7) & 0x9D2C5680
            y ^= (y << 15) & 0xEFC60000
            y ^= y >> 18
            out.append(y & 0xFFFFFFFF)
    return out[:n]


def test_mt19937_known_answer():
    # C++ [rand.predef]: the 10000th invocation of a default-constructed
    # std::mt19937 (seed 5489) produces 4123659995
    w = tf.mt19937_windows(5489, 9999, 1, 1)[0]
    assert _outputs_from_window(w, 1)[0] == 4123659995


def test_mt19937_windows_match_host_synth_noise():
    # synth_noise bytes are the top 8 bits of consecutive outputs
    width, height = 1536, 1000
    for seed in (1, 2, 7):
        ref = tf.synth_noise(width, height, seed).pixels
        first, stride, count = 5, 123_457, 12
        wins = tf.mt19937_windows(seed, first, stride, count)
        for s in range(count):
            k = first + s * stride
            got = np.array([v >> 24 for v in _outputs_from_window(wins[s], 700)], dtype=np.uint8)
            assert np.array_equal(got, ref[k:k + 700]), (seed, s)


@pytest.mark.gpu
@pytest.mark.parametrize("width,height,pitch", [(512, 512, 0), (1000, 777, 1008), (4099, 3001, 0), (16384, 4096, 0)])
def test_synth_noise_device_bit_identical(engine, width, height, pitch):
    for seed in (1, 3):
        out = engine.synth_noise_device(width, height, seed, pitch=pitch)
        p = pitch or width
        got = out.cpu().numpy().reshape(height, p)[:, :width]
        ref = tf.synth_noise(width, height, seed).pixels.reshape(height, width)
        assert np.array_equal(got, ref), (width, height, seed)


def test_parallel_host_noise_equals_sequential():
    # tfg_synth_noise_parallel (jump-ahead segments, any thread count) vs the
    # sequential std::mt19937 path (images < 4 Mpixel take it)
    import ctypes as C
    from paper_1710_06189_b200 import _lib as L
    lib = L.load()
    seq = tf.synth_noise(1999, 1003, 11).pixels
    for threads in (1, 3, 16):
        out = np.empty(seq.size, dtype=np.uint8)
        L.check(lib.tfg_synth_noise_parallel(seq.size, 11, out.ctypes.data_as(C.POINTER(C.c_uint8)), threads))
        assert np.array_equal(out, seq), threads


@pytest.mark.gpu
def test_synth_noise_device_golden_hashes(engine, golden_hashes):
    # the reference's own synth_noise bytes (tests/golden: FNV-1a of its output)
    for r in golden_hashes["synth"]:
        if r["kind"] != "noise":
            continue
        img = engine.synth_noise_device(r["w"], r["h"], r["seed"]).cpu().numpy()
        assert O.fnv1a64_image(img) == r["fnv_u64view"], r
