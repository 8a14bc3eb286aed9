"""CPU checks of the C-ABI library: it loads, exports every symbol that
include/texforge_cuda.h declares, and its host-only entry points (geometry,
plan, partition, input generators) match the reference KATs and the oracle.
No compute call needs a GPU here."""
import ctypes as C
import os
import re
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O
from paper_1710_06189_b200 import _lib as L
from paper_1710_06189_b200 import texforge as tf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "texforge_cuda.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:[A-Za-z_][\w\s\*]*?)\b(tfg_\w+)\s*\(", src, re.M)))


def test_header_symbols_exported():
    syms = declared_symbols()
    assert len(syms) >= 20
    lib = L.load()
    for s in syms:
        assert hasattr(lib, s), s
    nm = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True).stdout
    for s in syms:
        assert re.search(rf"\bT {s}$", nm, re.M), s
    bound = {n for n, _, _ in L.SIGNATURES}
    assert set(syms) == bound, set(syms) ^ bound


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_link_time_nccl_and_torch_imports_after_the_library():
    """NCCL is dlopened on the first multi-GPU call (csrc/tfg_nccl_dl.h). A
    link-time libnccl.so.2 (the system 2.27) would be the copy a later
    `import torch` binds to, and libtorch_cuda fails on a 2.28-only symbol —
    the order smoke() and the drop-in take (library first, torch second)."""
    needed = subprocess.run(["readelf", "-d", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "libnccl" not in needed
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_1710_06189_b200 import _lib; _lib.load()\n"
            "import torch; print('ok', torch.__version__)\n") % ROOT
    env = {k: v for k, v in os.environ.items() if k != "TEXFORGE_NCCL_LIB"}
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stderr[-2000:]


def test_abi_version():
    assert L.load().tfg_abi_version() == 1


def test_neighbor_offsets():  # R/tests/test_glcm.cpp:20-26
    assert tf.neighbor_offset(tf.GlcmParams(1, tf.Angle.deg0, 8)) == tf.PixelOffset(0, 1)
    assert tf.neighbor_offset(tf.GlcmParams(4, tf.Angle.deg90, 8)) == tf.PixelOffset(4, 0)
    assert tf.neighbor_offset(tf.GlcmParams(2, tf.Angle.deg45, 8)) == tf.PixelOffset(2, -2)
    assert tf.neighbor_offset(tf.GlcmParams(3, tf.Angle.deg135, 8)) == tf.PixelOffset(3, 3)
    with pytest.raises(ValueError, match="angle must be one of"):
        tf.angle_from_degrees(30)


def test_valid_pair_count_vs_oracle():
    assert tf.valid_pair_count(1024, 1024, tf.GlcmParams(4, tf.Angle.deg135, 8)) == 1040400
    rng = np.random.default_rng(1)
    for _ in range(200):
        w, h = int(rng.integers(2, 5000)), int(rng.integers(2, 5000))
        d = int(rng.integers(1, min(w, h)))
        a = int(rng.choice([0, 45, 90, 135]))
        assert tf.valid_pair_count(w, h, tf.GlcmParams(d, tf.Angle(a), 8)) == O.valid_pair_count(w, h, d, a)
    with pytest.raises(ValueError, match="degenerate geometry"):
        tf.valid_pair_count(4, 4, tf.GlcmParams(4, tf.Angle.deg0, 8))


def test_partition_vs_oracle_and_kats():
    specs = tf.partition(1024, 1024, tf.GlcmParams(1, tf.Angle.deg90, 8), 4)
    assert [(s.owned_row_start, s.owned_row_end, s.buffer_row_end) for s in specs] == \
        [(0, 256, 257), (256, 512, 513), (512, 768, 769), (768, 1024, 1024)]
    rng = np.random.default_rng(37)
    for trial in range(200):
        h = int(rng.integers(4, 64))
        d = int(rng.integers(1, 4))
        if d >= h:
            continue
        k = int(rng.integers(1, max(2, h // (d + 1) + 1)))
        a = (0, 45, 90, 135)[trial % 4]
        got = tf.partition(64, h, tf.GlcmParams(d, tf.Angle(a), 8), k)
        assert [[s.owned_row_start, s.owned_row_end, s.buffer_row_end] for s in got] == \
            O.partition(64, h, d, a, k).tolist()
    for args, msg in [((8, 8, 1, 0), "chunk count"), ((8, 8, 1, 9), "chunk count"),
                      ((8, 8, 4, 2), "too many chunks"), ((8, 8, 8, 1), "degenerate")]:
        w, h, d, k = args
        with pytest.raises(ValueError, match=msg):
            tf.partition(w, h, tf.GlcmParams(d, tf.Angle.deg90, 8), k)


def test_plan_unchanged():  # R/tests/test_parallel.cpp:22-56 + acceptance criterion 6
    p32 = tf.plan(32, 49152, 8)
    assert (p32.copies, p32.groups_per_unit, p32.group_size, p32.degraded) == (6, 2, 512, False)
    assert tf.plan(8, 49152, 8).copies == 8
    p256 = tf.plan(256, 49152, 8)
    assert p256.copies == 1 and p256.degraded
    with pytest.raises(ValueError):
        tf.plan(1, 49152, 8)
    with pytest.raises(ValueError):
        tf.plan(300, 49152, 8)
    rng = np.random.default_rng(2026)
    for _ in range(1000):
        L_ = int(rng.integers(2, 257))
        sub = L_ * L_ * 4
        budget = sub + int(rng.integers(0, 8 * sub + 131072))
        p = tf.plan(L_, budget, int(rng.integers(1, 33)))
        assert p.copies >= 1 and p.copies * sub * p.groups_per_unit <= budget
        assert (p.copies, p.groups_per_unit, p.degraded) == O.plan(L_, budget)


def test_types_validate_like_reference():
    with pytest.raises(ValueError, match="pixel value exceeds gray level"):
        tf.QuantizedImage(2, 2, 2, [0, 1, 2, 0])
    with pytest.raises(ValueError, match="dimensions must be positive"):
        tf.GrayImage(0, 2, [])
    with pytest.raises(ValueError, match="levels must be in"):
        tf.Glcm(1)
    with pytest.raises(ValueError, match="levels\\^2"):
        tf.Glcm(2, [1, 2, 3])
    assert tf.reduce_subglcms([[1, 0, 0, 1], [2, 3, 0, 0]], 2) == tf.Glcm(2, [3, 3, 0, 1])
    with pytest.raises(ValueError, match="length mismatch"):
        tf.reduce_subglcms([[1, 2, 3]], 2)
    a, b = tf.Glcm(2, [1, 2, 3, 4]), tf.Glcm(2, [10, 0, 0, 1])
    assert tf.merge_chunk_glcms([a, b]) == tf.Glcm(2, [11, 2, 3, 5])
    with pytest.raises(ValueError):
        tf.merge_chunk_glcms([a, tf.Glcm(3)])
    with pytest.raises(ValueError):
        tf.merge_chunk_glcms([])


def test_synth_rejects_degenerate():
    with pytest.raises(ValueError):
        tf.synth_smooth(1, 64, 1)
    with pytest.raises(ValueError):
        tf.synth_noise(64, 1, 1)


def test_engine_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(Exception):
        tf.Engine(0)
