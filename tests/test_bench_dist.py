"""bench.py's N>1 paths end to end on one GPU: N ranks share the device and
the collectives are staged through gloo (TFG_DIST_BACKEND=gloo). bench.py
launches the ranks itself (--gpus N without torchrun). After halo exchange +
one reduce, rank 0's gate requires every GLCM to equal the whole image voted
on one GPU; this test also checks the dumped GLCMs against the C oracle
(oracle/glcm_oracle.c, pinned to the reference) on the same global image."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def global_image(wl, kind):
    """The global image of a test workload, from the reference generators."""
    from paper_1710_06189_b200 import texforge as tf
    import bench
    cfg = bench.WORKLOADS[wl]
    gen = tf.synth_noise if kind == "noise" else tf.synth_smooth
    if cfg["layout"] == "rows-strong":
        return gen(cfg["width"], cfg["height"], 1).pixels
    raise AssertionError(wl)


def weak_image(wl, kind, n):
    from paper_1710_06189_b200 import texforge as tf
    import bench
    cfg = bench.WORKLOADS[wl]
    gen = tf.synth_noise if kind == "noise" else tf.synth_smooth
    return np.concatenate([gen(cfg["width"], cfg["block_rows"], 1 + b).pixels for b in range(n)])


@pytest.mark.gpu
@pytest.mark.parametrize("wl,n", [("t3", 2), ("t5", 3), ("t5", 2), ("t4", 2)])
def test_bench_partitioned_layouts(wl, n, tmp_path):
    from oracle import oracle as O
    import bench
    dump = str(tmp_path / "glcms.npz")
    env = dict(os.environ, TFG_DIST_BACKEND="gloo", TFG_BENCH_DUMP=dump)
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--workload", wl, "--steps", "2",
           "--warmup", "3", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == n
    chk = line["config"]["check"]
    assert chk["conservation"] is True
    assert line["e2e"]["value"] > 0
    cfg = bench.WORKLOADS[wl]
    if cfg["layout"].startswith("rows"):
        assert chk["single_gpu_recompute"].startswith(f"{len(cfg['kinds']) * len(cfg['ds']) * 4}/")
        z = np.load(dump)
        counts, offs, jobs = z["counts"], z["offsets"], z["jobs"]
        kinds = cfg["kinds"]
        imgs = {}
        for j, (L, k, d, a) in enumerate(jobs):
            kind = kinds[k]
            if kind not in imgs:
                imgs[kind] = (global_image(wl, kind) if cfg["layout"] == "rows-strong"
                              else weak_image(wl, kind, n))
            h = imgs[kind].size // cfg["width"]
            want = O.glcm_gray(imgs[kind], cfg["width"], h, int(L), int(d), int(a))
            got = counts[offs[j]:offs[j] + L * L]
            assert np.array_equal(got, want), f"{wl} N={n} {kind} L={L} d={d} theta={a}"
