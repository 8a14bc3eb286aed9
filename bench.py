"""Benchmark of the B200 GLCM engine (contract in DESIGN.md §6).

Metric (BASELINE.json): GLCM Gpixel-pairs/s per (d, theta) = valid pixel
pairs voted per second, whole job, summed over every (image, d, theta) GLCM.

Workloads (BASELINE.json configs; --workload, default c3):
  c3  16384^2 per GPU, L=256, d in {1,2,4} x 4 theta, uniform-noise AND
      smooth-gradient (the collision worst case): 24 GLCMs per step, one
      engine launch each, image device-resident. N>1: the image is
      (N*16384) x 16384, row-partitioned (partition(), pipeline.hpp:48-73):
      each GPU owns 16384 rows + a 4-row halo received from its neighbour,
      votes its owned anchors, and the 24 partial GLCMs are summed with ONE
      NCCL reduce per step inside the timed region (weak scaling).
  c5  65536^2 (4 GiB), L=64, d=1, 4 theta, noise, row-partitioned over N
      GPUs with d-row halos + one NCCL reduce per step (strong scaling).
  c4  256 bands of 2048^2, L=32, d=1, 4 theta, bands sharded over N GPUs,
      one launch per theta for all of a GPU's bands, no collective (strong).
  c2  4096^2, L=16 and 32, d=1, 4 theta, noise+smooth (replicas for N>1).
  c1  512^2, L=8, d=1, 0 deg (the reference's CPU case; replicas).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--workload c3]

Every input is larger than L2 (126 MB) except c1/c2/c4-per-band, where the
L2 is flushed between timed steps (config.l2 says which). --impl reference
times the reference's own CPU path (oracle/_ref/libtexforge_ref.so = the
UNMODIFIED reference headers, compute_glcm_privatized on all host threads)
on a bounded sample of the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GLCM Gpixel-pairs/s per (d,theta)"
UNIT = "Gpairs/s"
ANGLES = (0, 45, 90, 135)
L2_BYTES = 126 * 1024 * 1024

# name: width, rows per GPU block (None: whole image of `height` rows split over N),
#       height, levels list, distances, kinds, layout, bands
WORKLOADS = {
    "c3": dict(width=16384, block_rows=16384, levels=(256,), ds=(1, 2, 4), kinds=("noise", "smooth"),
               layout="rows-weak", bands=1),
    "c5": dict(width=65536, height=65536, levels=(64,), ds=(1,), kinds=("noise",), layout="rows-strong", bands=1),
    "c4": dict(width=2048, height=2048, levels=(32,), ds=(1,), kinds=("noise",), layout="bands", bands=256),
    "c2": dict(width=4096, height=4096, levels=(16, 32), ds=(1,), kinds=("noise", "smooth"), layout="replica",
               bands=1),
    "c1": dict(width=512, height=512, levels=(8,), ds=(1,), kinds=("noise",), layout="replica", bands=1,
               angles=(0,)),
    # small test-only variants of the partitioned layouts (tests/test_bench_dist.py)
    "t3": dict(width=4096, block_rows=1024, levels=(256,), ds=(1, 4), kinds=("noise", "smooth"),
               layout="rows-weak", bands=1),
    "t5": dict(width=4096, height=4096, levels=(64,), ds=(1,), kinds=("noise",), layout="rows-strong", bands=1),
    "t4": dict(width=1024, height=1024, levels=(32,), ds=(1,), kinds=("noise",), layout="bands", bands=10),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def valid_pairs(w, h, d, a):
    if a == 0:
        return h * (w - d)
    if a == 90:
        return (h - d) * w
    return (h - d) * (w - d)


def fnv1a64(counts: np.ndarray) -> str:
    h = 0xcbf29ce484222325
    for b in np.ascontiguousarray(counts, dtype="<u8").tobytes():
        h = ((h ^ b) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return "%016x" % h


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region (NVML every
    ~2 ms; nvidia-smi as fallback)."""
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device):
        self.device = device
        self.samples = []
        self.sm_max = None
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.sm_max = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nvml = None

    def _sample(self):
        if self._nvml:
            n = self._nvml
            return (n.nvmlDeviceGetClockInfo(self._h, n.NVML_CLOCK_SM),
                    n.nvmlDeviceGetCurrentClocksEventReasons(self._h))
        out = subprocess.run(["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5).stdout
        sm, mx = [float(x) for x in out.strip().split(",")]
        self.sm_max = mx
        return (sm, 0)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._sample())
            except Exception:
                pass
            self._stop.wait(0.002)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.01)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.sm_max, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples]
        reasons = sorted({name for _, m in self.samples for bit, name in self.REASONS.items() if m & bit})
        return {"sm_mhz": statistics.median(sm), "sm_min_mhz": min(sm), "sm_max_mhz": self.sm_max, "reasons": reasons,
                "samples": len(self.samples), "source": "nvml" if self._nvml else "nvidia-smi"}


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def committed_traffic(workload):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


# --------------------------------------------------------------------------- inputs
def noise_pixels(tf, width, height, seed):
    """synth_noise(width, height, seed) pixels, generated on the device
    (tfg_synth_noise_device: mt19937 jump-ahead, bit-identical to the host
    generator) and copied back; inputs are untimed, this only shortens setup."""
    import torch
    if torch.cuda.is_available():
        dev = torch.cuda.current_device()
        eng = _GEN_ENGINES.get(dev) or _GEN_ENGINES.setdefault(dev, tf.Engine(dev))
        return eng.synth_noise_device(width, height, seed).cpu().numpy()
    return tf.synth_noise(width, height, seed).pixels


_GEN_ENGINES = {}


def gen_rows(tf, kind, width, row0, rows, block_rows, seed0, height=None):
    """Rows [row0, row0+rows) of the workload image. block_rows=None: the one
    image synth_<kind>(width, height, seed0) (rows-strong; noise rows come
    straight from the device generator jumped to output row0*width). Else an
    image of generator blocks of `block_rows` rows, block b =
    synth_<kind>(width, block_rows, seed0 + b) (rows-weak). The content does
    not depend on how the rows are later partitioned."""
    if block_rows is None:
        import torch
        if kind == "noise" and torch.cuda.is_available():
            dev = torch.cuda.current_device()
            eng = _GEN_ENGINES.get(dev) or _GEN_ENGINES.setdefault(dev, tf.Engine(dev))
            return eng.synth_noise_rows_device(width, row0, rows, seed0).cpu().numpy()
        full = (tf.synth_noise if kind == "noise" else tf.synth_smooth)(width, height, seed0).pixels
        return full[row0 * width:(row0 + rows) * width].copy()
    out = np.empty(rows * width, dtype=np.uint8)
    r = row0
    while r < row0 + rows:
        b = r // block_rows
        if kind == "noise":
            blk = noise_pixels(tf, width, block_rows, seed0 + b)
        else:
            blk = tf.synth_smooth(width, block_rows, seed0 + b).pixels
        lo = r - b * block_rows
        hi = min(block_rows, row0 + rows - b * block_rows)
        out[(r - row0) * width:(r - row0 + hi - lo) * width] = blk[lo * width:hi * width]
        r += hi - lo
    return out


class Plan:
    """What this rank holds and computes for a workload at world size N."""

    def __init__(self, wl, world, rank, tf, D):
        cfg = WORKLOADS[wl]
        self.wl, self.cfg = wl, cfg
        self.width = cfg["width"]
        self.levels_list = cfg["levels"]
        angles = cfg.get("angles", ANGLES)
        self.dts = [(d, a) for d in cfg["ds"] for a in angles]
        self.kinds = cfg["kinds"]
        self.layout = cfg["layout"]
        # rows of halo below a shard (pipeline.hpp:60-61: d for the downward angles, none at 0 degrees)
        self.halo = max([d for d, a in self.dts if a != 0], default=0) if self.layout.startswith("rows") else 0
        self.bands = 1
        if self.layout == "rows-weak":
            self.height = cfg["block_rows"] * world          # global image
            self.owned0, self.owned = rank * cfg["block_rows"], cfg["block_rows"]
            self.gen_block = cfg["block_rows"]
        elif self.layout == "rows-strong":
            self.height = cfg["height"]
            spec = D.shard_rows(self.width, self.height, self.dts, self.levels_list[0], world, rank) \
                if world > 1 else None
            self.owned0 = spec.owned_row_start if spec else 0
            self.owned = spec.owned_rows() if spec else self.height
            self.gen_block = None  # one synth image, BASELINE config 5
        elif self.layout == "bands":
            self.height = cfg["height"]
            base, extra = divmod(cfg["bands"], world)  # contiguous blocks (distributed.bands_for_rank)
            start = rank * base + min(rank, extra)
            self.band_ids = list(range(start, start + base + (1 if rank < extra else 0)))
            self.bands = len(self.band_ids)
            self.owned0, self.owned = 0, self.height
        else:  # replica
            self.height = cfg["height"]
            self.owned0, self.owned = 0, self.height
        self.world, self.rank = world, rank
        self.scaling = "weak" if self.layout in ("rows-weak", "replica") else "strong"

    def buffer_rows_alloc(self):
        return self.owned + (self.halo if self.layout.startswith("rows") else 0)

    def pairs_per_step(self):
        """Valid pairs of every GLCM the WHOLE job computes in one step."""
        p = 0
        for _L in self.levels_list:
            for _k in self.kinds:
                for d, a in self.dts:
                    if self.layout == "bands":
                        p += self.cfg["bands"] * valid_pairs(self.width, self.height, d, a)
                    elif self.layout == "replica":
                        p += self.world * valid_pairs(self.width, self.height, d, a)
                    else:
                        p += valid_pairs(self.width, self.height, d, a)
        return p

    def describe(self):
        c = self.cfg
        kinds = "+".join(self.kinds)
        Ls = "/".join(str(x) for x in self.levels_list)
        th = "/".join(str(a) for a in c.get("angles", ANGLES))
        if self.layout == "rows-weak":
            return (f"{self.wl}: {self.height}x{self.width} ({self.world} x {c['block_rows']}-row blocks) {kinds}, "
                    f"L={Ls}, d={list(c['ds'])}, theta={th}, device-resident; row-partitioned, one {c['block_rows']}"
                    f"x{self.width} block + {self.halo}-row halo per GPU, one NCCL reduce per step")
        if self.layout == "rows-strong":
            return (f"{self.wl}: {self.height}x{self.width} {kinds}, L={Ls}, d={list(c['ds'])}, theta={th}, "
                    f"device-resident; row-partitioned over {self.world} GPU(s) with {self.halo}-row halos, "
                    f"one NCCL reduce per step")
        if self.layout == "bands":
            return (f"{self.wl}: {c['bands']} bands of {self.width}x{self.height} {kinds}, L={Ls}, d={list(c['ds'])},"
                    f" theta={th}, device-resident; bands sharded over {self.world} GPU(s), one launch per theta")
        return (f"{self.wl}: {self.width}x{self.height} {kinds}, L={Ls}, d={list(c['ds'])}, theta={th}, "
                f"device-resident, replica per GPU")


def make_host_inputs(plan, tf):
    """Pinned-able numpy buffers for this rank: {kind: array}. Rows layouts:
    owned rows only (the halo arrives over NCCL). Bands: concatenated bands."""
    imgs = {}
    for kind in plan.kinds:
        if plan.layout == "bands":
            imgs[kind] = np.concatenate([noise_pixels(tf, plan.width, plan.height, b + 1)
                                         for b in plan.band_ids])
        elif plan.layout.startswith("rows"):
            imgs[kind] = gen_rows(tf, kind, plan.width, plan.owned0, plan.owned, plan.gen_block, 1, plan.height)
        elif kind == "noise":
            imgs[kind] = noise_pixels(tf, plan.width, plan.height, 1)
        else:
            imgs[kind] = tf.synth_smooth(plan.width, plan.height, 1).pixels
    return imgs


# --------------------------------------------------------------------------- reference arm
def ref_image(r, gray, w, h, L):
    """A reference QuantizedImage: the reference's own quantize(gray, L)
    (image.hpp:55-62), untimed like in its CLI bench (texforge.cpp:190-236)."""
    q = np.empty(w * h, dtype=np.uint8)
    rc = r.ref_quantize(gray.ctypes.data_as(C.POINTER(C.c_uint8)), w, h, L, q.ctypes.data_as(C.POINTER(C.c_uint8)))
    if rc:
        raise RuntimeError("reference quantize failed")
    hd = r.ref_image_new(q.ctypes.data_as(C.POINTER(C.c_uint8)), w, h, L)
    if not hd:
        raise RuntimeError("reference QuantizedImage construction failed")
    return hd


def ref_synth(r, kind, w, h, seed):
    """The reference's own synth_noise / synth_smooth (image.hpp:76-116)."""
    out = np.empty(w * h, dtype=np.uint8)
    fn = r.ref_synth_noise if kind == "noise" else r.ref_synth_smooth
    if fn(w, h, seed, out.ctypes.data_as(C.POINTER(C.c_uint8))):
        raise RuntimeError("reference synth failed")
    return out


def run_reference(args, wl):
    """The reference's own CPU path on this box's host cores, nothing of the
    engine loaded: inputs from the reference's generators, its quantize, and
    compute_glcm_privatized (parallel.hpp:240-254) on all host threads for
    every (input, L, d, theta) GLCM of one step of the workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as O
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtexforge_ref.so not built"}))
        return
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    plan = Plan(wl, 1, 0, None, None)
    threads = os.cpu_count() or 1
    r = O.ref()
    w = plan.width
    t0 = time.time()
    if plan.layout == "rows-weak":
        h, units = plan.cfg["block_rows"], [1]  # one generator block (seed 1); N blocks = N x the same work
    elif plan.layout == "bands":
        h, units = plan.height, [b + 1 for b in range(plan.cfg["bands"])]
    else:
        h, units = plan.height, [1]
    handles = {}
    for kind in plan.kinds:
        for u in units:
            gray = ref_synth(r, kind, w, h, u)
            for L in plan.levels_list:
                handles[(kind, u, L)] = ref_image(r, gray, w, h, L)
            del gray
    log(f"[reference] inputs ready in {time.time() - t0:.1f}s")
    jobs = [(k, u, L, d, a) for L in plan.levels_list for k in plan.kinds for u in units for (d, a) in plan.dts]
    outs = {L: np.zeros(L * L, dtype=np.uint64) for L in plan.levels_list}

    def step():
        p = 0
        for kind, u, L, d, a in jobs:
            if r.ref_image_glcm(handles[(kind, u, L)], d, a, threads, 1,
                                outs[L].ctypes.data_as(C.POINTER(C.c_uint64))):
                raise RuntimeError("reference compute_glcm_privatized failed")
            p += valid_pairs(w, h, d, a)
        return p

    for _ in range(args.warmup):
        step()
    t = time.perf_counter()
    pairs = sum(step() for _ in range(args.steps))
    el = time.perf_counter() - t
    v = pairs / el / 1e9
    n_img = len(units) * len(plan.kinds)
    sample = (f"every GLCM of one step: {len(jobs)} (input, L, d, theta) jobs over {n_img} {w}x{h} image(s)"
              + (f" (one of the {world} row blocks a step covers at N={world}; each block is the same work)"
                 if plan.layout == "rows-weak" and world > 1 else "")
              + f"; reference compute_glcm_privatized (unmodified headers), {threads} workers")
    for hd in handles.values():
        r.ref_image_free(hd)
    print(json.dumps({
        "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3, "higher_is_better": True,
        "scaling": Plan(wl, world, 0, None, None).scaling if plan.layout != "rows-strong" else "strong",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic (reference synth_noise / synth_smooth)",
        "impl": "reference",
        "config": {"workload": Plan(wl, 1, 0, None, None).describe(), "host_threads": threads,
                   "pairs_per_step": pairs // args.steps, "glcms_per_step": len(jobs)},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def cpu_baseline(plan, imgs, seconds, threads):
    """The reference's compute_glcm_privatized on all host threads, ~`seconds`
    of work over (input, d, theta) GLCMs of this rank's images."""
    from oracle import oracle as O
    if not O.ref_available():
        return None
    r = O.ref()
    w = plan.width
    h = plan.owned if plan.layout != "bands" else plan.height
    L = plan.levels_list[-1]
    handles = {k: ref_image(r, v[: w * h], w, h, L) for k, v in imgs.items()}
    out = np.zeros(L * L, dtype=np.uint64)
    jobs = [(k, d, a) for (d, a) in plan.dts for k in imgs]
    pairs, el, calls = 0, 0.0, 0
    while el < seconds or calls < 2:
        kind, d, a = jobs[calls % len(jobs)]
        t = time.perf_counter()
        assert r.ref_image_glcm(handles[kind], d, a, threads, 1, out.ctypes.data_as(C.POINTER(C.c_uint64))) == 0
        el += time.perf_counter() - t
        pairs += valid_pairs(w, h, d, a)
        calls += 1
    for hd in handles.values():
        r.ref_image_free(hd)
    return {"value": pairs / el / 1e9, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{calls} single-(d,theta) GLCMs of {w}x{h} L={L} inputs (reference "
                      f"compute_glcm_privatized, unmodified headers, {threads} workers, ~{seconds:.0f}s)"}


# --------------------------------------------------------------------------- correctness gate
def golden_for(plan):
    """{(kind, L, d, theta): fnv} of the reference's own GLCMs of this plan's
    GLOBAL image, where tests/golden holds them."""
    out = {}
    gdir = os.path.join(ROOT, "tests", "golden")
    if plan.wl in ("c3", "c1", "c2", "c5"):
        with open(os.path.join(gdir, "golden_hashes.json")) as f:
            small = json.load(f)["glcm"]
        if plan.layout != "rows-weak" or plan.world == 1:
            for g in small:
                if g["size"] == plan.width and g["size"] == plan.height and g.get("seed", 1) == 1:
                    out[(g["kind"], g["levels"], g["d"], g["theta"])] = g["fnv"]
    try:
        with open(os.path.join(gdir, "golden_large.json")) as f:
            large = json.load(f)
    except OSError:
        return out
    if plan.wl == "c5":
        for g in large.get("c5", []):
            out[(g["kind"], g["levels"], g["d"], g["theta"])] = g["fnv"]
    if plan.wl == "c3" and plan.world == 1:
        for g in large.get("c3_smooth_d", []):
            out[(g["kind"], g["levels"], g["d"], g["theta"])] = g["fnv"]
    if plan.wl == "c3" and plan.world > 1:
        for g in large.get("c3_blocks", []):
            if g["blocks"] == plan.world:
                out[(g["kind"], g["levels"], g["d"], g["theta"])] = g["fnv"]
    return out


def single_gpu_recompute(plan, tf, eng, lib, jobs, out_off, cells, reduced):
    """Rank 0: the global image of a row-partitioned plan on this one GPU,
    voted with the N=1 path; returns how many reduced GLCMs equal it."""
    import torch
    from paper_1710_06189_b200 import _lib as Lb
    W, H = plan.width, plan.height
    want = torch.zeros(reduced.size, dtype=torch.int64, device="cuda")
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for kind in plan.kinds:
        img = torch.from_numpy(gen_rows(tf, kind, W, 0, H, plan.gen_block, 1, H)).cuda()
        for j, (L, k, d, a) in enumerate(jobs):
            if k != kind:
                continue
            Lb.check(lib.tfg_glcm_async(eng.handle, C.c_void_p(img.data_ptr()), W, H, W, H, 256, L, d, a, 0,
                                        C.c_void_p(want.data_ptr() + out_off[j] * 8), s))
        torch.cuda.synchronize()
        del img
    want = want.cpu().numpy().view(np.uint64)
    return sum(int(np.array_equal(reduced[out_off[j]:out_off[j] + cells[L]], want[out_off[j]:out_off[j] + cells[L]]))
               for j, (L, _k, _d, _a) in enumerate(jobs))


# --------------------------------------------------------------------------- engine arm
def run_engine(args, wl):
    import torch

    from paper_1710_06189_b200 import _lib as Lb
    from paper_1710_06189_b200 import distributed as D
    from paper_1710_06189_b200 import texforge as tf

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # TFG_DIST_BACKEND=gloo: test mode for the N>1 logic on fewer GPUs than
    # ranks (ranks share devices round-robin; collectives staged via the host)
    backend = os.environ.get("TFG_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl" and torch.cuda.device_count() < world:
            raise SystemExit(f"bench: {world} ranks need {world} GPUs for NCCL, this box has "
                             f"{torch.cuda.device_count()} (TFG_DIST_BACKEND=gloo runs the N>1 logic on one GPU)")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        dist.barrier()  # every rank's communicator is up before the first P2P batch (halo exchange)

    plan = Plan(wl, world, rank, tf, D)
    eng = tf.Engine(local)
    lib = Lb.load()
    # N>1 over NCCL: the library's own communicator (tfg_comm_*: ncclSend/Recv
    # halo rows, one ncclReduce per step) from a uid rank 0 ships over the
    # torch.distributed store; gloo test mode keeps torch's collectives.
    comm = None
    if dist is not None and backend == "nccl":
        box = [tf.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        comm = tf.Comm(eng, world, rank, box[0])
    t0 = time.time()
    imgs = make_host_inputs(plan, tf)
    log(f"[rank {rank}] inputs ready in {time.time() - t0:.1f}s")
    W = plan.width
    stream = torch.cuda.current_stream()
    sptr = C.c_void_p(stream.cuda_stream)

    # device-resident inputs: owned rows + halo (rows layouts; halo over NCCL).
    # Image layouts at L <= 64 keep every input in ONE allocation, a fixed
    # stride apart, so a step votes all inputs and all (L, d, theta) in one
    # multi-job launch (c2: 2 launches -> 1, +3%). L=256 keeps one call per
    # input: two images as bands of one cooperative launch measured 4% slower.
    merge_kinds = plan.layout != "bands" and max(plan.levels_list) <= 64
    dev, buf_rows = {}, {}
    kstride = 0
    if merge_kinds:
        kstride = (plan.buffer_rows_alloc() * W + 64 + 127) // 128 * 128
        allk = torch.zeros(kstride * len(imgs) + 64, dtype=torch.uint8, device="cuda")
    for ki, (kind, px) in enumerate(imgs.items()):
        alloc = plan.buffer_rows_alloc() * W if plan.layout != "bands" else px.size
        if merge_kinds:
            t = allk[ki * kstride: ki * kstride + alloc + 64]
        else:
            t = torch.zeros(alloc + 64, dtype=torch.uint8, device="cuda")
        t[: px.size].copy_(torch.from_numpy(px))
        if plan.layout.startswith("rows") and world > 1 and comm is not None:
            comm.exchange_halo(t.data_ptr(), W, plan.owned, plan.halo, torch.cuda.current_stream().cuda_stream)
            buf_rows[kind] = plan.owned + (plan.halo if rank + 1 < world else 0)
        elif plan.layout.startswith("rows") and world > 1:
            buf_rows[kind] = D.exchange_halo(t, plan.owned, W, plan.halo, world, rank)
        else:
            buf_rows[kind] = plan.owned
        dev[kind] = t
    torch.cuda.synchronize()

    cells = {L: L * L for L in plan.levels_list}
    kinds_all = list(plan.kinds)
    if merge_kinds:
        # one tfg_glcm_jobs_async call per step: job = (L, d, theta), band =
        # input; its output layout is [job][input][L*L]
        assert len(set(buf_rows.values())) == 1, "inputs of one step share their geometry"
        jobs, out_off, o = [], [], 0
        for L in plan.levels_list:
            for (d, a) in plan.dts:
                for b, kind in enumerate(kinds_all):
                    jobs.append((L, kind, d, a))
                    out_off.append(o + b * cells[L])
                o += len(kinds_all) * cells[L]
    else:
        # input-major: every GLCM of one input is contiguous in `acc`, so one
        # tfg_glcm_jobs_async call per input covers all its (L, d, theta)
        jobs = [(L, kind, d, a) for kind in plan.kinds for L in plan.levels_list for (d, a) in plan.dts]
        out_off, o = [], 0
        for (L, _k, _d, _a) in jobs:
            out_off.append(o)
            o += plan.bands * cells[L]
    acc = torch.zeros(o, dtype=torch.int64, device="cuda")
    pairs_per_step = plan.pairs_per_step()
    flush = torch.empty(0, dtype=torch.uint8, device="cuda")
    per_gpu_bytes = sum(v.numel() for v in dev.values())
    if per_gpu_bytes < 2 * L2_BYTES:
        flush = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device="cuda")
    launches = []
    record = {"on": False, "single": False}  # single: one engine call per job; on: time each call

    # timed steps: one engine call per input with every (L, d, theta) of it
    # (tfg_glcm_jobs_async); the roofline pass below times single launches
    groups = []  # (kind, first job, [(L, d, theta)])
    for j, (L, kind, d, a) in enumerate(jobs):
        if groups and groups[-1][0] == kind:
            groups[-1][2].append((L, d, a))
        else:
            groups.append((kind, j, [(L, d, a)]))
    gargs = []
    for kind, j0, g in groups:
        n = len(g)
        gargs.append((kind, out_off[j0], n, (C.c_int * n)(*[x[0] for x in g]), (C.c_int * n)(*[x[1] for x in g]),
                      (C.c_int * n)(*[x[2] for x in g])))

    cur = {"s": sptr}  # stream the engine calls enqueue on (the capture stream while recording a graph)

    if merge_kinds:
        jl = [(L, d, a) for L in plan.levels_list for (d, a) in plan.dts]
        nj = len(jl)
        step_args = ((C.c_int * nj)(*[x[0] for x in jl]), (C.c_int * nj)(*[x[1] for x in jl]),
                     (C.c_int * nj)(*[x[2] for x in jl]), nj)

    def vote_grouped():
        if merge_kinds:
            # every input as a band of one call: all (L, d, theta) x inputs
            ll, dd, aa, nj_ = step_args
            rows = buf_rows[kinds_all[0]]
            rc = lib.tfg_glcm_jobs_async(eng.handle, C.c_void_p(dev[kinds_all[0]].data_ptr()), W, rows, W, kstride,
                                         len(kinds_all), plan.owned, 256, ll, dd, aa, nj_, 0,
                                         C.c_void_p(acc.data_ptr()), cur["s"])
            if rc:
                Lb.check(rc)
            return
        # one engine call per input: every (L, d, theta) of it (tfg_glcm_jobs_async)
        for kind, off, n, ll, dd, aa in gargs:
            bands = plan.bands if plan.layout == "bands" else 1
            rows = plan.height if plan.layout == "bands" else buf_rows[kind]
            rc = lib.tfg_glcm_jobs_async(eng.handle, C.c_void_p(dev[kind].data_ptr()), W, rows, W, W * rows, bands,
                                         plan.owned if plan.layout != "bands" else rows, 256, ll, dd, aa, n, 0,
                                         C.c_void_p(acc.data_ptr() + off * 8), cur["s"])
            if rc:
                Lb.check(rc)

    def vote_all():
        if not record["single"]:
            vote_grouped()
            return
        for j, (L, kind, d, a) in enumerate(jobs):
            if record["on"]:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            dst = C.c_void_p(acc.data_ptr() + out_off[j] * 8)
            if plan.layout == "bands":
                rc = lib.tfg_glcm_bands_async(eng.handle, C.c_void_p(dev[kind].data_ptr()), W, plan.height, W,
                                              W * plan.height, plan.bands, 256, L, d, a, 0, dst, sptr)
            else:
                rc = lib.tfg_glcm_async(eng.handle, C.c_void_p(dev[kind].data_ptr()), W, buf_rows[kind], W,
                                        plan.owned, 256, L, d, a, 0, dst, sptr)
            if rc:
                Lb.check(rc)
            if record["on"]:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(stream)
                launches.append((e0, e1))

    def step():
        acc.zero_()
        vote_all()
        if dist is not None and plan.layout.startswith("rows"):
            if comm is not None:  # ONE ncclReduce of every partial GLCM, issued by the library
                comm.reduce_counts(acc.data_ptr(), acc.numel(), 0, cur["s"].value or 0)
            else:
                D.reduce_sum_(acc)

    # correctness gate (first step, untimed, rank 0 after the reduce):
    #  * conservation: every GLCM sums to valid_pair_count of the global image;
    #  * golden: the reference's own FNV-1a hashes of the same global image
    #    (tests/golden: Appendix A, golden_large.json for c5 and the N-block c3);
    #  * at N > 1, a single-GPU recompute: rank 0 builds the whole global image
    #    and votes it with the N=1 path (golden-pinned), and every reduced GLCM
    #    must equal it bit for bit (catches halo / ownership / reduce errors).
    step()
    torch.cuda.synchronize()
    check = {"conservation": None, "golden": None}
    if rank == 0:
        host = acc.cpu().numpy().view(np.uint64)
        ok = True
        for j, (L, kind, d, a) in enumerate(jobs):
            for b in range(plan.bands):
                seg = host[out_off[j] + b * cells[L]: out_off[j] + (b + 1) * cells[L]]
                ok &= int(seg.sum()) == valid_pairs(W, plan.height, d, a)
        check["conservation"] = bool(ok)
        gold = golden_for(plan)
        if gold:
            n_ok = n_all = 0
            for j, (L, kind, d, a) in enumerate(jobs):
                key = (kind, L, d, a)
                if key in gold:
                    n_all += 1
                    n_ok += fnv1a64(host[out_off[j]: out_off[j] + cells[L]]) == gold[key]
            check["golden"] = f"{n_ok}/{n_all} reference FNV-1a hashes of the global image match"
            ok &= n_ok == n_all
        if plan.layout == "bands":
            with open(os.path.join(ROOT, "tests", "golden", "golden_hashes.json")) as f:
                gb = {(g["kind"], g["seed"], g["levels"], g["d"], g["theta"]): g["fnv"]
                      for g in json.load(f)["glcm"] if g["size"] == W == plan.height}
            n_ok = n_all = 0
            for j, (L, kind, d, a) in enumerate(jobs):
                for b, band in enumerate(plan.band_ids):
                    key = (kind, band + 1, L, d, a)
                    if key in gb:
                        n_all += 1
                        seg = host[out_off[j] + b * cells[L]: out_off[j] + (b + 1) * cells[L]]
                        n_ok += fnv1a64(seg) == gb[key]
            check["golden"] = f"{n_ok}/{n_all} reference FNV-1a hashes of this rank's bands match"
            ok &= n_ok == n_all
        if world > 1 and plan.layout.startswith("rows"):
            same = single_gpu_recompute(plan, tf, eng, lib, jobs, out_off, cells, host)
            check["single_gpu_recompute"] = f"{same}/{len(jobs)} GLCMs equal the whole image voted on one GPU"
            ok &= same == len(jobs)
        if os.environ.get("TFG_BENCH_DUMP"):  # tests: the gated GLCMs, for an independent oracle check
            np.savez(os.environ["TFG_BENCH_DUMP"], counts=host, offsets=np.array(out_off),
                     jobs=np.array([(L, plan.kinds.index(k), d, a) for (L, k, d, a) in jobs]))
        if not ok:
            raise SystemExit(f"bench correctness gate failed: {check}")
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()

    # The step is replayed as ONE CUDA graph, so the timed region measures the
    # device, not the host's launch rate or the gaps between launches
    # (cooperative L > 64 launches capture too: c3 +0.7%). Not for steps with
    # an NCCL reduce. TFG_BENCH_GRAPH=0: eager engine calls.
    graph, graph_launches = None, 0
    nccl_step = dist is not None and plan.layout.startswith("rows")
    if not nccl_step and os.environ.get("TFG_BENCH_GRAPH", "1") != "0":
        cap = torch.cuda.Stream()
        cap.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        l_before = eng.launches
        cur["s"] = C.c_void_p(cap.cuda_stream)
        with torch.cuda.graph(graph, stream=cap):
            step()
        cur["s"] = sptr
        graph_launches = eng.launches - l_before
        torch.cuda.synchronize()
        graph.replay()
        torch.cuda.synchronize()
        if rank == 0 and not np.array_equal(acc.cpu().numpy().view(np.uint64), host):
            raise SystemExit("bench correctness gate failed: CUDA-graph replay differs from the eager step")
    run_step = graph.replay if graph is not None else step

    # timed region: K steps (L2 flushed between steps when the inputs fit in L2)
    l0 = eng.launches
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush_ms = 0.0
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        if flush.numel():
            fe0, fe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            steps_ms = 0.0
            for s in range(args.steps):
                flush.fill_(s & 0xFF)
                fe0.record(stream)
                run_step()
                fe1.record(stream)
                while not fe1.query():
                    time.sleep(0.0002)
                torch.cuda.synchronize()
                steps_ms += fe0.elapsed_time(fe1)
            ms = steps_ms / args.steps
        else:
            start.record(stream)
            for s in range(args.steps):
                run_step()
            end.record(stream)
            # wait by polling (sleep releases the GIL, so the clock sampler
            # thread runs during the timed region); the time is the events'
            while not end.query():
                time.sleep(0.0005)
            torch.cuda.synchronize()
            ms = start.elapsed_time(end) / args.steps
    gpu_launches = graph_launches * args.steps if graph is not None else eng.launches - l0
    if dist:
        t = torch.tensor([ms], device="cuda")
        D.all_reduce_max_(t)
        ms = float(t.item())
        dist.barrier()
    value = pairs_per_step / (ms / 1e3) / 1e9

    # per-call durations for the roofline (separate pass, same stream); one
    # untimed pass first: the timed steps may not have used the one-job
    # kernels, and their first (lazy) module load would land in the events
    record["single"] = True
    acc.zero_()
    vote_all()
    torch.cuda.synchronize()
    record["on"] = True
    for s in range(max(2, min(args.steps, 5))):
        acc.zero_()
        vote_all()
    torch.cuda.synchronize()
    durs = [a.elapsed_time(b) for a, b in launches]
    avg_ms = sum(durs) / len(durs)
    peak, peak_src = hbm_peak()
    bytes_per_call = sum(
        (plan.bands * W * plan.height if plan.layout == "bands" else buf_rows[k] * W) + plan.bands * cells[L] * 8
        for (L, k, _d, _a) in jobs) / len(jobs)
    per_call_achieved = bytes_per_call / (avg_ms / 1e3) / 1e9
    # the roofline figure comes from the TIMED region: every vote launch of a
    # step moves bytes_per_call algorithmic bytes; the
    # step's kernel time is ms_per_step (launch gaps and the accumulator
    # memset included, so this is the conservative figure). The separate
    # per-call pass above explains it (per_call).
    achieved = bytes_per_call * len(jobs) / (ms / 1e3) / 1e9
    # SURVEY.md §8(d)'s clause for fused launches: "if one launch computes
    # n_out (d, theta) pairs from a single read, the image bytes count once".
    # Each engine call's launches each read its input once (c3: 4 launches
    # per input, 3 (d, theta) each), so this basis credits far fewer bytes
    # than the per-job one; reported beside it, not instead of it.
    calls_per_step = 1 if merge_kinds else len(gargs)
    launches_per_call = (gpu_launches / max(args.steps, 1)) / max(calls_per_step, 1)
    input_bytes = sum((plan.bands * W * plan.height if plan.layout == "bands" else buf_rows[k] * W)
                      for k in plan.kinds)
    glcm_bytes = sum(plan.bands * cells[L] * 8 for (L, _k, _d, _a) in jobs)
    read_once_achieved = (launches_per_call * input_bytes + glcm_bytes) / (ms / 1e3) / 1e9

    # end-to-end through the public C ABI from pinned host memory: H2D of this
    # step's inputs inside the region, counts back to the host, NCCL reduce
    e2e = None
    if not args.no_e2e:
        # every input of the step in ONE pinned buffer (rows layouts: each
        # kind's owned + halo rows), so one call streams them all through a
        # single copy/vote pipeline
        kinds = list(plan.kinds)
        if plan.layout == "bands":
            pinned = {k: torch.from_numpy(imgs[k]).pin_memory() for k in kinds}
            rows_e2e = plan.height
        else:
            rows_e2e = buf_rows[kinds[0]]
            allk = torch.empty(len(kinds) * rows_e2e * W, dtype=torch.uint8).pin_memory()
            for i, k in enumerate(kinds):
                src = dev[k][: rows_e2e * W].cpu() if plan.layout.startswith("rows") else torch.from_numpy(imgs[k])
                allk[i * rows_e2e * W:(i + 1) * rows_e2e * W].copy_(src)
            pinned = {"all": allk}
        first = next(iter(pinned.values()))
        in_kind = lib.tfg_memory_kind(C.c_void_p(first.data_ptr()))  # 1 = pinned (tfg_memory_kind)
        probe = torch.empty(first.numel(), dtype=torch.uint8, device="cuda")
        h2d_gbs = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            probe.copy_(first, non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            h2d_gbs.append(probe.numel() / (e0.elapsed_time(e1) / 1e3) / 1e9)
        del probe
        red = torch.zeros(o, dtype=torch.int64, device="cuda") if dist else None
        # results land by DMA in a pinned output buffer, one slice per call
        out_host = torch.zeros(o, dtype=torch.int64).pin_memory().numpy().view(np.uint64)

        multi_level = plan.layout != "bands" and len(plan.levels_list) > 1
        e2e_jobs = [(L, d, a) for L in plan.levels_list for (d, a) in plan.dts]

        def e2e_step():
            off = 0
            if multi_level:
                # every (L, d, theta) of the step from ONE upload of each input
                # (tfg_glcm_shard_jobs)
                eng.shard_jobs(pinned["all"].numpy(), W, rows_e2e, plan.owned, e2e_jobs, n_bands=len(kinds),
                               band_stride=rows_e2e * W, out=out_host)
            for L in (() if multi_level else plan.levels_list):
                dts = plan.dts
                if plan.layout == "bands":
                    for kind in kinds:
                        n = plan.bands * len(dts) * L * L
                        eng.glcm(pinned[kind].numpy(), W, plan.height, L, dts, n_bands=plan.bands,
                                 out=out_host[off:off + n])
                        off += n
                else:
                    n = len(kinds) * len(dts) * L * L
                    eng.shard(pinned["all"].numpy(), W, rows_e2e, plan.owned, L, dts, n_bands=len(kinds),
                              band_stride=rows_e2e * W, out=out_host[off:off + n])
                    off += n
            host = out_host
            if dist is not None and plan.layout.startswith("rows"):
                red.copy_(torch.from_numpy(host.view(np.int64)))
                if comm is not None:
                    comm.reduce_counts(red.data_ptr(), red.numel(), 0, torch.cuda.current_stream().cuda_stream)
                else:
                    D.reduce_sum_(red)
                if rank == 0:
                    host = red.cpu().numpy().view(np.uint64)
            return host

        e2e_step()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        # median of per-step wall times (every step ends with its results on
        # the host, so steps do not overlap); short steps get more samples
        n_e2e = max(2, min(args.steps, 10))
        t = time.perf_counter()
        e2e_step()
        first = time.perf_counter() - t
        if first < 0.01:
            n_e2e = max(n_e2e, 30)
        samples = []
        with ClockSampler(local) as e2e_clocks:  # short steps leave the GPU mostly idle (clock governor)
            for _ in range(n_e2e):
                t = time.perf_counter()
                e2e_step()
                torch.cuda.synchronize()
                samples.append(time.perf_counter() - t)
        e2e_s = statistics.median(samples)
        if dist:
            tt = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
            D.all_reduce_max_(tt)
            e2e_s = float(tt.item())
        h2d = sum(v.numel() for v in pinned.values()) * (1 if multi_level else len(plan.levels_list))
        e2e = {"value": pairs_per_step / e2e_s / 1e9, "unit": UNIT, "h2d_bytes_per_step": world * h2d,
               "d2h_bytes_per_step": world * o * 8,
               "api": ("tfg_glcm_shard_jobs: every input of the step in one pinned host buffer, uploaded once for "
                       "all its (L, d, theta)" if multi_level else
                       "tfg_glcm_shard / tfg_glcm_bands: every input of the step in one pinned host buffer") +
                      ", one call = one continuous Scheme-3 copy/vote stream pipeline, counts to host" +
                      (", + NCCL reduce" if dist else ""),
               "pinned_h2d_GBps": max(h2d_gbs), "ms_per_step": e2e_s * 1e3,
               "h2d_bound_ms_per_step": h2d / (max(h2d_gbs) * 1e9) * 1e3,
               "spread_ms": [min(samples) * 1e3, max(samples) * 1e3], "clocks": e2e_clocks.summary(),
               "host_memory_kind": {"input": in_kind,
                                    "counts": lib.tfg_memory_kind(out_host.ctypes.data_as(C.c_void_p))}}

    # Secondary end-to-end line through the C++ drop-in's hottest call, in the
    # reference CLI's calling convention (R/tools/texforge.cpp:218-236): a
    # pageable QuantizedImage per input, compute_glcm_privatized(img, p,
    # plan(L, 49152, nproc)) per (d, theta) -> counts + per_copy_hottest on the
    # host. The drop-in header forwards it to ONE C-ABI call, tfg_subglcms
    # (include/texforge/parallel.hpp), which is what is timed here.
    e2e_dropin = None
    if not args.no_e2e and world == 1 and plan.layout != "bands":
        nproc = os.cpu_count() or 1
        Hd = plan.height
        qimgs = {}
        for L in plan.levels_list:
            pl = tf.plan(L, 49152, nproc)
            groups = tf._resolve_group_count(0, pl, W, Hd)
            for kind in plan.kinds:
                px = imgs[kind][: W * Hd]
                qimgs[(kind, L)] = (np.array(px) if L == 256 else eng.quantize(px, L), pl, groups)
        cnt = np.zeros(max(plan.levels_list) ** 2, dtype=np.uint64)

        def dropin_step():
            for L in plan.levels_list:
                for kind in plan.kinds:
                    q, pl, groups = qimgs[(kind, L)]
                    hot = np.zeros(groups * pl.copies, dtype=np.uint64)
                    for d, a in plan.dts:
                        Lb.check(lib.tfg_subglcms(eng.handle, q.ctypes.data_as(C.c_void_p), W, Hd, L, L, d, a,
                                                  pl.group_size, pl.copies, groups, 0, None,
                                                  cnt.ctypes.data_as(C.POINTER(C.c_uint64)),
                                                  hot.ctypes.data_as(C.POINTER(C.c_uint64))))

        dropin_step()
        samples = []
        for _ in range(max(2, min(args.steps, 5))):
            t = time.perf_counter()
            dropin_step()
            samples.append(time.perf_counter() - t)
        el = statistics.median(samples)

        # the same calls through compute_glcm_serial's C-ABI call (tfg_glcm, one
        # (d, theta), same pageable image): the drop-in's reference point
        def serial_step():
            for L in plan.levels_list:
                for kind in plan.kinds:
                    q, _pl, _g = qimgs[(kind, L)]
                    for d, a in plan.dts:
                        dd, aa = C.c_int(d), C.c_int(a)
                        Lb.check(lib.tfg_glcm(eng.handle, q.ctypes.data_as(C.c_void_p), W, Hd, W, L, L,
                                              C.byref(dd), C.byref(aa), 1, 0,
                                              cnt.ctypes.data_as(C.POINTER(C.c_uint64)), None, None))

        serial_step()
        ss = []
        for _ in range(max(2, min(args.steps, 5))):
            t = time.perf_counter()
            serial_step()
            ss.append(time.perf_counter() - t)
        el_serial = statistics.median(ss)
        e2e_dropin = {"value": pairs_per_step / el / 1e9, "unit": UNIT, "ms_per_step": el * 1e3,
                      "serial_value": pairs_per_step / el_serial / 1e9, "serial_ms_per_step": el_serial * 1e3,
                      "privatized_over_serial_time": el / el_serial,
                      "h2d_bytes_per_step": len(jobs) * W * Hd,
                      "d2h_bytes_per_step": sum(L * L * 8 for (L, _k, _d, _a) in jobs),
                      "api": "texforge::compute_glcm_privatized (C++ drop-in) = tfg_subglcms on a pageable image, "
                             "plan(L, 49152, nproc), one call per (input, d, theta) as in the reference CLI bench"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(plan, imgs, args.cpu_seconds, os.cpu_count() or 1)
        except Exception as e:  # reported, never required
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": plan.scaling,
            "vs_baseline": None, "dtype": "u8", "data": "synthetic (reference synth_noise / synth_smooth generators)",
            "config": {"workload": plan.describe(), "pairs_per_step": pairs_per_step,
                       "glcms_per_step": len(jobs) * plan.bands * (world if plan.layout in ("bands", "replica")
                                                                   else 1),
                       "l2": ("inputs larger than L2 (126 MB); no flush" if not flush.numel()
                              else "L2 flushed (256 MiB write) before every timed step; flush excluded"),
                       "parallelism": {"rows-weak": f"row partition x{world} + NCCL reduce",
                                       "rows-strong": f"row partition x{world} + NCCL reduce",
                                       "bands": f"band shards x{world}", "replica": f"replica x{world}"}[plan.layout],
                       "launch": ("one CUDA graph of the step, replayed per timed step" if graph is not None
                                  else "eager engine calls"),
                       "check": check},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": committed_traffic(wl),
                         "kernel": ("glcm_vote_jobs_kernel / glcm_vote_jobs1_kernel (multi-(d, theta) launches; "
                                    "glcm_vote_kernel for a lone (d, theta))"),
                         "bytes_per_job": bytes_per_call, "jobs_per_step": len(jobs),
                         "launches_per_step": gpu_launches / max(args.steps, 1),
                         "basis": ("bytes_per_job x jobs_per_step / ms_per_step (timed region, per GPU); a job is one "
                                   "(L, input, d, theta) over all its bands; traffic: ncu DRAM bytes per job"),
                         "read_once": {"achieved": read_once_achieved, "frac": read_once_achieved / peak,
                                       "launches_per_call": launches_per_call,
                                       "how": ("SURVEY.md §8(d) fused-launch basis: each launch's image bytes once "
                                               "+ every GLCM write, over the timed region")},
                         "per_call": {"avg_launch_ms": avg_ms, "achieved": per_call_achieved,
                                      "frac": per_call_achieved / peak,
                                      "how": "separate pass, CUDA events around each engine call on its stream"},
                         "peak_source": peak_src},
            "e2e": e2e,
            "e2e_dropin": e2e_dropin,
            "gpu_launches": gpu_launches,
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    if comm is not None:
        comm.close()
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        log("note: warmup raised to the contract minimum of 3")
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torch.distributed.run
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.run(cmd).returncode)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, args.workload)
    else:
        run_engine(args, args.workload)


if __name__ == "__main__":
    main()
