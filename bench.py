"""Benchmark of the B200 GLCM engine (contract in DESIGN.md §6).

Metric (BASELINE.json): GLCM Gpixel-pairs/s per (d, theta).
Default workload = BASELINE config 3: 16384x16384, L=256, d in {1,2,4} x four
theta, on BOTH the uniform-noise and the smooth-gradient input (the collision
worst case). One step = the 24 GLCMs (2 images x 12 (d, theta)), each a
separate single-(d, theta) engine launch over the device-resident image.
Each input (256 MiB) is larger than L2 (126 MB), so no L2 flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--workload c3|c2|c4]

N>1 (under torchrun): every rank runs the same per-GPU workload on its own
B200 (weak scaling: independent images, no data-path collective); time = max
over ranks. --impl reference times the reference's own CPU path
(oracle/_ref/libtexforge_ref.so = the unmodified reference headers,
compute_glcm_privatized on all host threads) on the same workload, rank 0 only.
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

WORKLOADS = {
    # name: (size, levels, distances, kinds, n_bands)
    "c3": (16384, 256, (1, 2, 4), ("noise", "smooth"), 1),
    "c2": (4096, 32, (1,), ("noise", "smooth"), 1),
    "c4": (2048, 32, (1,), ("noise",), 32),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def valid_pairs(w, h, d, a):
    if a == 0:
        return h * (w - d)
    if a == 90:
        return (h - d) * w
    return (h - d) * (w - d)


def make_images(tf, n, kinds, n_bands, rank):
    imgs = {}
    for kind in kinds:
        if n_bands == 1:
            gen = tf.synth_noise if kind == "noise" else tf.synth_smooth
            imgs[kind] = gen(n, n, 1).pixels
        else:
            imgs[kind] = np.concatenate([tf.synth_noise(n, n, b + 1 + rank * n_bands).pixels
                                         for b in range(n_bands)])
    return imgs


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region (NVML every
    ~2 ms; nvidia-smi as fallback)."""
    # nvmlClocksEventReason* bits
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device):
        self.device = device
        self.samples = []  # (sm_mhz, reasons_mask)
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
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.sm_max, "reasons": reasons,
                "samples": len(self.samples), "source": "nvml" if self._nvml else "nvidia-smi"}


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def committed_traffic(workload):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


# --------------------------------------------------------------------------- reference arm
def cpu_reference_rate(imgs, n, levels, dts, seconds_budget, threads, n_bands=1, rotate=0):
    """Times the reference's own compute_glcm_privatized (all host threads) on a
    bounded sample: GLCMs over (image, (d, theta)) pairs until the budget."""
    from oracle import oracle as O
    r = O.ref()
    handles = {}
    for kind, px in imgs.items():
        band = px[: n * n]
        handles[kind] = r.ref_image_new(band.ctypes.data_as(C.POINTER(C.c_uint8)), n, n, levels)
    out = np.zeros(levels * levels, dtype=np.uint64)
    pairs, elapsed, calls = 0, 0.0, 0
    jobs = [(k, d, a) for (d, a) in dts for k in imgs]
    i = rotate
    while elapsed < seconds_budget or calls < 2:
        kind, d, a = jobs[i % len(jobs)]
        i += 1
        t = time.perf_counter()
        rc = r.ref_image_glcm(handles[kind], d, a, threads, 1, out.ctypes.data_as(C.POINTER(C.c_uint64)))
        elapsed += time.perf_counter() - t
        assert rc == 0
        pairs += valid_pairs(n, n, d, a)
        calls += 1
    for h in handles.values():
        r.ref_image_free(h)
    return pairs / elapsed / 1e9, calls


def run_reference(args, wl):
    n, levels, ds, kinds, n_bands = WORKLOADS[wl]
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1710_06189_b200 import texforge as tf
    from oracle import oracle as O
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtexforge_ref.so not built"}))
        return
    threads = os.cpu_count() or 1
    imgs = make_images(tf, n, kinds, 1, 0)
    dts = [(d, a) for d in ds for a in ANGLES]
    jobs = [(k, d, a) for (d, a) in dts for k in imgs]
    r = O.ref()
    handles = {k: r.ref_image_new(px.ctypes.data_as(C.POINTER(C.c_uint8)), n, n, levels) for k, px in imgs.items()}
    out = np.zeros(levels * levels, dtype=np.uint64)
    per_step = min(len(jobs), 2)  # bounded sample per step: one GLCM per input kind

    def step(s):
        p = 0
        for j in range(per_step):
            kind, d, a = jobs[(s * per_step + j) % len(jobs)]
            assert r.ref_image_glcm(handles[kind], d, a, threads, 1, out.ctypes.data_as(C.POINTER(C.c_uint64))) == 0
            p += valid_pairs(n, n, d, a)
        return p

    for s in range(args.warmup):
        step(s)
    t = time.perf_counter()
    pairs = sum(step(args.warmup + s) for s in range(args.steps))
    el = time.perf_counter() - t
    v = pairs / el / 1e9
    sample = (f"{per_step} GLCMs/step (rotating over {len(jobs)} (input, d, theta) jobs) of the {n}x{n} "
              f"L={levels} images; reference compute_glcm_privatized, {threads} workers")
    print(json.dumps({
        "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": f"{wl}: {n}x{n} {'+'.join(kinds)}, L={levels}, d={list(ds)}, theta=0/45/90/135",
                   "host_threads": threads},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))
    for h in handles.values():
        r.ref_image_free(h)


# --------------------------------------------------------------------------- engine arm
def run_engine(args, wl):
    import torch

    from paper_1710_06189_b200 import _lib as L
    from paper_1710_06189_b200 import texforge as tf

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    n, levels, ds, kinds, n_bands = WORKLOADS[wl]
    eng = tf.Engine(local)
    lib = L.load()
    t0 = time.time()
    imgs = make_images(tf, n, kinds, n_bands, rank)
    log(f"[rank {rank}] inputs ready in {time.time() - t0:.1f}s")
    dts = [(d, a) for d in ds for a in ANGLES]
    cells = levels * levels
    dev = {k: torch.from_numpy(v).cuda() for k, v in imgs.items()}
    n_out = len(kinds) * len(dts) * n_bands
    acc = torch.zeros((n_out, cells), dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream()
    sptr = C.c_void_p(stream.cuda_stream)
    pairs_per_step = sum(valid_pairs(n, n, d, a) for (d, a) in dts) * len(kinds) * n_bands
    bytes_per_launch = n * n + cells * 8  # algorithmic: image read once + u64 GLCM write

    launches = []  # (start_event, end_event) per hot-path call
    record = {"on": False}

    def step():
        acc.zero_()
        o = 0
        for kind in kinds:
            base = dev[kind]
            for b in range(n_bands):
                for (d, a) in dts:
                    if record["on"]:
                        e0 = torch.cuda.Event(enable_timing=True)
                        e0.record(stream)
                    rc = lib.tfg_glcm_async(eng.handle, C.c_void_p(base.data_ptr() + b * n * n), n, n, n, n, 256,
                                            levels, d, a, 0, C.c_void_p(acc[o].data_ptr()), sptr)
                    if rc:
                        L.check(rc)
                    if record["on"]:
                        e1 = torch.cuda.Event(enable_timing=True)
                        e1.record(stream)
                        launches.append((e0, e1))
                    o += 1

    # correctness gate on the first step (cheap: the L2-sized accumulators)
    step()
    torch.cuda.synchronize()
    for w_ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    l0 = eng.launches
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        start.record(stream)
        for s in range(args.steps):
            step()
        end.record(stream)
        torch.cuda.synchronize()
    gpu_launches = eng.launches - l0
    ms = start.elapsed_time(end) / args.steps
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    value = world * pairs_per_step / (ms / 1e3) / 1e9

    # per-launch durations for the roofline (separate pass, same stream)
    record["on"] = True
    for s in range(max(2, min(args.steps, 5))):
        step()
    torch.cuda.synchronize()
    durs = [a.elapsed_time(b) for a, b in launches]
    avg_ms = sum(durs) / len(durs)
    peak, peak_src = hbm_peak()
    achieved = bytes_per_launch / (avg_ms / 1e3) / 1e9

    # end-to-end through the public API from pinned host memory
    pinned = {k: torch.from_numpy(v).pin_memory() for k, v in imgs.items()}
    probe = torch.empty(pinned[kinds[0]].numel(), dtype=torch.uint8, device="cuda")
    h2d_gbs = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        probe.copy_(pinned[kinds[0]], non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        h2d_gbs.append(probe.numel() / (e0.elapsed_time(e1) / 1e3) / 1e9)
    del probe
    e2e_steps = max(2, min(args.steps, 10))
    h2d = sum(v.numel() for v in pinned.values())
    d2h = n_out * cells * 8
    eng.glcm(pinned[kinds[0]].numpy(), n, n, levels, dts[:1], n_bands=n_bands)  # warm the pinned ring
    torch.cuda.synchronize()
    t = time.perf_counter()
    for s in range(e2e_steps):
        for kind in kinds:
            eng.glcm(pinned[kind].numpy(), n, n, levels, dts, n_bands=n_bands)
    e2e_s = (time.perf_counter() - t) / e2e_steps
    if dist:
        tt = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    e2e_value = world * pairs_per_step / e2e_s / 1e9

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import oracle as O
            if O.ref_available():
                threads = os.cpu_count() or 1
                v, calls = cpu_reference_rate({k: v for k, v in imgs.items()}, n, levels, dts,
                                              args.cpu_seconds, threads)
                cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                       "sample": f"{calls} single-(d,theta) GLCMs of the {n}x{n} L={levels} inputs "
                                 f"(reference compute_glcm_privatized, {threads} workers, ~{args.cpu_seconds:.0f}s)"}
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": f"{wl}: {n}x{n}{' x' + str(n_bands) + ' bands' if n_bands > 1 else ''} "
                                   f"{'+'.join(kinds)}, L={levels}, d={list(ds)}, theta=0/45/90/135, "
                                   f"device-resident, one launch per (d,theta)",
                       "pairs_per_step": pairs_per_step, "l2": "inputs (256 MiB each) larger than L2; no flush",
                       "parallelism": f"replica x{world}"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": committed_traffic(wl),
                         "kernel": "glcm_vote_kernel (+ glcm_reduce_partials_kernel for L*L > 4096)",
                         "bytes_per_launch": bytes_per_launch, "avg_launch_ms": avg_ms, "peak_source": peak_src},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "tfg_glcm (host pinned input, Scheme-3 stream pipeline, counts to host)",
                    "pinned_h2d_GBps": max(h2d_gbs), "ms_per_step": e2e_s * 1e3,
                    "h2d_bound_ms_per_step": h2d / (max(h2d_gbs) * 1e9) * 1e3},
            "gpu_launches": gpu_launches,
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
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
    args = ap.parse_args()
    if args.warmup < 3:
        log("note: warmup raised to the contract minimum of 3")
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args, args.workload)
    else:
        run_engine(args, args.workload)


if __name__ == "__main__":
    main()
