"""Pinned H2D time of 32 MiB on 12 fresh streams, 8 copies each, in order
(profiles/r02_e2e/h2d_ramp_probe.txt): shows the host link ramping from
~17 GB/s to ~55 GB/s under sustained traffic.
python tools/copy_engine_probe.py"""
import torch, time, statistics, json
w = 4096
buf = torch.empty(2 * w * w, dtype=torch.uint8).pin_memory()
dst = torch.empty_like(buf, device="cuda")
res = []
for k in range(12):
    s = torch.cuda.Stream()
    ts = []
    for _ in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s); dst.copy_(buf, non_blocking=True); e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res.append(round(statistics.median(ts), 3))
print(json.dumps({"per_stream_ms_32MiB": res}))
