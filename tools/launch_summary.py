"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_*)
into per-kernel rows: launches, mean/total device time, share of the total,
DRAM bytes per launch.  python tools/launch_summary.py launches.csv [--skip-torch]"""
import collections
import csv
import io
import json
import sys


def main():
    path = sys.argv[1]
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    launches = collections.defaultdict(set)
    for r in rows:
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        if "--skip-torch" in sys.argv and name.startswith("at::"):
            continue
        launches[name].add(r["ID"])
        v = float(r["Metric Value"].replace(",", "") or 0)
        unit = r["Metric Unit"]
        m = r["Metric Name"]
        if m == "gpu__time_duration.sum":
            v = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
            per[name]["time_us"] += v
        elif m.startswith("dram__bytes"):
            scale = {"byte": 1, "B": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9}.get(unit, 1)
            per[name]["dram_bytes"] += v * scale
    total = sum(p["time_us"] for p in per.values())
    out = []
    for name, p in sorted(per.items(), key=lambda kv: -kv[1]["time_us"]):
        n = len(launches[name])
        out.append({"kernel": name, "launches": n, "mean_us": p["time_us"] / n, "total_us": p["time_us"],
                    "share": p["time_us"] / total if total else 0.0,
                    "dram_bytes_per_launch": p["dram_bytes"] / n if p["dram_bytes"] else None})
    print(json.dumps({"source": path, "total_us": total, "kernels": out}, indent=1))


if __name__ == "__main__":
    main()
