"""Per-opcode stall attribution from an ncu source page (SASS) CSV(.gz):
python tools/sass_stalls.py file.sass.csv.gz [--top N] [--window ADDR N]"""
import csv
import gzip
import io
import sys
from collections import defaultdict


def load(path):
    f = io.TextIOWrapper(gzip.open(path)) if path.endswith(".gz") else open(path)
    rows = list(csv.reader(f))
    hdr = rows[1]
    return hdr, [r for r in rows[2:] if len(r) == len(hdr)]


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


def main():
    hdr, data = load(sys.argv[1])
    ix = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    by_op = defaultdict(lambda: defaultdict(float))
    tot = 0.0
    for r in data:
        op = r[ix["Source"]].split()[0] if r[ix["Source"]] else "?"
        if op.startswith("@"):
            op = r[ix["Source"]].split()[1]
        op = op.split(".")[0]
        s = num(r[ix["Warp Stall Sampling (All Samples)"]])
        tot += s
        by_op[op]["samples"] += s
        by_op[op]["exec"] += num(r[ix["Instructions Executed"]])
        by_op[op]["wf"] += num(r[ix["L1 Wavefronts Shared"]])
        for c in stall_cols:
            by_op[op][c] += num(r[ix[c]])
    print(f"total samples {tot:.0f}")
    top = sorted(by_op.items(), key=lambda kv: -kv[1]["samples"])[:int(sys.argv[sys.argv.index('--top') + 1]) if '--top' in sys.argv else 20]
    for op, d in top:
        st = sorted(((d[c], c[6:]) for c in stall_cols), reverse=True)[:4]
        print(f"{op:10s} {d['samples'] / tot * 100:5.1f}%  exec {d['exec']:12.0f}  smem_wf {d['wf']:11.0f}  " +
              ", ".join(f"{n} {v / max(d['samples'], 1) * 100:.0f}%" for v, n in st))


if __name__ == "__main__":
    main()
