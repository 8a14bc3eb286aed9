"""Prints the per-(input, d, theta) times of gpurun_out/abq_TAG/*.json side by side."""
import glob, json, os, sys
d = sys.argv[1]
for f in sorted(glob.glob(os.path.join(d, "*.json"))):
    try:
        r = json.load(open(f))
    except Exception as e:
        print(os.path.basename(f), "ERR", open(f).read()[-300:]); continue
    tot = sum(v["ms"] for v in r.values())
    print("%-16s sum %7.1f  " % (os.path.basename(f)[:-5], tot * 1000) +
          " ".join("%s:%.1f" % (k.replace("noise ", "n").replace("smooth ", "s").replace("d1 ", ""), v["ms"] * 1000) for k, v in r.items()))
