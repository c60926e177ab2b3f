"""Dev tool: an ncu `--page source --csv --print-source cuda,sass` export
aggregated by enclosing device function (file:function), with instructions
executed, thread instructions, stall samples.  The function of a line is the
nearest preceding definition line (__device__ / __global__ / PP_HD / struct
member functions) in that source file.
usage: python tools/ncu_regions.py export.csv [top]"""
import csv
import os
import re
import sys
from collections import defaultdict

DEF = re.compile(r"^\s*(template\s*<.*>\s*)?(__device__|__global__|PP_HD|__host__)[^;]*?(\w+)\s*\(")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def func_map(path):
    names = {}
    cur = "?"
    try:
        lines = open(path).read().split("\n")
    except OSError:
        return names
    for i, ln in enumerate(lines, 1):
        m = DEF.match(ln)
        if m:
            cur = m.group(3)
        names[i] = cur
    return names


rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = defaultdict(lambda: [0, 0, 0])
fname = None
fmap = {}
for r in rows:
    if r and r[0] in ("File Name", "File Path"):
        fname = r[1]
        p = fname if os.path.exists(fname) else os.path.join(ROOT, fname.split("/repo/")[-1])
        fmap = func_map(p)
        continue
    if fname is None or len(r) < 9 or not r[0].isdigit():
        continue
    try:
        stall, inst, tinst = int(r[4]), int(r[7]), int(r[8])
    except ValueError:
        continue
    key = f"{os.path.basename(fname)}:{fmap.get(int(r[0]), '?')}"
    a = agg[key]
    a[0] += inst
    a[1] += tinst
    a[2] += stall
ti = sum(a[0] for a in agg.values()) or 1
ts = sum(a[2] for a in agg.values()) or 1
print(f"total warp instructions {ti}, stall samples {ts}")
print(f"{'function':48s} {'inst%':>6s} {'thr/inst':>8s} {'stall%':>6s}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k:48s} {100 * a[0] / ti:6.1f} {a[1] / max(a[0], 1):8.1f} {100 * a[2] / ts:6.1f}")
