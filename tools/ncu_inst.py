"""Dev tool: instructions executed per CUDA source line (all files) from an
ncu `--page source --csv --print-source cuda,sass` export; top N."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
f = "?"
out = []
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) > 7 and r[0].isdigit() and r[2] == "-":
        try:
            out.append((int(r[7]), int(r[4]), f, int(r[0]), r[1][:80]))
        except ValueError:
            pass
tot = sum(o[0] for o in out) or 1
print(f"total inst {tot}")
for ins, s, fn, ln, src in sorted(out, reverse=True)[:n]:
    print(f"{100*ins/tot:5.1f}% {ins:9d} inst {s:6d} smp {fn}:{ln} {src}")
