"""Dev tool: aggregate an ncu `--page source --print-source cuda,sass` CSV by
CUDA source line (stall samples, instructions executed), top N."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = []
hdr = None
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or r[0] == "" or r[0] in ("File Path", "Function Name"):
        continue
    try:
        out.append((int(r[4]), int(r[7]), int(r[0]), r[1][:90]))
    except (ValueError, IndexError):
        pass
tot = sum(o[0] for o in out) or 1
print(f"total stall samples {tot}")
for s, ins, ln, src in sorted(out, reverse=True)[:n]:
    print(f"{100*s/tot:5.1f}% samples  {ins:9d} inst  L{ln:4d}  {src}")
