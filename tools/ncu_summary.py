"""Dev tool: condense an ncu --set full report into profiles/<name>.json + .txt
(key throughput/occupancy metrics, DRAM traffic, top source lines by stall
samples).  Usage: python tools/ncu_summary.py gpurun_out/prof.ncu-rep name"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg", "sm__cycles_elapsed.avg.per_second",
        "smsp__thread_inst_executed_per_inst_executed.ratio"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3}


def run(args):
    return subprocess.run(args, capture_output=True, text=True, check=True).stdout


def main(rep, name, kernel=None):
    raw = list(csv.reader(io.StringIO(run(["ncu", "-i", rep, "--page", "raw", "--csv"]))))
    hdr, unit = raw[0], raw[1]
    rows = raw[2:]
    if kernel:
        rows = [r for r in rows if kernel in r[hdr.index("Kernel Name")]]
    val = rows[0]
    out = {"report": os.path.basename(rep), "kernel": val[hdr.index("Kernel Name")][:120]}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            try:
                v = float(val[i].replace(",", ""))
            except ValueError:
                v = val[i]
            out[k] = {"value": v, "unit": unit[i]}
    def to_bytes(k):
        m = out.get(k)
        return m["value"] * SCALE.get(m["unit"], 1) if m else 0.0
    out["dram_bytes_per_launch"] = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
    dur = out.get("gpu__time_duration.sum")
    if dur:
        out["duration_us"] = dur["value"] * SCALE.get(dur["unit"], 1)
    src_cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kernel:
        src_cmd += ["--kernel-name", f"regex:{kernel}"]
    src = run(src_cmd)
    rows = list(csv.reader(io.StringIO(src)))
    lines, hdr2 = [], None
    for r in rows:
        if r and r[0] == "Line No":
            hdr2 = r
            continue
        if hdr2 is None or not r or r[0] in ("", "File Path", "Function Name"):
            continue
        try:
            lines.append((int(r[4]), int(r[7]), int(r[0]), r[1].strip()[:100]))
        except (ValueError, IndexError):
            pass
    tot = sum(x[0] for x in lines) or 1
    out["top_lines"] = [{"stall_pct": round(100 * s / tot, 2), "inst": i, "line": ln, "src": t}
                        for s, i, ln, t in sorted(lines, reverse=True)[:25]]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{name}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "top_lines"}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
