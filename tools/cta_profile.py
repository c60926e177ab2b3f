"""Dev tool: per-CTA timing records of the scan and value kernels from the
profiling build (lib/libpassplan_b200_prof.so, -DPP_PHASE_CLOCKS).  Shows the
span of each kernel, the CTA duration distribution, the per-phase cycles and
the robot-warp imbalance inside scan CTAs.  Not used by tests/bench."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1909_07717_b200 import abi  # noqa: E402
from helpers import case_inputs  # noqa: E402

lib = abi._declare(C.CDLL(os.path.join(ROOT, "paper_1909_07717_b200", "lib",
                                       "libpassplan_b200_prof.so")))
NREC = 8192
P = C.POINTER(C.c_longlong)
lib.pp_debug_cta_records.argtypes = [P, P, P]
g = np.load(os.path.join(ROOT, "tests", "golden", "grids.npz"))
ctx = C.c_void_p()
assert lib.pp_ctx_create(0, C.byref(ctx)) == 0


def records():
    s = np.zeros((NREC, 8), np.int64)
    v = np.zeros((NREC, 8), np.int64)
    r = np.zeros((NREC, 16), np.int64)
    assert lib.pp_debug_cta_records(s.ctypes.data_as(P), v.ctypes.data_as(P),
                                    r.ctypes.data_as(P)) == 0
    return s, v, r


def pct(a):
    return f"mean={a.mean():.0f} p50={np.median(a):.0f} p90={np.percentile(a, 90):.0f} max={a.max():.0f}"


def report(label, n_scan, n_value, n_robots):
    s, v, r = records()
    s, v, r = s[:n_scan], v[:n_value], r[:n_scan, :n_robots]
    v = v[v[:, 0] > 0]
    t0 = s[:, 0].min()
    print(f"== {label}")
    print(f" scan: {n_scan} CTAs span {(s[:, 7].max() - t0) / 1e3:.1f} us; "
          f"CTA us {pct((s[:, 7] - s[:, 0]) / 1e3)}")
    print(f"   start offsets us: {pct((s[:, 0] - t0) / 1e3)}; SMs used {len(set(s[:, 6]))}")
    print(f"   lane-per-cell cyc {pct(s[:, 1])}\n   leftovers cyc {pct(s[:, 2])}\n"
          f"   champions cyc {pct(s[:, 3])}\n   leftover pairs {pct(s[:, 4])}\n"
          f"   window (A, part of phase 1) cyc {pct(s[:, 5])}")
    lib.pp_debug_champ_records.argtypes = [C.POINTER(C.c_longlong)]
    CR = np.zeros((8192, 4), np.int64)
    lib.pp_debug_champ_records(CR.ctypes.data_as(C.POINTER(C.c_longlong)))
    CR = CR[:n_scan]
    print(f"   champ outside marks {pct(s[:, 3] - (CR[:, 3] - CR[:, 0]))}\n   entry+argmin {pct(CR[:, 1] - CR[:, 0])} rx+stores "
          f"{pct(CR[:, 2] - CR[:, 1])} atomics+queue {pct(CR[:, 3] - CR[:, 2])}")
    lib.pp_debug_win_records.argtypes = [C.POINTER(C.c_longlong)]
    WR = np.zeros((8192, 4), np.int64)
    lib.pp_debug_win_records(WR.ctypes.data_as(C.POINTER(C.c_longlong)))
    WR = WR[:n_scan]
    print(f"   window incl. frame-field loads (warp 0, from CTA start) {pct(WR[:, 0] - WR[:, 3])}")
    lib.pp_debug_round_records.argtypes = [C.POINTER(C.c_longlong)]
    RR = np.zeros((8192, 8, 2), np.int64)
    lib.pp_debug_round_records(RR.ctypes.data_as(C.POINTER(C.c_longlong)))
    RR = RR[:n_scan]
    sl = np.argsort(s[:, 7] - s[:, 0])[-5:]
    for i in sl:
        nr = int(s[i, 4] // 10000) + 1
        parts = [f"{RR[i, r, 0]}@{RR[i, r + 1, 1] - RR[i, r, 1] if r + 1 < nr else 0}" for r in range(min(nr, 8))]
        print(f"   slow CTA {i} rounds (open pairs@cycles): {' '.join(parts)}")
    for i in sl:
        print(f"   slow CTA {i}: us {(s[i, 7] - s[i, 0]) / 1e3:.1f} phase1 {s[i, 1]} left {s[i, 2]} "
              f"champ {s[i, 3]} n_left {s[i, 4]}")
    rm = r.max(1)
    print(f"   robot-warp cyc {pct(r.ravel())}; per-CTA max/mean {np.mean(rm / r.mean(1)):.2f}")
    if len(v):
        print(f" value: {len(v)} CTAs start {(v[:, 0].min() - t0) / 1e3:.1f} us, end "
              f"{(v[:, 7].max() - t0) / 1e3:.1f} us (gap after scan "
              f"{(v[:, 0].min() - s[:, 7].max()) / 1e3:.1f} us); CTA us {pct((v[:, 7] - v[:, 0]) / 1e3)}")
        print(f"   D1 {pct(v[:, 1])}\n   D2 {pct(v[:, 2])}\n   D3a {pct(v[:, 5])}\n   D3b {pct(v[:, 3])}\n   red {pct(v[:, 4])}")
        late = np.argsort(v[:, 7])[-5:]
        for i in late:
            print(f"   late CTA: start {(v[i, 0] - t0) / 1e3:.1f} end {(v[i, 7] - t0) / 1e3:.1f} us "
                  f"D1 {v[i, 1]} D2 {v[i, 2]} D3 {v[i, 3]} red {v[i, 4]}")


w, p, grid, k, _ = case_inputs(g, "f8")
for chip in (1, 0):
    grid.chip = chip
    n = 128 * 64 * (1 + chip)
    blk = abi.GridBlock(n)
    for _ in range(5):
        lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), k, 1, blk.ptr())
    nq = blk.summary.n_feasible[0]
    report(f"F8 chip={chip} dev_ms={blk.summary.device_ms:.3f} feasible={nq}", n // 32,
           (nq + 31) // 32, w.n_ours - 1 + w.n_theirs)

# per-lane scan counters of the last (chip=0) launch
lib.pp_debug_lane_records.argtypes = [C.POINTER(C.c_int)]
L = np.zeros((1024, 16, 32, 6), np.int32)
lib.pp_debug_lane_records(L.ctypes.data_as(C.POINTER(C.c_int)))
nr = w.n_ours - 1 + w.n_theirs
L = L[:256, :nr]
_, _, R = records()
R = R[:256, :nr]
it = L[..., 0]
print("lane steps:", pct(it.ravel()), " skips", pct(L[..., 1].ravel()), " lbrej", pct(L[..., 2].ravel()))
print("warp max-lane steps:", pct(it.max(-1).ravel()), " rounds", pct(L[..., 0, 5].ravel()))
print("exact per lane", pct(L[..., 4].ravel()), " ub", pct(L[..., 3].ravel()))
# correlate warp cycles with max steps and rounds
ms = it.max(-1).ravel().astype(float)
rd = L[..., 0, 5].ravel().astype(float)
cy = R.ravel().astype(float)
A = np.stack([ms, rd, np.ones_like(ms)], 1)
coef = np.linalg.lstsq(A, cy, rcond=None)[0]
print(f"fit cycles ~= {coef[0]:.0f}*maxsteps + {coef[1]:.0f}*rounds + {coef[2]:.0f}")
top = np.argsort(cy)[-8:]
for i in top:
    t, r = divmod(i, nr)
    print(f" slow: tile {t} robot {r} cyc {cy[i]:.0f} maxsteps {ms[i]:.0f} rounds {rd[i]:.0f} "
          f"lbrej max {L[t, r, :, 2].max()} skip max {L[t, r, :, 1].max()}")
lib.pp_debug_warp_records.argtypes = [C.POINTER(C.c_longlong)]
W = np.zeros((1024, 16, 4), np.int64)
lib.pp_debug_warp_records(W.ctypes.data_as(C.POINTER(C.c_longlong)))
W = W[:256, :nr]
print("warp plain steps", pct(W[..., 0].ravel()), " coop steps", pct(W[..., 1].ravel()))
print("cyc/plain step (no coop warps)", pct((W[..., 3] / np.maximum(W[..., 0], 1))[W[..., 1] == 0]))
for i in top:
    t, r = divmod(i, nr)
    print(f" slow: tile {t} robot {r} plain {W[t, r, 0]} coop {W[t, r, 1]} first coop at cyc "
          f"{W[t, r, 2]} total {W[t, r, 3]}")
# by robot
print("per robot mean cycles:", np.round(R.mean(0)).astype(int).tolist())
print("per robot mean maxsteps:", np.round(it.max(-1).mean(0), 1).tolist())

# per-tile durations of the chip=1 frame for cost-model fitting (tools/tile_cost.py)
grid.chip = 1
blk = abi.GridBlock(16384)
for _ in range(3):
    lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), k, 1, blk.ptr())
s_, v_, r_ = records()
np.save(os.path.join(ROOT, "gpurun_out", "tile_cycles.npy"), r_[:512, :15])
np.save(os.path.join(ROOT, "gpurun_out", "tile_dur.npy"), (s_[:512, 7] - s_[:512, 0]))
