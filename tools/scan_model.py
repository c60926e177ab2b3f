"""Dev tool (CPU): numpy model of the scan kernel's per-lane step counts on a
golden frame, to try skip/filter rules offline before writing them in CUDA.
float64 throughout; approximations are fine here (nothing is checked
against it).  Not used by tests/bench."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from helpers import case_inputs  # noqa: E402

g = np.load(os.path.join(ROOT, "tests", "golden", "grids.npz"))
case = sys.argv[1] if len(sys.argv) > 1 else "f8"
w, p, grid, kicker, _ = case_inputs(g, case)
SL, RO, RATIO = p.ball.slide_decel, p.ball.roll_decel, p.ball.transition_ratio
DT, RAD = p.thresholds.sbip_dt, p.thresholds.robot_radius
ND, NP = grid.n_directions, grid.n_powers


def one_d(v0, dist, a, b, vmax):
    brake = v0 * v0 / (2 * b)
    over = (v0 < 0) | (brake > dist)
    gap = brake - np.copysign(dist, v0)
    pk_r = np.sqrt(np.maximum(2 * a * b * gap / (a + b), 0))
    rr = np.where(pk_r <= vmax, pk_r / a + pk_r / b,
                  vmax / a + vmax / b + (gap - (vmax**2 / (2 * a) + vmax**2 / (2 * b))) / vmax)
    t_over = np.abs(v0) / b + rr
    pk = np.sqrt(np.maximum((2 * a * b * dist + b * v0 * v0) / (a + b), 0))
    t1 = (pk - v0) / a + pk / b
    t2 = (vmax - v0) / a + vmax / b + (dist - ((vmax**2 - v0**2) / (2 * a) + vmax**2 / (2 * b))) / vmax
    t3 = (v0 - vmax) / b + vmax / b + (dist - ((v0**2 - vmax**2) / (2 * b) + vmax**2 / (2 * b))) / vmax
    t_fwd = np.where(pk <= vmax, t1, np.where(v0 <= vmax, t2, t3))
    return np.where(over, t_over, t_fwd)


def arrival(qx, qy, vx, vy, a, b, vmax):
    d = np.hypot(qx, qy)
    deff = np.maximum(d - RAD, 0)
    dn = np.maximum(d, 1e-30)
    ex, ey = qx / dn, qy / dn
    va = vx * ex + vy * ey
    vc = vx * ey - vy * ex
    return np.maximum(one_d(va, deff, a, b, vmax), np.abs(vc) / b)


def reach_D(t, u, a, b, vmax):
    """ReachBound.reach (pp_kernels.cuh) in float64."""
    tb = u / b
    k = a * b / (a + b)
    tc0 = (vmax - u) / a + vmax / b
    d_used = (vmax**2 - u**2) / (2 * a) + vmax**2 / (2 * b)
    peak = (t + u / a) * k
    r = np.where(t <= tb, 0.5 * b * t * t,
                 np.where(u > vmax, u * u / (2 * b) + vmax * (t - tb),
                          np.where(t <= tc0, peak * peak / (2 * k) - u * u / (2 * a),
                                   d_used + vmax * (t - tc0))))
    return r


# cells (flat kick only), samples
ang = 2 * np.pi * np.arange(ND) / ND
ux, uy = np.cos(ang), np.sin(ang)
speed = p.grid.power_min + np.arange(NP) * (p.grid.power_max - p.grid.power_min) / max(NP - 1, 1)
v1 = RATIO * speed
t_se = (speed - v1) / SL
d_se = (speed**2 - v1**2) / (2 * SL)
t_stop = t_se + v1 / RO
d_stop = d_se + v1**2 / (2 * RO)
count = np.floor(t_stop / DT + 1e-9).astype(int) + 1
K = count.max()
k = np.arange(K)
t = k * DT
T, KK = np.meshgrid(t, k, indexing="ij")[0], None
s = np.where(t[None, :] < t_se[:, None], speed[:, None] * t - 0.5 * SL * t * t,
             np.where(t[None, :] < t_stop[:, None],
                      d_se[:, None] + v1[:, None] * (t - t_se[:, None]) - 0.5 * RO * (t - t_se[:, None])**2,
                      d_stop[:, None]))                    # [NP, K]
spd = np.where(t[None, :] < t_se[:, None], speed[:, None] - SL * t,
               np.where(t[None, :] < t_stop[:, None], v1[:, None] - RO * (t - t_se[:, None]), 0))
ox, oy = w.ball_px, w.ball_py
hx, hy = w.field.length / 2, w.field.width / 2
with np.errstate(divide="ignore"):
    ex_x = np.where(ux > 0, (hx - ox) / ux, np.where(ux < 0, (-hx - ox) / ux, np.inf))
    ex_y = np.where(uy > 0, (hy - oy) / uy, np.where(uy < 0, (-hy - oy) / uy, np.inf))
d_exit = np.minimum(ex_x, ex_y)                              # [ND]
# window end per cell: samples with s <= d_exit (approx)
ke = np.minimum(count[None, :], (s[None, :, :] <= d_exit[:, None, None] + 1e-12).sum(-1))
valid_k = k[None, None, :] < ke[:, :, None]                  # [ND, NP, K]

robots = []
ours = sorted([w.ours[i] for i in range(w.n_ours)], key=lambda r: r.id)
theirs = sorted([w.theirs[i] for i in range(w.n_theirs)], key=lambda r: r.id)
for r in ours:
    if r.id != kicker:
        robots.append((0, r, p.motion_ours))
for r in theirs:
    robots.append((1, r, p.motion_theirs))

bx = ox + ux[:, None, None] * s[None, :, :]
by = oy + uy[:, None, None] * s[None, :, :]
res = []
for team, r, m in robots:
    a, b, vmax = m.max_accel, m.max_decel, m.max_speed
    u = np.hypot(r.vx, r.vy)
    vb = max(u, vmax)
    qx, qy = bx - r.px, by - r.py
    d = np.hypot(qx, qy)
    T_arr = arrival(qx, qy, r.vx, r.vy, a, b, vmax)
    hit = valid_k & (T_arr <= t) & (d <= RAD + vb * t)
    thr = RAD + reach_D(t, u, a, b, vmax) * 1.0001 + 1e-4
    reach_ok = d <= thr
    first = np.where(hit.any(-1), hit.argmax(-1), 10**6)
    # closest approach coordinate on each ray
    s0 = (r.px - ox) * ux + (r.py - oy) * uy                 # [ND]
    h = np.abs(-(r.px - ox) * uy + (r.py - oy) * ux)
    res.append(dict(team=team, d=d, thr=thr, reach_ok=reach_ok, hit=hit, first=first,
                    s0=s0, h=h, vb=vb, T=T_arr))

cap = np.full((2, ND, NP), 10**6)
for R in res:
    cap[R["team"]] = np.minimum(cap[R["team"]], R["first"])


def simulate(R, rule):
    """Step count per lane of the current kernel loop (rule='cur') or a variant."""
    d, thr, T = R["d"], R["thr"], R["T"]
    c = cap[R["team"]]
    kcur = np.zeros((ND, NP), int)
    steps = np.zeros((ND, NP), int)
    done = np.zeros((ND, NP), bool) | (ke <= 0)
    ii, jj = np.meshgrid(np.arange(ND), np.arange(NP), indexing="ij")
    s0 = R["s0"][:, None] + 1e-3
    for _ in range(400):
        act = ~done
        if not act.any():
            break
        kk = np.minimum(kcur, K - 1)
        end = (kcur >= ke) | (kcur > c)
        done |= act & end
        act &= ~end
        steps += act
        dd, th = d[ii, jj, kk], thr[kk]
        tt = kk * DT
        sk = s[jj, kk]
        out = dd > th
        gap = dd - th
        if rule == "cur":
            appr = np.where(sk < s0, spd[jj, kk], 0)
            j = np.floor(gap / ((appr + R["vb"]) * DT * 1.0001) * 0.9999)
            adv = (1 + np.where(j > 1, np.minimum(j, 4096) - 1, 0)).astype(int)
        else:
            # Lipschitz skip, then interval certificates for far samples
            appr = np.where(sk < s0, spd[jj, kk], 0)
            j = np.floor(gap / ((appr + R["vb"]) * DT * 1.0001) * 0.9999)
            adv = (1 + np.where(j > 1, np.minimum(j, 4096) - 1, 0)).astype(int)
            s0lo = R["s0"][:, None] - 1e-3
            h = R["h"][:, None]
            for jc in CANDS[rule]:
                kb_ = np.minimum(kk + jc, K - 1)
                sb = s[jj, kb_]
                db = d[ii, jj, kb_]
                thb = thr[kb_]
                # approach: s_b <= s0 -> d_min = d_b
                ok_app = (sb <= s0lo) & (db > thb)
                # containing s0: d_min >= h
                ok_mid = (h > thb)
                # chase: s_a >= s0: tangent at s_b, check both ends
                cb = (sb - R["s0"][:, None]) / np.maximum(db, 1e-9)
                ok_ch = (sk >= s0) & (db > thb) & (db - cb * (sb - sk) > th)
                ok = out & (ok_app | ok_mid | ok_ch) & (kk + jc <= ke)
                adv = np.where(ok, np.maximum(adv, jc + 1), adv)
        lbrej = ~out & (T[ii, jj, kk] > tt)
        hitn = ~out & ~lbrej
        kcur = np.where(act & out, kcur + adv, np.where(act & lbrej, kcur + 1, kcur))
        done |= act & hitn
    return steps


def cand_adv(R, di, pj, kk, cands):
    """Largest certified advance from an out-of-reach sample kk using
    far-sample interval certificates (approach / contains-s0 / chase)."""
    d, thr = R["d"], R["thr"]
    s0 = R["s0"][di]
    h = R["h"][di]
    sa = s[pj, kk]
    best = 0
    for jc in cands:
        kb_ = kk + jc
        if kb_ >= ke[di, pj]:
            break
        sb, db, thb = s[pj, kb_], d[di, pj, kb_], thr[kb_]
        if sb <= s0 - 1e-3:
            ok = db > thb
        elif sa >= s0 + 1e-3:
            cb = (sb - s0) / max(db, 1e-9)
            ok = db > thb and db - cb * (sb - sa) > thr[kk]
        else:
            ok = h > thb
        if ok:
            best = max(best, jc + 1)
    return best


def simulate_coop(R, coop_max=16, cands=()):
    """Warp-level model: when <= coop_max lanes of a warp are still scanning,
    idle lanes evaluate the next samples of the active cells (m = 32 // n_a
    consecutive samples per active cell per step)."""
    d, thr, T = R["d"], R["thr"], R["T"]
    c = cap[R["team"]]
    s0 = R["s0"][:, None] + 1e-3
    steps_w = np.zeros((ND, NP // 32), int)
    for di in range(ND):
        for wg in range(NP // 32):
            lanes = np.arange(wg * 32, wg * 32 + 32)
            kc = np.zeros(32, int)
            done = ke[di, lanes] <= 0
            n = 0
            while not done.all() and n < 500:
                act = np.flatnonzero(~done)
                n += 1
                m = 32 // len(act) if len(act) <= coop_max else 1
                for L in act:
                    pj = lanes[L]
                    adv = 0
                    for i in range(m):
                        kk = kc[L] + i
                        if kk >= ke[di, pj] or kk > c[di, pj]:
                            done[L] = True
                            break
                        if d[di, pj, kk] > thr[kk]:
                            sk = s[pj, kk]
                            appr = spd[pj, kk] if sk < s0[di, 0] else 0
                            gap = d[di, pj, kk] - thr[kk]
                            j = np.floor(gap / ((appr + R["vb"]) * DT * 1.0001) * 0.9999)
                            a_i = 1 + (min(j, 4096) - 1 if j > 1 else 0)
                            if cands:
                                a_i = max(a_i, cand_adv(R, di, pj, kk, cands))
                            adv = max(adv, i + int(a_i))
                            continue
                        if T[di, pj, kk] > kk * DT:
                            adv = max(adv, i + 1)
                            continue
                        done[L] = True  # hit / candidate (exact round, ignored here)
                        break
                    if not done[L]:
                        kc[L] += max(adv, m if m > 1 else adv)
            steps_w[di, wg] = n
    return steps_w


if "--coop" in sys.argv:
    for cm, cands in ((0, ()), (16, ()), (0, (4, 16, 64)), (16, (4, 16, 64)), (16, (8, 32)),
                      (16, (2, 8, 32, 128)), (32, (4, 16, 64))):
        tot = np.array([simulate_coop(R, cm, cands) for R in res])
        print(f"coop<= {cm} cands {cands}: warp steps mean {tot.mean():.2f} p90 {np.percentile(tot, 90)} max {tot.max()}")
    sys.exit(0)

CANDS = {"c1": [8], "c2": [4, 16], "c3": [2, 8, 32], "c6": [2, 4, 8, 16, 32, 64]}
for rule in ["cur"] + list(CANDS):
    tot = np.array([simulate(R, rule).reshape(ND, NP // 32, 32).max(-1) for R in res])
    lanes = np.array([simulate(R, rule) for R in res])
    print(f"{rule}: lane mean {lanes.mean():.2f} warp max-steps mean {tot.mean():.2f} p90 {np.percentile(tot, 90)} max {tot.max()}")
tot = []
for i, R in enumerate(res):
    st = simulate(R, "cur")
    # warp = 32 consecutive powers of one direction
    wmax = st.reshape(ND, NP // 32, 32).max(-1)
    tot.append(wmax)
    print(f"robot {i} team {R['team']}: lane steps mean {st.mean():.1f} max {st.max()} | "
          f"warp max-steps mean {wmax.mean():.1f} max {wmax.max()} | hits {np.mean(R['first'] < 10**6):.2f}")
tot = np.array(tot)
print("all robot-warps: mean max-steps", tot.mean(), "p90", np.percentile(tot, 90), "max", tot.max())

if "--trace" in sys.argv:
    ri = int(sys.argv[sys.argv.index("--trace") + 1])
    R = res[ri]
    st = simulate(R, "cur")
    di, pj = np.unravel_index(st.argmax(), st.shape)
    team, r, m = robots[ri]
    print(f"robot {ri} pos ({r.px:.2f},{r.py:.2f}) vel ({r.vx:.2f},{r.vy:.2f}); dir {di} power {pj} "
          f"speed {speed[pj]:.2f} ke {ke[di, pj]} first {R['first'][di, pj]} cap {cap[team][di, pj]} s0 {R['s0'][di]:.2f}")
    for kk in range(0, min(ke[di, pj], 200)):
        print(f"  k {kk:3d} s {s[pj, kk]:.3f} d {R['d'][di, pj, kk]:.3f} thr {R['thr'][kk]:.3f} "
              f"T {R['T'][di, pj, kk]:.3f} t {kk * DT:.3f} {'REACH' if R['d'][di, pj, kk] <= R['thr'][kk] else ''}")
