// pp_value.cuh -- value_kernel: score_pass + best_pass over the queued cells
// (pass_eval.cpp:148-187), chunk argmax and the frame fold.
#pragma once

#include "pp_scan.cuh"

namespace pp {

// ---- value: one CTA per chunk of a frame's queue ---------------------------
struct ValueSmem {
  FrameDev frame;
  double q_rx[kChunk], q_ry[kChunk], q_ot[kChunk], q_pt[kChunk];
  int32_t q_cell[kChunk];
  int8_t q_slot[kChunk];
  // goal-view work items
  int iv_n;
  uint8_t iv_e[kIvCap];
  int8_t iv_j[kIvCap];
  int16_t iv_first[kIvCap], iv_last[kIvCap];
  uint8_t iv_fast[kIvCap];
  double iv_y1[kIvCap], iv_y2[kIvCap], iv_lo[kIvCap], iv_hi[kIvCap], iv_margin[kIvCap];
  double iv_alo[kIvCap], iv_ahi[kIvCap];  // atan2 of the edges seen from the cell
  double gap_lo[kIvCap], gap_w[kIvCap];   // the sweep's gap ending at each interval
  uint8_t gap_ok[kIvCap];
  double ch_am[kChunk], ch_ap[kChunk];    // ... and of the two posts
  uint8_t ch_zero[kChunk], ch_over[kChunk];
  int ch_n[kChunk];                    // intervals of each cell ...
  int16_t ch_iv[kChunk][kMaxTeamIv];   // ... and their slots
  double feat[kChunk][5];
  double heights[kMaxHeights];
  int hts_ok, n_half;
  double w_score[kMaxWarps][2];
  int64_t w_cell[kMaxWarps][2];
  int32_t w_idx[kMaxWarps][2];
  unsigned last;
  int n_act;  // streaming: queue size seen at start (-1 full chunk) / final chunk count
  int n_keep;  // batch pruning: cells of the chunk left after the score bounds
};

// Warp partials of a frame fold (last chunk done).
struct FoldSmem {
  double w_score[kMaxWarps][2];
  int64_t w_cell[kMaxWarps][2];
  int32_t w_idx[kMaxWarps][2];
};

// The view heights (pass_eval.cpp:65-71) of a frame, once per CTA; the
// caller syncs.
__device__ __forceinline__ void value_heights(ValueSmem& sm, const DevParams& P) {
  const ViewCtx V0 = make_view_ctx(0.0, 0.0, sm.frame, P.radius, P.r_lt2, P.mb_le2);
  const bool ok = V0.nh <= kMaxHeights;
  if (ok)
    for (int i = threadIdx.x; i < V0.nh; i += blockDim.x)
      sm.heights[i] = view_height(i, V0.n_half, V0.gh).v;
  if (threadIdx.x == 0) {
    sm.hts_ok = ok;
    sm.n_half = V0.n_half;
  }
}

// D1  thread per (cell, opponent): on-point test, gates, first/last blocked
//     height -> an interval slot
// D2  thread per (interval slot, edge): the edge bisection
// D3  thread per cell: sort + sweep (atan2), score_pass, score map store
// then the chunk's argmax per kick slot and a last-chunk-done reduction.
// One value chunk: queue entries [e0, e0 + m) of frame f (sm.frame loaded).
// Thread 0 writes the chunk's Partial to *dst.
// lb0/lb1 (batches, !kCells): the frame's score lower-bound keys per kick
// slot; a cell whose score upper bound is below its slot's key is dropped
// before the goal view (it cannot be best_pass), 0 = keep every cell.
template <bool kCells>
__device__ __forceinline__ void value_chunk(ValueSmem& sm, const DevParams& P, const CellQueue& q,
                                            const CellOut& out, int f, int e0, int m,
                                            Partial* dst, unsigned long long lb0 = 0ull,
                                            unsigned long long lb1 = 0ull) {
  PP_CLOCK_INIT();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x < m) {
    PP_CHECK(e0 + static_cast<int64_t>(threadIdx.x) < q.cap);
    const int64_t pos = static_cast<int64_t>(f) * q.cap + e0 + threadIdx.x;
    sm.q_rx[threadIdx.x] = __ldcg(&q.rx[pos]);
    sm.q_ry[threadIdx.x] = __ldcg(&q.ry[pos]);
    sm.q_ot[threadIdx.x] = __ldcg(&q.ot[pos]);
    sm.q_pt[threadIdx.x] = __ldcg(&q.pt[pos]);
    sm.q_cell[threadIdx.x] = __ldcg(&q.cell[pos]);
    sm.q_slot[threadIdx.x] = __ldcg(&q.slot[pos]);
  }
  if (threadIdx.x < kChunk) {
    sm.ch_zero[threadIdx.x] = 0;
    sm.ch_over[threadIdx.x] = 0;
    sm.ch_n[threadIdx.x] = 0;
  }
  if (threadIdx.x == 0) sm.iv_n = 0;
  __syncthreads();
  if (!kCells && (lb0 | lb1)) {
    // Batch pruning (warp 0, lane = queued cell; m <= 32): keep the cells
    // whose score upper bound reaches their slot's best lower bound,
    // compacted in queue order.
    if (warp == 0) {
      const int e = lane;
      double rx = 0.0, ry = 0.0, ot = 0.0, pt = 0.0;
      int32_t cell = 0;
      int8_t slot = 0;
      bool keep = false;
      if (e < m) {
        rx = sm.q_rx[e];
        ry = sm.q_ry[e];
        ot = sm.q_ot[e];
        pt = sm.q_pt[e];
        cell = sm.q_cell[e];
        slot = sm.q_slot[e];
        double lo, hi;
        score_bounds(rx, ry, ot, pt, sm.frame, P, &lo, &hi);
        keep = score_key(hi) >= (slot ? lb1 : lb0);
      }
      const unsigned km = __ballot_sync(0xffffffffu, keep);
      __syncwarp();
      if (keep) {
        const int at = __popc(km & ((1u << lane) - 1u));
        sm.q_rx[at] = rx;
        sm.q_ry[at] = ry;
        sm.q_ot[at] = ot;
        sm.q_pt[at] = pt;
        sm.q_cell[at] = cell;
        sm.q_slot[at] = slot;
      }
      if (lane == 0) sm.n_keep = __popc(km);
    }
    __syncthreads();
    m = sm.n_keep;
  }
  const FrameDev& F = sm.frame;
  const int nt = F.n_theirs;
  const xd radius = P.radius;
  // view heights (pass_eval.cpp:65-71), filled by value_heights
  const double* hts = sm.hts_ok ? sm.heights : nullptr;
  // D1
  for (int pr = threadIdx.x; pr < m * nt; pr += blockDim.x) {
    const int e = pr / nt, j = pr % nt;
    const ViewCtx V =
        make_view_ctx(sm.q_rx[e], sm.q_ry[e], F, radius, P.r_lt2, P.mb_le2, hts, sm.n_half,
                      P.exact_only != 0);
    if ((V.gx - V.px).v < 1e-9) continue;  // behind the goal line: zero view
    PP_D1_T0();
    const PairInfo pi = pair_info(V, F.px[kTheirs + j], F.py[kTheirs + j]);
    PP_D1_T1(pr, pi);
    if (pi.status == 2) {
      sm.ch_zero[e] = 1;
    } else if (pi.status == 1) {
      const int slot = atomicAdd(&sm.iv_n, 1);
      if (slot >= kIvCap) {
        sm.ch_over[e] = 1;  // rare: this cell's view is recomputed whole in D3
      } else {
        sm.iv_e[slot] = static_cast<uint8_t>(e);
        sm.iv_j[slot] = static_cast<int8_t>(j);
        sm.iv_first[slot] = static_cast<int16_t>(pi.first);
        sm.iv_last[slot] = static_cast<int16_t>(pi.last);
        sm.iv_fast[slot] = pi.fast;
        sm.iv_y1[slot] = pi.y1.v;
        sm.iv_y2[slot] = pi.y2.v;
        sm.iv_margin[slot] = pi.margin;
        const int at = atomicAdd(&sm.ch_n[e], 1);
        PP_CHECK(at < kMaxTeamIv);
        sm.ch_iv[e][at] = static_cast<int16_t>(slot);
      }
    }
  }
  __syncthreads();
  PP_MARK(3);
  // D2
  const int ns = sm.iv_n < kIvCap ? sm.iv_n : kIvCap;
  PP_D2_DECL();
  for (int job = threadIdx.x; job < 2 * ns + 2 * m; job += blockDim.x) {
    if (job >= 2 * ns) {  // post angles of cell e (the sweep's fixed ends)
      const int e = (job - 2 * ns) >> 1, side = job & 1;
      const xd py = sm.q_ry[e];
      const xd gh = xd(0.5) * xd(F.gw);
      const xd x_off = xd(0.5) * xd(F.L) - xd(sm.q_rx[e]);
      const double a = atan2(((side ? gh : -gh) - py).v, x_off.v);
      if (side) {
        sm.ch_ap[e] = a;
      } else {
        sm.ch_am[e] = a;
      }
      continue;
    }
    const int slot = job >> 1, edge = job & 1;
    const int e = sm.iv_e[slot];
    if (sm.ch_zero[e] || sm.ch_over[e]) continue;
    const ViewCtx V =
        make_view_ctx(sm.q_rx[e], sm.q_ry[e], F, radius, P.r_lt2, P.mb_le2, hts, sm.n_half,
                      P.exact_only != 0);
    const int j = sm.iv_j[slot];
    PP_D2_JOB(sm.iv_fast[slot]);
    const xd y = interval_edge_split(V, F.px[kTheirs + j], F.py[kTheirs + j], edge, sm.iv_first[slot],
                               sm.iv_last[slot], sm.iv_fast[slot], sm.iv_y1[slot], sm.iv_y2[slot],
                               sm.iv_margin[slot], PP_D2_ST);
    const double a = atan2((y - V.py).v, (V.gx - V.px).v);
    if (edge == 0) {
      sm.iv_lo[slot] = y.v;
      sm.iv_alo[slot] = a;
    } else {
      sm.iv_hi[slot] = y.v;
      sm.iv_ahi[slot] = a;
    }
  }

  PP_D2_FLUSH();
  __syncthreads();
  PP_MARK(4);
  // D3a  thread per interval slot: the sweep's gap ending at this interval
  //      (pass_eval.cpp:96-125).  In lo order the cursor before interval q
  //      is the largest hi of the intervals with a smaller lo (equal-lo
  //      intervals cannot open a gap at q), so each gap is found without
  //      sorting; its width uses the atan2 values from D2.
  for (int slot = threadIdx.x; slot < ns; slot += blockDim.x) {
    const int e = sm.iv_e[slot];
    if (sm.ch_zero[e] || sm.ch_over[e]) continue;
    const xd lo_q = sm.iv_lo[slot];
    xd cur = -(xd(0.5) * xd(F.gw));
    double a_cur = sm.ch_am[e];
    const int n = sm.ch_n[e];
    for (int q = 0; q < n; ++q) {
      const int p = sm.ch_iv[e][q];
      const double hp = sm.iv_hi[p];
      if (sm.iv_lo[p] < lo_q.v && hp > cur.v) {
        cur = hp;
        a_cur = sm.iv_ahi[p];
      }
    }
    sm.gap_ok[slot] = lo_q > cur;
    sm.gap_lo[slot] = cur.v;
    sm.gap_w[slot] = (xd(sm.iv_alo[slot]) - xd(a_cur)).v;
  }
  __syncthreads();
  PP_MARK(7);
  // D3b  thread per cell: the widest gap (first in lo order on ties, the
  //      final gap up to the post last), score_pass, score map store
  double bs[2] = {0.0, 0.0};
  int64_t bc[2] = {-1, -1};
  if (threadIdx.x < m) {
    const int e = threadIdx.x;
    View v{0.0, 0.0, 0.0, 0.0};
    if (sm.ch_over[e]) {
      v = goal_view_thread(sm.q_rx[e], sm.q_ry[e], F, radius, P.r_lt2, P.mb_le2,
                           P.exact_only != 0);
    } else if (!sm.ch_zero[e] && !((xd(0.5) * xd(F.L) - xd(sm.q_rx[e])).v < 1e-9)) {
      const xd gh = xd(0.5) * xd(F.gw);
      xd best_lo = 0.0, best_hi = 0.0, best_w = -1.0;
      xd cursor = -gh;
      double a_fin = sm.ch_am[e];
      const int n = sm.ch_n[e];
      for (int q = 0; q < n; ++q) {
        const int slot = sm.ch_iv[e][q];
        const double hq = sm.iv_hi[slot];
        if (hq > cursor.v) {
          cursor = hq;
          a_fin = sm.iv_ahi[slot];
        }
        if (!sm.gap_ok[slot]) continue;
        const xd w = sm.gap_w[slot];
        const xd b = sm.iv_lo[slot];
        if (w > best_w || (w.v == best_w.v && b < best_hi)) {
          best_w = w;
          best_lo = sm.gap_lo[slot];
          best_hi = b;
        }
      }
      if (cursor < gh) {
        const xd w = xd(sm.ch_ap[e]) - xd(a_fin);
        if (w > best_w) {
          best_w = w;
          best_lo = cursor;
          best_hi = gh;
        }
      }
      if (best_w.v > 0.0) {
        v.angle = best_w.v;
        v.lo = best_lo.v;
        v.hi = best_hi.v;
        v.ty = (xd(0.5) * (best_lo + best_hi)).v;
      }
    }
    double* feat = sm.feat[e];
    const double sc = score_from_view(v, sm.q_rx[e], sm.q_ry[e], sm.q_ot[e], sm.q_pt[e], F, P,
                                      feat);
    const int64_t c = sm.q_cell[e];
    PP_CHECK(c >= 0 && c < static_cast<int64_t>(P.n_kt) * P.n_dirs * P.n_pows);
    if (kCells) out.score[c] = static_cast<float>(sc);
    // (selects, not a runtime-indexed store: bs/bc stay in registers)
    const bool s1 = sm.q_slot[e] != 0;
    bs[0] = s1 ? bs[0] : sc;
    bc[0] = s1 ? bc[0] : c;
    bs[1] = s1 ? sc : bs[1];
    bc[1] = s1 ? c : bc[1];
  }
  PP_MARK(5);
  // The chunk's argmax per kick slot: D3 ran on warp 0 only (m <= 32), so one
  // warp-wide redux picks the max score (as an order-preserving key; +0.0
  // folds -0.0 so ties compare like `better`), then the lowest cell among the
  // ties -- the same winner as best_pass's first strict max in cell order.
  static_assert(kChunk <= 32, "D3 must fit one warp");
  if (warp == 0) {
    __syncwarp();  // sm.feat rows of the other lanes
    Partial p;
    reset_partial(p);
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const bool valid = bc[s] >= 0;
      const long long bits = __double_as_longlong(__dadd_rn(bs[s], 0.0));
      const unsigned long long key =
          valid ? (bits < 0 ? ~static_cast<unsigned long long>(bits)
                            : static_cast<unsigned long long>(bits) | (1ull << 63))
                : 0ull;
      const unsigned hi = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(key >> 32));
      const unsigned lo = __reduce_max_sync(
          0xffffffffu, static_cast<unsigned>(key >> 32) == hi ? static_cast<unsigned>(key) : 0u);
      const bool cand = valid && key == ((static_cast<unsigned long long>(hi) << 32) | lo);
      const unsigned cmin =
          __reduce_min_sync(0xffffffffu, cand ? static_cast<unsigned>(bc[s]) : 0xffffffffu);
      const unsigned win = __ballot_sync(0xffffffffu, cand && static_cast<unsigned>(bc[s]) == cmin);
      if (win) {
        const int wl = __ffs(win) - 1;
        p.score[s] = __shfl_sync(0xffffffffu, bs[s], wl);
        p.cell[s] = cmin;
        for (int k = 0; k < 5; ++k) p.feat[s][k] = sm.feat[wl][k];  // written by lane wl
      }
    }
    if (lane == 0) *dst = p;
  }
  PP_MARK(6);
  PP_FLUSH(9);
}

// Batches, between scan and value: per frame (one warp), the largest lower
// bound of a queued cell's score per kick slot (score_bounds), into
// FrameCounters::lb_key -- value_chunk then drops every cell whose upper
// bound is below its slot's key before the goal view (it cannot be the
// slot's best_pass).  The queue is complete: this grid runs after the scan.
#ifndef PP_SCORE_LB_MINB
#define PP_SCORE_LB_MINB 4  // 64 registers: 4 CTAs/SM (C5 -1.5 % against 128 registers, 2 CTAs)
#endif
__global__ void __launch_bounds__(256, PP_SCORE_LB_MINB) score_lb_kernel(const FrameDev* __restrict__ frames,
                                                       DevParams P, CellQueue q,
                                                       FrameCounters* __restrict__ fc,
                                                       int64_t n_frames) {
  const int64_t f = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  // (the value grid, launched programmatically after this one, waits for it)
  asm volatile("griddepcontrol.launch_dependents;");
  if (f >= n_frames) return;
  const FrameDev& F = frames[f];
  const int n = static_cast<int>(fc[f].q_count);
  unsigned long long best[2] = {0ull, 0ull};
  int at[2] = {-1, -1};
  for (int e = lane; e < n; e += 32) {
    const int64_t pos = f * q.cap + e;
    double lo;
    score_bounds<true>(q.rx[pos], q.ry[pos], q.ot[pos], q.pt[pos], F, P, &lo, nullptr);
    const unsigned long long k = score_key(lo);
    const int s = q.slot[pos];
    if (k > best[s]) {
      best[s] = k;
      at[s] = e;
    }
  }
  for (int s = 0; s < 2; ++s) {
    const unsigned hi = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(best[s] >> 32));
    const unsigned lo = __reduce_max_sync(
        0xffffffffu, static_cast<unsigned>(best[s] >> 32) == hi ? static_cast<unsigned>(best[s]) : 0u);
    const unsigned long long key = (static_cast<unsigned long long>(hi) << 32) | lo;
    // The slot's most promising cell gets its exact score (the same
    // goal_view + score_pass the value kernel runs): the slot's best_pass is
    // at least that, so it is a far tighter bound than the cell's own lower
    // bound.  (A small slack keeps it a bound even if a last ulp differed.)
    const unsigned owner = __ballot_sync(0xffffffffu, key != 0ull && best[s] == key);
    unsigned long long out = key;
    if (owner && lane == __ffs(owner) - 1) {
      const int64_t pos = f * q.cap + at[s];
      const double rx = q.rx[pos], ry = q.ry[pos];
      const View v = goal_view_thread(rx, ry, F, P.radius, P.r_lt2, P.mb_le2, P.exact_only != 0);
      double feat[5];
      const double sc = score_from_view(v, rx, ry, q.ot[pos], q.pt[pos], F, P, feat);
      const unsigned long long k2 = score_key(sc - (1e-9 + 1e-12 * fabs(sc)));
      out = k2 > key ? k2 : key;
    }
    out = __shfl_sync(0xffffffffu, out, owner ? __ffs(owner) - 1 : 0);
    if (lane == 0) fc[f].lb_key[s] = out;
  }
}

// Fold the n chunk partials of frame f into its summary (all threads of the
// CTA).  `better` is a strict total order on (score desc, cell asc), so the
// fold order cannot change the winner.  Resets the frame's counters.
__device__ __forceinline__ void fold_frame(FoldSmem& fs, const Partial* base, int n,
                                           FrameCounters* fcf, const DevParams& P,
                                           pp_dpps_summary* S, int f) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  __threadfence();
  double rs[2] = {0.0, 0.0};
  int64_t rc[2] = {-1, -1};
  int rb[2] = {-1, -1};
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const volatile Partial* p = base + i;
    for (int s = 0; s < 2; ++s) {
      const double ps = p->score[s];
      const int64_t pc = p->cell[s];
      if (better(ps, pc, rs[s], rc[s])) {
        rs[s] = ps;
        rc[s] = pc;
        rb[s] = i;
      }
    }
  }
  for (int s = 0; s < 2; ++s) {
    for (int off = 16; off > 0; off >>= 1) {
      const double os = __shfl_down_sync(0xffffffffu, rs[s], off);
      const int64_t oc = __shfl_down_sync(0xffffffffu, rc[s], off);
      const int ob = __shfl_down_sync(0xffffffffu, rb[s], off);
      if (better(os, oc, rs[s], rc[s])) {
        rs[s] = os;
        rc[s] = oc;
        rb[s] = ob;
      }
    }
    if (lane == 0) {
      fs.w_score[warp][s] = rs[s];
      fs.w_cell[warp][s] = rc[s];
      fs.w_idx[warp][s] = rb[s];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    Partial acc;
    reset_partial(acc);
    for (int s = 0; s < 2; ++s) {
      int b = -1;
      for (int w = 0; w < nwarps; ++w) {
        if (better(fs.w_score[w][s], fs.w_cell[w][s], acc.score[s], acc.cell[s])) {
          acc.score[s] = fs.w_score[w][s];
          acc.cell[s] = fs.w_cell[w][s];
          b = fs.w_idx[w][s];
        }
      }
      if (b >= 0) {
        const volatile Partial* p = base + b;
        for (int k = 0; k < 5; ++k) acc.feat[s][k] = p->feat[s][k];
      }
      acc.n_feasible[s] = fcf->n_feas[s];
    }
    if (P.compact) {
      write_compact(P.compact + f, acc, P);
    } else {
      write_summary(S, acc, P);
      // kernel span of this frame: first scan CTA start -> this fold
      S->device_ms = fcf->t0_inv ? static_cast<double>(pp_now_ns() - ~fcf->t0_inv) * 1e-6 : 0.0;
    }
    fcf->t0_inv = 0ull;
    fcf->q_count = 0;  // self-cleaning for the next launch / graph replay
    fcf->n_feas[0] = 0;
    fcf->n_feas[1] = 0;
    fcf->chunks_done = 0;
    fcf->lb_key[0] = 0ull;
    fcf->lb_key[1] = 0ull;
  }
}

// D1  thread per (cell, opponent): on-point test, gates, first/last blocked
//     height -> an interval slot
// D2  thread per (interval slot, edge): the edge bisection
// D3  thread per cell: sort + sweep (atan2), score_pass, score map store
// then the chunk's argmax per kick slot; the last chunk of a frame folds.
// Register caps (min resident CTAs per SM): the 128-thread batch shape at 6
// (80 registers: C5 value time 20.8 -> 13.8 ms per 16k frames against the
// uncapped 158-179), the 256-thread single-frame shape at 2 (128 registers;
// 3-4 only lengthen the D2 chains).  Measured with tools/variant_*.py.
#ifndef PP_VALUE_MINB
#define PP_VALUE_MINB 6
#endif
#ifndef PP_VALUE_MINB_WIDE
#define PP_VALUE_MINB_WIDE 2
#endif
template <bool kCells, int kThreads>
__global__ void __launch_bounds__(kThreads, kThreads == kValueThreadsWide ? PP_VALUE_MINB_WIDE
                                                                          : PP_VALUE_MINB)
    value_kernel(const FrameDev* __restrict__ frames, DevParams P, CellQueue q,
                 FrameCounters* __restrict__ fc, CellOut out, Partial* __restrict__ partials,
                 pp_dpps_summary* __restrict__ summaries, int chunks_per_frame,
                 int ctas_per_frame, const __grid_constant__ FrameDev fa) {
  __shared__ ValueSmem sm;
  __shared__ FoldSmem fs;
  const int f = blockIdx.x / ctas_per_frame;
  const int c0 = blockIdx.x % ctas_per_frame;
  // The frame (copied in before the scan started) and its view heights do
  // not depend on the scan.  Single-frame launches (the wide shape, at most
  // a wave of CTAs, one chunk per CTA) stage them while the scan's last CTAs
  // still run; batches (ctas_per_frame CTAs per frame, each taking chunks
  // c0, c0 + ctas_per_frame, ... of the frame's queue) only once a CTA has
  // work.
  constexpr bool kEarly = kThreads == kValueThreadsWide;
  if (kEarly) {
    load_frame(&sm.frame, P.frame_in_arg ? &fa : frames + f);
    __syncthreads();
    value_heights(sm, P);
  }
  const bool stream = kEarly && P.chunk_fill != nullptr;
  // Streaming: every value CTA of the frame counts itself out when it leaves;
  // the last one zeroes the streaming counters (see FrameCounters).
  auto leave = [&]() {
    if (stream && threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(&fc[f].value_out, 1u) == static_cast<unsigned>(ctas_per_frame - 1)) {
        fc[f].tiles_done = 0;
        fc[f].value_out = 0;
      }
    }
  };
  int n_q;
  unsigned long long lb_key0 = 0ull, lb_key1 = 0ull;  // batch pruning bounds
  if (stream) {
    // Scan -> value streaming (single frame): start as soon as this chunk's
    // entries are written, or once every tile is done (the last, partial
    // chunk, or a chunk that stays empty).
    if (threadIdx.x == 0) {
      volatile unsigned* fill = P.chunk_fill + c0;
      volatile unsigned* tiles = &fc[f].tiles_done;
      int nq = -1;
      for (unsigned spins = 0;; ++spins) {
        if (*fill == static_cast<unsigned>(kChunk)) break;
        if (*tiles == static_cast<unsigned>(P.n_tiles)) {
          __threadfence();
          nq = static_cast<int>(*reinterpret_cast<volatile unsigned*>(&fc[f].q_count));
          break;
        }
        if (spins > kSpinLimit) {
          nq = -2;  // stalled pipeline: leave without folding
          break;
        }
        __nanosleep(256);
      }
      __threadfence();
      sm.n_act = nq;  // -1: a full chunk, the final count not known yet
    }
    __syncthreads();
    if (sm.n_act == -2) return;
    n_q = sm.n_act < 0 ? (c0 + 1) * kChunk : sm.n_act;
  } else {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // scan grid done and visible
    n_q = static_cast<int>(fc[f].q_count);
    if (!kCells) {
      lb_key0 = fc[f].lb_key[0];
      lb_key1 = fc[f].lb_key[1];
    }
  }
  const int n_active_lb = n_q > 0 ? (n_q + kChunk - 1) / kChunk : 1;
  if (c0 >= n_active_lb) {
    leave();
    return;
  }
  if (!kEarly) {
    load_frame(&sm.frame, P.frame_in_arg ? &fa : frames + f);
    __syncthreads();
    value_heights(sm, P);
  }
  Partial* base = partials + static_cast<int64_t>(f) * chunks_per_frame;
  // (streaming CTAs take exactly one chunk: ctas_per_frame == chunks_per_frame)
  for (int ch = c0; ch < n_active_lb; ch += ctas_per_frame) {
    const int e0 = ch * kChunk;
    const int m = n_q - e0 < kChunk ? (n_q - e0 > 0 ? n_q - e0 : 0) : kChunk;
    PP_CHECK(ch < chunks_per_frame && e0 < q.cap + kChunk);
    value_chunk<kCells>(sm, P, q, out, f, e0, m, base + ch, lb_key0, lb_key1);
    if (threadIdx.x == 0) {
      int n_active = n_active_lb;
      bool stalled = false;
      if (stream) {
        P.chunk_fill[ch] = 0;  // consumed (self-cleaning for the next launch)
        // the fold needs the final chunk count: wait for the scan's last tile
        volatile unsigned* tiles = &fc[f].tiles_done;
        for (unsigned spins = 0; *tiles != static_cast<unsigned>(P.n_tiles); ++spins) {
          if (spins > kSpinLimit) {
            stalled = true;
            break;
          }
          __nanosleep(256);
        }
        __threadfence();
        const int nq = static_cast<int>(*reinterpret_cast<volatile unsigned*>(&fc[f].q_count));
        n_active = nq > 0 ? (nq + kChunk - 1) / kChunk : 1;
      }
      sm.last = 0;
      sm.n_act = -2;
      if (!stalled) {
        __threadfence();
        const unsigned prev = atomicAdd(&fc[f].chunks_done, 1u);
        sm.last = prev == static_cast<unsigned>(n_active - 1);
        sm.n_act = n_active;
      }
    }
    __syncthreads();
    if (sm.n_act == -2) return;  // stalled: no fold (the host reports it)
    if (sm.last) fold_frame(fs, base, sm.n_act, fc + f, P, summaries ? summaries + f : nullptr, f);
    __syncthreads();  // (sm reused by the next chunk)
  }
  leave();  // after the fold: the fold reads the frame's counters
}

}  // namespace pp
