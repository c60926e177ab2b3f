// pp_scan.cuh -- scan_kernel: the SBIP search per tile (dpps.cpp:106-215), its shared
// memory, leftover rounds, champions and the value queue; profiling hooks.
#pragma once

#include "pp_view.cuh"

namespace pp {

// ---------------------------------------------------------------------------
// The DPPS pipeline: scan_kernel (search, dpps.cpp:106-215) appends every
// feasible cell to a per-frame queue; value_kernel (score_pass + best_pass,
// pass_eval.cpp:148-187) drains the queue in chunks.  Splitting the two keeps
// every CTA's threads busy: a scan CTA is one tile with one warp per robot,
// a value CTA is a full chunk of goal views broken into independent items.

// Two scan CTA shapes (64 registers each): 16 warps x 2 CTAs/SM minimises a
// single frame's latency (one robot per warp); 4 warps x 8 CTAs/SM maximises
// throughput when there are many tiles (batches, 1 cm grids).
constexpr int kScanWarpsWide = 16, kScanCtasWide = 2;
#ifndef PP_SCAN_WARPS_NARROW
#define PP_SCAN_WARPS_NARROW 4
#endif
#ifndef PP_SCAN_CTAS_NARROW
#define PP_SCAN_CTAS_NARROW 8
#endif
constexpr int kScanWarpsNarrow = PP_SCAN_WARPS_NARROW, kScanCtasNarrow = PP_SCAN_CTAS_NARROW;
constexpr int kScanWarpsMid = 8, kScanCtasMid = 4;  // one wave of up to 4 x 148 tiles
#ifndef PP_TILE_PRUNE
#define PP_TILE_PRUNE 1
#endif
#ifndef PP_SCAN_WARP_W
#define PP_SCAN_WARP_W 4
#endif
#ifndef PP_SCAN_WARP_C
#define PP_SCAN_WARP_C 7
#endif
// scan_warp_kernel (batches): warps per CTA and CTAs per SM
constexpr int kScanWarpWarps = PP_SCAN_WARP_W, kScanWarpCtas = PP_SCAN_WARP_C;
constexpr bool kTilePrune = PP_TILE_PRUNE != 0;  // warp-tile scan: per-tile robot prune
#ifndef PP_REST_RANK
#define PP_REST_RANK 1  // warp-tile scan: rest rule in rank order (dev knob)
#endif
#ifndef PP_EARLY_CAP
#define PP_EARLY_CAP 1
#endif
#ifndef PP_REST_X
#define PP_REST_X 1
#endif
constexpr bool kRestX = PP_REST_X != 0;  // batches: our rest rules behind their champion too
#ifndef PP_REST_LB
#define PP_REST_LB 1
#endif
constexpr bool kRestLB = PP_REST_LB != 0;  // warp-tile scan: rest rule behind a lower bound
#ifndef PP_VALUE_CHUNK
#define PP_VALUE_CHUNK 32
#endif
#ifndef PP_VALUE_THREADS
#define PP_VALUE_THREADS 128
#endif
constexpr int kChunk = PP_VALUE_CHUNK;           // queued cells per value CTA
// A warp appends at most 32 queue entries, so they touch at most two chunks
// (tile_champions' chunk_fill split), and D3 runs one cell per lane of warp 0.
static_assert(kChunk == 32, "value chunks are one warp wide");
constexpr int kMaxWarps = 16;                    // largest CTA of any pipeline kernel
constexpr int kValueThreads = PP_VALUE_THREADS;  // threads per value CTA (pair/edge items) ...
constexpr int kValueThreadsWide = 256;           // ... and for launches of at most a wave
constexpr int kIvCap = 8 * kChunk;               // blocking-opponent intervals per chunk
constexpr int kMaxHeights = 129;                 // view heights cached in shared memory
constexpr int kMaxTeamIv = 16;                  // at most one interval per opponent

// Per-frame counters, self-cleaning: the frame fold (last active value CTA)
// zeroes q_count / n_feas / chunks_done / t0_inv; in streaming launches the
// last value CTA of the frame to LEAVE (idle chunks included) zeroes
// tiles_done / value_out, so no CTA still polling tiles_done can see it reset.
struct FrameCounters {
  unsigned q_count;     // feasible cells queued
  unsigned n_feas[2];   // per kick slot
  unsigned chunks_done;
  unsigned tiles_done;  // scan tiles whose queue entries are written (streaming value)
  unsigned value_out;   // streaming: value CTAs of the frame that have left
  unsigned long long t0_inv;  // ~(earliest scan CTA start, globaltimer ns); 0 = none
  // batches: per kick slot, the largest lower bound of a queued cell's score
  // (score_key; 0 = none) -- cells whose upper bound is below it cannot be
  // the slot's best_pass and skip the value function (value_chunk)
  unsigned long long lb_key[2];
};

// Streaming waits give up after this many polls (~4 s): the CTA leaves
// without folding, the host sees the fold missing, reports PP_INTERNAL and
// zeroes the counters (no __trap: the context stays usable).
constexpr unsigned kSpinLimit = 1u << 24;

__device__ __forceinline__ unsigned long long pp_now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Feasible cells awaiting score_pass; frame f owns entries [f*cap, f*cap+cap).
struct CellQueue {
  double* rx;
  double* ry;
  double* ot;
  double* pt;
  int32_t* cell;
  int8_t* slot;
  int64_t cap;
};

struct CellLane {
  Traj tr;
  double ux, uy;          // unit direction
  double s_lo, s_hi;      // ray distances of the window's first / last sample
  double rest_x, rest_y;  // rest point
  int kb, ke;             // window [kb, ke)
  bool valid, rif;        // power exists / ball rests in the field
};

struct __align__(16) RobotK {
  ReachBound rb;
  ArrivalLB lb;
  double vbound;   // max(|v|, vmax), intercept.cpp:97
  float bxf, byf;  // ball - robot in FP32 (sample offsets q = b + u s)
  float vbf;       // vbound in FP32
};

// A single frame as a kernel parameter: the world state and the scanned
// robots' filter constants (5.4 KB of the 32 KB parameter space).
struct __align__(16) FrameArg {
  FrameDev frame;
  RobotK rk[kMaxRobots];
};

// FP32 filter constants of scanned robot `ri` (once per tile, lane = robot).
PP_HD void robot_consts(const FrameDev& F, const DevParams& P, int ri,
                                             RobotK* out) {
  const int slot = F.scan_slot[ri];
  const bool theirs = slot >= kTheirs;
  const xd rvx = F.vx[slot], rvy = F.vy[slot];
  const xd a = theirs ? P.a_t : P.a_o;
  const xd b = theirs ? P.b_t : P.b_o;
  const xd vmax = theirs ? P.vmax_t : P.vmax_o;
  const xd speed_r = xsqrt(rvx * rvx + rvy * rvy);
  out->vbound = (speed_r > vmax ? speed_r : vmax).v;
  out->vbf = static_cast<float>(out->vbound);
  out->bxf = static_cast<float>((xd(F.ball_x) - xd(F.px[slot])).v);
  out->byf = static_cast<float>((xd(F.ball_y) - xd(F.py[slot])).v);
  out->rb = ReachBound(static_cast<float>(speed_r.v), static_cast<float>(a.v),
                       static_cast<float>(b.v), static_cast<float>(vmax.v));
  out->lb = ArrivalLB(static_cast<float>(rvx.v), static_cast<float>(rvy.v),
                      static_cast<float>(speed_r.v), static_cast<float>(a.v),
                      static_cast<float>(b.v), static_cast<float>(vmax.v));
}

struct ScanSmem {
  // A: per-cell window (lane = cell), raw storage (xd has a constructor)
  __align__(16) unsigned char cl_raw[32 * sizeof(CellLane)];
  int32_t ke[32];
  // earliest hit sample per team and cell (team cap); row 2: batches' cross
  // cap of our team (cross_cap of their earliest hit)
  int32_t cap[3][32];
  TrajF trf[32];  // FP32 trajectory per cell
  float2 win_s[32];  // FP32 ray distances of each cell's first / last window sample
  float2 tile_uf;  // FP32 unit direction of the tile
  // per scanned robot: FP32 filter constants and the FP64 speed bound
  RobotK rk[kMaxRobots];
  // B: per (robot, cell) results
  double res_t[kMaxRobots][32];
  int32_t res_k[kMaxRobots][32];
  // (robot, cell) pairs left for scan_leftovers
  uint16_t left[kMaxRobots * 32];  // ri << 5 | cell; the next sample waits in res_k
  unsigned n_left, next_pair;
  long long tph[4];  // profiling build: phase end clocks
  FrameDev frame;
};

__device__ __forceinline__ bool better(double s_new, int64_t c_new, double s_old, int64_t c_old) {
  // best_pass keeps the first strict max in cell order (pass_eval.cpp:178-185).
  if (c_old < 0) return c_new >= 0;
  if (c_new < 0) return false;
  return s_new > s_old || (s_new == s_old && c_new < c_old);
}

__device__ __forceinline__ void reset_partial(Partial& p) {
  for (int s = 0; s < 2; ++s) {
    p.score[s] = 0.0;
    p.cell[s] = -1;
    for (int q = 0; q < 5; ++q) p.feat[s][q] = 0.0;
    p.n_feasible[s] = 0;
  }
}

// Summary rows: 0 = all kick types, 1 = flat, 2 = chip (best_pass x3,
// passplan_main.cpp:102-104).
__device__ void write_summary(pp_dpps_summary* S, const Partial& B, const DevParams& P) {
  for (int k = 0; k < 3; ++k) {
    S->best_cell[k] = -1;
    S->best_score[k] = 0.0;
    S->n_feasible[k] = 0;
    S->best_features[k] = pp_pass_features{0, 0, 0, 0, 0};
  }
  for (int s = 0; s < P.n_kt; ++s) {
    const int row = (s == 0 ? P.kt_chip0 : P.kt_chip1) ? 2 : 1;
    S->n_feasible[row] = B.n_feasible[s];
    S->n_feasible[0] += B.n_feasible[s];
    if (B.cell[s] < 0) continue;
    S->best_cell[row] = B.cell[s];
    S->best_score[row] = B.score[s];
    S->best_features[row] = pp_pass_features{B.feat[s][0], B.feat[s][1], B.feat[s][2],
                                              B.feat[s][3], B.feat[s][4]};
    if (better(B.score[s], B.cell[s], S->best_score[0], S->best_cell[0])) {
      S->best_cell[0] = B.cell[s];
      S->best_score[0] = B.score[s];
      S->best_features[0] = S->best_features[row];
    }
  }
}

// The compact per-frame result of a batch (pp_frame_summary).
__device__ void write_compact(pp_frame_summary* C, const Partial& B, const DevParams& P) {
  pp_frame_summary o;
  for (int k = 0; k < 3; ++k) {
    o.best_cell[k] = -1;
    o.best_score[k] = 0.0;
    o.n_feasible[k] = 0;
  }
  int64_t c0 = -1;
  double s0 = 0.0;
  for (int s = 0; s < P.n_kt; ++s) {
    const int row = (s == 0 ? P.kt_chip0 : P.kt_chip1) ? 2 : 1;
    o.n_feasible[row] = static_cast<int32_t>(B.n_feasible[s]);
    o.n_feasible[0] += static_cast<int32_t>(B.n_feasible[s]);
    if (B.cell[s] < 0) continue;
    o.best_cell[row] = static_cast<int32_t>(B.cell[s]);
    o.best_score[row] = B.score[s];
    if (better(B.score[s], B.cell[s], s0, c0)) {
      c0 = B.cell[s];
      s0 = B.score[s];
    }
  }
  o.best_cell[0] = static_cast<int32_t>(c0);
  o.best_score[0] = s0;
  *C = o;
}

// Optional per-phase cycle accounting (build with -DPP_PHASE_CLOCKS).
#ifdef PP_PHASE_CLOCKS
__device__ unsigned long long g_phase_cycles[16];
constexpr int kRecCtas = 8192;
__device__ long long g_cta_rec[2][kRecCtas][8];   // [scan|value][cta]: t0, phases, smid, t1
__device__ long long g_robot_rec[kRecCtas][16];   // scan: cycles per robot-warp
__device__ __forceinline__ long long pp_gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PP_CLOCK_INIT() \
  long long ph_[8] = {0, 0, 0, 0, 0, 0, 0, 0}; \
  const long long gt0_ = pp_gtimer(); \
  long long ph_last_ = clock64()
#define PP_MARK(i)                              \
  if (threadIdx.x == 0) {                       \
    const long long now_ = clock64();           \
    ph_[i] += now_ - ph_last_;                  \
    ph_last_ = now_;                            \
  }
#define PP_FLUSH(slot0)                                                            \
  if (threadIdx.x == 0) {                                                          \
    for (int i_ = 0; i_ < 8; ++i_) atomicAdd(&g_phase_cycles[i_], (unsigned long long)ph_[i_]); \
    atomicAdd(&g_phase_cycles[slot0], 1ull);                                       \
    if (blockIdx.x < kRecCtas) {                                                   \
      long long* r_ = g_cta_rec[slot0 - 8][blockIdx.x];                            \
      unsigned smid_;                                                              \
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid_));                           \
      r_[0] = gt0_;                                                                \
      for (int i_ = 0; i_ < 5; ++i_) r_[1 + i_] = ph_[(slot0 == 8 ? 0 : 3) + i_];   \
      r_[6] = smid_;                                                               \
      r_[7] = pp_gtimer();                                                         \
    }                                                                              \
  }
__device__ long long g_d1_rec[512][256][2];
#define PP_D1_T0() const long long d1t0_ = clock64()
#define PP_D1_T1(pr, pi)                                                         \
  {                                                                              \
    long long d1t1_;                                                             \
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(d1t1_) : "r"(pi.status), "r"(pi.first) : "memory"); \
    if (blockIdx.x < 512 && pr < 256) {                                          \
      g_d1_rec[blockIdx.x][pr][0] = d1t1_ - d1t0_;                               \
      g_d1_rec[blockIdx.x][pr][1] = pi.status + 4 * pi.fast + 8 * (pi.first >= 0); \
    }                                                                            \
  }
// per value CTA and thread: D2 jobs, non-fast edges, band steps, exact
// rounds, setup + first band run cycles, exact-round cycles
__device__ long long g_d2_rec[512][256][6];
#define PP_D2_DECL() \
  long long d2st_[4] = {0, 0, 0, 0}; \
  int d2jobs_ = 0, d2nf_ = 0
#define PP_D2_ST d2st_
#define PP_D2_JOB(fast) (++d2jobs_, d2nf_ += !(fast))
#define PP_D2_FLUSH()                                                     \
  if (blockIdx.x < 512 && threadIdx.x < 256) {                            \
    long long* r_ = g_d2_rec[blockIdx.x][threadIdx.x];                    \
    r_[0] = d2jobs_; r_[1] = d2nf_; r_[2] = d2st_[1]; r_[3] = d2st_[2];   \
    r_[4] = d2st_[0]; r_[5] = d2st_[3];                                   \
  }
#define PP_TMARK(i) \
  if (threadIdx.x == 0) sm.tph[i] = clock64()
__device__ long long g_champ_rec[kRecCtas][4];
__device__ long long g_round_rec[kRecCtas][8][2];  // leftover rounds: open pairs, clock
__device__ long long g_win_rec[kRecCtas][4];  // window end, consts end, frame in, start
#define PP_CMARK_W(i) \
  if ((threadIdx.x & 31) == 0 && blockIdx.x < kRecCtas) g_win_rec[blockIdx.x][i] = clock64()
#define PP_CMARK(i) \
  if (threadIdx.x == 0 && blockIdx.x < kRecCtas) g_champ_rec[blockIdx.x][i] = clock64()
#define PP_ROBOT_START() const long long rb_clk_ = clock64()
#define PP_ROBOT_END(ri)                                                           \
  if ((threadIdx.x & 31) == 0 && blockIdx.x < kRecCtas && ri < 16)                 \
    g_robot_rec[blockIdx.x][ri] = clock64() - rb_clk_
// per-lane scan counters of the first kLaneRecCtas CTAs: steps, skips,
// lower-bound rejects, upper-bound accepts, exact tests, warp rounds
constexpr int kLaneRecCtas = 1024;
__device__ int g_lane_rec[kLaneRecCtas][16][32][6];
__device__ long long g_warp_rec[kLaneRecCtas][16][4];  // plain / coop steps, cycle of 1st coop
#define PP_CNT_DECL() \
  int c_it = 0, c_skip = 0, c_lbrej = 0, c_ub = 0, c_exact = 0, c_rounds = 0, c_plain = 0, \
      c_coop = 0;                                                                     \
  long long c_clk0 = clock64(), c_clk_coop = 0
#define PP_WCLK(i)
#define PP_CNT(v) (++(v))
#define PP_STEP_PLAIN() (++c_plain)
#define PP_STEP_COOP() \
  if (!c_coop++) c_clk_coop = clock64()
#define PP_CNT_FLUSH()                                                              \
  if (blockIdx.x < kLaneRecCtas && ri < 16) {                                      \
    int* l_ = g_lane_rec[blockIdx.x][ri][threadIdx.x & 31];                        \
    l_[0] = c_it; l_[1] = c_skip; l_[2] = c_lbrej; l_[3] = c_ub; l_[4] = c_exact;  \
    l_[5] = c_rounds;                                                              \
    if ((threadIdx.x & 31) == 0) {                                                 \
      long long* w_ = g_warp_rec[blockIdx.x][ri];                                  \
      w_[0] = c_plain; w_[1] = c_coop; w_[2] = c_clk_coop ? c_clk_coop - c_clk0 : -1; \
      w_[3] = clock64() - c_clk0;                                                  \
    }                                                                              \
  }
#else
#define PP_CLOCK_INIT()
#define PP_MARK(i)
#define PP_FLUSH(slot0)
#define PP_CNT_DECL()
#define PP_WCLK(i)
#define PP_TMARK(i)
#define PP_D1_T0()
#define PP_D1_T1(pr, pi)
#define PP_D2_DECL()
#define PP_D2_ST nullptr
#define PP_D2_JOB(fast)
#define PP_D2_FLUSH()
#define PP_CMARK(i)
#define PP_CMARK_W(i)
#define PP_ROBOT_START()
#define PP_ROBOT_END(ri)
#define PP_CNT(v)
#define PP_CNT_FLUSH()
#define PP_STEP_PLAIN()
#define PP_STEP_COOP()
#endif

__device__ __forceinline__ void load_frame(FrameDev* dst_, const FrameDev* src_) {
  const int n = sizeof(FrameDev) / 16;
  const int4* src = reinterpret_cast<const int4*>(src_);
  int4* dst = reinterpret_cast<int4*>(dst_);
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

// ---- scan: one tile (kick slot, direction, 32 powers) per CTA -------------
// The frame is in sm.frame.
// Per-lane (cell) scan window of one tile: A of the scan (ball_model.cpp:
// 12-43, intercept.cpp:12-25, 47-69; dpps.cpp:119-138).  Lane = power.


// ray_exit_distance / travel_time_to_distance (passplan/detail/pp_math.hpp) with xdiv.
__device__ __forceinline__ xd ray_exit_distance_d(xd L, xd W, xd ox, xd oy, xd ux, xd uy) {
  const xd hx = xd(0.5) * L;
  const xd hy = xd(0.5) * W;
  if (!(ox.v >= -hx.v && ox.v <= hx.v && oy.v >= -hy.v && oy.v <= hy.v)) return CUDART_NAN;
  xd s_exit = kInfD;
  if (ux.v != 0.0) {
    const xd c = xdiv((ux.v > 0.0 ? hx : -hx) - ox, ux);
    if (c < s_exit) s_exit = c;
  }
  if (uy.v != 0.0) {
    const xd c = xdiv((uy.v > 0.0 ? hy : -hy) - oy, uy);
    if (c < s_exit) s_exit = c;
  }
  return s_exit.v < 0.0 ? xd(0.0) : s_exit;
}

__device__ __forceinline__ xd travel_time_d(const Traj& tr, xd slide, xd roll, xd d) {
  if (d.v == 0.0) return 0.0;
  if (d > tr.d_stop) return CUDART_NAN;
  if (d <= tr.d_se) {
    const xd rad = tr.speed * tr.speed - xd(2.0) * slide * d;
    return xdiv(xd(2.0) * d, tr.speed + xsqrt(rad.v < 0.0 ? xd(0.0) : rad));
  }
  const xd rem = d - tr.d_se;
  const xd rad = tr.v1 * tr.v1 - xd(2.0) * roll * rem;
  return tr.t_se + xdiv(xd(2.0) * rem, tr.v1 + xsqrt(rad.v < 0.0 ? xd(0.0) : rad));
}

// dd / pr: the tile's direction row and this lane's power row, loaded by the
// caller ahead of the frame (they do not depend on it).
__device__ __forceinline__ CellLane cell_window(const FrameDev& F, const DevParams& P,
                                                const double4& dd, const PowRow& pr, bool valid) {
  const xd dt = P.dt, slide = P.slide, roll = P.roll;
  CellLane c;
  c.valid = valid;
  c.tr.speed = pr.speed;
  c.tr.v1 = pr.v1;
  c.tr.t_se = pr.t_se;
  c.tr.d_se = pr.d_se;
  c.tr.t_stop = pr.t_stop;
  c.tr.d_stop = pr.d_stop;
  const Traj& tr = c.tr;
  const xd ux = dd.z, uy = dd.w;
  const xd ox = F.ball_x, oy = F.ball_y;
  const xd d_exit = ray_exit_distance_d(F.L, F.W, ox, oy, dd.x, dd.y);
  int kb = 0, ke = 0;
  bool rif = false;
  if (!isnan(d_exit.v)) {
    ke = pr.count;
    kb = pr.kb;
    if (d_exit < tr.d_stop) {
      const xd t_exit = travel_time_d(tr, slide, roll, d_exit);
      const int k_last = !isnan(t_exit.v)
                             ? static_cast<int>(floor((xdiv(t_exit, dt) + xd(1e-9)).v))
                             : pr.count - 1;
      ke = ke < k_last + 1 ? ke : k_last + 1;
    } else {
      rif = true;
    }
  }
  c.ux = ux.v;
  c.uy = uy.v;
  c.kb = kb;
  c.ke = ke;
  c.rif = rif;
  c.rest_x = (ox + ux * tr.d_stop).v;
  c.rest_y = (oy + uy * tr.d_stop).v;
  c.s_lo = c.s_hi = 0.0;
  if (kb < ke) {
    const xd s_lo = distance_at(tr, slide, roll, xd(double(kb)) * dt);
    const xd s_hi = distance_at(tr, slide, roll, xd(double(ke - 1)) * dt);
    c.s_lo = s_lo.v;
    c.s_hi = s_hi.v;
  }
  return c;
}

// Dev statistics of the filters (variant build -DPP_SCAN_STATS only; read
// with pp_debug_scan_stats): sample outcomes, skipped samples, warp steps.
#ifdef PP_SCAN_STATS
// [24..39]: pairs by tests (bucket min(tests, 15) ... ), [40..55]: their tests;
// [56]: lower-bound rejects in a run of >= 4 consecutive ones
__device__ unsigned long long g_scan_stats[64];
__device__ unsigned long long g_act_hist[33];  // warp steps by active lanes
#define PP_STAT(i) atomicAdd(&g_scan_stats[i], 1ull)
#define PP_STATN(i, n) atomicAdd(&g_scan_stats[i], static_cast<unsigned long long>(n))
#else
#define PP_STAT(i)
#define PP_STATN(i, n)
#endif

// FP32 sample filter outcome (scan_robot / scan_leftovers).
enum SampleCode { kNone = 0, kRej = 1, kEnd = 2, kCap = 3, kHit = 4, kCand = 5 };

// Per (robot, tile) FP32 filter constants: the robot's offset from the ball,
// speed bound and the tile's direction; rb / lb stay in shared memory (rk).
struct SampleF {
  float bxf, byf, vbf;  // ball - robot, vbound
  float uxf, uyf;       // the tile's direction
  float dtf, radf;
  float s0;             // ray coordinate of the robot's closest approach
  bool exact;           // DevParams::exact_only: no filtering at all
};

__device__ __forceinline__ SampleF sample_f(const RobotK& rk, float2 uf, const DevParams& P) {
  SampleF S;
  S.bxf = rk.bxf;
  S.byf = rk.byf;
  S.vbf = rk.vbf;
  S.uxf = uf.x;
  S.uyf = uf.y;
  S.dtf = P.dtf;
  S.radf = P.radf;
  S.s0 = -(S.bxf * S.uxf + S.byf * S.uyf);
  S.exact = P.exact_only != 0;
  return S;
}

// One sample kk of a (robot, cell): kRej with the next sample worth looking
// at in *next (every sample in [kk, *next) certainly infeasible), else the
// first non-rejected outcome: kEnd (window over), kCap (past the team cap),
// kHit (certainly feasible), kCand (needs the exact test).
__device__ __forceinline__ int test_sample(const RobotK& rk, const SampleF& S, int kk,
                                           const TrajF& tf_, int ke_s, int cap_c, int* next) {
  PP_STAT(0);
  // one compare against min(window end, cap + 1) (loop-invariant in a robot's
  // scan), then which of the two it was
  const int lim = cap_c < ke_s ? cap_c + 1 : ke_s;
  if (kk >= lim) {
    if (kk >= ke_s) {
      PP_STAT(1);
      return kEnd;
    }
    PP_STAT(2);
    return kCap;
  }
  if (S.exact) return kCand;
  const float tf = static_cast<float>(kk) * S.dtf;
  const float sf = tf_.distance_at(tf);
  const float qxf = fmaf(S.uxf, sf, S.bxf);
  const float qyf = fmaf(S.uyf, sf, S.byf);
  const float d2f = fmaf(qxf, qxf, qyf * qyf);
  const float thr = S.radf + fmaf(rk.rb.reach(tf), 1.0001f, 1e-4f);
  const float inv_d = rsqrt_ftz(fmaxf(d2f, 1e-30f));
  const float df = d2f * inv_d;
  if (d2f > thr * thr) {
    // Cannot get there.  Skip ahead: the gap d - thr shrinks by at most
    // (ball approach speed + vbound) * dt per sample; past the closest
    // approach (s >= s0) the distance cannot shrink.
    const float gap = df - thr;
    const float approach = sf < S.s0 + 1e-3f ? tf_.speed_at(tf) : 0.f;
    const float rate = (approach + S.vbf) * S.dtf * 1.0001f;
    const float j = floorf(gap * rcp_ftz(rate) * 0.9999f);
    // skip j - 1 samples, clamped to [0, 4095] (NaN: 0)
    *next = kk + 1 + static_cast<int>(fminf(fmaxf(j - 1.f, 0.f), 4095.f));
    PP_STAT(3);
    PP_STATN(4, *next - kk - 1);
    return kRej;
  }
  if (rk.lb.lower_bound(qxf, qyf, df, inv_d, S.radf) > fmaf(tf, 1.000001f, 1e-6f)) {
    *next = kk + 1;
    PP_STAT(5);
    return kRej;
  }
  // certainly feasible: arrival <= t with margin (and then the reference's
  // quick reject cannot fire: reach - deff >= vbound t / 2)
  if (rk.lb.upper_bound(qxf, qyf, df, inv_d, S.radf) < fmaf(tf, 0.999999f, -1e-6f)) {
    PP_STAT(6);
    return kHit;
  }
  PP_STAT(7);
  return kCand;
}

// FP64 state of scanned robot ri for the exact test and the rest rule.
struct RobotX {
  xd px, py, vx, vy, a, b, vmax, vbound;
  int team;
};

__device__ __forceinline__ RobotX robot_x(const FrameDev& F, const DevParams& P, const RobotK& rk,
                                          int ri) {
  RobotX X;
  const int slot = F.scan_slot[ri];
  const bool theirs = slot >= kTheirs;
  X.team = theirs ? 1 : 0;
  X.px = F.px[slot];
  X.py = F.py[slot];
  X.vx = F.vx[slot];
  X.vy = F.vy[slot];
  X.a = theirs ? P.a_t : P.a_o;
  X.b = theirs ? P.b_t : P.b_o;
  X.vmax = theirs ? P.vmax_t : P.vmax_o;
  X.vbound = rk.vbound;
  return X;
}

// The reference's test of sample k (kernel.hpp:33-44, intercept.cpp:96-113).
__device__ __forceinline__ bool exact_hit(const CellLane& c, const FrameDev& F, const DevParams& P,
                                          const RobotX& X, int k) {
  const xd dt = P.dt, radius = P.radius;
  const xd t = xd(double(k)) * dt;
  const xd sx = distance_at(c.tr, P.slide, P.roll, t);
  const xd qx = (xd(F.ball_x) + xd(c.ux) * sx) - X.px;
  const xd qy = (xd(F.ball_y) + xd(c.uy) * sx) - X.py;
  const xd d2 = qx * qx + qy * qy;
  const xd reach = radius + X.vbound * t;
  return !(d2 > reach * reach) &&
         arrival_given(qx, qy, d2, X.vx, X.vy, X.a, X.b, X.vmax, radius) <= t;
}

// Result of a finished (robot, cell) scan: hit sample, team-capped, else the
// rest rule (dpps.cpp:177-190).  time +inf = never; code -2 never, -1 rest,
// -3 capped out, >= 0 hit sample.
__device__ __forceinline__ void pair_result(const CellLane& c, const DevParams& P, const RobotX& X,
                                            int hit, bool capped, double* t_out, int* code_out) {
  double time = CUDART_INF;
  int code = -2;
  if (c.valid) {
    if (hit >= 0) {
      time = (xd(double(hit)) * xd(P.dt)).v;
      code = hit;
    } else if (capped) {
      code = -3;  // another robot of the team hit strictly earlier
    } else if (c.rif) {
      const xd arr = arrival_to_point(c.rest_x, c.rest_y, X.px, X.py, X.vx, X.vy, X.a, X.b,
                                      X.vmax, P.radius);
      const xd ts = c.tr.t_stop;
#ifdef PP_SCAN_STATS
      PP_STAT(57);
      if (arr <= ts) PP_STAT(58);
      if (X.team == 0) PP_STAT(59);
#endif
      time = (arr > ts ? arr : ts).v;
      code = -1;
    }
  }
  *t_out = time;
  *code_out = code;
}

// Result of a finished (robot, cell) scan (dpps.cpp:177-190): a hit, capped
// out, else the rest rule -- skipped, as (+inf, never), where a robot of the
// same team has already hit strictly before the ball comes to rest: the
// rest-rule time max(arrival, t_stop) >= t_stop is then later than that
// hit, so it can neither win nor tie the team's champion (the only robot
// whose time and id reach the outputs, dpps.cpp:192-213).  The team cap only
// decreases, so reading it early is conservative.  cap_lane points at this
// cell's entry of the team-cap table (cap_lane[team * 32]).
template <bool kX = false>
__device__ __forceinline__ void pair_finish(const CellLane& c, const FrameDev& F,
                                            const DevParams& P, const RobotK& rk, int ri,
                                            int hit, bool capped, const int* cap_lane,
                                            double* t_out, int* code_out) {
  if (hit < 0 && !capped && c.valid && c.rif) {
    const int team = F.scan_slot[ri] >= kTheirs ? 1 : 0;
    const int k_team = *reinterpret_cast<const volatile int*>(cap_lane + team * 32);
    if (k_team != 0x7fffffff && xd(double(k_team)) * xd(P.dt) < c.tr.t_stop) {
      *t_out = CUDART_INF;
      *code_out = -2;
      return;
    }
    if (kX && team == 0) {
      // batches (see cross_cap): their hit at sample k_t leaves our rest-rule
      // time t >= t_stop useless once fl(t_stop + safety) > k_t * dt
      const int k_t = *reinterpret_cast<const volatile int*>(cap_lane + 32);
      if (k_t != 0x7fffffff &&
          c.tr.t_stop + xd(P.safety) > xd(double(k_t)) * xd(P.dt)) {
        *t_out = CUDART_INF;
        *code_out = -2;
        return;
      }
    }
  }
  pair_result(c, P, robot_x(F, P, rk, ri), hit, capped, t_out, code_out);
}

// The scan's own outcome of a finished pair: a hit, capped out, or kNoHit --
// no sample hit, the rest rule decides (resolved by rest_rule_pass once every
// robot of the tile is done).
constexpr int kNoHit = -4;
__device__ __forceinline__ void pair_outcome(int hit, bool capped, const DevParams& P,
                                             double* t_out, int* code_out) {
  *t_out = hit >= 0 ? (xd(double(hit)) * xd(P.dt)).v : CUDART_INF;
  *code_out = hit >= 0 ? hit : (capped ? -3 : kNoHit);
}

// The rest rule (dpps.cpp:177-190) for every kNoHit pair of the tile, all
// threads, after the scan phase.  Skipped -- (+inf, never) -- where a robot
// of the same team hit strictly before the ball comes to rest: the rest-rule
// time max(arrival, t_stop) >= t_stop is then later than that hit, so it can
// neither win nor tie the team's champion (the only robot whose time and id
// reach the outputs, dpps.cpp:192-213).
template <class ResT, class ResK>
__device__ __forceinline__ void rest_rule_pass(const CellLane* cl, const FrameDev& F,
                                               const DevParams& P, const RobotK* rk_s,
                                               const int (*cap)[32], ResT res_t, ResK res_k) {
  for (int e = threadIdx.x; e < F.n_scan * 32; e += blockDim.x) {
    const int ri = e >> 5, cell = e & 31;
    if (res_k[ri][cell] != kNoHit) continue;
    const CellLane& c = cl[cell];
    const int team = F.scan_slot[ri] >= kTheirs ? 1 : 0;
    const int k_team = cap[team][cell];
    double t;
    int cd;
    if (k_team != 0x7fffffff && xd(double(k_team)) * xd(P.dt) < c.tr.t_stop) {
      t = CUDART_INF;
      cd = -2;
    } else {
      pair_result(c, P, robot_x(F, P, rk_s[ri], ri), -1, false, &t, &cd);
    }
    res_t[ri][cell] = t;
    res_k[ri][cell] = cd;
  }
}

// First sample worth testing for robot ri on cell c (ke when none):
// scan_robot's prunes (intercept.cpp:89-113) in FP32 with 1e-3 m of slack --
// the window is skipped, or the scan starts late, only where every sample
// certainly fails the quick reject.  Exact-only mode: the window start.
__device__ __forceinline__ int scan_start(const CellLane& c, const SampleF& S, float2 win_s) {
  const int kb = c.kb;
  const int ke = c.valid ? c.ke : 0;
  if (!(c.valid && kb < ke)) return ke;
  if (S.exact) return kb;
  // segment_distance(robot, a, b) for a, b on the ray (a = ball + u s_lo,
  // b = ball + u s_hi): the distance to the ray point at the robot's own ray
  // coordinate s0 clamped to [s_lo, s_hi]
  const float sc = fminf(fmaxf(S.s0, win_s.x), win_s.y);
  const float ex = fmaf(S.uxf, sc, S.bxf), ey = fmaf(S.uyf, sc, S.byf);
  const float gap = sqrt_a(ex * ex + ey * ey) - 1e-3f - S.radf;
  if (gap > S.vbf * static_cast<float>(ke - 1) * S.dtf * 1.0001f) return ke;
  int k = kb;
  if (S.vbf > 0.f && gap > 0.f) {
    // (approximate reciprocal, ~2 ulp; the 1e-6 shrink keeps the quotient
    // at or below the exact one, so the start is never later)
    const int kk =
        static_cast<int>(floorf(gap * rcp_ftz(S.vbf * S.dtf * 1.0001f) * (1.f - 1e-6f))) - 1;
    k = kk > kb ? (kk < ke ? kk : ke) : kb;
  }
  return k;
}

// Batches only (the outputs are the per-frame summary: feasible cells and the
// best of them): once their team hits a cell at sample k (time tau =
// k * dt), our robots need no sample j with fl(fl(j * dt) + safety) > tau --
// a hit there, or the rest rule after it (time >= t_stop >= t_j), leaves
// our time t with fl(t + safety) > tau >= their final time, an infeasible
// cell (dpps.cpp:207-212) whatever our champion is; and where the cell is
// feasible its champion hits at a sample j with fl(t_j + safety) <= their
// final time <= tau, never cut.  Returns that largest useful j (-1: none;
// every j when the safety margin allows all), rounding-exact: the estimate
// is corrected with the reference's own FP64 comparison.
__device__ __forceinline__ int cross_cap(int k, const DevParams& P) {
  const xd dt = P.dt, sm = P.safety;
  const xd tau = xd(double(k)) * dt;
  auto ok = [&](int j) { return j < 0 || xd(double(j)) * dt + sm <= tau; };
  const double est = floor((tau.v - sm.v) / dt.v);
  if (!(est < 1e8)) return 0x7fffffff;  // (huge or NaN: no cut)
  int j = est < -1.0 ? -1 : static_cast<int>(est);
  for (int it = 0; it < 8; ++it) {
    if (!ok(j)) {
      --j;
    } else if (ok(j + 1)) {
      ++j;
    } else {
      return j;
    }
  }
  return 0x7fffffff;  // (not settled: no cut)
}

// cross_cap from the launch's table (DevParams::xcap, built by
// xcap_table_kernel with cross_cap itself) where it covers k.
__device__ __forceinline__ int cross_cap_t(int k, const DevParams& P) {
  return k < P.n_xcap ? __ldg(P.xcap + k) : cross_cap(k, P);
}

__global__ void xcap_table_kernel(DevParams P, int32_t* __restrict__ tab, int n) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) tab[k] = cross_cap(k, P);
}

// B of the scan for robot `ri` (one warp, lane = cell): scan_robot
// (intercept.cpp:87-115) + first feasible sample (kernel.hpp:33-44) + rest
// rule (dpps.cpp:177-190).  Two exact-safe accelerations, neither of which
// can change a result:
//  * team cap (dpps.cpp:142-153): robots of a team share the earliest hit
//    index per cell (cap[team * 32 + cell], shared memory); a robot stops
//    once its next sample is past it (it can no longer win or tie).
//  * FP32 filters: a sample is tested exactly only if the robot could
//    possibly get there (ReachBound, ArrivalLB); runs of samples are skipped
//    only when certified infeasible.
// Lane-per-cell steps, at most max_steps of them: a lane still searching
// after that returns its next sample in *left_k (the CTA finishes it in
// scan_leftovers with many lanes per cell); otherwise *left_k = -1 and the
// result is in *t_out / *code_out.
// kEager: resolve the rest rule here (throughput shape, no extra pass);
// else leave kNoHit for rest_rule_pass (latency shapes, final team caps).
// kSolo (scan_warp_kernel): the warp is the cell's only scanner, so the
// caps cannot move during this robot's scan except by its own hit (which
// ends it): they are read once, and updated without atomics.
template <bool kEager, bool kX = false, bool kSolo = false>
__device__ __forceinline__ void scan_robot(const CellLane& c, const TrajF& trf_in, float2 win_s,
                                           const SampleF& S, const FrameDev& F, const DevParams& P,
                                           const RobotK& rk, int* cap,
                                           int ri, int max_steps, double* t_out,
                                           int* code_out, int* left_k) {
  const int lane = threadIdx.x & 31;
  const int ke = c.valid ? c.ke : 0;
  int k = scan_start(c, S, win_s);
  PP_STAT(10);
  if (k >= ke) PP_STAT(11);
#ifdef PP_SCAN_STATS
  if (F.scan_slot[ri] >= kTheirs) PP_STAT(22);  // their pairs
#endif
  const TrajF trf = trf_in;
  int hit = -1;
  bool capped = false;
  int state = k >= ke ? 2 : 0;  // 0 scanning, 1 candidate pending, 2 finished
#ifdef PP_SCAN_STATS
  int n_tests = 0, lb_run = 0;
#endif
  PP_CNT_DECL();
  // Warp-synchronous: each step every scanning lane examines one sample (or
  // certifies a run of them infeasible); lanes the FP32 bounds cannot decide
  // wait as candidates and get the exact FP64 test together when no lane is
  // scanning.  Team caps are re-read from shared memory every step.
  const int team = F.scan_slot[ri] >= kTheirs ? 1 : 0;
  volatile int* vcap = cap + team * 32 + lane;
  // kX (batches): our robots also stop past the cross cap (cap row 2)
  volatile int* vxcap = cap + (kX && team == 0 ? 2 : team) * 32 + lane;
  auto hit_at = [&](int kh) {
    if (kSolo) {
      int* ct = &cap[team * 32 + lane];
      *ct = min(*ct, kh);
      if (kX && team == 1) {
        int* cx = &cap[2 * 32 + lane];
        *cx = min(*cx, cross_cap_t(kh, P));
      }
    } else {
      atomicMin(&cap[team * 32 + lane], kh);
      if (kX && team == 1) atomicMin(&cap[2 * 32 + lane], cross_cap_t(kh, P));
    }
  };
  const int cap_solo = kSolo ? (kX ? min(*vcap, *vxcap) : *vcap) : 0;
#if PP_EARLY_CAP
  // solo scans: a start already past the (fixed) cap ends as the first
  // test would (kCap), before the loop
  if (kSolo && state == 0 && k > cap_solo) {
    capped = true;
    state = 2;
  }
#endif
  for (int n_step = 0; n_step < max_steps; ++n_step) {
    const unsigned act = __ballot_sync(0xffffffffu, state == 0);
#ifdef PP_SCAN_STATS
    if (lane == 0) {
      PP_STAT(12);
      PP_STATN(13, __popc(act));
      atomicAdd(&g_act_hist[__popc(act)], 1ull);
      if (team) PP_STAT(23);  // their warp steps
    }
#endif
    if (act == 0u) {
      const bool pend = state == 1;
      if (!__any_sync(0xffffffffu, pend)) break;
      PP_CNT(c_rounds);
      if (pend) {
        PP_CNT(c_exact);
        PP_STAT(8);
        if (exact_hit(c, F, P, robot_x(F, P, rk, ri), k)) {
          PP_STAT(9);
          hit = k;
          hit_at(k);
          state = 2;
        } else {
          ++k;
          state = 0;
        }
      }
      continue;
    }
    PP_STEP_PLAIN();
    if (state == 0) {
      PP_CNT(c_it);
#ifdef PP_SCAN_STATS
      ++n_tests;
      if (team) PP_STAT(15);  // their tests
#endif
      int next = k;
      const int cap_c = kSolo ? cap_solo : (kX ? min(*vcap, *vxcap) : *vcap);
      const int code = test_sample(rk, S, k, trf, ke, cap_c, &next);
      switch (code) {
        case kRej:
          PP_CNT(c_skip);
#ifdef PP_SCAN_STATS
          if (next == k + 1) {
            if (++lb_run >= 4) PP_STAT(56);
          } else {
            lb_run = 0;
          }
#endif
          k = next;
          break;
        case kEnd: state = 2; break;
        case kCap: capped = true; state = 2; break;
        case kHit:
          PP_CNT(c_ub);
          hit = k;
          hit_at(k);
          state = 2;
          break;
        default: state = 1; break;  // kCand
      }
    }
  }
  PP_CNT_FLUSH();
#ifdef PP_SCAN_STATS
  if (state == 2) {
    const int b = n_tests < 4 ? n_tests : (n_tests < 8 ? 4 + (n_tests - 4) / 2
                                                       : (n_tests < 16 ? 6 + (n_tests - 8) / 4
                                                                       : (n_tests < 64 ? 8 + (n_tests - 16) / 16
                                                                                       : (n_tests < 256 ? 11 + (n_tests - 64) / 64 : 15))));
    PP_STAT(24 + b);
    PP_STATN(40 + b, n_tests);
  }
  // tests by outcome: 16/17 hit (count, tests), 18/19 capped, 20/21 window end
  {
    const int o = hit >= 0 ? 16 : (capped ? 18 : 20);
    if (state == 2 && k < ke + 1 && n_tests > 0) {
      PP_STAT(o);
      PP_STATN(o + 1, n_tests);
    }
  }
#endif
  if (state != 2) {
    PP_STAT(14);
    *left_k = k;
    return;
  }
  *left_k = -1;
  if (kEager) {
    pair_finish<kX>(c, F, P, rk, ri, hit, capped, cap + lane, t_out, code_out);
  } else {
    pair_outcome(hit, capped, P, t_out, code_out);
  }
}

// Scan pairs left over by scan_robot: left[] holds ri << 5 | cell and
// res_k[ri][cell] the pair's next sample.
// Each pair gets a group of g lanes (a power of two, 4..32) testing g
// consecutive samples per step: the first non-rejected one decides (exact
// test for a candidate), else the pair advances past every sample the group
// certified infeasible.  Groups take pairs from the shared list dynamically.
// All warps of the CTA take part; results go to res_t / res_k.
__device__ __forceinline__ void scan_leftovers(const CellLane* cl, const TrajF* trf_s,
                                               const int* ke_s, float2 uf, const FrameDev& F,
                                               const DevParams& P, const RobotK* rk_s, int* cap,
                                               const uint16_t* left, int n_left,
                                               unsigned* next_pair, double (*res_t)[32],
                                               int32_t (*res_k)[32], int max_steps) {
  const int lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  int g = 32;
  while (g > 4 && n_left * g > nwarps * 32) g >>= 1;
  const int gbase = lane & ~(g - 1);
  const int o = lane - gbase;
  const unsigned gmask = g == 32 ? 0xffffffffu : ((1u << g) - 1u) << gbase;
  int pi = -1;      // pair of this group (-1 none / finished the list)
  int ri = 0, cell = 0, k = 0;
  int hit = -1, ns = 0;
  bool capped = false;
  // every lane calls take(); groups with need == false keep their pair
  auto take = [&](bool need) {
    unsigned nx = 0;
    if (need && o == 0) nx = atomicAdd(next_pair, 1u);
    nx = __shfl_sync(0xffffffffu, nx, gbase);
    if (need) {
      pi = nx < static_cast<unsigned>(n_left) ? static_cast<int>(nx) : -1;
      if (pi >= 0) {
        const unsigned w = left[pi];
        PP_CHECK(pi < n_left);
        ri = static_cast<int>(w >> 5);
        cell = static_cast<int>(w & 31u);
        k = res_k[ri][cell];
        hit = -1;
        ns = 0;
        capped = false;
      }
    }
  };
  take(true);
  while (__any_sync(0xffffffffu, pi >= 0)) {
    int code = kNone, nxt = 0;
    const RobotK& rk = rk_s[ri];
    const int team = F.scan_slot[ri] >= kTheirs ? 1 : 0;
    if (pi >= 0) {
      const SampleF S = sample_f(rk, uf, P);
      const int cap_c = *(volatile int*)(cap + team * 32 + cell);
      code = test_sample(rk, S, k + o, trf_s[cell], ke_s[cell], cap_c, &nxt);
    }
    const unsigned nonrej = __ballot_sync(0xffffffffu, code > kRej) & gmask;
    int reach = code == kRej ? nxt : 0;
    for (int s = 1; s < g; s <<= 1) reach = max(reach, __shfl_xor_sync(0xffffffffu, reach, s));
    bool done = false;
    if (pi >= 0) {
      if (nonrej) {
        const int f = __ffs(nonrej) - 1 - gbase;
        const int gcode = __shfl_sync(gmask, code, gbase + f);
        const int kk = k + f;
        if (gcode == kEnd) {
          done = true;
        } else if (gcode == kCap) {
          capped = true;
          done = true;
        } else if (gcode == kHit) {
          hit = kk;
          done = true;
        } else {  // kCand: the exact test (same arguments in every lane of the group)
          const RobotX X = robot_x(F, P, rk, ri);
          if (exact_hit(cl[cell], F, P, X, kk)) {
            hit = kk;
            done = true;
          } else {
            k = kk + 1;
          }
        }
      } else {
        k = max(k + g, reach);
      }
    }
    if (done) {
      if (o == 0) {
        if (hit >= 0) atomicMin(&cap[team * 32 + cell], hit);
        double t;
        int cd;
        pair_outcome(hit, capped, P, &t, &cd);
        res_t[ri][cell] = t;
        res_k[ri][cell] = cd;
      }
    }
    // a pair still open after max_steps goes back to the list (next round,
    // with more lanes per pair once fewer pairs remain)
    bool release = done;
    if (pi >= 0 && !done && ++ns >= max_steps) {
      if (o == 0) res_k[ri][cell] = k;
      release = true;
    }
    if (__any_sync(0xffffffffu, release)) take(release);
  }
}

template <bool kCells>
__device__ __forceinline__ void tile_publish(const CellLane& c, const FrameDev& F,
                                             const DevParams& P, unsigned long long bt_o_bits,
                                             int bk_o, int bs_o, unsigned long long bt_t_bits,
                                             int bs_t, const CellOut& out, const CellQueue& q,
                                             FrameCounters* __restrict__ fc, int f, int kt,
                                             int64_t cell);

// C of the scan (dpps.cpp:140-213), one warp, lane = cell: our and their
// champion (strict (time, id) lexicographic argmin seeded with (kNever, -1),
// so visiting order does not matter), receive point, feasibility; cell
// outputs, and feasible cells appended to the frame's value queue.
// res_t(ri) / res_k(ri): this lane's time and code for scanned robot ri.
template <bool kCells, class ResT, class ResK>
__device__ __forceinline__ void tile_champions(const CellLane& c, const FrameDev& F,
                                               const DevParams& P, ResT res_t, ResK res_k,
                                               const CellOut& out, const CellQueue& q,
                                               FrameCounters* __restrict__ fc, int f, int kt,
                                               int64_t cell0) {
      // Times are >= 0 or +inf (never NaN, never -0), so their bit patterns
      // order like the values: the (time, id) argmin runs on integers.
      const int n_ours_scan = F.n_ours - 1;  // kicker excluded
      unsigned long long bt_o_bits = 0x7ff0000000000000ull;  // +inf
      int bid_o = -1, bri_o = -1, bs_o = -1;
      for (int s = 0; s < F.n_ours; ++s) {
        if (s == F.kicker_slot) continue;
        const int ri = s - (s > F.kicker_slot ? 1 : 0);
        const unsigned long long tb = __double_as_longlong(res_t(ri));
        const int id = F.id[s];
        if (tb < bt_o_bits || (tb == bt_o_bits && id < bid_o)) {
          bt_o_bits = tb;
          bid_o = id;
          bri_o = ri;
          bs_o = s;
        }
      }
      unsigned long long bt_t_bits = 0x7ff0000000000000ull;
      int bid_t = -1, bs_t = -1;
      for (int s = 0; s < F.n_theirs; ++s) {
        const int ri = n_ours_scan + s;
        const unsigned long long tb = __double_as_longlong(res_t(ri));
        const int id = F.id[kTheirs + s];
        if (tb < bt_t_bits || (tb == bt_t_bits && id < bid_t)) {
          bt_t_bits = tb;
          bid_t = id;
          bs_t = s;
        }
      }
      PP_CMARK(1);
      tile_publish<kCells>(c, F, P, bt_o_bits, bri_o >= 0 ? res_k(bri_o) : -2, bs_o, bt_t_bits,
                           bs_t, out, q, fc, f, kt, cell0 + (threadIdx.x & 31));
}

// The end of C for one lane (cell): from its champions -- our (time bits,
// hit code, slot) and theirs (time bits, index among theirs) -- the receive
// point and feasibility (dpps.cpp:192-213), the append of a feasible cell to
// the frame's value queue, and the cell outputs.
template <bool kCells>
__device__ __forceinline__ void tile_publish(const CellLane& c, const FrameDev& F,
                                             const DevParams& P, unsigned long long bt_o_bits,
                                             int bk_o, int bs_o, unsigned long long bt_t_bits,
                                             int bs_t, const CellOut& out, const CellQueue& q,
                                             FrameCounters* __restrict__ fc, int f, int kt,
                                             int64_t cell) {
      const int lane = threadIdx.x & 31;
      const xd dt = P.dt, slide = P.slide, roll = P.roll;
      const xd bt_o = __longlong_as_double(static_cast<long long>(bt_o_bits));
      const xd bt_t = __longlong_as_double(static_cast<long long>(bt_t_bits));
      xd rx = 0.0, ry = 0.0;
      bool feas = false;
      if (bt_o.v < CUDART_INF) {
        if (bk_o >= 0) {
          const xd s = distance_at(c.tr, slide, roll, xd(double(bk_o)) * dt);
          rx = xd(F.ball_x) + xd(c.ux) * s;
          ry = xd(F.ball_y) + xd(c.uy) * s;
        } else {
          rx = c.rest_x;
          ry = c.rest_y;
        }
        feas = isinf(bt_t.v) || (bt_o + xd(P.safety) <= bt_t);
      }
      feas = feas && c.valid;
      PP_CMARK(2);
      const unsigned fm = __ballot_sync(0xffffffffu, feas);
      unsigned base = 0;
      if (lane == 0 && fm) {
        base = atomicAdd(&fc[f].q_count, static_cast<unsigned>(__popc(fm)));
        atomicAdd(&fc[f].n_feas[kt], static_cast<unsigned>(__popc(fm)));
      }
      base = __shfl_sync(0xffffffffu, base, 0);
      const unsigned n_new = static_cast<unsigned>(__popc(fm));
      const unsigned rank = __popc(fm & ((1u << lane) - 1u));
      // (base + rank < cap always: a frame queues at most its cells; the
      // guard keeps dirty counters from writing past the frame's region)
      PP_CHECK(!feas || base + rank < static_cast<unsigned>(q.cap));
      if (feas && base + rank < static_cast<unsigned>(q.cap)) {
        const int64_t pos = static_cast<int64_t>(f) * q.cap + base + rank;
        q.rx[pos] = rx.v;
        q.ry[pos] = ry.v;
        q.ot[pos] = bt_o.v;
        q.pt[pos] = bt_t.v;
        q.cell[pos] = static_cast<int32_t>(cell);
        q.slot[pos] = static_cast<int8_t>(kt);
      }
      if (P.chunk_fill) {
        // publish: entries first (every lane's, ordered by the warp barrier
        // and lane 0's fence), then the chunks' fill counts, then the tile
        __syncwarp();
        if (lane == 0) {
          __threadfence();
          if (n_new) {
            const unsigned c0 = base / kChunk, c1 = (base + n_new - 1) / kChunk;
            const unsigned in0 = min(n_new, (c0 + 1) * kChunk - base);
            PP_CHECK(c1 * kChunk < static_cast<unsigned>(q.cap) + kChunk);
            atomicAdd(&P.chunk_fill[c0], in0);
            if (c1 != c0) atomicAdd(&P.chunk_fill[c1], n_new - in0);
          }
          __threadfence();
          atomicAdd(&fc[f].tiles_done, 1u);
        }
      }
      // The cell outputs last: they may go to host memory (pinned result
      // block), and the fences above need not wait for those writes.
      PP_CHECK(!c.valid || cell < static_cast<int64_t>(P.n_kt) * P.n_dirs * P.n_pows);
      PP_CHECK(bs_o < 16 && bs_t < 16);
      if (kCells && c.valid) {
        out.our_time[cell] = bt_o.v;
        out.opp_time[cell] = bt_t.v;
        out.rx[cell] = rx.v;
        out.ry[cell] = ry.v;
        out.our_slot[cell] = static_cast<int8_t>(bs_o);
        out.opp_slot[cell] = static_cast<int8_t>(bs_t);
        out.feasible[cell] = feas;
        if (!feas) out.score[cell] = -CUDART_INF_F;
      }
      PP_CMARK(3);
}

#ifndef PP_CROSS_CAP
#define PP_CROSS_CAP 1
#endif
constexpr bool kCrossCap = PP_CROSS_CAP != 0;  // dev knob: batches' cross-team cap

template <bool kCells, bool kLeftovers>
__device__ __forceinline__ void scan_tile(ScanSmem& sm, const DevParams& P, const CellOut& out,
                                          const CellQueue& q, FrameCounters* __restrict__ fc,
                                          int f, int tile, const double4& dd, const PowRow& pr,
                                          const FrameDev* src, const RobotK* rk_arg) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const FrameDev& F = sm.frame;
  const xd dt = P.dt, slide = P.slide, roll = P.roll, radius = P.radius;
  {
    const int kt = tile / (P.n_dirs * P.n_ptiles);
    const int dir = (tile / P.n_ptiles) % P.n_dirs;
    const int ptile = tile % P.n_ptiles;
    const int64_t cell0 = (static_cast<int64_t>(kt) * P.n_dirs + dir) * P.n_pows + ptile * 32;

    // ---- A: trajectory + scan window per cell (ball_model.cpp:12-43,
    //      intercept.cpp:12-25, 47-69; dpps.cpp:119-138) by warp 0, reading
    //      the ball and field from the frame's source, while the other warps
    //      stage the frame and the robots' filter constants.
    if (nwarps == 1) {
      load_frame(&sm.frame, src);
      __syncwarp();
    } else if (warp > 0) {
      const int4* fs = reinterpret_cast<const int4*>(src);
      int4* fd = reinterpret_cast<int4*>(&sm.frame);
      for (int i = threadIdx.x - 32; i < static_cast<int>(sizeof(FrameDev) / 16);
           i += blockDim.x - 32)
        fd[i] = fs[i];
    }
    if (warp == 0) {
      const CellLane c = cell_window(*src, P, dd, pr, ptile * 32 + lane < P.n_pows);
      reinterpret_cast<CellLane*>(sm.cl_raw)[lane] = c;
      sm.cap[0][lane] = 0x7fffffff;
      sm.cap[1][lane] = 0x7fffffff;
      sm.cap[2][lane] = 0x7fffffff;
      if (lane == 0) {
        sm.n_left = 0;
        sm.next_pair = 0;
      }
      sm.ke[lane] = c.ke;
      sm.trf[lane] = TrajF(c.tr, static_cast<float>(slide.v), static_cast<float>(roll.v));
      sm.win_s[lane] = make_float2(static_cast<float>(c.s_lo), static_cast<float>(c.s_hi));
      if (lane == 0) sm.tile_uf = make_float2(static_cast<float>(c.ux), static_cast<float>(c.uy));
      PP_CMARK_W(0);
    }
    if (rk_arg || P.rk_pre) {
      // the frame's robot constants (host- or pre-computed): the other warps
      // stage them while warp 0 computes the windows
      if (warp > 0 || nwarps == 1) {
        const int4* rks = rk_arg ? reinterpret_cast<const int4*>(rk_arg)
                                 : static_cast<const int4*>(P.rk_pre) +
                                       static_cast<int64_t>(f) * (kMaxRobots * sizeof(RobotK) / 16);
        int4* dst = reinterpret_cast<int4*>(sm.rk);
        const int n16 = src->n_scan * static_cast<int>(sizeof(RobotK) / 16);
        const int t0 = nwarps == 1 ? lane : threadIdx.x - 32;
        const int nt = nwarps == 1 ? 32 : blockDim.x - 32;
        for (int i = t0; i < n16; i += nt) dst[i] = rks[i];
      }
    } else if (warp == (nwarps > 1 ? 1 : 0)) {
      for (int ri = lane; ri < src->n_scan; ri += 32) robot_consts(*src, P, ri, &sm.rk[ri]);
      PP_CMARK_W(1);
    }
    __syncthreads();
    PP_TMARK(2);

  // ---- B: SBIP scan per (robot, cell): scan_robot (intercept.cpp:87-115)
    //      + first feasible sample (kernel.hpp:33-44) + rest rule
    //      (dpps.cpp:177-190).
    //      Two exact-safe accelerations, neither of which can change a result:
    //      * team cap (dpps.cpp:142-153): robots of a team share the earliest
    //        hit index per cell in shared memory; a robot stops once its next
    //        sample is past it (it can no longer win or tie).
    //      * FP32 reach filter: a sample is only tested exactly if the robot
    //        could possibly get there, d <= radius + D(t) (ReachBound).
    const CellLane* cl = reinterpret_cast<const CellLane*>(sm.cl_raw);
    const int max_steps = kLeftovers ? P.scan_steps : 1 << 30;
    // Robot order (throughput shape): the robots nearest the tile's ray
    // first -- the longest scans, and the earliest team caps -- pulled
    // dynamically by the warps (sm.next_pair counts robots here), so the
    // warps reach the barrier together.  Every warp ranks the robots the
    // same way (lane = robot; concurrently, which measured faster than
    // one ranking behind a barrier); order does not change results.
#ifndef PP_SCAN_STATIC_ORDER
    constexpr bool kDyn = !kLeftovers;
#else
    constexpr bool kDyn = false;  // dev knob: round-robin robots (round-1 order)
#endif
    int my_rank = 0;
    if (kDyn) {
      float key = 3.0e38f;
      if (lane < F.n_scan) {
        const RobotK& rk = sm.rk[lane];
        const float2 u = sm.tile_uf;
        const float along = fmaxf(-(rk.bxf * u.x + rk.byf * u.y), 0.f);  // robot - ball on u
        const float ex = -rk.bxf - along * u.x, ey = -rk.byf - along * u.y;
        key = ex * ex + ey * ey;
        // batches: their robots first, so the cross cap is set early
        // (ours then still go nearest first among themselves)
        if (kCrossCap && !kCells && F.scan_slot[lane] < kTheirs) key += 1e6f;
      }
      // (lanes >= n_scan hold the largest key: ranks of the scanned robots
      // only count the scanned robots)
      for (int j = 0; j < F.n_scan; ++j) {
        const float kj = __shfl_sync(0xffffffffu, key, j);
        my_rank += (kj < key || (kj == key && j < lane)) ? 1 : 0;
      }
    }
    for (int it = warp;; it = kDyn ? it : it + nwarps) {
      int ri = it;
      if (kDyn) {
        unsigned i = 0;
        if (lane == 0) i = atomicAdd(&sm.next_pair, 1u);
        i = __shfl_sync(0xffffffffu, i, 0);
        if (i >= static_cast<unsigned>(F.n_scan)) break;
        ri = __ffs(__ballot_sync(0xffffffffu, my_rank == static_cast<int>(i))) - 1;
      } else if (ri >= F.n_scan) {
        break;
      }
      const RobotK& rk = sm.rk[ri];
      const SampleF S = sample_f(rk, sm.tile_uf, P);
      double time;
      int code, lk;
      PP_ROBOT_START();
      scan_robot<!kLeftovers, !kCells && !kLeftovers && kCrossCap>(
                 cl[lane], sm.trf[lane], sm.win_s[lane], S, F, P, rk, &sm.cap[0][0], ri,
                 max_steps, &time,
                 &code, &lk);
      // an open pair: NaN time (no result is NaN) and its next sample
      PP_CHECK(ri >= 0 && ri < kMaxRobots);
      sm.res_t[ri][lane] = lk < 0 ? time : CUDART_NAN;
      sm.res_k[ri][lane] = lk < 0 ? code : lk;
      PP_ROBOT_END(ri);
    }
    __syncthreads();
    PP_TMARK(0);
    if (kLeftovers) {
      // rounds over the open pairs until none is left
      const int n_pairs = F.n_scan * 32;
      for (int round = 0;; ++round) {
        if (threadIdx.x == 0) {
          sm.n_left = 0;
          sm.next_pair = 0;
        }
        __syncthreads();
        for (int e0 = warp * 32; e0 < n_pairs; e0 += nwarps * 32) {
          const int e = e0 + lane;
          const bool open = e < n_pairs && isnan(sm.res_t[e >> 5][e & 31]);
          const unsigned om = __ballot_sync(0xffffffffu, open);
          if (om) {
            unsigned at = 0;
            if (lane == 0) at = atomicAdd(&sm.n_left, static_cast<unsigned>(__popc(om)));
            at = __shfl_sync(0xffffffffu, at, 0);
            if (open) sm.left[at + __popc(om & ((1u << lane) - 1u))] = static_cast<uint16_t>(e);
          }
        }
        __syncthreads();
        const int n_left = static_cast<int>(sm.n_left);
        PP_CHECK(n_left <= kMaxRobots * 32);
#ifdef PP_PHASE_CLOCKS
        if (threadIdx.x == 0) sm.tph[3] = round == 0 ? n_left : sm.tph[3] + 10000;
        if (threadIdx.x == 0 && blockIdx.x < kRecCtas && round < 8) {
          g_round_rec[blockIdx.x][round][0] = n_left;
          g_round_rec[blockIdx.x][round][1] = clock64();
        }
#endif
        if (n_left == 0) break;
        scan_leftovers(cl, sm.trf, sm.ke, sm.tile_uf, F, P, sm.rk, &sm.cap[0][0], sm.left, n_left,
                       &sm.next_pair, sm.res_t, sm.res_k, P.scan_round_steps);
        __syncthreads();
      }
    }
    if (kLeftovers) {
      rest_rule_pass(cl, F, P, sm.rk, sm.cap, sm.res_t, sm.res_k);
      __syncthreads();
    }
    PP_TMARK(1);
    PP_CMARK(0);

    // ---- C: champions (dpps.cpp:140-213).  The update is a strict (time, id)
    //      lexicographic argmin seeded with (kNever, -1), so visiting order
    //      does not matter.  Feasible cells go to the frame's value queue.
    if (warp == 0) {
      const CellLane& c = reinterpret_cast<const CellLane*>(sm.cl_raw)[lane];
      tile_champions<kCells>(
          c, F, P, [&](int ri) { return sm.res_t[ri][lane]; },
          [&](int ri) { return sm.res_k[ri][lane]; }, out, q, fc, f, kt, cell0);
    }
  }
}

template <bool kCells, int kWarps, int kCtas, bool kLeftovers = (kCtas <= 2)>
__global__ void __launch_bounds__(kWarps * 32, kCtas)
    scan_kernel(const FrameDev* __restrict__ frames, DevParams P, CellOut out, CellQueue q,
                FrameCounters* __restrict__ fc, const __grid_constant__ FrameArg fa) {
  __shared__ ScanSmem sm;
  PP_CLOCK_INIT();
  const int f = blockIdx.x / P.n_tiles;
  // Heavy tiles first: slow kick speeds (low power tiles) before fast ones,
  // flat before chip, then by direction.  Co-resident CTAs of one SM are
  // launched about an SM count apart, so the grid order (power tile
  // fastest-varying, 148 even) put heavy tiles on SMs with heavy tiles; this
  // order gives the slowest tiles lighter neighbours (measured: C2 frame
  // kernel span 51.1 -> 49.1 us, C1 41.9 -> 39.7 us).  Not for multi-wave
  // single frames (C3): their cell outputs stream into the result block,
  // possibly host memory, and grid order keeps those writes sequential
  // (C3 with the block in pinned memory: 1.58 vs 1.93 ms).  Results do not
  // depend on the order.
  const int b = blockIdx.x % P.n_tiles;
  const int per_pt = P.n_kt * P.n_dirs;
  const int tile = (kLeftovers || !kCells) ? (b % per_pt) * P.n_ptiles + b / per_pt : b;
  // Let the value kernel (launched with programmatic stream serialization)
  // get its CTAs resident while the last scan CTAs run; it waits for this
  // grid's completion before reading anything (griddepcontrol.wait).
  asm volatile("griddepcontrol.launch_dependents;");
  if (threadIdx.x == 0) atomicMax(&fc[f].t0_inv, ~pp_now_ns());
  // warp 0's table rows (window phase) are requested before the frame
  double4 dd = make_double4(0.0, 0.0, 0.0, 0.0);
  PowRow pr{};
  if (threadIdx.x < 32) {
    const int kt = tile / (P.n_dirs * P.n_ptiles);
    const int dir = (tile / P.n_ptiles) % P.n_dirs;
    const int pw = (tile % P.n_ptiles) * 32 + threadIdx.x;
    dd = P.dirs[dir];
    pr = P.pows[kt * P.n_pows + (pw < P.n_pows ? pw : P.n_pows - 1)];
  }
#ifdef PP_PHASE_CLOCKS
  if (threadIdx.x == 0 && blockIdx.x < kRecCtas) g_win_rec[blockIdx.x][3] = ph_last_;
#endif
  // (the frame is staged to shared memory inside scan_tile, overlapped with
  // warp 0's windows, which read the few frame fields they need directly)
  scan_tile<kCells, kLeftovers>(sm, P, out, q, fc, f, tile, dd, pr,
                                P.frame_in_arg ? &fa.frame : frames + f,
                                P.frame_in_arg ? fa.rk : nullptr);
#ifdef PP_PHASE_CLOCKS
  if (threadIdx.x == 0) {
    const long long now_ = clock64();
    ph_[0] = sm.tph[0] - ph_last_;       // window + lane-per-cell phase
    ph_[1] = sm.tph[1] - sm.tph[0];      // leftovers
    ph_[2] = now_ - sm.tph[1];           // champions + queue
    ph_[3] = sm.tph[3];  // first-round open pairs + 10000 x rounds
    ph_[4] = sm.tph[2] - ph_last_;       // window (A) alone
  }
#endif
  PP_FLUSH(8);
}

// ---- throughput scan: a warp per tile ------------------------------------
// Batches (and other launches of many tiles) have more tiles than the GPU
// has warps, so a tile needs no more than one warp: the warp computes its
// cells' windows (lane = cell), scans the tile's robots one after another,
// keeps each cell's champions as it goes, and publishes the cells -- with no
// CTA barrier between the phases (in the 4-warp-per-tile form, 3 of 4 warps
// waited at barriers through the window and champion phases, and for the
// tile's slowest robot).  Robots scanned in sequence also see their team's
// final cap from every robot before them.  A CTA stages one frame and its
// robots' constants once and its warps pull that frame's tiles (group g of
// G: tiles g, g + G, ... in heavy-first order) from a shared counter.
struct WarpTile {
  __align__(16) unsigned char cl_raw[32 * sizeof(CellLane)];
  TrajF trf[32];
  float2 win_s[32];
  int32_t cap[3][32];  // team caps (ours, theirs) and our cross cap, per cell
  int8_t order[32];    // the tile's robots by rank
};


template <int kWarps>
struct ScanWarpSmem {
  RobotK rk[kMaxRobots];
  FrameDev frame;
  unsigned next_tile;
  WarpTile w[kWarps];
};

template <bool kCells>
__device__ __forceinline__ void warp_tile(const FrameDev& F, const RobotK* rk_s, WarpTile& ws,
                                          const DevParams& P, const CellOut& out,
                                          const CellQueue& q, FrameCounters* __restrict__ fc,
                                          int f, int tile) {
  const int lane = threadIdx.x & 31;
  // lane = power: tile = (kick slot, direction, 32 powers)
  const int kt = tile / (P.n_dirs * P.n_ptiles);
  const int dir = (tile / P.n_ptiles) % P.n_dirs;
  const bool valid = (tile % P.n_ptiles) * 32 + lane < P.n_pows;
  const int pw = valid ? (tile % P.n_ptiles) * 32 + lane : P.n_pows - 1;
  const int64_t cell = (static_cast<int64_t>(kt) * P.n_dirs + dir) * P.n_pows + pw;
  // A: the window of this lane's cell (as scan_tile)
  {
    const double4 dd = P.dirs[dir];
    const PowRow pr = P.pows[kt * P.n_pows + pw];
    const CellLane c = cell_window(F, P, dd, pr, valid);
    reinterpret_cast<CellLane*>(ws.cl_raw)[lane] = c;
    ws.trf[lane] = TrajF(c.tr, static_cast<float>(P.slide), static_cast<float>(P.roll));
    ws.win_s[lane] = make_float2(static_cast<float>(c.s_lo), static_cast<float>(c.s_hi));
    ws.cap[0][lane] = ws.cap[1][lane] = ws.cap[2][lane] = 0x7fffffff;
  }
  const float2 uf = make_float2(static_cast<float>(P.dirs[dir].z), static_cast<float>(P.dirs[dir].w));
  __syncwarp();
  const CellLane& c = reinterpret_cast<const CellLane*>(ws.cl_raw)[lane];
  // Robot order: their robots first (their hits set our cross cap), then
  // nearest the tile's ray first (the longest scans and earliest team caps).
  // Lane = robot; order does not change results.
  int my_rank = 0;
  {
    float key = 3.0e38f;
    if (lane < F.n_scan) {
      const RobotK& rk = rk_s[lane];
      const float along = fmaxf(-(rk.bxf * uf.x + rk.byf * uf.y), 0.f);
      const float ex = -rk.bxf - along * uf.x, ey = -rk.byf - along * uf.y;
      key = ex * ex + ey * ey;
      if (kCrossCap && !kCells && F.scan_slot[lane] < kTheirs) key += 1e6f;
    }
    for (int j = 0; j < F.n_scan; ++j) {
      const float kj = __shfl_sync(0xffffffffu, key, j);
      my_rank += (kj < key || (kj == key && j < lane)) ? 1 : 0;
    }
  }
  // Robots no cell of the tile can need: scan_start's window prune (the
  // quick reject over the whole window, intercept.cpp:89-95, in FP32 with
  // 1 mm of slack) applied to the union of the cells' windows -- the segment
  // from the nearest first sample to the farthest last one, the latest last
  // sample time -- so it prunes only robots every cell's own prune drops.
  // One pass with lane = robot instead of a scan per robot.
  unsigned pruned = 0u;
  if (kTilePrune && !P.exact_only) {
    const bool has = c.valid && c.kb < c.ke;
    float lo = has ? ws.win_s[lane].x : 3.0e38f;
    float hi = has ? ws.win_s[lane].y : -3.0e38f;
    float tk = has ? static_cast<float>(c.ke - 1) * P.dtf : 0.f;
    for (int sh = 16; sh > 0; sh >>= 1) {
      lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, sh));
      hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, sh));
      tk = fmaxf(tk, __shfl_xor_sync(0xffffffffu, tk, sh));
    }
    bool drop = false;
    if (lane < F.n_scan) {
      if (hi < lo) {
        drop = true;  // no cell has a window
      } else {
        const RobotK& rk = rk_s[lane];
        const float s0 = -(rk.bxf * uf.x + rk.byf * uf.y);
        const float sc = fminf(fmaxf(s0, lo), hi);
        const float ex = fmaf(uf.x, sc, rk.bxf), ey = fmaf(uf.y, sc, rk.byf);
        const float gap = sqrt_a(ex * ex + ey * ey) - 1e-3f - P.radf;
        drop = gap > rk.vbf * tk * 1.0001f;
      }
    }
    pruned = __ballot_sync(0xffffffffu, drop);
  }
  // B: every robot in rank order, this lane's champions -- (time bits, id)
  // argmin per team, as tile_champions -- updated after each
  unsigned long long bt_o = 0x7ff0000000000000ull, bt_t = 0x7ff0000000000000ull;  // +inf
  int bid_o = -1, bk_o = -2, bs_o = -1, bid_t = -1, bs_t = -1;
  auto champion = [&](int ri, double time, int code) {
    const int slot = F.scan_slot[ri];
    const int id = F.id[slot];
    const unsigned long long tb = __double_as_longlong(time);
    if (slot < kTheirs) {
      if (tb < bt_o || (tb == bt_o && id < bid_o)) {
        bt_o = tb;
        bid_o = id;
        bk_o = code;
        bs_o = slot;
      }
    } else if (tb < bt_t || (tb == bt_t && id < bid_t)) {
      bt_t = tb;
      bid_t = id;
      bs_t = slot - kTheirs;
    }
  };
  constexpr bool kX = !kCells && kCrossCap;
#if PP_REST_RANK
  // robots (bit = rank) whose pair ended without a hit: the rest rule runs
  // nearest first, so the champion it sets early filters the others
  if (my_rank < F.n_scan) ws.order[my_rank] = static_cast<int8_t>(lane);
  __syncwarp();
#define PP_REST_BIT(i, ri) (1u << (i))
#else
#define PP_REST_BIT(i, ri) (1u << (ri))
#endif
  unsigned rest_mask = 0;  // robots whose pair ended without a hit
  for (int i = 0; i < F.n_scan; ++i) {
    const int ri = __ffs(__ballot_sync(0xffffffffu, my_rank == i)) - 1;
    PP_CHECK(ri >= 0 && ri < F.n_scan);
    if ((pruned >> ri) & 1u) {  // every cell's window pruned: no hit, rest rule
      if (c.valid && c.rif) rest_mask |= PP_REST_BIT(i, ri);
      continue;
    }
    const RobotK& rk = rk_s[ri];
    const SampleF S = sample_f(rk, uf, P);
    double time;
    int code, lk;
    scan_robot<false, kX, true>(c, ws.trf[lane], ws.win_s[lane], S, F, P, rk, &ws.cap[0][0], ri,
                          1 << 30, &time, &code, &lk);
    if (code >= 0) {
      champion(ri, time, code);
    } else if (code == kNoHit && c.valid && c.rif) {
      rest_mask |= PP_REST_BIT(i, ri);
    }
    // (capped out, or no hit with the rest outside the field: +inf, which
    // never displaces a champion)
  }
  // The rest rule (dpps.cpp:177-190) of the pairs without a hit, after every
  // robot, with the lane's final caps: skipped where the robot's team hit
  // strictly before the ball rests, and (batches) for ours where their hit
  // leaves the cell infeasible anyway (pair_finish's rules; caps only
  // decrease, so the final ones skip at least as much).
  {
    const int cap_o = ws.cap[0][lane], cap_t = ws.cap[1][lane];
    while (rest_mask) {
#if PP_REST_RANK
      const int rj = ws.order[__ffs(rest_mask) - 1];
#else
      const int rj = __ffs(rest_mask) - 1;
#endif
      rest_mask &= rest_mask - 1;
      const bool theirs = F.scan_slot[rj] >= kTheirs;
      const int k_team = theirs ? cap_t : cap_o;
      if ((k_team != 0x7fffffff && xd(double(k_team)) * xd(P.dt) < c.tr.t_stop) ||
          (kX && !theirs && cap_t != 0x7fffffff &&
           c.tr.t_stop + xd(P.safety) > xd(double(cap_t)) * xd(P.dt)))
        continue;
      if (kRestLB && !P.exact_only) {
        // the FP32 arrival lower bound at the rest point (the sample test's
        // ArrivalLB): above the team's champion time, this robot's rest-rule
        // time max(arrival, t_stop) can neither beat nor tie it
        const unsigned long long bt = theirs ? bt_t : bt_o;
        // batches, ours: their champion so far ends the cell's chances once
        // fl(bound + safety) > it (dpps.cpp:207-212) -- then this robot is
        // not the champion of a feasible cell
        const bool vs_theirs = kX && kRestX && !theirs && bt_t != 0x7ff0000000000000ull;
        if (bt != 0x7ff0000000000000ull || vs_theirs) {
          const RobotK& rk = rk_s[rj];
          const float ds = static_cast<float>(c.tr.d_stop.v);
          const float qx = fmaf(uf.x, ds, rk.bxf), qy = fmaf(uf.y, ds, rk.byf);
          const float d2 = fmaf(qx, qx, qy * qy);
          const float inv = rsqrt_ftz(fmaxf(d2, 1e-30f));
          const double lbd =
              static_cast<double>(rk.lb.lower_bound(qx, qy, d2 * inv, inv, P.radf));
          if (lbd > __longlong_as_double(static_cast<long long>(bt))) continue;
          if (vs_theirs &&
              (xd(lbd) + xd(P.safety)).v > __longlong_as_double(static_cast<long long>(bt_t)))
            continue;
        }
      }
      double t;
      int cd;
      pair_result(c, P, robot_x(F, P, rk_s[rj], rj), -1, false, &t, &cd);
      champion(rj, t, cd);
    }
  }
  // C: receive point, feasibility, queue, cell outputs
  tile_publish<kCells>(c, F, P, bt_o, bk_o, bs_o, bt_t, bs_t, out, q, fc, f, kt, cell);
  __syncwarp();  // (ws is reused by the warp's next tile)
}

// Grid: n_frames x P.scan_groups CTAs; CTA (f, g) runs its share of frame
// f's tiles (below).
template <bool kCells, int kWarps, int kCtas>
__global__ void __launch_bounds__(kWarps * 32, kCtas)
    scan_warp_kernel(const FrameDev* __restrict__ frames, DevParams P, CellOut out, CellQueue q,
                     FrameCounters* __restrict__ fc, const __grid_constant__ FrameArg fa) {
  __shared__ ScanWarpSmem<kWarps> sm;
  const int groups = P.scan_groups;
  const int f = blockIdx.x / groups;
  const int g = blockIdx.x % groups;
  asm volatile("griddepcontrol.launch_dependents;");
  const FrameDev* src = P.frame_in_arg ? &fa.frame : frames + f;
  const RobotK* rk_arg = P.frame_in_arg ? fa.rk : nullptr;
  if (threadIdx.x == 0) {
    atomicMax(&fc[f].t0_inv, ~pp_now_ns());
    sm.next_tile = 0;
  }
  {
    const int4* fs = reinterpret_cast<const int4*>(src);
    int4* fd = reinterpret_cast<int4*>(&sm.frame);
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(FrameDev) / 16); i += blockDim.x)
      fd[i] = fs[i];
  }
  const int n_scan = src->n_scan;
  if (rk_arg || P.rk_pre) {
    const int4* rks = rk_arg ? reinterpret_cast<const int4*>(rk_arg)
                             : static_cast<const int4*>(P.rk_pre) +
                                   static_cast<int64_t>(f) * (kMaxRobots * sizeof(RobotK) / 16);
    int4* dst = reinterpret_cast<int4*>(sm.rk);
    const int n16 = n_scan * static_cast<int>(sizeof(RobotK) / 16);
    for (int i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = rks[i];
  } else if (static_cast<int>(threadIdx.x) < n_scan) {
    robot_consts(*src, P, threadIdx.x, &sm.rk[threadIdx.x]);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  WarpTile& ws = sm.w[threadIdx.x >> 5];
  // CTA g runs tiles g, g + groups, ...: batches in heavy-first order (each
  // CTA gets a mix of heavy and light tiles, heaviest first); cell outputs (a
  // single multi-wave frame) in grid order, so the tiles running at any time
  // are neighbours and the result block (possibly host memory) is written
  // about sequentially.
  const int n_mine = (P.n_tiles - g + groups - 1) / groups;
  const int per_pt = P.n_kt * P.n_dirs;
  for (;;) {
    unsigned j = 0;
    if (lane == 0) j = atomicAdd(&sm.next_tile, 1u);
    j = __shfl_sync(0xffffffffu, j, 0);
    if (static_cast<int>(j) >= n_mine) break;
    const int b = g + groups * static_cast<int>(j);
    const int tile = kCells ? b : (b % per_pt) * P.n_ptiles + b / per_pt;
    PP_CHECK(tile >= 0 && tile < P.n_tiles && (threadIdx.x >> 5) < kWarps);
    warp_tile<kCells>(sm.frame, sm.rk, ws, P, out, q, fc, f, tile);
  }
}

// robot_consts of every scanned robot of every frame of a batch, once
// (instead of once per tile): thread per (frame, robot).
__global__ void __launch_bounds__(256) robot_consts_kernel(const FrameDev* __restrict__ frames,
                                                           DevParams P, RobotK* __restrict__ out,
                                                           int64_t n_frames) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t f = i / kMaxRobots;
  const int ri = static_cast<int>(i % kMaxRobots);
  if (f >= n_frames || ri >= frames[f].n_scan) return;
  robot_consts(frames[f], P, ri, &out[i]);
}

}  // namespace pp
