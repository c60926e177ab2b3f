// pp_cabi.cu -- host side of the C-ABI declared in include/passplan_b200.h.
//
// Owns validation (config.cpp:172-200, dpps.cpp:22-28, 219-223), the staging
// of world state into the kernels' FrameDev layout (id-sorted teams,
// dpps.cpp:79-92), the direction table (dpps.cpp:30-48, computed here with the
// host libm so it is bit-identical to the reference's), and the launches.
// Host code is compiled with -ffp-contract=off like the reference.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "passplan_b200.h"
#include "passplan_b200_layout.h"
#include "pp_kernels.cuh"

// NVTX ranges around the C-ABI entry points (profiler ranges);
// header-only NVTX v3, a no-op unless a profiler is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define PP_NVTX(name) const NvtxRange pp_nvtx_range_(name)

namespace {

constexpr double kPi = 3.14159265358979323846;  // == std::numbers::pi

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  // Grow-only; new memory is zeroed on the context's stream `s`, so the
  // kernels queued after it on that stream see the zeros.
  cudaError_t reserve(cudaStream_t s, size_t want) {
    if (want <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) {
      bytes = want;
      e = cudaMemsetAsync(p, 0, want, s);
    }
    return e;
  }
};

struct PinnedBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  cudaError_t reserve(size_t want) {
    if (want <= bytes) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaHostAlloc(&p, want, cudaHostAllocDefault);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
};

}  // namespace

// The arguments and launch shapes of a single-frame pipeline, recorded when
// pp_dpps captures its graph: per call only the FrameArg parameter changes,
// so the call updates the two kernel nodes' parameters instead of copying
// the frame to the device.
using ScanFn = void (*)(const pp::FrameDev*, pp::DevParams, pp::CellOut, pp::CellQueue,
                        pp::FrameCounters*, pp::FrameArg);
using ValueFn = void (*)(const pp::FrameDev*, pp::DevParams, pp::CellQueue, pp::FrameCounters*,
                         pp::CellOut, pp::Partial*, pp_dpps_summary*, int, int, pp::FrameDev);
struct PipeRec {
  const pp::FrameDev* frames;
  pp::DevParams P;
  pp::CellOut co;
  pp::CellQueue q;
  pp::FrameCounters* fc;
  pp::Partial* parts;
  pp_dpps_summary* sums;
  int nch, per_frame;
  ScanFn scan_fn;
  ValueFn value_fn;
  dim3 sgrid, sblock, vgrid, vblock;
};

struct pp_ctx {
  int device = 0;
  // Device shape, queried once: SM count and the resident CTAs per SM of the
  // pipeline kernels (launch-shape thresholds derive from these, not from an
  // assumed 148 SMs).
  int n_sms = 0;
  int occ_scan_wide = 0, occ_scan_mid = 0, occ_scan_narrow = 0, occ_value_wide = 0;
  // PP_OPT_EXACT_ONLY: every FP32 filter off (verification switch)
  int exact_only = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evm = nullptr;
  // pp_dpps as one CUDA graph (scan, value; a D2H only for pageable
  // blocks), rebuilt when its key (params, output pointers, copy flags, ...)
  // changes; each call only rewrites the two kernel nodes' FrameArg.
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  cudaGraphNode_t scan_node = nullptr, value_node = nullptr;
  PipeRec rec{};
  std::vector<unsigned char> gkey;
  std::string err;
  // single frame
  DevBuf frame, block, partials, counters, dirs, pows, scratch_in, scratch_out;
  DevBuf queue, fcount;  // scan -> value pipeline (per-frame cell queues, counters)
  DevBuf chunk_fill;     // single frame: entries written per value chunk (streaming)
  PinnedBuf frame_h;
  int dirs_n = -1;
  std::vector<double> pows_key;  // inputs the power table was built from
  int max_count = 0;             // most samples of any power row
  DevBuf xcap;                   // batches: cross_cap table (xcap_table_kernel)
  std::vector<double> xcap_key;  // (dt, safety, entries) it was built for
  // run map
  DevBuf run_block, run_partials, run_counter;
  // batch: raw worlds (+ caller's kicker ids) uploaded, staged FrameDevs,
  // chosen kickers, first bad frame, robot constants, per-frame results
  DevBuf batch_worlds, batch_kick_in, batch_frames, batch_kickers, batch_bad, batch_rk;
  DevBuf batch_compact, batch_full;
  int64_t batch_n = 0;
  int64_t batch_frame0 = 0;  // index of the first uploaded frame in the caller's array (messages)
  int batch_max_scan = 1;      // widest scan list of the uploaded frames
  bool batch_has_kickers = false;
  bool batch_ran = false;
  // last single-frame launch (pp_dpps_relaunch)
  bool last_valid = false;
  pp::DevParams last_P{};
  pp::CellOut last_co{};
  pp_dpps_summary* last_dsum = nullptr;
  int last_threads = 0;
  std::unique_ptr<pp::FrameArg> last_fa{new pp::FrameArg()};  // the frame, as a parameter

  pp_ctx() = default;
  pp_ctx(const pp_ctx&) = delete;
  pp_ctx& operator=(const pp_ctx&) = delete;
  // Releases whatever a (possibly partial) pp_ctx_create acquired.
  ~pp_ctx() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (evm) cudaEventDestroy(evm);
    if (gexec) cudaGraphExecDestroy(gexec);
    if (graph) cudaGraphDestroy(graph);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

// single-frame staging: FrameDev, then the frame's RobotK[kMaxRobots]
constexpr size_t kFrameBytes = sizeof(pp::FrameDev) + sizeof(pp::RobotK) * pp::kMaxRobots;

pp_status fail(pp_ctx* ctx, pp_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  return st;
}

#define PP_CUDA_TRY(ctx, expr)                                                              \
  do {                                                                                      \
    const cudaError_t e_ = (expr);                                                          \
    if (e_ != cudaSuccess)                                                                  \
      return fail((ctx), PP_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                                \
  } while (0)

// Zero the pipeline's counters after a failed or stalled launch, so the
// next call does not start from dirty queue bases (they are otherwise
// self-cleaning, see FrameCounters).
void reset_pipeline(pp_ctx* ctx) {
  if (ctx->fcount.p) cudaMemsetAsync(ctx->fcount.p, 0, ctx->fcount.bytes, ctx->stream);
  if (ctx->chunk_fill.p) cudaMemsetAsync(ctx->chunk_fill.p, 0, ctx->chunk_fill.bytes, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
}

#define PP_PIPE_TRY(ctx, expr)                                                              \
  do {                                                                                      \
    const cudaError_t e_ = (expr);                                                          \
    if (e_ != cudaSuccess) {                                                                \
      reset_pipeline(ctx);                                                                  \
      return fail((ctx), PP_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                                \
    }                                                                                       \
  } while (0)

void put(char* msg, size_t len, const std::string& s) {
  if (msg && len) std::snprintf(msg, len, "%s", s.c_str());
}

// PlannerConfig::validate (config.cpp:172-200) minus SvgStyle, plus
// BallModelParams/MotionLimits::validate (ball_model.cpp:47-60, motion.cpp:10-14)
// and SearchGrid::validate (dpps.cpp:22-28).
// BallModelParams::validate (ball_model.cpp:47-60).
bool validate_ball(const pp_ball_model& b, std::string* why) {
  if (!(b.slide_decel > b.roll_decel) || !(b.roll_decel > 0.0)) {
    *why = "ball model requires slide_decel > roll_decel > 0";
    return false;
  }
  if (!(b.transition_ratio > 0.0) || !(b.transition_ratio < 1.0)) {
    *why = "transition_ratio must lie in (0,1)";
    return false;
  }
  if (!(b.power_min > 0.0) || !(b.power_min < b.power_max)) {
    *why = "ball model requires 0 < power_min < power_max";
    return false;
  }
  if (!(b.chip_flight_fraction > 0.0) || !(b.chip_flight_fraction < 1.0)) {
    *why = "chip_flight_fraction must lie in (0,1)";
    return false;
  }
  return true;
}

bool validate_params(const pp_params& p, std::string* why) {
  if (!validate_ball(p.ball, why)) return false;
  for (const pp_motion_limits* m : {&p.motion_ours, &p.motion_theirs}) {
    if (!(m->max_speed > 0.0) || !(m->max_accel > 0.0) || !(m->max_decel > 0.0)) {
      *why = "motion limits must all be positive";
      return false;
    }
  }
  const pp_search_grid& g = p.grid;
  if (g.n_directions < 1) {
    *why = "grid.n_directions must be >= 1";
    return false;
  }
  if (g.n_powers < 1) {
    *why = "grid.n_powers must be >= 1";
    return false;
  }
  if (!(g.power_min > 0.0) || !(g.power_min <= g.power_max)) {
    *why = "grid requires 0 < power_min <= power_max";
    return false;
  }
  const pp_thresholds& t = p.thresholds;
  struct Rule {
    bool ok;
    const char* msg;
  };
  const Rule rules[] = {
      {t.sbip_dt > 0.0, "thresholds.sbip_dt must be > 0"},
      {t.possession_dt > 0.0, "thresholds.possession_dt must be > 0"},
      {t.robot_radius >= 0.0, "thresholds.robot_radius must be >= 0"},
      {t.safety_margin >= 0.0, "thresholds.safety_margin must be >= 0"},
      {t.buffer_time >= 0.0, "thresholds.buffer_time must be >= 0"},
      {t.possession_radius > 0.0, "thresholds.possession_radius must be > 0"},
      {t.angle_threshold >= 0.0, "thresholds.angle_threshold must be >= 0"},
      {t.shot_power >= 0.0, "thresholds.shot_power must be >= 0"},
      {t.margin_cap > 0.0, "thresholds.margin_cap must be > 0"},
      {t.contest_epsilon >= 0.0, "thresholds.contest_epsilon must be >= 0"},
      {t.grid_step > 0.0, "thresholds.grid_step must be > 0"},
      {t.min_zone_width > 0.0, "thresholds.min_zone_width must be > 0"},
      {t.guard_time_cap > 0.0, "thresholds.guard_time_cap must be > 0"},
      {t.drag_v_min >= 0.0, "thresholds.drag_v_min must be >= 0"},
      {t.marking_radius > 0.0, "thresholds.marking_radius must be > 0"},
      {p.norm.length_upper >= 0.0, "norm.length_upper must be >= 0"},
      {p.norm.angle_upper > 0.0, "norm.angle_upper must be > 0"},
  };
  for (const Rule& r : rules) {
    if (!r.ok) {
      *why = r.msg;
      return false;
    }
  }
  const pp_angle_band& a = p.angle_band;
  if (!(a.full_lo <= a.peak_lo && a.peak_lo <= a.peak_hi && a.peak_hi <= a.full_hi)) {
    *why = "angle_band knots must be non-decreasing";
    return false;
  }
  return true;
}

bool validate_grid(const pp_search_grid& g, std::string* why) {
  if (g.n_directions < 1) {
    *why = "grid.n_directions must be >= 1";
    return false;
  }
  if (g.n_powers < 1) {
    *why = "grid.n_powers must be >= 1";
    return false;
  }
  if (!(g.power_min > 0.0) || !(g.power_min <= g.power_max)) {
    *why = "grid requires 0 < power_min <= power_max";
    return false;
  }
  return true;
}

// direction_table (dpps.cpp:30-48) with the host libm, bit-identical.
std::vector<double> direction_table(int n) {
  std::vector<double> xy(2 * static_cast<size_t>(n));
  pp::direction_table_xy(n, xy.data());
  return xy;
}

// Team slots in id order (dpps.cpp:79-92; stable for equal ids).
std::vector<int> id_order(const pp_robot* robots, int n) {
  std::vector<int> idx(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) idx[i] = i;
  std::stable_sort(idx.begin(), idx.end(),
                   [&](int a, int b) { return robots[a].id < robots[b].id; });
  return idx;
}

// Stages one world into FrameDev.  Returns false (validation) when the kicker
// is not on team ours (dpps.cpp:221-223).
// Scan list of a packed frame: the DPPS search scans ours minus the kicker
// then theirs; interception scans everybody or the opponents only.
enum class ScanList { kDpps, kAll, kTheirs };

bool pack_frame(const pp_world& w, int32_t kicker_id, pp::FrameDev* F, int32_t* kicker_slot_out,
                std::string* why, ScanList list = ScanList::kDpps) {
  std::memset(F, 0, sizeof(*F));
  if (w.n_ours < 0 || w.n_ours > PP_MAX_TEAM || w.n_theirs < 0 || w.n_theirs > PP_MAX_TEAM) {
    *why = "team size outside [0, 16]";
    return false;
  }
  bool found = false;
  for (int i = 0; i < w.n_ours; ++i) found = found || w.ours[i].id == kicker_id;
  if (!found && list == ScanList::kDpps) {
    *why = "kicker id " + std::to_string(kicker_id) + " is not on team ours";
    return false;
  }
  const std::vector<int> so = id_order(w.ours, w.n_ours);
  const std::vector<int> st = id_order(w.theirs, w.n_theirs);
  int kicker_slot = -1;
  for (int s = 0; s < w.n_ours; ++s) {
    const pp_robot& r = w.ours[so[s]];
    F->px[s] = r.px;
    F->py[s] = r.py;
    F->vx[s] = r.vx;
    F->vy[s] = r.vy;
    F->id[s] = r.id;
    if (r.id == kicker_id) kicker_slot = s;  // last match, like dpps.cpp:250-252
  }
  for (int s = 0; s < w.n_theirs; ++s) {
    const pp_robot& r = w.theirs[st[s]];
    F->px[pp::kTheirs + s] = r.px;
    F->py[pp::kTheirs + s] = r.py;
    F->vx[pp::kTheirs + s] = r.vx;
    F->vy[pp::kTheirs + s] = r.vy;
    F->id[pp::kTheirs + s] = r.id;
  }
  F->ball_x = w.ball_px;
  F->ball_y = w.ball_py;
  F->L = w.field.length;
  F->W = w.field.width;
  F->gw = w.field.goal_width;
  F->dd = w.field.defense_depth;
  F->dw = w.field.defense_width;
  F->n_ours = w.n_ours;
  F->n_theirs = w.n_theirs;
  F->kicker_slot = kicker_slot;
  int n = 0;
  if (list != ScanList::kTheirs)
    for (int s = 0; s < w.n_ours; ++s)
      if (s != kicker_slot || list == ScanList::kAll) F->scan_slot[n++] = static_cast<int8_t>(s);
  for (int s = 0; s < w.n_theirs; ++s) F->scan_slot[n++] = static_cast<int8_t>(pp::kTheirs + s);
  F->n_scan = n;
  *kicker_slot_out = kicker_slot;
  return true;
}

const pp_robot* find_ours(const pp_world& w, int32_t id) {
  for (int i = 0; i < w.n_ours; ++i)
    if (w.ours[i].id == id) return &w.ours[i];
  return nullptr;
}

double host_distance(double ax, double ay, double bx, double by) {
  const double dx = ax - bx, dy = ay - by;
  return std::sqrt(dx * dx + dy * dy);
}

// Smallest double x >= 0 with sqrt_rn(x) >= r, so that for every double x:
// sqrt_rn(x) < r  <=>  x < sqrt_lt_threshold(r)   (sqrt_rn is monotone).
double sqrt_lt_threshold(double r) {
  if (!(r > 0.0)) return 0.0;
  double x = r * r;
  while (x > 0.0 && std::sqrt(x) >= r) x = std::nextafter(x, 0.0);
  while (std::sqrt(x) < r) x = std::nextafter(x, HUGE_VAL);
  return x;
}

// Largest double x with sqrt_rn(x) <= m:  sqrt_rn(x) <= m  <=>  x <= result.
double sqrt_le_threshold(double m) {
  if (m < 0.0) return -1.0;
  double x = m * m;
  while (std::sqrt(x) > m) x = std::nextafter(x, 0.0);
  while (std::sqrt(std::nextafter(x, HUGE_VAL)) <= m) x = std::nextafter(x, HUGE_VAL);
  return x;
}

pp::DevParams make_dev_params(const pp_ctx* ctx, const pp_params& p, const pp_search_grid& g) {
  pp::DevParams d{};
  d.exact_only = ctx->exact_only;
  d.r_lt2 = sqrt_lt_threshold(p.thresholds.robot_radius);
  d.mb_le2 = sqrt_le_threshold(p.thresholds.robot_radius + 1e-9);
  d.slide = p.ball.slide_decel;
  d.roll = p.ball.roll_decel;
  d.ratio = p.ball.transition_ratio;
  d.chip_frac = p.ball.chip_flight_fraction;
  d.dt = p.thresholds.sbip_dt;
  d.radius = p.thresholds.robot_radius;
  d.safety = p.thresholds.safety_margin;
  d.margin_cap = p.thresholds.margin_cap;
  d.a_o = p.motion_ours.max_accel;
  d.b_o = p.motion_ours.max_decel;
  d.vmax_o = p.motion_ours.max_speed;
  d.a_t = p.motion_theirs.max_accel;
  d.b_t = p.motion_theirs.max_decel;
  d.vmax_t = p.motion_theirs.max_speed;
  d.pw_t = p.pass_weights.teammate_time;
  d.pw_s = p.pass_weights.shoot_angle;
  d.pw_d = p.pass_weights.dist_goal;
  d.pw_r = p.pass_weights.refraction;
  d.pw_m = p.pass_weights.margin;
  d.len_upper_cfg = p.norm.length_upper;
  d.ang_upper = p.norm.angle_upper;
  d.power_min = g.power_min;
  d.power_max = g.power_max;
  d.dtf = static_cast<float>(d.dt);
  d.radf = static_cast<float>(d.radius);
  d.n_dirs = g.n_directions;
  d.n_pows = g.n_powers;
  d.n_kt = (g.flat ? 1 : 0) + (g.chip ? 1 : 0);
  d.kt_chip0 = g.flat ? 0 : 1;
  d.kt_chip1 = 1;
  d.n_ptiles = (g.n_powers + 31) / 32;
  d.n_tiles = d.n_kt * g.n_directions * d.n_ptiles;
  // Leftover-round schedule (tuned on C1/C2; PP_SCAN_STEPS / PP_SCAN_ROUND
  // override it for experiments, read once)
  static const int steps = [] {
    const char* e = getenv("PP_SCAN_STEPS");
    return e ? atoi(e) : 6;
  }();
  static const int round_steps = [] {
    const char* e = getenv("PP_SCAN_ROUND");
    return e ? atoi(e) : 4;
  }();
  d.scan_steps = steps;
  d.scan_round_steps = round_steps;
  return d;
}

void fill_summary_host(pp_dpps_summary* s, const pp_world& w, const pp_search_grid& g,
                       int32_t kicker_id, int32_t kicker_slot, int32_t possession) {
  s->n_cells = pp_grid_cells(&g);
  s->n_kick_types = (g.flat ? 1 : 0) + (g.chip ? 1 : 0);
  s->kick_types[0] = g.flat ? 0 : 1;
  s->kick_types[1] = 1;
  s->n_directions = g.n_directions;
  s->n_powers = g.n_powers;
  s->kicker_id = kicker_id;
  s->kicker_slot = kicker_slot;
  s->kicker_in_possession = possession;
  s->n_ours = w.n_ours;
  s->n_theirs = w.n_theirs;
  // id-sorted teams (stable insertion sort: at most 16 robots, no allocation)
  auto sorted_ids = [](const pp_robot* r, int n, int32_t* out) {
    for (int i = 0; i < PP_MAX_TEAM; ++i) out[i] = -1;
    for (int i = 0; i < n && i < PP_MAX_TEAM; ++i) {
      int j = i;
      while (j > 0 && out[j - 1] > r[i].id) {
        out[j] = out[j - 1];
        --j;
      }
      out[j] = r[i].id;
    }
  };
  sorted_ids(w.ours, w.n_ours, s->ours_ids);
  sorted_ids(w.theirs, w.n_theirs, s->theirs_ids);
  s->sbip_calls = static_cast<uint64_t>(s->n_cells) *
                  static_cast<uint64_t>(w.n_ours + w.n_theirs);  // dpps.cpp:148-153
}

int32_t possession_of(const pp_world& w, int32_t kicker_id, const pp_params& p) {
  const pp_robot* k = find_ours(w, kicker_id);
  if (!k) return 0;
  return host_distance(w.ball_px, w.ball_py, k->px, k->py) <= p.thresholds.possession_radius;
}

// World-independent tables of a (params, grid): unit directions and the
// per-(kick slot, power) trajectory rows.  Built on the host with the same
// FP64 operations as the kernels (passplan/detail/pp_math.hpp is host/device) and uploaded
// only when the inputs change.  Fills P.dirs / P.pows.
cudaError_t ensure_tables(pp_ctx* ctx, pp::DevParams* P) {
  using pp::xd;
  cudaError_t e = cudaSuccess;
  if (ctx->dirs_n != P->n_dirs) {
    const std::vector<double> xy = direction_table(P->n_dirs);
    std::vector<double4> d(static_cast<size_t>(P->n_dirs));
    for (int i = 0; i < P->n_dirs; ++i) {
      const xd dx = xy[2 * i], dy = xy[2 * i + 1];
      const xd n = pp::xsqrt(dx * dx + dy * dy);  // dpps.cpp:120-122 normalized()
      xd ux = 1.0, uy = 0.0;
      if (n.v != 0.0) {
        ux = dx / n;
        uy = dy / n;
      }
      d[i] = make_double4(dx.v, dy.v, ux.v, uy.v);
    }
    e = ctx->dirs.reserve(ctx->stream, d.size() * sizeof(double4));
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(ctx->dirs.p, d.data(), d.size() * sizeof(double4), cudaMemcpyHostToDevice,
                          ctx->stream);
    if (e != cudaSuccess) return e;
    ctx->dirs_n = P->n_dirs;
    ctx->last_valid = false;
  }
  const std::vector<double> key = {P->slide, P->roll, P->ratio, P->chip_frac, P->dt,
                                   P->power_min, P->power_max, double(P->n_pows),
                                   double(P->n_kt), double(P->kt_chip0), double(P->kt_chip1)};
  if (key != ctx->pows_key) {
    std::vector<pp::PowRow> rows(static_cast<size_t>(P->n_kt) * P->n_pows);
    const xd dt = P->dt, slide = P->slide, roll = P->roll;
    for (int s = 0; s < P->n_kt; ++s) {
      const bool chip = (s == 0 ? P->kt_chip0 : P->kt_chip1) != 0;
      for (int pw = 0; pw < P->n_pows; ++pw) {
        const xd speed = pp::power_at(pw, P->n_pows, P->power_min, P->power_max);
        const pp::Traj tr = pp::resolve_kick(speed, chip, slide, roll, P->ratio, P->chip_frac);
        pp::PowRow& r = rows[static_cast<size_t>(s) * P->n_pows + pw];
        r.speed = tr.speed.v;
        r.v1 = tr.v1.v;
        r.t_se = tr.t_se.v;
        r.d_se = tr.d_se.v;
        r.t_stop = tr.t_stop.v;
        r.d_stop = tr.d_stop.v;
        r.count = static_cast<int32_t>(std::floor((tr.t_stop / dt + xd(1e-9)).v)) + 1;
        r.kb = 0;
        if (tr.from.v > 0.0) {  // chip: skip the airborne stretch (intercept.cpp:47-69)
          const xd t_air = pp::travel_time_to_distance(tr, slide, roll, tr.from);
          if (!std::isnan(t_air.v)) r.kb = static_cast<int32_t>(std::ceil((t_air / dt - xd(1e-9)).v));
        }
      }
    }
    e = ctx->pows.reserve(ctx->stream, rows.size() * sizeof(pp::PowRow));
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(ctx->pows.p, rows.data(), rows.size() * sizeof(pp::PowRow),
                          cudaMemcpyHostToDevice, ctx->stream);
    if (e != cudaSuccess) return e;
    ctx->pows_key = key;
    ctx->max_count = 0;
    for (const pp::PowRow& r : rows) ctx->max_count = std::max(ctx->max_count, r.count);
    ctx->last_valid = false;
  }
  P->dirs = static_cast<const double4*>(ctx->dirs.p);
  P->pows = static_cast<const pp::PowRow*>(ctx->pows.p);
  return cudaSuccess;
}

// Resident CTAs per SM of the pipeline kernels (pp_ctx_create).
cudaError_t query_occupancy(pp_ctx* ctx) {
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &ctx->occ_scan_wide, pp::scan_kernel<true, pp::kScanWarpsWide, pp::kScanCtasWide>,
      32 * pp::kScanWarpsWide, 0);
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &ctx->occ_scan_mid, pp::scan_kernel<true, pp::kScanWarpsMid, pp::kScanCtasMid, true>,
        32 * pp::kScanWarpsMid, 0);
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &ctx->occ_scan_narrow, pp::scan_kernel<true, pp::kScanWarpsNarrow, pp::kScanCtasNarrow>,
        32 * pp::kScanWarpsNarrow, 0);
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &ctx->occ_value_wide, pp::value_kernel<true, pp::kValueThreadsWide>,
        pp::kValueThreadsWide, 0);
  if (e == cudaSuccess && (ctx->occ_scan_wide < 1 || ctx->occ_scan_mid < 1 ||
                           ctx->occ_scan_narrow < 1 || ctx->occ_value_wide < 1))
    e = cudaErrorInvalidConfiguration;
  return e;
}

// Largest value grid launched with the wide (single-frame, streaming) CTA
// shape: up to 4 chunks per SM the 256-thread CTAs' shorter item chains pay
// (measured: C1/C2 frames); beyond that the 128-thread shape packs better.
// Correctness does not depend on residency: streaming CTAs only wait for scan
// tiles, and every scan CTA has started before any value CTA runs (the scan
// triggers griddepcontrol.launch_dependents first thing), so they all finish.
// Value CTAs per frame of a batch launch (each loops over the frame's chunks).
#ifndef PP_VALUE_CTAS_PER_FRAME
#define PP_VALUE_CTAS_PER_FRAME 8
#endif
constexpr int kValueCtasPerFrame = PP_VALUE_CTAS_PER_FRAME;

int64_t value_wide_limit(const pp_ctx* ctx) {
  return static_cast<int64_t>(ctx->n_sms) * std::max(ctx->occ_value_wide, 4);
}

// Robots scanned per tile (passed on as the scan CTA width request).
int warps_for(int n_scan) { return n_scan < 1 ? 1 : n_scan; }

int64_t chunks_for(const pp::DevParams& P) {
  const int64_t n_cells = static_cast<int64_t>(P.n_kt) * P.n_dirs * P.n_pows;
  return (n_cells + pp::kChunk - 1) / pp::kChunk;
}

// Queue + counters + partials for `n_frames` frames of this grid shape.
cudaError_t reserve_pipeline(pp_ctx* ctx, const pp::DevParams& P, int64_t n_frames) {
  const int64_t n_cells = static_cast<int64_t>(P.n_kt) * P.n_dirs * P.n_pows;
  const size_t n = static_cast<size_t>(n_frames * n_cells);
  cudaError_t e = ctx->queue.reserve(ctx->stream, n * (4 * sizeof(double) + sizeof(int32_t) + 1) + 64);
  if (e != cudaSuccess) return e;
  e = ctx->fcount.reserve(ctx->stream, sizeof(pp::FrameCounters) * static_cast<size_t>(n_frames));
  if (e != cudaSuccess) return e;
  return ctx->partials.reserve(ctx->stream, sizeof(pp::Partial) * static_cast<size_t>(n_frames * chunks_for(P)));
}



pp::CellQueue make_queue(pp_ctx* ctx, const pp::DevParams& P, int64_t n_frames) {
  const int64_t n_cells = static_cast<int64_t>(P.n_kt) * P.n_dirs * P.n_pows;
  const size_t n = static_cast<size_t>(n_frames * n_cells);
  char* b = static_cast<char*>(ctx->queue.p);
  pp::CellQueue q;
  q.rx = reinterpret_cast<double*>(b);
  q.ry = q.rx + n;
  q.ot = q.ry + n;
  q.pt = q.ot + n;
  q.cell = reinterpret_cast<int32_t*>(q.pt + n);
  q.slot = reinterpret_cast<int8_t*>(q.cell + n);
  q.cap = n_cells;
  return q;
}

// scan_kernel -> value_kernel for `n_frames` frames (buffers reserved).
// fa: the single frame as a kernel parameter (P.frame_in_arg), else unused.
template <bool kCells>
cudaError_t launch_pipeline(pp_ctx* ctx, const pp::FrameDev* frames, int64_t n_frames,
                            const pp::DevParams& P, int scan_threads, const pp::CellOut& co,
                            pp_dpps_summary* sums, cudaEvent_t mid = nullptr,
                            const pp::FrameArg* fa = nullptr, PipeRec* rec = nullptr) {
  static const pp::FrameArg kNoArg{};
  const pp::FrameArg& arg = fa ? *fa : kNoArg;
  const int n_scan = scan_threads / 32;
  const int64_t ctas = n_frames * P.n_tiles;
  const pp::CellQueue q = make_queue(ctx, P, n_frames);
  auto* fc = static_cast<pp::FrameCounters*>(ctx->fcount.p);
  const int64_t chunks = chunks_for(P);
  auto* parts = static_cast<pp::Partial*>(ctx->partials.p);
  static const int force_shape = [] {  // dev: PP_SCAN_SHAPE=w|m|n
    const char* e = getenv("PP_SCAN_SHAPE");
    return e ? (e[0] == 'n' ? 2 : e[0] == 'w' ? 1 : e[0] == 'm' ? 3 : 0) : 0;
  }();
  ScanFn sfn;
  int w;
  const int64_t sms = ctx->n_sms;
  if (force_shape == 2 || (force_shape == 0 && ctas >= 2 * sms * ctx->occ_scan_narrow)) {
    // Throughput (>= 2 waves of the narrow shape): 4-warp CTAs, 8 per SM,
    // robots round-robin over the warps.
    w = n_scan < pp::kScanWarpsNarrow ? n_scan : pp::kScanWarpsNarrow;
    sfn = pp::scan_kernel<kCells, pp::kScanWarpsNarrow, pp::kScanCtasNarrow>;
  } else if (force_shape == 3 || (force_shape == 0 && ctas > sms * ctx->occ_scan_wide)) {
    // More tiles than one wave of the wide shape: 8-warp CTAs, 4 per SM
    // (one wave up to 592 tiles), robots two per warp, same leftover rounds.
    w = n_scan < pp::kScanWarpsMid ? n_scan : pp::kScanWarpsMid;
    sfn = pp::scan_kernel<kCells, pp::kScanWarpsMid, pp::kScanCtasMid, true>;
  } else {
    // Latency: 16-warp CTAs, one robot per warp.
    w = n_scan < pp::kScanWarpsWide ? n_scan : pp::kScanWarpsWide;
    sfn = pp::scan_kernel<kCells, pp::kScanWarpsWide, pp::kScanCtasWide>;
  }
  cudaLaunchConfig_t scfg{};
  scfg.gridDim = dim3(static_cast<unsigned>(ctas));
  scfg.blockDim = dim3(32 * w);
  scfg.stream = ctx->stream;
  // Batches (the throughput shape): a warp per tile (scan_warp_kernel),
  // ~warp_tiles tiles per CTA.  Not for a single multi-wave frame (the 1 cm
  // grid): there it is no faster, and with the result block in pinned host
  // memory the later, burstier tile completions cost (C3 1.48 -> 1.71 ms).
  // Dev knobs: PP_WARP_TILES=n (0: the 4-warp tile CTAs of scan_kernel),
  // PP_WARP_CELLS=1 (single frames too).
  static const int warp_tiles = [] {
    const char* e = getenv("PP_WARP_TILES");
    return e ? atoi(e) : 128;
  }();
  static const bool warp_cells = [] {
    const char* e = getenv("PP_WARP_CELLS");
    return e ? atoi(e) != 0 : false;
  }();
  pp::DevParams Ps = P;
  if (!kCells) {
    // the cross caps of every sample index a hit can have (batches)
    const std::vector<double> xkey = {P.dt, P.safety, double(ctx->max_count)};
    if (xkey != ctx->xcap_key && ctx->max_count > 0) {
      cudaError_t xe = ctx->xcap.reserve(ctx->stream, sizeof(int32_t) * ctx->max_count);
      if (xe != cudaSuccess) return xe;
      pp::xcap_table_kernel<<<(ctx->max_count + 255) / 256, 256, 0, ctx->stream>>>(
          P, static_cast<int32_t*>(ctx->xcap.p), ctx->max_count);
      xe = cudaGetLastError();
      if (xe != cudaSuccess) return xe;
      ctx->xcap_key = xkey;
    }
    if (ctx->xcap_key == xkey) {
      Ps.xcap = static_cast<const int32_t*>(ctx->xcap.p);
      Ps.n_xcap = ctx->max_count;
    }
  }
  if (warp_tiles > 0 && (!kCells || warp_cells) &&
      sfn == pp::scan_kernel<kCells, pp::kScanWarpsNarrow, pp::kScanCtasNarrow>) {
    // ~warp_tiles tiles per CTA (C5, 65,536 frames: 32 -> 350.6 ms, 64 ->
    // 344.2, 128 -> 342.7, 256 -> 344.9), but at least ~8 waves of CTAs
    // for smaller batches, and at least one tile per warp
    const int64_t want = (8 * sms * pp::kScanWarpCtas + n_frames - 1) / n_frames;
    int64_t groups = std::max<int64_t>(1, P.n_tiles / warp_tiles);
    groups = std::min<int64_t>(std::max(groups, want),
                               std::max<int64_t>(1, P.n_tiles / pp::kScanWarpWarps));
    Ps.scan_groups = static_cast<int32_t>(groups);
    sfn = pp::scan_warp_kernel<kCells, pp::kScanWarpWarps, pp::kScanWarpCtas>;
    scfg.gridDim = dim3(static_cast<unsigned>(n_frames * Ps.scan_groups));
    scfg.blockDim = dim3(32 * pp::kScanWarpWarps);
  }
  cudaError_t e = cudaLaunchKernelEx(&scfg, sfn, frames, Ps, co, q, fc, arg);
  if (e != cudaSuccess) return e;
  if (mid) cudaEventRecord(mid, ctx->stream);
  if (!kCells) {
    // batches: the per-frame score lower bounds the value grid prunes with
    // (timed with the value grid)
    pp::score_lb_kernel<<<static_cast<unsigned>((n_frames * 32 + 255) / 256), 256, 0,
                          ctx->stream>>>(frames, P, q, fc, n_frames);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  // Few chunks (one frame): wider CTAs shorten each chunk's chain of
  // dependent items; many chunks: narrower CTAs pack the SMs better.
  const unsigned vctas = static_cast<unsigned>(n_frames * chunks);
  // Programmatic dependent launch: the value grid is launched while the scan
  // grid drains and waits on it in-kernel.
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(vctas);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = ctx->stream;
  cfg.attrs = attr;
  cfg.numAttrs = mid ? 0 : 1;  // (kernel timing splits the two grids)
  const int nch = static_cast<int>(chunks);
  const bool wide = static_cast<int64_t>(vctas) <= value_wide_limit(ctx);
  // Batches: a few CTAs per frame, each looping over the frame's chunks (most
  // of a frame's chunks are empty: C5 frames fill ~45 of 256), instead of a
  // CTA per chunk.  Single frames: one CTA per chunk (streaming).
  // (at least ~2 waves of CTAs over the whole launch: a single huge frame,
  // e.g. a 1 cm grid, still gets a CTA per few chunks)
  const int64_t min_per_frame = (2 * 8 * static_cast<int64_t>(ctx->n_sms) + n_frames - 1) / n_frames;
  const int per_frame =
      wide ? nch
           : static_cast<int>(std::min<int64_t>(
                 nch, std::max<int64_t>(kValueCtasPerFrame, min_per_frame)));
  cfg.gridDim = dim3(static_cast<unsigned>(n_frames * per_frame));
  const ValueFn vfn = wide ? pp::value_kernel<kCells, pp::kValueThreadsWide>
                           : pp::value_kernel<kCells, pp::kValueThreads>;
  cfg.blockDim = dim3(wide ? pp::kValueThreadsWide : pp::kValueThreads);
  if (rec)
    *rec = PipeRec{frames, Ps, co, q, fc, parts, sums, nch, per_frame, sfn, vfn,
                   scfg.gridDim, scfg.blockDim, cfg.gridDim, cfg.blockDim};
  return cudaLaunchKernelEx(&cfg, vfn, frames, P, q, fc, co, parts, sums, nch, per_frame,
                            arg.frame);
}


// The single-frame launch of the last pp_dpps call.
cudaError_t launch_single(pp_ctx* ctx, cudaEvent_t mid = nullptr) {
  return launch_pipeline<true>(ctx, static_cast<const pp::FrameDev*>(ctx->frame.p), 1,
                               ctx->last_P, ctx->last_threads, ctx->last_co, ctx->last_dsum, mid,
                               ctx->last_fa.get());
}

}  // namespace


// Dev-only host stage timing of pp_dpps (PP_HOST_TRACE=1): mean microseconds
// between stages, printed to stderr every 1000 calls.
static bool g_ht_on = std::getenv("PP_HOST_TRACE") != nullptr;
static double g_ht_acc[8];
static std::chrono::steady_clock::time_point g_ht_last;
static int g_ht_n = 0;
#define HT(k)                                                                   \
  if (g_ht_on) {                                                                \
    const auto now_ = std::chrono::steady_clock::now();                         \
    if (k > 0) g_ht_acc[k] += std::chrono::duration<double, std::micro>(now_ - g_ht_last).count(); \
    g_ht_last = now_;                                                           \
  }
static void ht_flush() {
  if (!g_ht_on || ++g_ht_n < 200) return;
  std::fprintf(stderr, "pp_dpps host stages (us):");
  for (int i = 1; i < 7; ++i) std::fprintf(stderr, " %.2f", g_ht_acc[i] / g_ht_n);
  std::fprintf(stderr, "\n");
  for (double& a : g_ht_acc) a = 0.0;
  g_ht_n = 0;
}

extern "C" {

int pp_abi_version(void) { return PP_ABI_VERSION; }

size_t pp_dpps_upload_bytes(void) { return sizeof(pp::FrameArg) + sizeof(pp::FrameDev); }

void* pp_ctx_stream(pp_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

pp_status pp_dpps_relaunch(pp_ctx* ctx) {
  if (!ctx || !ctx->last_valid) return fail(ctx, PP_INTERNAL, "no previous pp_dpps launch");
  PP_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  PP_CUDA_TRY(ctx, launch_single(ctx));
  return PP_OK;
}

pp_status pp_dpps_kernel_times(pp_ctx* ctx, int32_t reps, float* scan_ms, float* value_ms) {
  if (!ctx || !ctx->last_valid || reps < 1) return fail(ctx, PP_INTERNAL, "no previous pp_dpps launch");
  PP_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  double a = 0.0, b = 0.0;
  for (int i = 0; i < reps; ++i) {
    PP_CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
    PP_CUDA_TRY(ctx, launch_single(ctx, ctx->evm));
    PP_CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
    PP_CUDA_TRY(ctx, cudaEventSynchronize(ctx->ev1));
    float x = 0.f, y = 0.f;
    cudaEventElapsedTime(&x, ctx->ev0, ctx->evm);
    cudaEventElapsedTime(&y, ctx->evm, ctx->ev1);
    a += x;
    b += y;
  }
  if (scan_ms) *scan_ms = static_cast<float>(a / reps);
  if (value_ms) *value_ms = static_cast<float>(b / reps);
  return PP_OK;
}
const char* pp_kernel_name(void) { return "sm100a"; }

void pp_params_default(pp_params* p) {
  std::memset(p, 0, sizeof(*p));
  p->ball = {3.4, 0.5, 5.0 / 7.0, 1.0, 6.5, 0.5};
  p->motion_ours = {3.25, 3.0, 3.0};
  p->motion_theirs = {3.25, 3.0, 3.0};
  p->grid = {128, 64, 1.0, 6.5, 1, 1};
  p->pass_weights = {1.0, 2.0, 1.0, 0.5, 1.0};
  p->run_weights = {1.0, 0.3, 1.0, 0.3, 0.5};
  p->norm = {0.0, kPi};
  p->angle_band = {0.0, 15.0 * kPi / 180.0, 45.0 * kPi / 180.0, 90.0 * kPi / 180.0};
  p->thresholds = {1.0 / 60.0, 0.09, 0.3, 0.3, 0.15, 0.1, 0.0, 10.0,
                   1e-3,       1e-3, 0.1, 1.0, 10.0, 1.0, 0.6};
}

pp_status pp_params_validate(const pp_params* params, char* msg, size_t msg_len) {
  std::string why;
  if (!params) {
    put(msg, msg_len, "null params");
    return PP_INTERNAL;
  }
  if (!validate_params(*params, &why)) {
    put(msg, msg_len, why);
    return PP_CONFIG;
  }
  return PP_OK;
}

size_t pp_grid_bytes(int64_t n_cells) { return pp_grid_offsets_for_(n_cells).total; }
void pp_grid_view_of(void* block, int64_t n_cells, pp_grid_view* out) {
  pp_grid_view_of_(block, n_cells, out);
}
size_t pp_runmap_bytes(int64_t n_vertices) { return pp_runmap_offsets_for_(n_vertices).total; }
void pp_runmap_view_of(void* block, int64_t n_vertices, pp_runmap_view* out) {
  pp_runmap_view_of_(block, n_vertices, out);
}

int64_t pp_grid_cells(const pp_search_grid* g) {
  if (!g || g->n_directions < 1 || g->n_powers < 1) return 0;
  return static_cast<int64_t>((g->flat ? 1 : 0) + (g->chip ? 1 : 0)) * g->n_directions *
         g->n_powers;
}

void* pp_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) return nullptr;
  return p;
}
void pp_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

pp_status pp_ctx_create(int device, pp_ctx** out) {
  if (!out) return PP_INTERNAL;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count <= device || device < 0)
    return PP_CUDA;
  if (cudaSetDevice(device) != cudaSuccess) return PP_CUDA;
  // every early return below releases what was acquired (~pp_ctx)
  std::unique_ptr<pp_ctx> ctx(new pp_ctx());
  ctx->device = device;
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess)
    return PP_CUDA;
  if (cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess ||
      cudaEventCreate(&ctx->evm) != cudaSuccess)
    return PP_CUDA;
  if (cudaDeviceGetAttribute(&ctx->n_sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess ||
      ctx->n_sms < 1)
    return PP_CUDA;
  if (query_occupancy(ctx.get()) != cudaSuccess) return PP_CUDA;
  if (ctx->frame.reserve(ctx->stream, kFrameBytes) != cudaSuccess) return PP_CUDA;
  if (ctx->frame_h.reserve(kFrameBytes) != cudaSuccess) return PP_CUDA;
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return PP_CUDA;
  if (const char* e = std::getenv("PP_EXACT_ONLY")) ctx->exact_only = std::atoi(e) != 0;
  *out = ctx.release();
  return PP_OK;
}

void pp_ctx_destroy(pp_ctx* ctx) { delete ctx; }

pp_status pp_ctx_set_option(pp_ctx* ctx, int32_t option, int32_t value) {
  if (!ctx) return PP_INTERNAL;
  switch (option) {
    case PP_OPT_EXACT_ONLY:
      ctx->exact_only = value != 0;
      ctx->last_valid = false;  // (pp_dpps_relaunch would replay the old setting)
      return PP_OK;
    default:
      return fail(ctx, PP_CONFIG, "unknown context option %d", option);
  }
}

const char* pp_last_error(const pp_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

pp_status pp_dpps(pp_ctx* ctx, const pp_world* world, const pp_params* params,
                  const pp_search_grid* grid_in, int32_t kicker_id, uint32_t copy_flags,
                  void* block) {
  PP_NVTX("pp_dpps");
  if (!ctx || !world || !params || !block) return fail(ctx, PP_INTERNAL, "null argument");
  HT(0);
  ctx->err.clear();
  const pp_search_grid& g = grid_in ? *grid_in : params->grid;
  std::string why;
  if (!validate_grid(g, &why)) return fail(ctx, PP_CONFIG, "%s", why.c_str());
  if (!validate_params(*params, &why)) return fail(ctx, PP_CONFIG, "%s", why.c_str());
  PP_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  pp::FrameDev* F = static_cast<pp::FrameDev*>(ctx->frame_h.p);
  int32_t kicker_slot = -1;
  if (!pack_frame(*world, kicker_id, F, &kicker_slot, &why))
    return fail(ctx, PP_VALIDATION, "%s", why.c_str());

  HT(1);
  const int64_t n_cells = pp_grid_cells(&g);
  const pp_grid_offsets_ off = pp_grid_offsets_for_(n_cells);
  pp_grid_view hv;
  pp_grid_view_of_(block, n_cells, &hv);
  if (n_cells == 0) {
    std::memset(hv.summary, 0, sizeof(pp_dpps_summary));
    for (int k = 0; k < 3; ++k) hv.summary->best_cell[k] = -1;
    fill_summary_host(hv.summary, *world, g, kicker_id, kicker_slot,
                      possession_of(*world, kicker_id, *params));
    return PP_OK;
  }
  pp::DevParams P = make_dev_params(ctx, *params, g);
  PP_CUDA_TRY(ctx, ensure_tables(ctx, &P));
  // The frame and its robots' filter constants (computed here once, not per
  // tile) travel in the kernels' FrameArg parameter: no host-to-device copy.
  pp::FrameArg* fa = ctx->last_fa.get();
  std::memcpy(&fa->frame, F, sizeof(pp::FrameDev));
  for (int ri = 0; ri < F->n_scan; ++ri) pp::robot_consts(*F, P, ri, &fa->rk[ri]);
  P.frame_in_arg = 1;
  PP_CUDA_TRY(ctx, ctx->block.reserve(ctx->stream, off.total));
  PP_CUDA_TRY(ctx, reserve_pipeline(ctx, P, 1));
  if (chunks_for(P) <= value_wide_limit(ctx)) {  // the value grid's wide (streaming) shape
    PP_CUDA_TRY(ctx, ctx->chunk_fill.reserve(ctx->stream, sizeof(unsigned) * static_cast<size_t>(chunks_for(P))));
    P.chunk_fill = static_cast<unsigned*>(ctx->chunk_fill.p);
  }
  HT(2);

  char* dblk = static_cast<char*>(ctx->block.p);
  pp::CellOut co;
  co.our_time = reinterpret_cast<double*>(dblk + off.our_time);
  co.opp_time = reinterpret_cast<double*>(dblk + off.opp_time);
  co.rx = reinterpret_cast<double*>(dblk + off.rx);
  co.ry = reinterpret_cast<double*>(dblk + off.ry);
  co.score = reinterpret_cast<float*>(dblk + off.score);
  co.our_slot = reinterpret_cast<int8_t*>(dblk + off.our_slot);
  co.opp_slot = reinterpret_cast<int8_t*>(dblk + off.opp_slot);
  co.feasible = reinterpret_cast<uint8_t*>(dblk + off.feasible);
  pp_dpps_summary* dsum = reinterpret_cast<pp_dpps_summary*>(dblk + off.summary);

  cudaStream_t s = ctx->stream;
  ctx->last_P = P;
  ctx->last_co = co;
  ctx->last_dsum = dsum;
  ctx->last_threads = 32 * warps_for(F->n_scan);
  ctx->last_valid = true;
  const bool all = (copy_flags & PP_COPY_ALL) != 0;
  char* hblk = static_cast<char*>(block);
  // A pinned block (pp_host_alloc) is device-addressable: the kernels then
  // write the per-cell outputs, the scores and the summary straight into it
  // over PCIe while they run, and the call has no device-to-host copy.
  bool pinned = false;
  {
    cudaPointerAttributes pa{};
    pinned = cudaPointerGetAttributes(&pa, block) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
             pa.devicePointer == block;
    cudaGetLastError();
  }
  const bool direct = all && pinned;
  pp::CellOut co_run = co;
  // a pinned block also takes the summary straight from the fold
  pp_dpps_summary* sum_run = pinned ? reinterpret_cast<pp_dpps_summary*>(block) : dsum;
  if (direct) {
    co_run.score = reinterpret_cast<float*>(hblk + off.score);
    co_run.our_time = reinterpret_cast<double*>(hblk + off.our_time);
    co_run.opp_time = reinterpret_cast<double*>(hblk + off.opp_time);
    co_run.rx = reinterpret_cast<double*>(hblk + off.rx);
    co_run.ry = reinterpret_cast<double*>(hblk + off.ry);
    co_run.our_slot = reinterpret_cast<int8_t*>(hblk + off.our_slot);
    co_run.opp_slot = reinterpret_cast<int8_t*>(hblk + off.opp_slot);
    co_run.feasible = reinterpret_cast<uint8_t*>(hblk + off.feasible);
  }
  HT(3);
  // (summary.device_ms is the kernels' own span, measured on the device)
  auto enqueue = [&]() -> cudaError_t {
    // (only a graph capture records its launch: the cached graph's node
    // updates read ctx->rec, which a plain pageable launch must not clobber)
    cudaError_t e = launch_pipeline<true>(ctx, static_cast<const pp::FrameDev*>(ctx->frame.p), 1,
                                          P, ctx->last_threads, co_run, sum_run, nullptr, fa,
                                          pinned ? &ctx->rec : nullptr);
    if (e == cudaSuccess && !pinned)
      e = cudaMemcpyAsync(block, dblk, sizeof(pp_dpps_summary), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && all && !direct)
      e = cudaMemcpyAsync(hblk + off.our_time, dblk + off.our_time, off.total - off.our_time,
                          cudaMemcpyDeviceToHost, s);
    return e;
  };
  if (!pinned) {  // pageable block: plain stream work (graphs copy pinned memory only)
    // fold sentinel: the final fold overwrites device_ms (NaN bytes until then)
    PP_PIPE_TRY(ctx, cudaMemsetAsync(&dsum->device_ms, 0xFF, sizeof(double), s));
    PP_PIPE_TRY(ctx, enqueue());
    PP_PIPE_TRY(ctx, cudaStreamSynchronize(s));
  } else {
  // The whole call is one graph: scan -> value (D2H only for pageable
  // blocks, which take the plain path above).
  struct Key {
    pp::DevParams P;
    pp::CellOut co;
    const void* block;
    const void* dblk;
    const void* bufs[4];  // pipeline buffers baked into the graph
    int64_t n_cells;
    uint32_t flags;
    int32_t threads, direct;
  } key;
  std::memset(&key, 0, sizeof(key));
  key.P = P;
  key.co = co_run;
  key.block = block;
  key.dblk = dblk;
  key.bufs[0] = ctx->queue.p;
  key.bufs[1] = ctx->fcount.p;
  key.bufs[2] = ctx->partials.p;
  key.bufs[3] = ctx->frame.p;
  key.n_cells = n_cells;
  key.flags = copy_flags;
  key.threads = ctx->last_threads;
  key.direct = direct;
  const unsigned char* kb = reinterpret_cast<const unsigned char*>(&key);
  if (!ctx->gexec || ctx->gkey.size() != sizeof(key) ||
      std::memcmp(ctx->gkey.data(), kb, sizeof(key)) != 0) {
    if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
    if (ctx->graph) cudaGraphDestroy(ctx->graph);
    ctx->gexec = nullptr;
    ctx->graph = nullptr;
    ctx->scan_node = ctx->value_node = nullptr;
    ctx->gkey.clear();
    PP_CUDA_TRY(ctx, cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    cudaError_t e = enqueue();
    const cudaError_t e2 = cudaStreamEndCapture(s, &ctx->graph);
    if (e == cudaSuccess) e = e2;
    if (e == cudaSuccess) e = cudaGraphInstantiate(&ctx->gexec, ctx->graph, 0);
    if (e == cudaSuccess) {  // the two kernel nodes whose FrameArg each call rewrites
      size_t n = 0;
      cudaGraphGetNodes(ctx->graph, nullptr, &n);
      std::vector<cudaGraphNode_t> nodes(n);
      e = cudaGraphGetNodes(ctx->graph, nodes.data(), &n);
      for (size_t i = 0; e == cudaSuccess && i < n; ++i) {
        cudaGraphNodeType t;
        cudaGraphNodeGetType(nodes[i], &t);
        if (t != cudaGraphNodeTypeKernel) continue;
        cudaKernelNodeParams kp{};
        e = cudaGraphKernelNodeGetParams(nodes[i], &kp);
        if (kp.func == reinterpret_cast<void*>(ctx->rec.scan_fn)) ctx->scan_node = nodes[i];
        if (kp.func == reinterpret_cast<void*>(ctx->rec.value_fn)) ctx->value_node = nodes[i];
      }
      if (e == cudaSuccess && (!ctx->scan_node || !ctx->value_node)) e = cudaErrorInvalidValue;
    }
    PP_PIPE_TRY(ctx, e);
    ctx->gkey.assign(kb, kb + sizeof(key));
  } else {
    // same graph: only this frame's FrameArg changes
    PipeRec& r = ctx->rec;
    void* sargs[] = {&r.frames, &r.P, &r.co, &r.q, &r.fc, fa};
    cudaKernelNodeParams kp{};
    kp.func = reinterpret_cast<void*>(r.scan_fn);
    kp.gridDim = r.sgrid;
    kp.blockDim = r.sblock;
    kp.kernelParams = sargs;
    PP_CUDA_TRY(ctx, cudaGraphExecKernelNodeSetParams(ctx->gexec, ctx->scan_node, &kp));
    void* vargs[] = {&r.frames, &r.P, &r.q, &r.fc, &r.co, &r.parts, &r.sums, &r.nch,
                     &r.per_frame, &fa->frame};
    kp.func = reinterpret_cast<void*>(r.value_fn);
    kp.gridDim = r.vgrid;
    kp.blockDim = r.vblock;
    kp.kernelParams = vargs;
    PP_CUDA_TRY(ctx, cudaGraphExecKernelNodeSetParams(ctx->gexec, ctx->value_node, &kp));
  }
  HT(4);
  hv.summary->device_ms = std::numeric_limits<double>::quiet_NaN();  // fold sentinel
  PP_PIPE_TRY(ctx, cudaGraphLaunch(ctx->gexec, s));
  PP_PIPE_TRY(ctx, cudaStreamSynchronize(s));
  }
  HT(5);
  const double dms = hv.summary->device_ms;
  if (std::isnan(dms)) {  // a streaming wait gave up: no fold ran
    reset_pipeline(ctx);
    return fail(ctx, PP_INTERNAL, "scan->value pipeline stalled (no fold); counters reset");
  }
  fill_summary_host(hv.summary, *world, g, kicker_id, kicker_slot,
                    possession_of(*world, kicker_id, *params));
  hv.summary->device_ms = dms;
  HT(6);
  ht_flush();
  return PP_OK;
}

pp_status pp_score_cells(pp_ctx* ctx, const pp_world* world, const pp_params* params, int64_t n,
                         const double* rx, const double* ry, const double* our_time,
                         const double* opp_time, const uint8_t* feasible, double* score_out,
                         pp_pass_features* features_out) {
  PP_NVTX("pp_score_cells");
  if (!ctx || !world || !params) return fail(ctx, PP_INTERNAL, "null argument");
  ctx->err.clear();
  for (int64_t i = 0; i < n; ++i)
    if (!feasible[i]) return fail(ctx, PP_DOMAIN, "score_pass: candidate is not feasible");
  if (n == 0) return PP_OK;
  std::string why;
  if (!validate_params(*params, &why)) return fail(ctx, PP_CONFIG, "%s", why.c_str());
  PP_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  pp::FrameDev* F = static_cast<pp::FrameDev*>(ctx->frame_h.p);
  int32_t ks = -1;
  pp_world w = *world;
  if (w.n_ours == 0) {  // score_pass needs no kicker; stage a placeholder
    w.n_ours = 1;
    w.ours[0] = pp_robot{0, 0, 0, 0, 0, 0, 0};
  }
  if (!pack_frame(w, w.ours[0].id, F, &ks, &why)) return fail(ctx, PP_VALIDATION, "%s", why.c_str());
  const pp::DevParams P = make_dev_params(ctx, *params, params->grid);
  std::vector<double> in(4 * static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    in[4 * i] = rx[i];
    in[4 * i + 1] = ry[i];
    in[4 * i + 2] = our_time[i];
    in[4 * i + 3] = opp_time[i];
  }
  PP_CUDA_TRY(ctx, ctx->scratch_in.reserve(ctx->stream, in.size() * 8));
  PP_CUDA_TRY(ctx, ctx->scratch_out.reserve(ctx->stream, 6 * static_cast<size_t>(n) * 8));
  cudaStream_t s = ctx->stream;
  PP_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->frame.p, F, sizeof(pp::FrameDev), cudaMemcpyHostToDevice, s));
  PP_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->scratch_in.p, in.data(), in.size() * 8, cudaMemcpyHostToDevice, s));
  const int blocks = static_cast<int>((n + 255) / 256);
  pp::score_cells_kernel<<<blocks, 256, 0, s>>>(static_cast<const pp::FrameDev*>(ctx->frame.p), P,
                                                n, static_cast<const double*>(ctx->scratch_in.p),
                                                static_cast<double*>(ctx->scratch_out.p));
  PP_CUDA_TRY(ctx, cudaGetLastError());
  std::vector<double> o(6 * static_cast<size_t>(n));
  PP_CUDA_TRY(ctx, cudaMemcpyAsync(o.data(), ctx->scratch_out.p, o.size() * 8, cudaMemcpyDeviceToHost, s));
  PP_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  for (int64_t i = 0; i < n; ++i) {
    score_out[i] = o[6 * i];
    if (features_out)
      features_out[i] = pp_pass_features{o[6 * i + 1], o[6 * i + 2], o[6 * i + 3], o[6 * i + 4],
                                         o[6 * i + 5]};
  }
  return PP_OK;
}

pp_status pp_goal_views(pp_ctx* ctx, const pp_world* world, double robot_radius, int64_t n,
                        const double* px, const double* py, double* angle, double* window_lo,
                        double* window_hi, double* target_y) {
  PP_NVTX("pp_goal_views");
  if (!ctx || !world) return fail(ctx, PP_INTERNAL, "null argument");
  ctx->err.clear();
  if (n == 0) return PP_OK;
  PP_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  pp::FrameDev* F = static_cast<pp::FrameDev*>(ctx->frame_h.p);
  pp_world w = *world;
  if (w.n_ours == 0) {
    w.n_ours = 1;
    w.ours[0] = pp_robot{0, 0, 0, 0, 0, 0, 0};
  }
  int32_t ks = -1;
  std::string why;
  if (!pack_frame(w, w.ours[0].id, F, &ks, &why)) return fail(ctx, PP_VALIDATION, "%s", why.c_str());
  std::vector<double> in(2 * static_cast<size_t>(n));
  std::memcpy(in.data(), px, n * 8);
  std::memcpy(in.data() + n, py, n * 8);
  PP_CUDA_TRY(ctx, ctx->scratch_in.reserve(ctx->stream, in.size() * 8));
  PP_CUDA_TRY(ctx, ctx->scratch_out.reserve(ctx->stream, 4 * static_cast<size_t>(n) * 8));
  cudaStream_t s = ctx->stream;
  PP_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->frame.p, F, sizeof(pp::FrameDev), cudaMemcpyHostToDevice, s));
  PP_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->scratch_in.p, in.data(), in.size() * 8, cudaMemcpyHostToDevice, s));
  const double* dpx = static_cast<const double*>(ctx->scratch_in.p);
  pp::goal_view_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, s>>>(
      static_cast<const pp::FrameDev*>(ctx->frame.p), robot_radius,
      sqrt_lt_threshold(robot_radius), sqrt_le_threshold(robot_radius + 1e-9), n, dpx, dpx + n,
      static_cast<double*>(ctx->scratch_out.p), ctx->exact_only != 0);
  PP_CUDA_TRY(ctx, cudaGetLastError());
  std::vector<double> o(4 * static_cast<size_t>(n));
  PP_CUDA_TRY(ctx, cudaMemcpyAsync(o.data(), ctx->scratch_out.p, o.size() * 8, cudaMemcpyDeviceToHost, s));
  PP_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  for (int64_t i = 0; i < n; ++i) {
    angle[i] = o[4 * i];
    window_lo[i] = o[4 * i + 1];
    window_hi[i] = o[4 * i + 2];
    target_y[i] = o[4 * i + 3];
  }
  return PP_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Running-point map host side (offball.cpp:69-123, 137-174, 215-258).

namespace {

struct HostZone {
  double x0, x1, y0, y1;
};

int axis_count(double span, double step) {
  const int n = static_cast<int>(std::floor(span / step + 1e-9)) + 1;
  return n > 0 ? n : 0;
}

double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

struct RunSetup {
  pp::RunParams R;
  double cut_x, cut_y;
  int64_t n_map;
};

// Frame constants of score_running_point (offball.cpp:176-201), including the
// point-independent parts hoisted per frame: nearest opponent to the ball
// (offball.cpp:188-191) and the guard ranking (offball.cpp:143-155).
void fill_run_common(const pp_world& w, const pp_params& p, pp::RunParams& R) {
  const pp_field& f = w.field;
  R.L = f.length;
  R.W = f.width;
  R.dd = f.defense_depth;
  R.dw = f.defense_width;
  R.gw = f.goal_width;
  R.ball_x = w.ball_px;
  R.ball_y = w.ball_py;
  R.a_t = p.motion_theirs.max_accel;
  R.b_t = p.motion_theirs.max_decel;
  R.vmax_t = p.motion_theirs.max_speed;
  R.cap = p.thresholds.guard_time_cap;
  R.w_dg = p.run_weights.dist_goal;
  R.w_db = p.run_weights.dist_ball;
  R.w_angle = p.run_weights.angle;
  R.w_guard = p.run_weights.guard_time;
  R.w_exp = p.run_weights.exposure;
  R.len_upper = p.norm.length_upper > 0.0 ? p.norm.length_upper : f.length;
  R.band_full_lo = p.angle_band.full_lo;
  R.band_peak_lo = p.angle_band.peak_lo;
  R.band_peak_hi = p.angle_band.peak_hi;
  R.band_full_hi = p.angle_band.full_hi;
  double nearest = std::numeric_limits<double>::infinity();
  for (int i = 0; i < w.n_theirs; ++i) {
    const double d = host_distance(w.theirs[i].px, w.theirs[i].py, w.ball_px, w.ball_py);
    nearest = std::min(nearest, d);
  }
  R.nearest_opp = nearest;
  const double bx0 = 0.5 * f.length - f.defense_depth, bx1 = 0.5 * f.length;
  const double by0 = -0.5 * f.defense_width, by1 = 0.5 * f.defense_width;
  struct Cand {
    double dist;
    int id;
    int idx;
  };
  std::vector<Cand> cands;
  for (int i = 0; i < w.n_theirs; ++i) {
    const pp_robot& r = w.theirs[i];
    const double cx = std::clamp(r.px, bx0, bx1);
    const double cy = std::clamp(r.py, by0, by1);
    cands.push_back({host_distance(r.px, r.py, cx, cy), r.id, i});
  }
  std::sort(cands.begin(), cands.end(), [](const Cand& a, const Cand& b) {
    if (a.dist != b.dist) return a.dist < b.dist;
    return a.id < b.id;
  });
  R.n_guards = static_cast<int32_t>(std::min<size_t>(cands.size(), 2));
  for (int g = 0; g < R.n_guards; ++g) {
    const pp_robot& r = w.theirs[cands[g].idx];
    R.g_px[g] = r.px;
    R.g_py[g] = r.py;
    R.g_vx[g] = r.vx;
    R.g_vy[g] = r.vy;
  }
}

bool setup_runmap(const pp_world& w, const pp_params& p, const pp_runmap_request& req,
                  RunSetup* out, std::string* why) {
  const pp_field& f = w.field;
  const double mzw = p.thresholds.min_zone_width;
  if (!(mzw > 0.0) || 2.0 * mzw > f.width) {
    *why = "min_zone_width must be positive and at most half the field width";
    return false;
  }
  const double step = p.thresholds.grid_step;
  if (!(step > 0.0)) {
    *why = "lattice step must be positive";
    return false;
  }
  pp::RunParams& R = out->R;
  std::memset(&R, 0, sizeof(R));
  const double cut_x = 0.25 * f.length;
  const double cut_y = clampd(w.ball_py, -0.5 * f.width + mzw, 0.5 * f.width - mzw);
  const double x_mid = 0.5 * f.length;
  const double y_top = 0.5 * f.width;
  const HostZone zones[4] = {{0.0, cut_x, cut_y, y_top},
                             {0.0, cut_x, -y_top, cut_y},
                             {cut_x, x_mid, cut_y, y_top},
                             {cut_x, x_mid, -y_top, cut_y}};
  out->cut_x = cut_x;
  out->cut_y = cut_y;
  // Zone selection (offball.cpp:221-233).
  uint32_t excluded = req.occupied_mask;
  if (req.has_best_pass_point) {
    const double px = req.best_pass_px, py = req.best_pass_py;
    const double x_lo = zones[0].x0, x_hi = zones[2].x1, y_lo = zones[1].y0, y_hi = zones[0].y1;
    if (!(px < x_lo || px > x_hi || py < y_lo || py > y_hi)) {
      const int z = px >= cut_x ? (py >= cut_y ? 2 : 3) : (py >= cut_y ? 0 : 1);
      excluded |= 1u << z;
    }
  }
  uint32_t selected = 0;
  int n_sel = 0;
  for (int z : {2, 3, 0, 1}) {
    if (n_sel >= req.n_runners) break;
    if (!(excluded & (1u << z))) {
      selected |= 1u << z;
      ++n_sel;
    }
  }
  int64_t at = 0;
  int max_blocks = 1;
  for (int z = 0; z < 4; ++z) {
    const HostZone& Z = zones[z];
    pp::RunZone& rz = R.zone[z];
    const bool upper = z == 0 || z == 2;
    rz.x0 = Z.x0;
    rz.y0 = upper ? Z.y0 : Z.y1;
    rz.ydir = upper ? 1.0 : -1.0;
    rz.nx = axis_count(Z.x1 - Z.x0, step);
    rz.ny = axis_count(Z.y1 - Z.y0, step);
    rz.selected = (selected >> z) & 1u;
    rz.in_map = (req.zone_mask >> z) & 1u;
    rz.offset = at;
    if (rz.in_map) at += static_cast<int64_t>(rz.nx) * rz.ny;
    const int64_t nv = static_cast<int64_t>(rz.nx) * rz.ny;
    const int b = static_cast<int>((nv + 255) / 256);
    R.blocks_per_zone[z] = (rz.in_map || rz.selected) ? b : 0;
    if (R.blocks_per_zone[z] > max_blocks) max_blocks = R.blocks_per_zone[z];
  }
  out->n_map = at;
  R.step = step;
  fill_run_common(w, p, R);
  (void)max_blocks;
  return true;
}

}  // namespace

extern "C" {

pp_status pp_runmap_count(const pp_world* world, const pp_params* params, uint32_t zone_mask,
                          int64_t* n_vertices) {
  if (!world || !params || !n_vertices) return PP_INTERNAL;
  pp_runmap_request req{zone_mask, 0, 0, 0, 0.0, 0.0, 1};
  RunSetup rs;
  std::string why;
  if (!setup_runmap(*world, *params, req, &rs, &why)) return PP_CONFIG;
  *n_vertices = rs.n_map;
  return PP_OK;
}

pp_status pp_runmap(pp_ctx* ctx, const pp_world* world, const pp_params* params,
                    const pp_runmap_request* req, void* block, int64_t block_vertices) {
  PP_NVTX("pp_runmap");
  if (!ctx || !world || !params || !req || !block) return fail(ctx, PP_INTERNAL, "null argument");
  ctx->err.clear();
  std::string why;
  if (!validate_params(*params, &why)) return fail(ctx, PP_CONFIG, "%s", why.c_str());
  RunSetup rs;
  if (!setup_runmap(*world, *params, *req, &rs, &why)) return fail(ctx, PP_CONFIG, "%s", why.c_str());
  const bool want_map = req->want_map != 0;
  const int64_t n_map = want_map ? rs.n_map : 0;
  if (want_map && block_vertices < rs.n_map)
    return fail(ctx, PP_INTERNAL, "runmap block holds %lld vertices, need %lld",
                static_cast<long long>(block_vertices), static_cast<long long>(rs.n_map));
  PP_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const pp_runmap_offsets_ off = pp_runmap_offsets_for_(n_map);
  PP_CUDA_TRY(ctx, ctx->run_block.reserve(ctx->stream, off.total));
  int max_blocks = 1;
  for (int z = 0; z < 4; ++z) max_blocks = std::max(max_blocks, rs.R.blocks_per_zone[z]);
  PP_CUDA_TRY(ctx, ctx->run_partials.reserve(ctx->stream, sizeof(pp::RunPartial) * 4 * max_blocks));
  PP_CUDA_TRY(ctx, ctx->run_counter.reserve(ctx->stream, sizeof(unsigned) * 4));  // done count, pad, u64 scorable
  // (the map is written in device memory and copied in one DMA transfer:
  // tens of MB of per-thread stores straight into host memory are slower)
  char* d = static_cast<char*>(ctx->run_block.p);
  pp::RunOut ro;
  ro.px = reinterpret_cast<double*>(d + off.px);
  ro.py = reinterpret_cast<double*>(d + off.py);
  ro.score = reinterpret_cast<double*>(d + off.score);
  ro.features = reinterpret_cast<pp_run_features*>(d + off.features);
  ro.scorable = reinterpret_cast<uint8_t*>(d + off.scorable);
  pp_runmap_summary* dsum = reinterpret_cast<pp_runmap_summary*>(d + off.summary);
  cudaStream_t s = ctx->stream;
  const dim3 grid(max_blocks, 4);
  if (want_map) {
    pp::runmap_kernel<true><<<grid, 256, 0, s>>>(rs.R, ro,
                                                 static_cast<pp::RunPartial*>(ctx->run_partials.p),
                                                 static_cast<unsigned*>(ctx->run_counter.p), dsum);
  } else {
    pp::runmap_kernel<false><<<grid, 256, 0, s>>>(rs.R, ro,
                                                  static_cast<pp::RunPartial*>(ctx->run_partials.p),
                                                  static_cast<unsigned*>(ctx->run_counter.p), dsum);
  }
  PP_CUDA_TRY(ctx, cudaGetLastError());
  const size_t bytes = want_map ? off.total : sizeof(pp_runmap_summary);
  PP_CUDA_TRY(ctx, cudaMemcpyAsync(block, d, bytes, cudaMemcpyDeviceToHost, s));
  PP_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  pp_runmap_view v;
  pp_runmap_view_of_(block, n_map, &v);
  pp_runmap_summary& S = *v.summary;
  S.cut_x = rs.cut_x;
  S.cut_y = rs.cut_y;
  S.n_vertices = n_map;  // (n_scorable: counted by the kernel)
  for (int z = 0; z < 4; ++z) {
    const bool in_map = (req->zone_mask >> z) & 1u;
    S.zone_nx[z] = in_map ? rs.R.zone[z].nx : 0;
    S.zone_ny[z] = in_map ? rs.R.zone[z].ny : 0;
    S.zone_offset[z] = rs.R.zone[z].offset;
  }
  S.n_best = 0;
  for (int z = 0; z < 4; ++z) {
    S.best_order[z] = -1;
    if (S.best[z].valid) S.best_order[S.n_best++] = z;
  }
  return PP_OK;
}

pp_status pp_score_running_points(pp_ctx* ctx, const pp_world* world, const pp_params* params,
                                  int64_t n, const double* px, const double* py,
                                  double* score_out, pp_run_features* features_out,
                                  uint8_t* ok_out) {
  PP_NVTX("pp_score_running_points");
  if (!ctx || !world || !params) return fail(ctx, PP_INTERNAL, "null argument");
  ctx->err.clear();
  std::string why;
  if (!validate_params(*params, &why)) return fail(ctx, PP_CONFIG, "%s", why.c_str());
  if (n == 0) return PP_OK;
  PP_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  pp::RunParams R;
  std::memset(&R, 0, sizeof(R));
  fill_run_common(*world, *params, R);
  std::vector<double> in(2 * static_cast<size_t>(n));
  std::memcpy(in.data(), px, n * 8);
  std::memcpy(in.data() + n, py, n * 8);
  PP_CUDA_TRY(ctx, ctx->scratch_in.reserve(ctx->stream, in.size() * 8));
  PP_CUDA_TRY(ctx, ctx->scratch_out.reserve(ctx->stream, 7 * static_cast<size_t>(n) * 8));
  cudaStream_t s = ctx->stream;
  PP_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->scratch_in.p, in.data(), in.size() * 8, cudaMemcpyHostToDevice, s));
  const double* d = static_cast<const double*>(ctx->scratch_in.p);
  pp::run_points_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, s>>>(
      R, n, d, d + n, static_cast<double*>(ctx->scratch_out.p));
  PP_CUDA_TRY(ctx, cudaGetLastError());
  std::vector<double> o(7 * static_cast<size_t>(n));
  PP_CUDA_TRY(ctx, cudaMemcpyAsync(o.data(), ctx->scratch_out.p, o.size() * 8, cudaMemcpyDeviceToHost, s));
  PP_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  for (int64_t i = 0; i < n; ++i) {
    if (ok_out) ok_out[i] = o[7 * i] != 0.0;
    if (score_out) score_out[i] = o[7 * i + 1];
    if (features_out)
      features_out[i] = pp_run_features{o[7 * i + 2], o[7 * i + 3], o[7 * i + 4], o[7 * i + 5],
                                        o[7 * i + 6]};
  }
  return PP_OK;
}

#ifdef PP_SCAN_STATS
// Dev variant only (not in the header): read and optionally reset the scan
// filter statistics (pp_scan.cuh g_scan_stats).
void pp_debug_scan_stats(unsigned long long* out16, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out16, pp::g_scan_stats, 64 * sizeof(unsigned long long));
  if (reset) {
    unsigned long long z[64] = {};
    cudaMemcpyToSymbol(pp::g_scan_stats, z, sizeof(z));
  }
}
void pp_debug_act_hist(unsigned long long* out33, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out33, pp::g_act_hist, 33 * sizeof(unsigned long long));
  if (reset) {
    unsigned long long z[33] = {};
    cudaMemcpyToSymbol(pp::g_act_hist, z, sizeof(z));
  }
}
#endif

pp_status pp_scan_first(pp_ctx* ctx, int64_t n, const pp_scan_batch* batches,
                        const pp_robot_kin* kins, int32_t* first_k) {
  PP_NVTX("pp_scan_first");
  if (!ctx || (n > 0 && (!batches || !kins || !first_k)) || n < 0)
    return fail(ctx, PP_INTERNAL, "null argument");
  ctx->err.clear();
  if (n == 0) return PP_OK;
  PP_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  std::vector<pp::ScanPair> pairs(static_cast<size_t>(n));
  std::vector<double> samples;
  for (int64_t i = 0; i < n; ++i) {
    const pp_scan_batch& b = batches[i];
    const pp_robot_kin& r = kins[i];
    pp::ScanPair& q = pairs[static_cast<size_t>(i)];
    q = pp::ScanPair{b.ox, b.oy, b.ux, b.uy, r.px, r.py, r.vx, r.vy, r.accel, r.decel, r.vmax,
                     r.radius, r.vbound, static_cast<int64_t>(samples.size() / 2), b.k_begin,
                     b.k_end};
    if (b.k_end > b.k_begin) {
      if (!b.ts || !b.ss) return fail(ctx, PP_INTERNAL, "null sample arrays");
      for (int32_t k = b.k_begin; k < b.k_end; ++k) {
        samples.push_back(b.ts[k]);
        samples.push_back(b.ss[k]);
      }
    }
  }
  if (samples.empty()) samples.assign(2, 0.0);
  // (samples start 16-byte aligned: they are read as double2)
  const size_t pb = (pairs.size() * sizeof(pp::ScanPair) + 15) / 16 * 16;
  const size_t sb = samples.size() * sizeof(double);
  PP_CUDA_TRY(ctx, ctx->scratch_in.reserve(ctx->stream, pb + sb));
  PP_CUDA_TRY(ctx, ctx->scratch_out.reserve(ctx->stream, static_cast<size_t>(n) * sizeof(int32_t)));
  cudaStream_t s = ctx->stream;
  char* din = static_cast<char*>(ctx->scratch_in.p);
  PP_CUDA_TRY(ctx, cudaMemcpyAsync(din, pairs.data(), pairs.size() * sizeof(pp::ScanPair),
                                   cudaMemcpyHostToDevice, s));
  PP_CUDA_TRY(ctx, cudaMemcpyAsync(din + pb, samples.data(), sb, cudaMemcpyHostToDevice, s));
  const int64_t threads = n * 32;
  pp::scan_first_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(
      reinterpret_cast<const pp::ScanPair*>(din), n, reinterpret_cast<const double2*>(din + pb),
      static_cast<int32_t*>(ctx->scratch_out.p));
  PP_CUDA_TRY(ctx, cudaGetLastError());
  PP_CUDA_TRY(ctx, cudaMemcpyAsync(first_k, ctx->scratch_out.p, static_cast<size_t>(n) * sizeof(int32_t),
                                   cudaMemcpyDeviceToHost, s));
  PP_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  return PP_OK;
}

pp_status pp_guard_points(pp_ctx* ctx, const pp_world* world, const pp_motion_limits* limits,
                          double cap, int64_t n, const double* px, const double* py,
                          double* guard_pq, double* guard_time, uint8_t* ok_out) {
  PP_NVTX("pp_guard_points");
  if (!ctx || !world || !limits) return fail(ctx, PP_INTERNAL, "null argument");
  ctx->err.clear();
  if (!(cap > 0.0) || !std::isfinite(cap))
    return fail(ctx, PP_DOMAIN, "guard time cap must be positive");
  if (n == 0) return PP_OK;
  if (n < 0 || !px || !py) return fail(ctx, PP_INTERNAL, "bad point arrays");
  PP_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  pp_params p;
  pp_params_default(&p);
  p.motion_theirs = *limits;
  p.thresholds.guard_time_cap = cap;
  pp::RunParams R;
  std::memset(&R, 0, sizeof(R));
  fill_run_common(*world, p, R);
  std::vector<double> in(2 * static_cast<size_t>(n));
  std::memcpy(in.data(), px, n * 8);
  std::memcpy(in.data() + n, py, n * 8);
  PP_CUDA_TRY(ctx, ctx->scratch_in.reserve(ctx->stream, in.size() * 8));
  PP_CUDA_TRY(ctx, ctx->scratch_out.reserve(ctx->stream, 6 * static_cast<size_t>(n) * 8));
  cudaStream_t s = ctx->stream;
  PP_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->scratch_in.p, in.data(), in.size() * 8,
                                   cudaMemcpyHostToDevice, s));
  const double* d = static_cast<const double*>(ctx->scratch_in.p);
  pp::guard_points_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, s>>>(
      R, n, d, d + n, static_cast<double*>(ctx->scratch_out.p));
  PP_CUDA_TRY(ctx, cudaGetLastError());
  std::vector<double> o(6 * static_cast<size_t>(n));
  PP_CUDA_TRY(ctx, cudaMemcpyAsync(o.data(), ctx->scratch_out.p, o.size() * 8,
                                   cudaMemcpyDeviceToHost, s));
  PP_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  for (int64_t i = 0; i < n; ++i) {
    if (ok_out) ok_out[i] = o[6 * i] != 0.0;
    if (guard_pq)
      for (int k = 0; k < 4; ++k) guard_pq[4 * i + k] = o[6 * i + 1 + k];
    if (guard_time) guard_time[i] = o[6 * i + 5];
  }
  return PP_OK;
}

// ---------------------------------------------------------------------------
// Batched frames (C5): raw worlds staged on the device, compact summaries.

}  // extern "C"

namespace {

// Stage + robot constants + the search pipeline for the uploaded frames,
// enqueued on the context's stream.  full != nullptr: full pp_dpps_summary
// per frame (pp_dpps_batch), else the compact pp_frame_summary.  With
// ev_stage / ev_scan / ev_value the pipeline runs group by group with
// events between its kernels (kernel timing; no PDL overlap).
struct BatchTimes {
  double stage_ms = 0.0, scan_ms = 0.0, value_ms = 0.0;
  int n_scan_launches = 0;
};

#ifndef PP_BATCH_CELLS_LOG2
#define PP_BATCH_CELLS_LOG2 28
#endif
cudaError_t enqueue_batch(pp_ctx* ctx, pp::DevParams P, pp_dpps_summary* full,
                          BatchTimes* times) {
  const int64_t n = ctx->batch_n;
  cudaStream_t s = ctx->stream;
  const int64_t n_cells = static_cast<int64_t>(P.n_kt) * P.n_dirs * P.n_pows;
  // Frames are independent: launch them in groups so the per-frame cell
  // queues stay a bounded working set (group x cells x 37 B, at most 2^28
  // cells = 9.9 GB of the 180 GB HBM).  Fewer, larger launches have fewer
  // tails: C5 65,536 frames 359.6 ms in groups of 4,096, 355.3 (8,192),
  // 352.0 (16,384), 350.5 (32,768 = the cell cap for the 128 x 64 grid).
  static const int64_t max_group = [] {
    const char* e = getenv("PP_BATCH_GROUP");  // dev knob
    return e ? std::max<int64_t>(1, atoll(e)) : int64_t(32768);
  }();
  int64_t group = (int64_t(1) << PP_BATCH_CELLS_LOG2) / std::max<int64_t>(n_cells, 1);
  group = std::max<int64_t>(1, std::min<int64_t>(group, std::min<int64_t>(n, max_group)));
  cudaError_t e = reserve_pipeline(ctx, P, group);
  if (e == cudaSuccess)
    e = ctx->batch_rk.reserve(ctx->stream, sizeof(pp::RobotK) * pp::kMaxRobots * static_cast<size_t>(n));
  if (e != cudaSuccess) return e;
  auto* frames = static_cast<pp::FrameDev*>(ctx->batch_frames.p);
  auto* rk = static_cast<pp::RobotK*>(ctx->batch_rk.p);
  if (times) cudaEventRecord(ctx->ev0, s);
  e = cudaMemsetAsync(ctx->batch_bad.p, 0xFF, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  pp::stage_frames_kernel<<<static_cast<unsigned>((n * 32 + 255) / 256), 256, 0, s>>>(
      static_cast<const pp_world*>(ctx->batch_worlds.p),
      ctx->batch_has_kickers ? static_cast<const int32_t*>(ctx->batch_kick_in.p) : nullptr, n,
      frames, static_cast<int32_t*>(ctx->batch_kickers.p),
      static_cast<unsigned long long*>(ctx->batch_bad.p));
  // every frame's robot filter constants once, not once per tile
  pp::robot_consts_kernel<<<static_cast<unsigned>((n * pp::kMaxRobots + 255) / 256), 256, 0, s>>>(
      frames, P, rk, n);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (times) {
    cudaEventRecord(ctx->ev1, s);
    e = cudaEventSynchronize(ctx->ev1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    times->stage_ms += ms;
  }
  const int threads = 32 * warps_for(ctx->batch_max_scan);
  pp::CellOut co{};
  auto* compact = static_cast<pp_frame_summary*>(ctx->batch_compact.p);
  for (int64_t f0 = 0; e == cudaSuccess && f0 < n; f0 += group) {
    const int64_t nf = std::min(group, n - f0);
    pp::DevParams Pg = P;
    Pg.rk_pre = rk + f0 * pp::kMaxRobots;
    Pg.compact = full ? nullptr : compact + f0;
    if (times) cudaEventRecord(ctx->ev0, s);
    e = launch_pipeline<false>(ctx, frames + f0, nf, Pg, threads, co, full ? full + f0 : nullptr,
                               times ? ctx->evm : nullptr);
    if (e == cudaSuccess && times) {
      cudaEventRecord(ctx->ev1, s);
      e = cudaEventSynchronize(ctx->ev1);
      float a = 0.f, b = 0.f;
      cudaEventElapsedTime(&a, ctx->ev0, ctx->evm);
      cudaEventElapsedTime(&b, ctx->evm, ctx->ev1);
      times->scan_ms += a;
      times->value_ms += b;
      times->n_scan_launches += 1;
    }
  }
  return e;
}

pp_status batch_prepare(pp_ctx* ctx, const pp_params* params, const pp_search_grid* grid_in,
                        pp::DevParams* P) {
  if (!ctx || !params) return fail(ctx, PP_INTERNAL, "null argument");
  ctx->err.clear();
  const pp_search_grid& g = grid_in ? *grid_in : params->grid;
  std::string why;
  if (!validate_grid(g, &why)) return fail(ctx, PP_CONFIG, "%s", why.c_str());
  if (!validate_params(*params, &why)) return fail(ctx, PP_CONFIG, "%s", why.c_str());
  PP_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  *P = make_dev_params(ctx, *params, g);
  PP_CUDA_TRY(ctx, ensure_tables(ctx, P));
  const size_t n = static_cast<size_t>(std::max<int64_t>(ctx->batch_n, 1));
  PP_CUDA_TRY(ctx, ctx->batch_frames.reserve(ctx->stream, sizeof(pp::FrameDev) * n));
  PP_CUDA_TRY(ctx, ctx->batch_kickers.reserve(ctx->stream, sizeof(int32_t) * n));
  PP_CUDA_TRY(ctx, ctx->batch_bad.reserve(ctx->stream, sizeof(unsigned long long)));
  PP_CUDA_TRY(ctx, ctx->batch_compact.reserve(ctx->stream, sizeof(pp_frame_summary) * n));
  return PP_OK;
}

// The first frame the device could not stage, as the host's pack_frame
// would have reported it.
pp_status batch_check(pp_ctx* ctx) {
  unsigned long long bad = ~0ull;
  PP_CUDA_TRY(ctx, cudaMemcpyAsync(&bad, ctx->batch_bad.p, sizeof(bad), cudaMemcpyDeviceToHost,
                                   ctx->stream));
  PP_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (bad == ~0ull) return PP_OK;
  const long long f = static_cast<long long>(bad >> 2);
  const long long fg = f + ctx->batch_frame0;
  if ((bad & 3ull) == pp::kStageTeamSize)
    return fail(ctx, PP_VALIDATION, "frame %lld: team size outside [0, 16]", fg);
  int32_t kid = -1;
  PP_CUDA_TRY(ctx, cudaMemcpy(&kid, static_cast<const int32_t*>(ctx->batch_kickers.p) + f,
                              sizeof(kid), cudaMemcpyDeviceToHost));
  return fail(ctx, PP_VALIDATION, "frame %lld: kicker id %d is not on team ours", fg, kid);
}

}  // namespace

extern "C" {

pp_status pp_batch_upload(pp_ctx* ctx, const pp_world* frames, int64_t n_frames,
                          const int32_t* kicker_ids) {
  PP_NVTX("pp_batch_upload");
  if (!ctx || (!frames && n_frames > 0) || n_frames < 0)
    return fail(ctx, PP_INTERNAL, "null argument");
  ctx->err.clear();
  PP_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  ctx->batch_ran = false;
  ctx->batch_n = n_frames;
  ctx->batch_frame0 = 0;
  const size_t n = static_cast<size_t>(std::max<int64_t>(n_frames, 1));
  PP_CUDA_TRY(ctx, ctx->batch_worlds.reserve(ctx->stream, sizeof(pp_world) * n));
  PP_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->batch_worlds.p, frames, sizeof(pp_world) * n_frames,
                                   cudaMemcpyHostToDevice, ctx->stream));
  ctx->batch_has_kickers = kicker_ids != nullptr;
  if (kicker_ids) {
    PP_CUDA_TRY(ctx, ctx->batch_kick_in.reserve(ctx->stream, sizeof(int32_t) * n));
    PP_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->batch_kick_in.p, kicker_ids,
                                     sizeof(int32_t) * n_frames, cudaMemcpyHostToDevice,
                                     ctx->stream));
  }
  // widest scan list (the scan CTA's width request): ours minus the kicker
  // plus theirs, from the team sizes alone
  int widest = 1;
  for (int64_t i = 0; i < n_frames; ++i) {
    const int no = frames[i].n_ours, nt = frames[i].n_theirs;
    if (no >= 0 && no <= PP_MAX_TEAM && nt >= 0 && nt <= PP_MAX_TEAM)
      widest = std::max(widest, no - 1 + nt);
  }
  ctx->batch_max_scan = widest;
  return PP_OK;
}

pp_status pp_batch_run(pp_ctx* ctx, const pp_params* params, const pp_search_grid* grid_in,
                       float* device_ms) {
  PP_NVTX("pp_batch_run");
  pp::DevParams P;
  pp_status st = batch_prepare(ctx, params, grid_in, &P);
  if (st != PP_OK) return st;
  ctx->batch_ran = true;
  if (ctx->batch_n == 0 || pp_grid_cells(grid_in ? grid_in : &params->grid) == 0) {
    PP_CUDA_TRY(ctx, cudaMemsetAsync(ctx->batch_bad.p, 0xFF, sizeof(unsigned long long),
                                     ctx->stream));
    PP_CUDA_TRY(ctx, cudaMemsetAsync(ctx->batch_compact.p, 0,
                                     sizeof(pp_frame_summary) * ctx->batch_n, ctx->stream));
    if (device_ms) *device_ms = 0.f;
    return PP_OK;
  }
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  if (device_ms) {
    PP_CUDA_TRY(ctx, cudaEventCreate(&t0));
    cudaEventCreate(&t1);
    cudaEventRecord(t0, ctx->stream);
  }
  const cudaError_t e = enqueue_batch(ctx, P, nullptr, nullptr);
  if (e != cudaSuccess) {
    if (t0) cudaEventDestroy(t0);
    if (t1) cudaEventDestroy(t1);
    PP_PIPE_TRY(ctx, e);
  }
  if (device_ms) {
    cudaEventRecord(t1, ctx->stream);
    const cudaError_t e2 = cudaEventSynchronize(t1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t0, t1);
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    PP_PIPE_TRY(ctx, e2);
    *device_ms = ms;
  }
  return PP_OK;
}

pp_status pp_batch_download(pp_ctx* ctx, pp_frame_summary* out) {
  PP_NVTX("pp_batch_download");
  if (!ctx || (!out && ctx->batch_n > 0)) return fail(ctx, PP_INTERNAL, "null argument");
  if (!ctx->batch_ran) return fail(ctx, PP_INTERNAL, "pp_batch_download before pp_batch_run");
  PP_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const int64_t n = ctx->batch_n;
  if (n > 0)
    PP_CUDA_TRY(ctx, cudaMemcpyAsync(out, ctx->batch_compact.p, sizeof(pp_frame_summary) * n,
                                     cudaMemcpyDeviceToHost, ctx->stream));
  return batch_check(ctx);
}

pp_status pp_batch_kernel_times(pp_ctx* ctx, const pp_params* params, const pp_search_grid* grid,
                                int32_t reps, float* stage_ms, float* scan_ms, float* value_ms,
                                int32_t* n_scan_launches) {
  pp::DevParams P;
  pp_status st = batch_prepare(ctx, params, grid, &P);
  if (st != PP_OK) return st;
  if (reps < 1 || ctx->batch_n == 0) return fail(ctx, PP_INTERNAL, "nothing to time");
  BatchTimes t;
  for (int r = 0; r < reps; ++r) PP_PIPE_TRY(ctx, enqueue_batch(ctx, P, nullptr, &t));
  if (stage_ms) *stage_ms = static_cast<float>(t.stage_ms / reps);
  if (scan_ms) *scan_ms = static_cast<float>(t.scan_ms / reps);
  if (value_ms) *value_ms = static_cast<float>(t.value_ms / reps);
  if (n_scan_launches) *n_scan_launches = t.n_scan_launches / reps;
  return PP_OK;
}

pp_status pp_dpps_frames(pp_ctx* ctx, const pp_world* frames, int64_t n_frames,
                         const pp_params* params, const pp_search_grid* grid,
                         const int32_t* kicker_ids, pp_frame_summary* out) {
  PP_NVTX("pp_dpps_frames");
  pp_status st = pp_batch_upload(ctx, frames, n_frames, kicker_ids);
  if (st == PP_OK) st = pp_batch_run(ctx, params, grid, nullptr);
  if (st == PP_OK) st = pp_batch_download(ctx, out);
  return st;
}

// One process, several devices (SURVEY 8(b)3's batch shape): contiguous
// frame ranges, one per context; every context's upload and search are
// enqueued before any result is read, so the devices run concurrently.
pp_status pp_dpps_frames_multi(pp_ctx* const* ctxs, int32_t n_ctx, const pp_world* frames,
                               int64_t n_frames, const pp_params* params,
                               const pp_search_grid* grid, const int32_t* kicker_ids,
                               pp_frame_summary* out) {
  PP_NVTX("pp_dpps_frames_multi");
  if (!ctxs || n_ctx < 1 || !ctxs[0]) return PP_INTERNAL;
  pp_ctx* c0 = ctxs[0];
  for (int i = 1; i < n_ctx; ++i)
    if (!ctxs[i] || ctxs[i] == ctxs[i - 1])
      return fail(c0, PP_INTERNAL, "context %d: null or repeated", i);
  if ((!frames || !out) && n_frames > 0) return fail(c0, PP_INTERNAL, "null argument");
  if (n_frames < 0) return fail(c0, PP_INTERNAL, "negative frame count");
  auto lo = [&](int i) { return n_frames * i / n_ctx; };
  auto relay = [&](int i, pp_status st) {  // the failing context's message, on ctxs[0]
    if (i != 0) c0->err = "context " + std::to_string(i) + ": " + ctxs[i]->err;
    return st;
  };
  for (int i = 0; i < n_ctx; ++i) {
    const int64_t a = lo(i), m = lo(i + 1) - a;
    pp_status st = pp_batch_upload(ctxs[i], frames + a, m, kicker_ids ? kicker_ids + a : nullptr);
    ctxs[i]->batch_frame0 = a;
    if (st == PP_OK) st = pp_batch_run(ctxs[i], params, grid, nullptr);
    if (st != PP_OK) return relay(i, st);
  }
  pp_status first = PP_OK;
  for (int i = 0; i < n_ctx; ++i) {  // (every context is drained, even after a failure)
    const pp_status st = pp_batch_download(ctxs[i], out + lo(i));
    if (st != PP_OK && first == PP_OK) first = relay(i, st);
  }
  return first;
}

// Full per-frame summaries (the single-frame pp_dpps_summary, best features
// included): the same device staging and search, then the host fills the
// per-frame team tables.
pp_status pp_dpps_batch(pp_ctx* ctx, const pp_world* frames, int64_t n_frames,
                        const pp_params* params, const pp_search_grid* grid_in,
                        const int32_t* kicker_ids, pp_dpps_summary* summaries) {
  PP_NVTX("pp_dpps_batch");
  if (!summaries && n_frames > 0) return fail(ctx, PP_INTERNAL, "null argument");
  pp_status st = pp_batch_upload(ctx, frames, n_frames, kicker_ids);
  if (st != PP_OK) return st;
  pp::DevParams P;
  st = batch_prepare(ctx, params, grid_in, &P);
  if (st != PP_OK) return st;
  ctx->batch_ran = true;
  const pp_search_grid& g = grid_in ? *grid_in : params->grid;
  const size_t n = static_cast<size_t>(std::max<int64_t>(n_frames, 1));
  PP_CUDA_TRY(ctx, ctx->batch_full.reserve(ctx->stream, sizeof(pp_dpps_summary) * n));
  auto* full = static_cast<pp_dpps_summary*>(ctx->batch_full.p);
  if (n_frames > 0 && pp_grid_cells(&g) > 0) {
    PP_PIPE_TRY(ctx, enqueue_batch(ctx, P, full, nullptr));
    PP_CUDA_TRY(ctx, cudaMemcpyAsync(summaries, full, sizeof(pp_dpps_summary) * n_frames,
                                     cudaMemcpyDeviceToHost, ctx->stream));
  } else {
    PP_CUDA_TRY(ctx, cudaMemsetAsync(ctx->batch_bad.p, 0xFF, sizeof(unsigned long long),
                                     ctx->stream));
    std::memset(summaries, 0, sizeof(pp_dpps_summary) * static_cast<size_t>(n_frames));
    for (int64_t i = 0; i < n_frames; ++i)
      for (int k = 0; k < 3; ++k) summaries[i].best_cell[k] = -1;
  }
  std::vector<int32_t> kick(n);
  if (n_frames > 0)
    PP_CUDA_TRY(ctx, cudaMemcpyAsync(kick.data(), ctx->batch_kickers.p, sizeof(int32_t) * n_frames,
                                     cudaMemcpyDeviceToHost, ctx->stream));
  st = batch_check(ctx);  // (synchronises)
  if (st != PP_OK) return st;
  for (int64_t i = 0; i < n_frames; ++i) {
    const double dms = summaries[i].device_ms;
    pp::FrameDev F;
    int32_t ks = -1;
    std::string why;
    pack_frame(frames[i], kick[i], &F, &ks, &why);
    fill_summary_host(&summaries[i], frames[i], g, kick[i], ks,
                      possession_of(frames[i], kick[i], *params));
    summaries[i].device_ms = dms;
  }
  return PP_OK;
}

}  // extern "C"


// ---- interception, possession, shot decision, free kick -----------------
namespace {

// BallTrajectory::resolve argument checks (ball_model.cpp:12-43).
bool kick_path(const pp_kick& k, const pp_ball_model& b, pp::BallPath* out, pp_status* st,
               std::string* why) {
  if (!validate_ball(b, why)) {
    *st = PP_CONFIG;
    return false;
  }
  using pp::xd;
  const bool roll = k.kind == 2;
  const xd speed = roll ? pp::xsqrt(xd(k.dir_x) * xd(k.dir_x) + xd(k.dir_y) * xd(k.dir_y))
                        : xd(k.speed);
  if (!(speed.v >= 0.0) || !std::isfinite(speed.v)) {
    *st = PP_DOMAIN;
    *why = "kick speed must be finite and non-negative";
    return false;
  }
  const xd n = pp::xsqrt(xd(k.dir_x) * xd(k.dir_x) + xd(k.dir_y) * xd(k.dir_y));
  if (n.v == 0.0 && speed.v > 0.0) {
    *st = PP_DOMAIN;
    *why = "kick direction must be non-zero";
    return false;
  }
  *out = pp::make_path(k.origin_x, k.origin_y, k.dir_x, k.dir_y, speed, k.kind == 1, !roll,
                       b.slide_decel, b.roll_decel, b.transition_ratio, b.chip_flight_fraction);
  return true;
}

pp::BallPath path_of(const pp_trajectory& t) {
  pp::BallPath b;
  b.ox = t.origin_x;
  b.oy = t.origin_y;
  b.ux = t.dir_x;
  b.uy = t.dir_y;
  b.slide = t.slide_decel;
  b.roll = t.roll_decel;
  b.tr.speed = t.kick_speed;
  b.tr.v1 = t.v1;
  b.tr.t_se = t.slide_end_time;
  b.tr.d_se = t.slide_end_distance;
  b.tr.t_stop = t.stop_time;
  b.tr.d_stop = t.stop_distance;
  b.tr.from = t.interceptable_from;
  return b;
}

// Runs intercept_kernel for the frame staged in ctx->frame_h (scan list set).
cudaError_t run_intercepts(pp_ctx* ctx, const pp::FrameDev& F, const pp::DevParams& P,
                           const pp::BallPath& B, double dt, std::vector<pp::InterceptOut>* res) {
  cudaStream_t s = ctx->stream;
  cudaError_t e = ctx->scratch_out.reserve(ctx->stream, sizeof(pp::InterceptOut) * pp::kMaxRobots);
  if (e != cudaSuccess) return e;
  e = cudaMemcpyAsync(ctx->frame.p, &F, sizeof(F), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  res->assign(static_cast<size_t>(F.n_scan), pp::InterceptOut{});
  if (F.n_scan == 0) return cudaStreamSynchronize(s);
  pp::intercept_kernel<<<1, 32 * F.n_scan, 0, s>>>(static_cast<const pp::FrameDev*>(ctx->frame.p),
                                                   P, B, dt,
                                                   static_cast<pp::InterceptOut*>(ctx->scratch_out.p));
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = cudaMemcpyAsync(res->data(), ctx->scratch_out.p, sizeof(pp::InterceptOut) * res->size(),
                      cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(s);
}

const pp_robot* find_robot(const pp_robot* r, int n, int32_t id) {
  for (int i = 0; i < n; ++i)
    if (r[i].id == id) return &r[i];
  return nullptr;
}

}  // namespace

extern "C" {

pp_status pp_kick_trajectory(const pp_kick* kick, const pp_ball_model* ball, pp_trajectory* out,
                             char* msg, size_t msg_len) {
  if (!kick || !ball || !out) {
    put(msg, msg_len, "null argument");
    return PP_INTERNAL;
  }
  pp::BallPath B;
  pp_status st = PP_OK;
  std::string why;
  if (!kick_path(*kick, *ball, &B, &st, &why)) {
    put(msg, msg_len, why);
    return st;
  }
  std::memset(out, 0, sizeof(*out));
  out->origin_x = B.ox;
  out->origin_y = B.oy;
  out->dir_x = B.ux;
  out->dir_y = B.uy;
  out->kick_speed = B.tr.speed.v;
  out->v1 = B.tr.v1.v;
  out->slide_decel = B.slide;
  out->roll_decel = B.roll;
  out->slide_end_time = B.tr.t_se.v;
  out->slide_end_distance = B.tr.d_se.v;
  out->stop_time = B.tr.t_stop.v;
  out->stop_distance = B.tr.d_stop.v;
  out->interceptable_from = B.tr.from.v;
  out->kick_type = kick->kind == 1 ? 1 : 0;
  return PP_OK;
}

pp_status pp_intercept_all(pp_ctx* ctx, const pp_world* world, const pp_params* params,
                           const pp_trajectory* traj, double dt, pp_intercept* out) {
  PP_NVTX("pp_intercept_all");
  if (!ctx || !world || !params || !traj || !out) return fail(ctx, PP_INTERNAL, "null argument");
  ctx->err.clear();
  std::string why;
  if (!(dt > 0.0)) return fail(ctx, PP_DOMAIN, "intercept_all: dt must be > 0");
  const pp::BallPath B = path_of(*traj);
  PP_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  pp::FrameDev* F = static_cast<pp::FrameDev*>(ctx->frame_h.p);
  int32_t ks = -1;
  if (!pack_frame(*world, -1, F, &ks, &why, ScanList::kAll))
    return fail(ctx, PP_VALIDATION, "%s", why.c_str());
  const pp::DevParams P = make_dev_params(ctx, *params, params->grid);
  std::vector<pp::InterceptOut> res;
  PP_CUDA_TRY(ctx, run_intercepts(ctx, *F, P, B, dt, &res));
  for (int i = 0; i < F->n_scan; ++i) {
    const int slot = F->scan_slot[i];
    pp_intercept& o = out[i];
    o.team = slot >= pp::kTheirs ? 1 : 0;
    o.robot_id = F->id[slot];
    o.finite = res[i].finite;
    o.pad = 0;
    o.time = res[i].finite ? res[i].time : 0.0;
    o.point_x = res[i].finite ? res[i].px : 0.0;
    o.point_y = res[i].finite ? res[i].py : 0.0;
  }
  return PP_OK;
}

pp_status pp_possession(pp_ctx* ctx, const pp_world* world, const pp_params* params,
                        pp_possession_report* out) {
  PP_NVTX("pp_possession");
  if (!ctx || !world || !params || !out) return fail(ctx, PP_INTERNAL, "null argument");
  const int n = world->n_ours + world->n_theirs;
  if (world->n_ours < 0 || world->n_theirs < 0 || n > 2 * PP_MAX_TEAM)
    return fail(ctx, PP_VALIDATION, "team size outside [0, 16]");
  const pp_kick roll{world->ball_px, world->ball_py, world->ball_vx, world->ball_vy, 0.0, 2, 0};
  pp_trajectory traj;
  char msg[256];
  pp_status st = pp_kick_trajectory(&roll, &params->ball, &traj, msg, sizeof(msg));
  if (st != PP_OK) return fail(ctx, st, "%s", msg);
  pp_intercept all[2 * PP_MAX_TEAM];
  st = pp_intercept_all(ctx, world, params, &traj, params->thresholds.possession_dt, all);
  if (st != PP_OK) return st;
  std::memset(out, 0, sizeof(*out));
  for (int i = 0; i < n; ++i) {  // fastest finite intercept per team (pass_eval.cpp:279-283)
    if (!all[i].finite) continue;
    int32_t* has = all[i].team == 0 ? &out->has_our : &out->has_their;
    double* t = all[i].team == 0 ? &out->our_time : &out->their_time;
    if (!*has || all[i].time < *t) {
      *has = 1;
      *t = all[i].time;
    }
  }
  if (!out->has_our && !out->has_their) {
    out->side = 2;
  } else if (!out->has_their) {
    out->side = 0;
  } else if (!out->has_our) {
    out->side = 1;
  } else {
    const double delta = out->our_time - out->their_time;
    out->side = std::fabs(delta) <= params->thresholds.contest_epsilon ? 2 : (delta < 0.0 ? 0 : 1);
  }
  return PP_OK;
}

pp_status pp_decide_shot(pp_ctx* ctx, const pp_world* world, const pp_params* params,
                         int32_t shooter_id, pp_shot_decision* out) {
  PP_NVTX("pp_decide_shot");
  if (!ctx || !world || !params || !out) return fail(ctx, PP_INTERNAL, "null argument");
  ctx->err.clear();
  std::string why;
  const pp_robot* shooter = find_robot(world->ours, world->n_ours, shooter_id);
  if (!shooter) return fail(ctx, PP_VALIDATION, "kicker id not on team ours");
  if (!validate_ball(params->ball, &why)) return fail(ctx, PP_CONFIG, "%s", why.c_str());
  const double shot_speed =
      params->thresholds.shot_power > 0.0 ? params->thresholds.shot_power : params->ball.power_max;
  if (!(shot_speed >= 0.0) || !std::isfinite(shot_speed))
    return fail(ctx, PP_DOMAIN, "kick speed must be finite and non-negative");
  PP_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  pp::FrameDev* F = static_cast<pp::FrameDev*>(ctx->frame_h.p);
  int32_t ks = -1;
  if (!pack_frame(*world, shooter_id, F, &ks, &why, ScanList::kTheirs))
    return fail(ctx, PP_VALIDATION, "%s", why.c_str());
  // origin: the ball when the shooter has it (pass_eval.cpp:196-199)
  const bool has_ball = host_distance(shooter->px, shooter->py, world->ball_px, world->ball_py) <=
                        params->thresholds.possession_radius;
  const double ox = has_ball ? world->ball_px : shooter->px;
  const double oy = has_ball ? world->ball_py : shooter->py;
  const pp::DevParams P = make_dev_params(ctx, *params, params->grid);
  cudaStream_t s = ctx->stream;
  PP_CUDA_TRY(ctx, ctx->scratch_out.reserve(ctx->stream, sizeof(pp_shot_decision)));
  PP_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->frame.p, F, sizeof(*F), cudaMemcpyHostToDevice, s));
  pp::shot_kernel<<<1, 32 * std::max(F->n_scan, 2), 0, s>>>(
      static_cast<const pp::FrameDev*>(ctx->frame.p), P, ox, oy, shot_speed,
      params->thresholds.angle_threshold, static_cast<pp_shot_decision*>(ctx->scratch_out.p));
  PP_CUDA_TRY(ctx, cudaGetLastError());
  PP_CUDA_TRY(ctx, cudaMemcpyAsync(out, ctx->scratch_out.p, sizeof(*out), cudaMemcpyDeviceToHost, s));
  PP_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  return PP_OK;
}

pp_status pp_plan_free_kick(pp_ctx* ctx, const pp_world* world, const pp_params* params,
                            int32_t kicker_id, const pp_candidate* target,
                            pp_free_kick_plan* out) {
  PP_NVTX("pp_plan_free_kick");
  if (!ctx || !world || !params || !target || !out)
    return fail(ctx, PP_INTERNAL, "null argument");
  ctx->err.clear();
  using pp::xd;
  if (!target->feasible)
    return fail(ctx, PP_DOMAIN, "plan_free_kick: target candidate is not feasible");
  if (!find_robot(world->ours, world->n_ours, kicker_id))
    return fail(ctx, PP_VALIDATION, "plan_free_kick: kicker id %d is not on team ours", kicker_id);
  const pp_robot* rcv = find_robot(world->ours, world->n_ours, target->our_id);
  if (!rcv)
    return fail(ctx, PP_VALIDATION, "plan_free_kick: receiver id %d is not on team ours",
                target->our_id);
  const pp_search_grid& g = params->grid;
  if (target->power_index < 0 || target->power_index >= g.n_powers)
    return fail(ctx, PP_DOMAIN,
                "plan_free_kick: candidate power index outside the configured grid");
  const xd power = pp::power_at(target->power_index, g.n_powers, g.power_min, g.power_max);
  pp_kick k{world->ball_px, world->ball_py, (xd(target->receive_x) - xd(world->ball_px)).v,
            (xd(target->receive_y) - xd(world->ball_py)).v, power.v, target->kick_type == 1 ? 1 : 0,
            0};
  pp::BallPath B;
  pp_status st = PP_OK;
  std::string why;
  if (!kick_path(k, params->ball, &B, &st, &why)) return fail(ctx, st, "%s", why.c_str());
  const xd dlen = pp::xsqrt(xd(k.dir_x) * xd(k.dir_x) + xd(k.dir_y) * xd(k.dir_y));
  const xd t_ball =
      pp::travel_time_to_distance(B.tr, params->ball.slide_decel, params->ball.roll_decel, dlen);
  if (std::isnan(t_ball.v))
    return fail(ctx, PP_DOMAIN, "plan_free_kick: receive point beyond the ball's rollout");
  const pp_motion_limits& m = params->motion_ours;
  const xd t_robot = pp::arrival_time(rcv->px, rcv->py, rcv->vx, rcv->vy, target->receive_x,
                                      target->receive_y, m.max_accel, m.max_decel, m.max_speed);
  out->t_ball = t_ball.v;
  out->t_robot = t_robot.v;
  out->order = t_robot <= t_ball ? 1 : 0;
  out->pad = 0;
  const xd wait = t_robot - t_ball;
  out->kick_delay = wait.v > 0.0 ? wait.v : 0.0;  // std::max(0.0, t_robot - t_ball)
  return PP_OK;
}

}  // extern "C"

#ifdef PP_PHASE_CLOCKS
// Profiling build only: cumulative SM cycles per phase (scan A/B/C in 0..2,
// value D1/D2/D3/reduce in 3..6) and CTA counts (scan [8], value [9]).
extern "C" int pp_debug_phase_cycles(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, pp::g_phase_cycles, 16 * sizeof(unsigned long long)) != cudaSuccess)
    return PP_CUDA;
  if (reset) {
    const unsigned long long z[16] = {0};
    if (cudaMemcpyToSymbol(pp::g_phase_cycles, z, sizeof(z)) != cudaSuccess) return PP_CUDA;
  }
  return PP_OK;
}
#endif

#ifdef PP_PHASE_CLOCKS
// Profiling build only: scan counters (iterations, skips, lower-bound
// rejects, upper-bound accepts, exact FP64 tests, FP64 rounds, sum of per-warp
// max iterations, robot-warp scans).
#endif

#ifdef PP_PHASE_CLOCKS
// Profiling build only: per-CTA records of the last launches (see PP_FLUSH).
extern "C" int pp_debug_cta_records(long long* scan, long long* value, long long* robots) {
  if (cudaMemcpyFromSymbol(scan, pp::g_cta_rec, sizeof(pp::g_cta_rec) / 2) != cudaSuccess ||
      cudaMemcpyFromSymbol(value, pp::g_cta_rec, sizeof(pp::g_cta_rec) / 2, sizeof(pp::g_cta_rec) / 2) != cudaSuccess ||
      cudaMemcpyFromSymbol(robots, pp::g_robot_rec, sizeof(pp::g_robot_rec)) != cudaSuccess)
    return PP_CUDA;
  return PP_OK;
}
#endif

#ifdef PP_PHASE_CLOCKS
extern "C" int pp_debug_champ_records(long long* out) {
  return cudaMemcpyFromSymbol(out, pp::g_champ_rec, sizeof(pp::g_champ_rec)) == cudaSuccess ? 0 : -1;
}
extern "C" int pp_debug_d1_records(long long* out) {
  return cudaMemcpyFromSymbol(out, pp::g_d1_rec, sizeof(pp::g_d1_rec)) == cudaSuccess ? 0 : -1;
}
extern "C" int pp_debug_d2_records(long long* out) {
  return cudaMemcpyFromSymbol(out, pp::g_d2_rec, sizeof(pp::g_d2_rec)) == cudaSuccess ? 0 : -1;
}
extern "C" int pp_debug_win_records(long long* out) {
  return cudaMemcpyFromSymbol(out, pp::g_win_rec, sizeof(pp::g_win_rec)) == cudaSuccess ? 0 : -1;
}
extern "C" int pp_debug_round_records(long long* out) {
  return cudaMemcpyFromSymbol(out, pp::g_round_rec, sizeof(pp::g_round_rec)) == cudaSuccess ? 0 : -1;
}
extern "C" int pp_debug_warp_records(long long* out) {
  return cudaMemcpyFromSymbol(out, pp::g_warp_rec, sizeof(pp::g_warp_rec)) == cudaSuccess ? 0 : -1;
}
extern "C" int pp_debug_lane_records(int* out) {
  return cudaMemcpyFromSymbol(out, pp::g_lane_rec, sizeof(pp::g_lane_rec)) == cudaSuccess ? PP_OK
                                                                                          : PP_CUDA;
}
#endif


#ifdef PP_PHASE_CLOCKS
#endif
