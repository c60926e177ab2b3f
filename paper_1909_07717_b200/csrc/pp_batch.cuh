// pp_batch.cuh -- staging of raw world states on the device for batched
// frames (the C5 log-replay path): the id-sorted team layout of run_dpps
// (dpps.cpp:74-92, 249-252) and the kicker choice, one warp per frame, so a
// batch costs one DMA of the caller's pp_world array and no host pass.
#pragma once

#include "pp_value.cuh"

namespace pp {

// Why a frame could not be staged (pp_dpps_frames reports the first one).
enum StageCode : unsigned { kStageTeamSize = 1, kStageKicker = 2 };

// One warp per frame; lanes 0-15 take team ours' entries, 16-31 theirs'.
// The same FrameDev as the host's pack_frame (pp_cabi.cu):
//  * slot = rank of the entry in its team by (id, entry index) -- a stable
//    id sort (dpps.cpp:79-92);
//  * kicker = kicker_ids[f], or the teammate nearest the ball: the first
//    strict minimum of |p - ball| in entry order (FP64, correctly rounded,
//    so identical to the host's), -1 with no teammates;
//  * kicker_slot = the last slot holding the kicker's id (dpps.cpp:250-252);
//    no such slot -> the frame is invalid (dpps.cpp:221-223);
//  * scan list = ours minus the kicker, then theirs.
// An invalid frame is staged with no scanned robots (its summary is then
// meaningless) and reported through *first_bad = min(f << 2 | code).
__global__ void __launch_bounds__(256)
    stage_frames_kernel(const pp_world* __restrict__ worlds, const int32_t* __restrict__ kicker_ids,
                        int64_t n_frames, FrameDev* __restrict__ out,
                        int32_t* __restrict__ kicker_out,
                        unsigned long long* __restrict__ first_bad) {
  const int lane = threadIdx.x & 31;
  const int64_t f = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (f >= n_frames) return;  // uniform per warp
  const pp_world& w = worlds[f];
  const int team = lane >> 4, j = lane & 15;
  const int n_ours = w.n_ours, n_theirs = w.n_theirs;
  const bool size_ok = n_ours >= 0 && n_ours <= kTheirs && n_theirs >= 0 && n_theirs <= kTheirs;
  const int nt = size_ok ? (team ? n_theirs : n_ours) : 0;
  const bool present = j < nt;
  pp_robot r{};
  if (present) r = team ? w.theirs[j] : w.ours[j];
  // stable rank by id within the team
  int rank = 0;
  for (int k = 0; k < 16; ++k) {
    const int idk = __shfl_sync(0xffffffffu, r.id, (team << 4) | k);
    rank += (k < nt && (idk < r.id || (idk == r.id && k < j))) ? 1 : 0;
  }
  // kicker
  int32_t kid;
  if (kicker_ids) {
    kid = kicker_ids[f];
  } else {
    // (d, entry) lexicographic argmin over the teammates; a NaN or infinite
    // distance never wins, like the host's `d < best` from best = +inf
    double d = CUDART_INF;
    int who = 1 << 30;
    if (present && team == 0) {
      const double dd = dist2d(r.px, r.py, w.ball_px, w.ball_py).v;
      if (dd < CUDART_INF) {
        d = dd;
        who = j;
      }
    }
    for (int s = 16; s > 0; s >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, d, s);
      const int ow = __shfl_xor_sync(0xffffffffu, who, s);
      if (od < d || (od == d && ow < who)) {
        d = od;
        who = ow;
      }
    }
    kid = who < 16 ? __shfl_sync(0xffffffffu, r.id, who) : -1;
  }
  const bool is_kicker = present && team == 0 && r.id == kid;
  int ks = is_kicker ? rank : -1;
  for (int s = 16; s > 0; s >>= 1) ks = max(ks, __shfl_xor_sync(0xffffffffu, ks, s));
  const bool ok = size_ok && ks >= 0;
  FrameDev& F = out[f];
  // robot slots: a present entry fills slot `rank`, an absent one zeroes
  // slot j (together they cover [0, 16) once per team)
  const int slot = (team << 4) | (present ? rank : j);
  F.px[slot] = present ? r.px : 0.0;
  F.py[slot] = present ? r.py : 0.0;
  F.vx[slot] = present ? r.vx : 0.0;
  F.vy[slot] = present ? r.vy : 0.0;
  F.id[slot] = present ? r.id : 0;
  // scan list: ours slots except the kicker's, then theirs
  const int n_scan = ok ? (n_ours - 1) + n_theirs : 0;
  F.scan_slot[lane] = 0;
  __syncwarp();
  if (ok && present) {
    const int pos = team ? (n_ours - 1) + rank : (rank == ks ? -1 : rank - (rank > ks ? 1 : 0));
    if (pos >= 0) F.scan_slot[pos] = static_cast<int8_t>(slot);
  }
  if (lane == 0) {
    F.ball_x = w.ball_px;
    F.ball_y = w.ball_py;
    F.L = w.field.length;
    F.W = w.field.width;
    F.gw = w.field.goal_width;
    F.dd = w.field.defense_depth;
    F.dw = w.field.defense_width;
    F.n_ours = size_ok ? n_ours : 0;
    F.n_theirs = size_ok ? n_theirs : 0;
    F.kicker_slot = ok ? ks : -1;
    F.n_scan = n_scan;
    kicker_out[f] = kid;
    if (!ok)
      atomicMin(first_bad, (static_cast<unsigned long long>(f) << 2) |
                               (size_ok ? kStageKicker : kStageTeamSize));
  }
}

}  // namespace pp
