// pp_queries.cuh -- Standalone goal_view / score_pass / score_running_point queries.
#pragma once

#include "pp_runmap.cuh"

namespace pp {

// ---------------------------------------------------------------------------
// Standalone goal views / score_pass on explicit candidates (one warp each).

__global__ void __launch_bounds__(256) goal_view_kernel(const FrameDev* __restrict__ frame,
                                                        double radius, double r_lt2,
                                                        double mb_le2, int64_t n,
                                                        const double* __restrict__ px,
                                                        const double* __restrict__ py,
                                                        double* __restrict__ out4, bool exact) {
  __shared__ FrameDev F;
  {
    const int nn = sizeof(FrameDev) / 16;
    const int4* src = reinterpret_cast<const int4*>(frame);
    int4* dst = reinterpret_cast<int4*>(&F);
    for (int i = threadIdx.x; i < nn; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const View v = goal_view_thread(px[q], py[q], F, radius, r_lt2, mb_le2, exact);
  out4[4 * q + 0] = v.angle;
  out4[4 * q + 1] = v.lo;
  out4[4 * q + 2] = v.hi;
  out4[4 * q + 3] = v.ty;
}

__global__ void __launch_bounds__(256) score_cells_kernel(const FrameDev* __restrict__ frame,
                                                          DevParams P, int64_t n,
                                                          const double* __restrict__ in4,
                                                          double* __restrict__ out6) {
  __shared__ FrameDev F;
  {
    const int nn = sizeof(FrameDev) / 16;
    const int4* src = reinterpret_cast<const int4*>(frame);
    int4* dst = reinterpret_cast<int4*>(&F);
    for (int i = threadIdx.x; i < nn; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const double rx = in4[4 * q], ry = in4[4 * q + 1], ot = in4[4 * q + 2], pt = in4[4 * q + 3];
  const View v = goal_view_thread(rx, ry, F, P.radius, P.r_lt2, P.mb_le2, P.exact_only != 0);
  double feat[5];
  const double s = score_from_view(v, rx, ry, ot, pt, F, P, feat);
  out6[6 * q] = s;
  for (int k = 0; k < 5; ++k) out6[6 * q + 1 + k] = feat[k];
}

// ---------------------------------------------------------------------------
// kernels::KernelBackend::scan_first (kernel.hpp:33-53) for n independent
// (ray, robot) pairs: one warp per pair, 32 consecutive samples per step with
// the reference's exact test (FP64, no FP32 filter: a plug-in call is a
// single pair, there is nothing to amortise), the first passing sample by
// ballot.  samples: every pair's [k_begin, k_end) (t, s) values, packed at
// off[i].
struct ScanPair {
  double ox, oy, ux, uy;
  double px, py, vx, vy, a, b, vmax, radius, vbound;
  int64_t off;
  int32_t k_begin, k_end;
};

__global__ void __launch_bounds__(256) scan_first_kernel(const ScanPair* __restrict__ pairs,
                                                         int64_t n,
                                                         const double2* __restrict__ samples,
                                                         int32_t* __restrict__ out) {
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const ScanPair& q = pairs[i];
  int first = -1;
  for (int k0 = q.k_begin; k0 < q.k_end; k0 += 32) {
    const int k = k0 + lane;
    bool ok = false;
    if (k < q.k_end) {
      const double2 ts = samples[q.off + (k - q.k_begin)];
      const xd t = ts.x, s = ts.y;
      const xd qx = (xd(q.ox) + xd(q.ux) * s) - xd(q.px);
      const xd qy = (xd(q.oy) + xd(q.uy) * s) - xd(q.py);
      const xd d2 = qx * qx + qy * qy;
      const xd reach = xd(q.radius) + xd(q.vbound) * t;
      ok = !(d2 > reach * reach) &&
           arrival_given(qx, qy, d2, q.vx, q.vy, q.a, q.b, q.vmax, q.radius) <= t;
    }
    const unsigned m = __ballot_sync(0xffffffffu, ok);
    if (m) {
      first = k0 + __ffs(m) - 1;
      break;
    }
  }
  if (lane == 0) out[i] = first;
}

}  // namespace pp
