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

}  // namespace pp
