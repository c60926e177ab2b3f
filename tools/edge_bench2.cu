// Dev tool: D2 (goal-view edge bisection) latency per warp with 32 active
// lanes of distinct blocking geometry: interval_edge (one divergent loop,
// defined here) vs the product's interval_edge_split (band steps, then exact
// rounds); checks both give identical edges.  Also times pair_info.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o tools/edge_bench2 tools/edge_bench2.cu
#include <cstdio>
#include "../paper_1909_07717_b200/csrc/pp_kernels.cuh"

using namespace pp;

// The straightforward replay of bisect_edge (one loop, band-decided or exact
// step by step): the reference the product's interval_edge_split is checked
// against here (same result, bit for bit).
// Interval edge `edge` (0 = lo, 1 = hi) of a blocking opponent: the end value
// or the 60-step bisection of bisect_edge (pass_eval.cpp:40-51, 88-92).
// Replayed exactly: each step's predicate is the reference's FP64 one,
// except where the fast-path band decides it; once the midpoint rounds onto
// an end point the state is a fixed point (the remaining steps are no-ops).
// Inside the band two steps are resolved per round: the midpoint and both
// possible next midpoints are evaluated together (independent FP64 chains).
__device__ __forceinline__ xd interval_edge(const ViewCtx& V, xd cx, xd cy, int edge, int first,
                                            int last, bool fast, xd y1, xd y2, double margin) {
  if (edge == 0 && first == 0) return -V.gh;
  if (edge == 1 && last == V.nh - 1) return V.gh;
  xd y_blocked = edge == 0 ? height_at(V, first) : height_at(V, last);
  xd y_free = edge == 0 ? height_at(V, first - 1) : height_at(V, last + 1);
  const double lo_in = y1.v + margin, hi_in = y2.v - margin;
  const double lo_out = y1.v - margin, hi_out = y2.v + margin;
  // 0 = surely free, 1 = surely blocked, 2 = needs the exact predicate
  auto decide = [&](double y) -> int {
    if (!fast) return 2;
    if (y > lo_in && y < hi_in) return 1;
    if (y < lo_out || y > hi_out) return 0;
    return 2;
  };
  int i = 0;
#pragma unroll 1
  while (i < 60) {
    const xd mid = xd(0.5) * (y_blocked + y_free);
    if (mid.v == y_blocked.v || mid.v == y_free.v) break;
    const int d0 = decide(mid.v);
    if (d0 != 2) {
      if (d0) {
        y_blocked = mid;
      } else {
        y_free = mid;
      }
      ++i;
      continue;
    }
    // speculate one level ahead
    const xd mid_b = xd(0.5) * (mid + y_free);     // next midpoint if `mid` is blocked
    const xd mid_f = xd(0.5) * (y_blocked + mid);  // next midpoint if `mid` is free
    bool k0, k1, k2;
    xd s0 = segment_dist_sq_f(cx, cy, V.px, V.py, V.gx, mid, &k0);
    xd sb = segment_dist_sq_f(cx, cy, V.px, V.py, V.gx, mid_b, &k1);
    xd sf = segment_dist_sq_f(cx, cy, V.px, V.py, V.gx, mid_f, &k2);
    if (!(k0 && k1 && k2)) {  // outside ddiv_fast's range: exact division
      s0 = segment_dist_sq(cx, cy, V.px, V.py, V.gx, mid);
      sb = segment_dist_sq(cx, cy, V.px, V.py, V.gx, mid_b);
      sf = segment_dist_sq(cx, cy, V.px, V.py, V.gx, mid_f);
    }
    const bool b0 = s0.v < V.r_lt2;
    xd nxt;
    bool bn;
    if (b0) {
      y_blocked = mid;
      nxt = mid_b;
      const int dn = decide(mid_b.v);
      bn = dn == 2 ? sb.v < V.r_lt2 : dn == 1;
    } else {
      y_free = mid;
      nxt = mid_f;
      const int dn = decide(mid_f.v);
      bn = dn == 2 ? sf.v < V.r_lt2 : dn == 1;
    }
    ++i;
    if (i >= 60) break;
    if (nxt.v == y_blocked.v || nxt.v == y_free.v) break;
    if (bn) {
      y_blocked = nxt;
    } else {
      y_free = nxt;
    }
    ++i;
  }
  return xd(0.5) * (y_blocked + y_free);
}



__device__ long long g_st[4];
template <int kMode, int kLanes>
__global__ void k(const FrameDev* F_, double r_lt2, double mb_le2, long long* cyc, double* out) {
  __shared__ FrameDev F;
  __shared__ double hts[kMaxHeights];
  __shared__ PairInfo pis[32];
  load_frame(&F, F_);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const ViewCtx V0 = make_view_ctx(0.0, 0.0, F, 0.09, r_lt2, mb_le2);
  for (int i = threadIdx.x; i < V0.nh; i += blockDim.x) hts[i] = view_height(i, V0.n_half, V0.gh).v;
  __syncthreads();
  const double t = lane + 32.0 * blockIdx.x;
  auto h = [&](double k) { const double x = sin(t * 12.9898 + k * 78.233) * 43758.5453; return x - floor(x); };
  const xd px = -2.0 + 5.0 * h(1), py = -2.0 + 4.0 * h(2);
  const double gy = -0.8 + 1.6 * h(3), f = 0.3 + 0.5 * h(4), off = (h(5) - 0.5) * 0.1;
  const xd cx = px.v + f * (6.0 - px.v), cy = py.v + f * (gy - py.v) + off;
  const ViewCtx V = make_view_ctx(px, py, F, 0.09, r_lt2, mb_le2, hts);
  pis[lane] = pair_info(V, cx, cy);
  __syncwarp();
  const PairInfo pi = pis[lane];
  const bool active = pi.status == 1 && lane < kLanes;
  __syncwarp();
  const long long t0 = clock64();
  double acc = 0.0;
  for (int edge = 0; edge < 2; ++edge) {
    xd y;
    if (kMode == 0) {
      y = active ? interval_edge(V, cx, cy, edge, pi.first, pi.last, pi.fast, pi.y1, pi.y2,
                                 pi.margin)
                 : xd(0.0);
    } else {
      long long st[4] = {0, 0, 0, 0};
      y = active ? interval_edge_split(V, cx, cy, edge, pi.first, pi.last, pi.fast, pi.y1, pi.y2,
                                       pi.margin, kLanes == 1 ? st : nullptr)
                 : xd(0.0);
      if (kLanes == 1 && active)
        for (int q = 0; q < 4; ++q) atomicAdd((unsigned long long*)&g_st[q], (unsigned long long)st[q]);
    }
    acc += y.v;
  }
  __syncwarp();
  const long long t1 = clock64();
  out[blockIdx.x * 32 + lane] = active ? acc : -999.0;
  if (lane == 0) cyc[blockIdx.x] = t1 - t0;
}


template <int kLanes>
__global__ void kp(const FrameDev* F_, double r_lt2, double mb_le2, long long* cyc, double* out) {
  __shared__ FrameDev F;
  __shared__ double hts[kMaxHeights];
  load_frame(&F, F_);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const ViewCtx V0 = make_view_ctx(0.0, 0.0, F, 0.09, r_lt2, mb_le2);
  for (int i = threadIdx.x; i < V0.nh; i += blockDim.x) hts[i] = view_height(i, V0.n_half, V0.gh).v;
  __syncthreads();
  const double t = lane + 32.0 * blockIdx.x;
  auto h = [&](double k) { const double x = sin(t * 12.9898 + k * 78.233) * 43758.5453; return x - floor(x); };
  const xd px = -2.0 + 5.0 * h(1), py = -2.0 + 4.0 * h(2);
  const double gy = -0.8 + 1.6 * h(3), f = 0.3 + 0.5 * h(4), off = (h(5) - 0.5) * 0.1;
  const xd cx = px.v + f * (6.0 - px.v), cy = py.v + f * (gy - py.v) + off;
  const ViewCtx V = make_view_ctx(px, py, F, 0.09, r_lt2, mb_le2, hts);
  __syncwarp();
  const long long t0 = clock64();
  int st = -1;
  if (lane < kLanes) {
    const PairInfo pi = pair_info(V, cx, cy);
    st = pi.status + 4 * pi.first;
  }
  __syncwarp();
  const long long t1 = clock64();
  out[blockIdx.x * 32 + lane] = st;
  if (lane == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  FrameDev F{};
  F.L = 12.0; F.W = 9.0; F.gw = 1.8;
  FrameDev* dF;
  cudaMalloc(&dF, sizeof(F));
  cudaMemcpy(dF, &F, sizeof(F), cudaMemcpyHostToDevice);
  const double r = 0.09, r_lt2 = r * r, mb_le2 = (r + 1e-9) * (r + 1e-9);
  long long* cyc; double* out;
  const int nb = 64;
  cudaMalloc(&cyc, nb * 8); cudaMalloc(&out, nb * 32 * 8);
  double ho[6][nb * 32]; long long hc[nb];
  for (int mode = 0; mode < 6; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k<0, 32><<<nb, 32>>>(dF, r_lt2, mb_le2, cyc, out);
      else if (mode == 1) k<1, 32><<<nb, 32>>>(dF, r_lt2, mb_le2, cyc, out);
      else if (mode == 2) k<0, 1><<<nb, 32>>>(dF, r_lt2, mb_le2, cyc, out);
      else if (mode == 3) k<1, 1><<<nb, 32>>>(dF, r_lt2, mb_le2, cyc, out);
      else if (mode == 4) k<0, 8><<<nb, 32>>>(dF, r_lt2, mb_le2, cyc, out);
      else k<1, 8><<<nb, 32>>>(dF, r_lt2, mb_le2, cyc, out);
    }
    cudaDeviceSynchronize();
    cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
    cudaMemcpy(ho[mode], out, sizeof(ho[0]), cudaMemcpyDeviceToHost);
    double s = 0; long long mx = 0; int act = 0;
    for (int i = 0; i < nb; ++i) { s += hc[i]; mx = hc[i] > mx ? hc[i] : mx; }
    for (int i = 0; i < nb * 32; ++i) act += ho[mode][i] != -999.0;
    printf("mode %d: active lanes %d/%d, warp cycles mean %.0f max %lld\n", mode, act, nb * 32, s / nb, mx);
  }
  long long hst[4];
  cudaMemcpyFromSymbol(hst, g_st, sizeof(hst));
  printf("1-lane totals (2 reps x 64 edges pairs): first-run cyc %lld cheap steps %lld exact rounds %lld exact-phase cyc %lld\n", hst[0], hst[1], hst[2], hst[3]);
  for (int m = 0; m < 2; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      if (m == 0) kp<1><<<nb, 32>>>(dF, r_lt2, mb_le2, cyc, out);
      else kp<32><<<nb, 32>>>(dF, r_lt2, mb_le2, cyc, out);
    }
    cudaDeviceSynchronize();
    cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < nb; ++i) s += hc[i];
    printf("pair_info %d lanes: warp cycles mean %.0f\n", m ? 32 : 1, s / nb);
  }
  int diff = 0;
  for (int i = 0; i < nb * 32; ++i) diff += ho[0][i] != ho[1][i];
  printf("mismatches %d; %s\n", diff, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
