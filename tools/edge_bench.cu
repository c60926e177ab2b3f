// Dev tool: latency of one goal-view interval-edge bisection (interval_edge)
// per warp, on synthetic tangent-geometry pairs.  Not used by tests/bench.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o tools/edge_bench tools/edge_bench.cu
#include <cstdio>
#define PP_EDGE_TRACE
__device__ long long g_trace[128];
__device__ double g_trace_w[64], g_trace_d[64];
#include "../paper_1909_07717_b200/csrc/pp_kernels.cuh"

using namespace pp;


__device__ xd edge_traced(const ViewCtx& V, xd cx, xd cy, int edge, int first, int last, bool fast,
                          xd y1, xd y2, double margin) {
  if (edge == 0 && first == 0) return -V.gh;
  if (edge == 1 && last == V.nh - 1) return V.gh;
  xd y_blocked = edge == 0 ? height_at(V, first) : height_at(V, last);
  xd y_free = edge == 0 ? height_at(V, first - 1) : height_at(V, last + 1);
  const double lo_in = y1.v + margin, hi_in = y2.v - margin;
  const double lo_out = y1.v - margin, hi_out = y2.v + margin;
  auto decide = [&](double y) -> int {
    if (!fast) return 2;
    if (y > lo_in && y < hi_in) return 1;
    if (y < lo_out || y > hi_out) return 0;
    return 2;
  };
  int i = 0, n = 0;
  while (i < 60) {
    g_trace[n++ & 127] = clock64();
    const xd mid = xd(0.5) * (y_blocked + y_free);
    if (mid.v == y_blocked.v || mid.v == y_free.v) break;
    const int d0 = decide(mid.v);
    if (d0 != 2) {
      if (d0) y_blocked = mid; else y_free = mid;
      ++i;
      continue;
    }
    y_free = mid;  // (trace only measures the cheap path)
    ++i;
  }
  g_trace[127] = n;
  return xd(0.5) * (y_blocked + y_free);
}

template <int kMode>
__global__ void k_edge(const FrameDev* F_, double r_lt2, double mb_le2, long long* cyc, double* out,
                       int* n_exact) {
  __shared__ FrameDev F;
  load_frame(&F, F_);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  // point on the field, opponent 1.5 m ahead toward the goal, lateral jitter
  const xd px = -1.0 + 0.05 * (threadIdx.x % 7), py = -0.8 + 0.05 * lane;
  const xd cx = px + 1.5, cy = py * 0.5 + 0.01 * (lane % 5);
  const ViewCtx V = make_view_ctx(px, py, F, 0.09, r_lt2, mb_le2);
  const PairInfo pi = pair_info(V, cx, cy);
  const bool active = pi.status == 1;
  double acc = 0.0;
  __syncwarp();
  const long long t0 = clock64();
  for (int edge = 0; edge < 2; ++edge) {
    xd y;
    if (kMode == 0) {
      y = active ? interval_edge(V, cx, cy, edge, pi.first, pi.last, pi.fast, pi.y1, pi.y2, pi.margin) : xd(0.0);
    } else if (kMode == 2) {
      y = active ? interval_edge(V, cx, cy, edge, pi.first, pi.last, pi.fast, pi.y1, pi.y2, 0.0) : xd(0.0);
    } else if (kMode == 4) {
      y = active ? edge_traced(V, cx, cy, edge, pi.first, pi.last, pi.fast, pi.y1, pi.y2, 0.0) : xd(0.0);
    } else if (kMode == 3) {
      y = active ? interval_edge(V, cx, cy, edge, pi.first, pi.last, false, pi.y1, pi.y2, pi.margin) : xd(0.0);
    } else {
      y = active ? interval_edge(V, cx, cy, edge, pi.first, pi.last, pi.fast, pi.y1, pi.y2, pi.margin) : xd(0.0);
    }
    acc += y.v;
  }
  __syncwarp();
  const long long t1 = clock64();
  if (active && kMode == 0 && blockIdx.x == 0) { g_trace[120] = t0; g_trace[121] = t1; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (lane == 0) cyc[blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5)] = t1 - t0;
  if (threadIdx.x == 0 && blockIdx.x == 0) *n_exact = __popc(__ballot_sync(0xffffffffu, active));

}

int main() {
  FrameDev F{};
  F.L = 12.0; F.W = 9.0; F.gw = 1.8;  // SSL division B
  F.n_theirs = 0;
  FrameDev* dF;
  cudaMalloc(&dF, sizeof(F));
  cudaMemcpy(dF, &F, sizeof(F), cudaMemcpyHostToDevice);
  const double r = 0.09;
  const double r_lt2 = r * r, mb_le2 = (r + 1e-9) * (r + 1e-9);
  long long* cyc; double* out; int* ne;
  cudaMalloc(&cyc, 1 << 20); cudaMalloc(&out, 1 << 20); cudaMalloc(&ne, 4);
  long long h[4096];
  int hn = 0;
  for (int mode = 4; mode >= 0; mode -= 2) {
    for (int cfg = 0; cfg < 1; ++cfg) {
      const int blocks = cfg == 0 ? 1 : 148 * 2, threads = cfg == 2 ? 256 : 32;
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) k_edge<0><<<blocks, threads>>>(dF, r_lt2, mb_le2, cyc, out, ne);
        else if (mode == 1) k_edge<1><<<blocks, threads>>>(dF, r_lt2, mb_le2, cyc, out, ne);
        else if (mode == 2) k_edge<2><<<blocks, threads>>>(dF, r_lt2, mb_le2, cyc, out, ne);
        else if (mode == 3) k_edge<3><<<blocks, threads>>>(dF, r_lt2, mb_le2, cyc, out, ne);
        else k_edge<4><<<blocks, threads>>>(dF, r_lt2, mb_le2, cyc, out, ne);
      }
      cudaDeviceSynchronize();
      const int nw = blocks * threads / 32;
      cudaMemcpy(h, cyc, sizeof(long long) * (nw < 4096 ? nw : 4096), cudaMemcpyDeviceToHost);
      cudaMemcpy(&hn, ne, 4, cudaMemcpyDeviceToHost);
      double s = 0; long long mx = 0;
      const int m = nw < 4096 ? nw : 4096;
      for (int i = 0; i < m; ++i) { s += h[i]; mx = h[i] > mx ? h[i] : mx; }
      printf("mode %d blocks %d threads %d: active lanes %d, cycles per warp (2 edges) mean %.0f max %lld\n",
             mode, blocks, threads, hn, s / m, mx);
    }
  }
  long long tr[128];
  cudaMemcpyFromSymbol(tr, g_trace, sizeof(tr));
  printf("trace n=%lld: first-t0 %lld  t1-last %lld |", tr[127], tr[0] - tr[120], tr[121] - tr[(tr[127] - 1) & 127]);
  for (int i = 1; i < 60 && i < tr[127]; ++i) printf(" %lld", tr[i] - tr[i - 1]);
  double tw[64], td[64];
  cudaMemcpyFromSymbol(tw, g_trace_w, sizeof(tw));
  cudaMemcpyFromSymbol(td, g_trace_d, sizeof(td));
  printf("\n");
  for (int i = 0; i < 60 && i < tr[127]; ++i) printf("it %d dt %lld width %.3g dist-to-edge %.3g\n", i, i ? tr[i] - tr[i-1] : 0, tw[i], td[i]);
  printf("\n%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
