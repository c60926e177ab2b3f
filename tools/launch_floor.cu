// Dev tool: host-measured launch+sync floor of the single-frame call shape --
// a CUDA graph of two kernels (PDL edge), with small or 5 KB by-value
// parameters, grids of 512 CTAs -- against plain launches.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/launch_floor tools/launch_floor.cu
#include <chrono>
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

struct Big { char b[5120]; };

__global__ void k_small(int* x) { if (threadIdx.x == 0 && x[blockIdx.x] == 12345) x[0] = 1; }
__global__ void k_big(int* x, const __grid_constant__ Big b) {
  if (threadIdx.x == 0 && x[blockIdx.x] == b.b[blockIdx.x % 5120]) x[0] = 1;
}
__global__ void k_small_pdl(int* x) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && x[blockIdx.x] == 12345) x[0] = 1;
}
__global__ void k_big_pdl(int* x, const __grid_constant__ Big b) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && x[blockIdx.x] == b.b[blockIdx.x % 5120]) x[0] = 1;
}

template <class F>
double p50(F f, int reps = 2000) {
  std::vector<double> t;
  for (int i = 0; i < reps + 50; ++i) {
    auto a = std::chrono::steady_clock::now();
    f();
    auto b = std::chrono::steady_clock::now();
    if (i >= 50) t.push_back(std::chrono::duration<double, std::micro>(b - a).count());
  }
  std::sort(t.begin(), t.end());
  return t[t.size() / 2];
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  int* x;
  cudaMalloc(&x, 4096 * sizeof(int));
  cudaMemset(x, 0, 4096 * sizeof(int));
  Big big{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  auto launch2 = [&](bool bigp, bool pdl) {
    cudaLaunchConfig_t c{};
    c.gridDim = 512; c.blockDim = 256; c.stream = s;
    if (bigp) cudaLaunchKernelEx(&c, k_big, x, big); else cudaLaunchKernelEx(&c, k_small, x);
    c.attrs = attr; c.numAttrs = pdl ? 1 : 0;
    if (bigp) cudaLaunchKernelEx(&c, k_big_pdl, x, big); else cudaLaunchKernelEx(&c, k_small_pdl, x);
  };
  for (int bigp = 0; bigp < 2; ++bigp) {
    for (int pdl = 0; pdl < 2; ++pdl) {
      double plain = p50([&] { launch2(bigp, pdl); cudaStreamSynchronize(s); });
      cudaGraph_t g; cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      launch2(bigp, pdl);
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaGraphUpload(ge, s);
      double gr = p50([&] { cudaGraphLaunch(ge, s); cudaStreamSynchronize(s); });
      std::printf("params=%s pdl=%d: plain launches+sync p50 %.1f us, graph launch+sync p50 %.1f us\n",
                  bigp ? "5KB" : "8B", pdl, plain, gr);
      cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    }
  }
  double one = p50([&] { k_small<<<1, 32, 0, s>>>(x); cudaStreamSynchronize(s); });
  std::printf("one 1-CTA kernel + sync p50 %.1f us\n", one);
  return 0;
}
