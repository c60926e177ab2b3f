// fp_peak.cu -- measured FP32 / FP64 pipe throughput of this B200 (the
// roofline denominators bench.py uses; MEASURED_PEAKS.json has only HBM and
// bf16 tensor figures).  Each thread runs kChains independent FMA chains so
// the pipes, not latency, bound the loop; the grid is a multiple of the SM
// count.  FLOP = 2 per FMA.  Timed with CUDA events after a warm-up.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp_peak tools/fp_peak.cu
//   tools/fp_peak > profiles/fp_peaks.json
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;

template <typename T>
__global__ void __launch_bounds__(256) fma_loop(T* out, int iters, T a, T b) {
  T x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = static_cast<T>(threadIdx.x + c);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int c = 0; c < kChains; ++c) x[c] = x[c] * a + b;  // one FMA (contracted)
    }
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == static_cast<T>(-1.2345)) out[threadIdx.x] = s;  // keep the chains alive
}

template <typename T>
double run(int sms, int blocks_per_sm, int iters, float* ms_out) {
  T* out;
  cudaMalloc(&out, 1024 * sizeof(T));
  const int blocks = sms * blocks_per_sm;
  const T a = static_cast<T>(0.999999), b = static_cast<T>(1e-7);
  fma_loop<T><<<blocks, 256>>>(out, iters, a, b);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    fma_loop<T><<<blocks, 256>>>(out, iters, a, b);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaFree(out);
  *ms_out = best;
  const double fmas = double(blocks) * 256 * iters * 16 * kChains;
  return 2.0 * fmas / (best * 1e-3) / 1e12;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int sms = prop.multiProcessorCount;
  float ms32, ms64;
  const double t32 = run<float>(sms, 8, 4096, &ms32);
  const double t64 = run<double>(sms, 8, 256, &ms64);
  std::printf(
      "{\"device\": \"%s\", \"sms\": %d, \"clock_mhz_attr\": %.0f, \"fp32_tflops\": %.2f, "
      "\"fp32_ms\": %.3f, \"fp64_tflops\": %.3f, \"fp64_ms\": %.3f, \"how\": \"tools/fp_peak.cu: "
      "%d independent FMA chains per thread, 256 threads x 8 CTAs per SM x %d SMs, best of 5 "
      "event-timed launches, 2 FLOP per FMA\"}\n",
      prop.name, sms, clk_khz / 1e3, t32, ms32, t64, ms64, kChains, sms);
  return 0;
}
