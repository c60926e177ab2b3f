// Dev tool: checks pp::ddiv_fast against __ddiv_rn bit for bit on random
// operands (wide exponent ranges, near-tie cases).  Not used by tests/bench.
#include <cstdio>
#include <cstdint>
#include "../paper_1909_07717_b200/csrc/pp_kernels.cuh"

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return x;
}

__global__ void k(unsigned long long* bad, unsigned long long* slow, long long n, int range) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const uint64_t r1 = mix(i * 2 + 1 + range * 0x9e3779b97f4a7c15ULL), r2 = mix(i * 2 + 2 + range);
    double a, b;
    if (range == 0) {         // geometry-like magnitudes
      a = (double)(int64_t)(r1 >> 11) * 1e-15;  // |a| up to ~1e3
      b = 1e-6 + (double)(r2 >> 11) * 1e-13;
    } else if (range == 1) {  // random bit patterns with exponents in [-300, 300]
      a = __longlong_as_double((long long)((r1 & 0x800fffffffffffffULL) | ((uint64_t)(1023 + (int)(r1 % 601) - 300) << 52)));
      b = __longlong_as_double((long long)((r2 & 0x800fffffffffffffULL) | ((uint64_t)(1023 + (int)(r2 % 601) - 300) << 52)));
    } else {                  // products of small integers (exact / tie-prone quotients)
      a = (double)((r1 % 1000003) + 1) * (double)((r2 % 4096) + 1);
      b = (double)((r2 % 1000003) + 1);
    }
    bool ok;
    const double q = pp::ddiv_fast(a, b, &ok);
    if (!ok) { atomicAdd(slow, 1ull); continue; }
    if (__double_as_longlong(q) != __double_as_longlong(__ddiv_rn(a, b))) atomicAdd(bad, 1ull);
  }
}

int main() {
  unsigned long long *bad, *slow, hb, hs;
  cudaMalloc(&bad, 8); cudaMalloc(&slow, 8);
  const long long n = 1LL << 32;
  for (int range = 0; range < 3; ++range) {
    cudaMemset(bad, 0, 8); cudaMemset(slow, 0, 8);
    k<<<148 * 16, 256>>>(bad, slow, n, range);
    cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&hs, slow, 8, cudaMemcpyDeviceToHost);
    printf("range %d: %lld quotients, %llu mismatches, %llu slow-path\n", range, n, hb, hs);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
