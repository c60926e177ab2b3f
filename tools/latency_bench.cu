// Dev tool: dependent-chain latency (cycles/op) of FP64 and FP32 ops on this
// GPU, one warp, clock64.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>

#define CHAIN(name, T, init, expr)                                             \
  __global__ void k_##name(T* out, long long* cyc, int n) {                    \
    T x = init + threadIdx.x * (T)1e-9;                                        \
    const T y = (T)1.0000001;                                                  \
    long long t0 = clock64();                                                  \
    for (int i = 0; i < n; ++i) { expr; }                                      \
    long long t1 = clock64();                                                  \
    out[threadIdx.x] = x;                                                      \
    if (threadIdx.x == 0) *cyc = t1 - t0;                                      \
  }

CHAIN(dadd, double, 1.0, x = __dadd_rn(x, y))
CHAIN(dmul, double, 1.0, x = __dmul_rn(x, y))
CHAIN(dfma, double, 1.0, x = fma(x, y, 1e-12))
CHAIN(ddiv, double, 1.0, x = __ddiv_rn(y, x))
CHAIN(dsqrt, double, 2.0, x = __dsqrt_rn(x + 1.0))
CHAIN(fadd, float, 1.0f, x = __fadd_rn(x, y))
CHAIN(ffma, float, 1.0f, x = fmaf(x, y, 1e-7f))
CHAIN(fdiv, float, 1.0f, x = y / x)
CHAIN(fsqrt, float, 2.0f, x = sqrtf(x + 1.0f))
CHAIN(frsq, float, 2.0f, x = rsqrtf(x) + 1.0f)
CHAIN(datan2, double, 0.5, x = atan2(x, y) + 0.5)
// compare-dependent chains: the select consumes the predicate
CHAIN(dsetp, double, 1.0, x = (x < y) ? __dadd_rn(x, 1e-9) : __dsub_rn(x, 1e-9))
CHAIN(fsetp, float, 1.0f, x = (x < y) ? __fadd_rn(x, 1e-7f) : __fsub_rn(x, 1e-7f))
CHAIN(dmidp, double, 1.0, x = __dmul_rn(0.5, __dadd_rn(x, y)); x = (x == y) ? 1.0 : x)
// one integer bisection step: midpoint of two int64 ends, compare, select
CHAIN(imid, long long, 1000000007LL, x = (x + (long long)y * 3 + 12345) >> 1; x = (x > 500000000LL) ? x : x + 777)
CHAIN(iadd, long long, 1LL, x = x + (x >> 7) + 3)

template <typename T>
void run(const char* name, void (*k)(T*, long long*, int), int warps) {
  T* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(T));
  cudaMalloc(&cyc, sizeof(long long));
  const int n = 2000;
  k<<<1, 32 * warps>>>(out, cyc, n);
  k<<<1, 32 * warps>>>(out, cyc, n);
  long long c = 0;
  cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  printf("%-7s warps=%2d  %.1f cycles/op\n", name, warps, double(c) / n);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {1, 16}) {
    run<double>("dadd", k_dadd, w);
    run<double>("dmul", k_dmul, w);
    run<double>("dfma", k_dfma, w);
    run<double>("ddiv", k_ddiv, w);
    run<double>("dsqrt", k_dsqrt, w);
    run<double>("datan2", k_datan2, w);
    run<double>("dsetp", k_dsetp, w);
    run<double>("dmidp", k_dmidp, w);
    run<float>("fsetp", k_fsetp, w);
    run<long long>("imid", k_imid, w);
    run<long long>("iadd", k_iadd, w);
    run<float>("fadd", k_fadd, w);
    run<float>("ffma", k_ffma, w);
    run<float>("fdiv", k_fdiv, w);
    run<float>("fsqrt", k_fsqrt, w);
    run<float>("frsq", k_frsq, w);
  }
  return 0;
}
