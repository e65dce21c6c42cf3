// Dependent-chain latency probe (tuning tool, not product): cycles per operation of
// the FP64 / shuffle / shared-memory operations on the rollout kernel's serial
// per-step chain (one warp, one CTA, clock64 around 1024 dependent operations).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_probe tools/lat_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 1024;

__global__ void probe(double *out, long long *cyc, double seed) {
  __shared__ double sh[64];
  __shared__ float shf[64];
  const int lane = threadIdx.x & 31;
  sh[lane] = seed + lane;
  sh[lane + 32] = seed - lane;
  shf[lane] = (float)lane;
  __syncwarp();
  double x = seed + lane * 1e-3, y = 1.0000001;
  float xf = (float)x;
  long long t0, t1;
  int k = 0;
#define MEASURE(...)                     \
  t0 = clock64();                        \
  _Pragma("unroll 16") for (int i = 0; i < N; ++i) { __VA_ARGS__; } \
  t1 = clock64();                        \
  if (lane == 0) cyc[k] = (t1 - t0);     \
  ++k;
  MEASURE(x = x + y)                                                  // 0 DADD
  MEASURE(x = x * y)                                                  // 1 DMUL
  MEASURE(x = fma(x, y, 1e-9))                                        // 2 DFMA
  MEASURE(x = __shfl_xor_sync(0xffffffffu, x, 1))                     // 3 SHFL f64 (2x32)
  MEASURE(xf = __shfl_xor_sync(0xffffffffu, xf, 1))                   // 4 SHFL f32
  MEASURE(x = sh[(int)x & 31])                                        // 5 LDS.64 + F2I
  MEASURE(x = sqrt(x + 2.0))                                          // 6 DSQRT (+DADD)
  MEASURE(x = 1.0 / (x + 2.0))                                        // 7 DDIV (+DADD)
  MEASURE({ double s_, c_; sincos(x, &s_, &c_); x = s_ + c_; })      // 8 sincos f64
  MEASURE(x = atan2(x, 1.5))                                          // 9 atan2 f64
  MEASURE(xf = xf * 1.0001f + 1e-7f)                                  // 10 FFMA f32
  MEASURE(x = (double)shf[(int)xf & 31] + x)                          // 11 LDS.32 + F2F + DADD
  MEASURE(x = x + (double)__shfl_xor_sync(0xffffffffu, xf, 1))       // 12
  out[threadIdx.x] = x + xf;
#undef MEASURE
}

int main() {
  double *out;
  long long *cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMallocManaged(&cyc, 64 * sizeof(long long));
  probe<<<1, 32>>>(out, cyc, 0.5);
  cudaDeviceSynchronize();
  probe<<<1, 32>>>(out, cyc, 0.5);
  cudaDeviceSynchronize();
  const char *names[] = {"DADD", "DMUL", "DFMA", "SHFL f64", "SHFL f32", "LDS.64 dep", "sqrt f64",
                         "div f64", "sincos f64", "atan2 f64", "FFMA f32", "LDS.32+F2F+DADD",
                         "SHFL f32 + F2F + DADD"};
  for (int i = 0; i < 13; ++i) printf("{\"op\":\"%s\",\"cycles\":%.1f}\n", names[i], cyc[i] / (double)N);
  return 0;
}
