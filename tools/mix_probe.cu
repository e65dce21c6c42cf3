// Pipe-mix probe: can the FMA pipe and the MUFU pipe run at their rates together?
// Kernel A: per "interaction" 4 packed FP32 ops (= 8 lane-ops) + 1 MUFU.RSQ on
// independent chains (the direct Biot-Savart mix).  Kernel B: the real sweep loop
// (packed pairs, LDS.128 broadcast sources) over n sources in shared memory.
// Reports interactions / clk / SM.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
// -o tools/mix_probe tools/mix_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float rsq(float v) {
  float r;
  asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

// NF packed FP32 ops and NM MUFU.RSQ per 2 "interactions", C independent chains.
template <int C, int NF, int NM>
__global__ void mix_kernel(float *out, int iters, float a) {
  float2 v[C], w[C];
  const float2 A = make_float2(a, a);
#pragma unroll
  for (int i = 0; i < C; ++i) {
    v[i] = make_float2(1.f + threadIdx.x * 1e-3f + i, 2.f + i);
    w[i] = make_float2(0.5f, 0.25f);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < C; ++i) {
      float2 t = v[i];
#pragma unroll
      for (int f = 0; f < NF - 1; ++f) t = __ffma2_rn(t, A, w[i]);
      if constexpr (NM == 2) t = make_float2(rsq(t.x), rsq(t.y));
      if constexpr (NM == 1) t.x = rsq(t.x);
      v[i] = __ffma2_rn(t, A, v[i]);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < C; ++i) s += v[i].x + v[i].y + w[i].x + w[i].y;
  if (s == 1.2345f) out[blockIdx.x] = s;
}

template <int KP, int UN>
__global__ void sweep_kernel(float *out, int n, int reps, float rc4) {
  extern __shared__ float4 src[];
  for (int j = threadIdx.x; j < n; j += blockDim.x)
    src[j] = make_float4(0.01f * j, 0.02f * (j & 7), 1e-3f * (j & 3), 0.f);
  __syncthreads();
  float2 px[KP], pz[KP], qx[KP], qz[KP];
#pragma unroll
  for (int p = 0; p < KP; ++p) {
    px[p] = make_float2(-0.013f * (threadIdx.x + p), -0.017f * p);
    pz[p] = make_float2(-0.011f * p, -0.019f * (threadIdx.x & 3));
    qx[p] = qz[p] = make_float2(0.f, 0.f);
  }
  const float2 rc = make_float2(rc4, rc4);
  for (int r = 0; r < reps; ++r) {
#pragma unroll UN
    for (int j = 0; j < n; ++j) {
      const float4 s = src[j];
      const float2 sx = make_float2(s.x, s.x), sz = make_float2(s.y, s.y), sg = make_float2(s.z, s.z);
#pragma unroll
      for (int p = 0; p < KP; ++p) {
        const float2 dx = __fadd2_rn(sx, px[p]);
        const float2 dz = __fadd2_rn(sz, pz[p]);
        const float2 r2 = __ffma2_rn(dx, dx, __fmul2_rn(dz, dz));
        const float2 q = __ffma2_rn(r2, r2, rc);
        const float2 rs = make_float2(rsq(q.x), rsq(q.y));
        const float2 c = __fmul2_rn(sg, rs);
        qx[p] = __ffma2_rn(c, dz, qx[p]);
        qz[p] = __ffma2_rn(c, dx, qz[p]);
      }
    }
    __syncthreads();
  }
  float s = 0.f;
#pragma unroll
  for (int p = 0; p < KP; ++p) s += qx[p].x + qx[p].y + qz[p].x + qz[p].y;
  if (s == 1.2345f) out[blockIdx.x] = s;
}

// Symmetric-pair tile: lane holds 2*KP "i" targets (packed pairs) and one rotating
// "j" particle whose data (x, z, g) and packed accumulator travel one lane per step
// (7 SHFL per step); every (i, j) pair is evaluated once and updates both sides.
template <int KP>
__global__ void sym_kernel(float *out, int reps, float rc4) {
  const int lane = threadIdx.x & 31;
  float2 px[KP], pz[KP], pg[KP], ax[KP], az[KP];
#pragma unroll
  for (int p = 0; p < KP; ++p) {
    px[p] = make_float2(0.013f * (lane + p), 0.017f * p);
    pz[p] = make_float2(0.011f * p, 0.019f * (lane & 3));
    pg[p] = make_float2(1e-3f * (p + 1), -1e-3f * (lane & 1));
    ax[p] = az[p] = make_float2(0.f, 0.f);
  }
  float jx = 0.021f * lane, jz = -0.01f * lane, jg = 2e-3f;
  float2 bx = make_float2(0.f, 0.f), bz = make_float2(0.f, 0.f);
  const float2 rc = make_float2(rc4, rc4);
  for (int r = 0; r < reps; ++r) {
#pragma unroll 4
    for (int k = 0; k < 32; ++k) {
      const float2 sx = make_float2(jx, jx), sz = make_float2(jz, jz), sg = make_float2(jg, jg);
#pragma unroll
      for (int p = 0; p < KP; ++p) {
        const float2 dx = __fadd2_rn(sx, px[p]);
        const float2 dz = __fadd2_rn(sz, pz[p]);
        const float2 r2 = __ffma2_rn(dx, dx, __fmul2_rn(dz, dz));
        const float2 q = __ffma2_rn(r2, r2, rc);
        const float2 rs = make_float2(rsq(q.x), rsq(q.y));
        const float2 ci = __fmul2_rn(sg, rs);
        ax[p] = __ffma2_rn(ci, dz, ax[p]);
        az[p] = __ffma2_rn(ci, dx, az[p]);
        const float2 cj = __fmul2_rn(pg[p], rs);
        bx = __ffma2_rn(cj, dz, bx);
        bz = __ffma2_rn(cj, dx, bz);
      }
      const int src = (lane + 1) & 31;
      jx = __shfl_sync(0xffffffffu, jx, src);
      jz = __shfl_sync(0xffffffffu, jz, src);
      jg = __shfl_sync(0xffffffffu, jg, src);
      bx.x = __shfl_sync(0xffffffffu, bx.x, src);
      bx.y = __shfl_sync(0xffffffffu, bx.y, src);
      bz.x = __shfl_sync(0xffffffffu, bz.x, src);
      bz.y = __shfl_sync(0xffffffffu, bz.y, src);
    }
  }
  float s = jx + bx.x + bx.y + bz.x + bz.y;
#pragma unroll
  for (int p = 0; p < KP; ++p) s += ax[p].x + ax[p].y + az[p].x + az[p].y;
  if (s == 1.2345f) out[blockIdx.x] = s;
}

static int g_sms, g_clk_khz;

template <typename F>
static float time_ms(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaEventRecord(a);
  f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

template <int C, int NF, int NM>
static void run_mix(float *out, int blocks_per_sm, int threads) {
  const int iters = 2048;
  const int grid = g_sms * blocks_per_sm * 4;
  float ms = time_ms([&] { mix_kernel<C, NF, NM><<<grid, threads>>>(out, iters, 0.999f); });
  const double pairs = (double)grid * threads * iters * C;
  const double clk = ms * 1e-3 * g_clk_khz * 1e3;
  printf("{\"probe\":\"mix\",\"packed_fp32\":%d,\"mufu\":%d,\"chains\":%d,\"ctas\":%d,"
         "\"lane_fp32_per_clk_sm\":%.1f,\"mufu_per_clk_sm\":%.2f,\"cyc_per_pair_smsp\":%.2f}\n",
         NF, NM, C, blocks_per_sm, pairs * NF * 2 / clk / g_sms, pairs * NM / clk / g_sms,
         clk * g_sms * 4 / (pairs / 32));
}

template <int KP, int UN = 2>
static void run_sweep(float *out, int n, int threads, int ctas_per_sm) {
  const int reps = 40;
  const int grid = g_sms * ctas_per_sm * 4;
  const size_t smem = n * 16;
  float ms = time_ms([&] { sweep_kernel<KP, UN><<<grid, threads, smem>>>(out, n, reps, 1e-4f); });
  const double inter = (double)grid * threads * 2 * KP * n * reps;
  const double clk = ms * 1e-3 * g_clk_khz * 1e3;
  printf("{\"probe\":\"sweep\",\"unroll\":%d,\"pairs\":%d,\"n\":%d,\"threads\":%d,\"ctas\":%d,\"inter_per_clk_sm\":%.2f}\n", UN, KP, n,
         threads, ctas_per_sm, inter / clk / g_sms);
}

template <int KP>
static void run_sym(float *out, int threads, int ctas_per_sm) {
  const int reps = 200;
  const int grid = g_sms * ctas_per_sm * 4;
  float ms = time_ms([&] { sym_kernel<KP><<<grid, threads>>>(out, reps, 1e-4f); });
  // directed interactions: 2 per (i, j) pair; 2*KP pairs per lane per step
  const double inter = (double)grid * threads * reps * 32 * 2 * KP * 2;
  const double clk = ms * 1e-3 * g_clk_khz * 1e3;
  printf("{\"probe\":\"sym\",\"pairs\":%d,\"threads\":%d,\"ctas\":%d,\"directed_per_clk_sm\":%.2f}\n", KP, threads,
         ctas_per_sm, inter / clk / g_sms);
}

int main() {
  cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&g_clk_khz, cudaDevAttrClockRate, 0);
  float *out;
  cudaMalloc(&out, 1 << 24);
  run_sweep<2, 8>(out, 512, 128, 7);
  for (int c : {4, 7}) {
    run_sym<1>(out, 128, c);
    run_sym<2>(out, 128, c);
    run_sym<3>(out, 128, c);
    run_sym<4>(out, 128, c);
  }
  printf("{\"sms\":%d,\"clk_mhz\":%d}\n", g_sms, g_clk_khz / 1000);
  return 0;
}
