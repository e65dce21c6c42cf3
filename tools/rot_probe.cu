// Symmetric-pair probe with lane rotation (tuning tool, not product).
//
//   direct : the rollout kernel's loop -- 4 targets per lane (2 packed pairs),
//            sources as LDS.128 broadcasts: 8 lane-ops + 1 MUFU.RSQ per directed
//            interaction.
//   rot    : each unordered pair once.  A lane holds 4 targets (2 packed pairs) and
//            one "packet" source of a 32-source block; the packet -- source
//            coordinates and the reaction accumulated on it so far -- moves one
//            lane per step, so after 32 steps every target met every source of the
//            block, each reaction was summed in a fixed lane order and the packet
//            is back in its home lane (no cross-lane reduction, no atomics).
//            ACC2=1: the reaction travels as two float2 partials (7 SHFL / step),
//            ACC2=0: folded to scalars every step (5 SHFL, 2 extra FADD).
//            NPK packets per step interleave independent rotations (ILP).
// Prints directed interactions / clk / SM (a symmetric pair counts twice).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/rot_probe tools/rot_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float rsq(float v) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

__device__ void fill(float4 *src, int n) {
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const float x = 0.01f * j, z = 0.02f * (j & 7), g = 1e-3f * ((j & 3) + 1);
    src[j] = make_float4(x, z, g, 0.f);
  }
  __syncthreads();
}

template <int MAXREG>
__global__ void __maxnreg__(MAXREG) direct_kernel(float *out, int n, int reps, float rc4) {
  extern __shared__ float4 src[];
  fill(src, n);
  float2 px[2], pz[2], qx[2], qz[2];
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    px[p] = make_float2(-0.013f * (threadIdx.x + p), -0.017f * p);
    pz[p] = make_float2(-0.011f * p, -0.019f * (threadIdx.x & 3));
    qx[p] = qz[p] = make_float2(0.f, 0.f);
  }
  const float2 rc = make_float2(rc4, rc4);
  for (int r = 0; r < reps; ++r) {
#pragma unroll 8
    for (int j = 0; j < n; ++j) {
      const float4 s = src[j];
      const float2 sx = make_float2(s.x, s.x), sz = make_float2(s.y, s.y), sg = make_float2(s.z, s.z);
#pragma unroll
      for (int p = 0; p < 2; ++p) {
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
  }
  float s = 0.f;
#pragma unroll
  for (int p = 0; p < 2; ++p) s += qx[p].x + qx[p].y + qz[p].x + qz[p].y;
  if (s == 1.2345f) out[blockIdx.x] = s;
}

template <int NPK, int ACC2, int MAXREG, int UNR, int KPT = 2>
__global__ void __maxnreg__(MAXREG) rot_kernel(float *out, int n, int reps, float rc4) {
  extern __shared__ float4 src[];
  fill(src, n);
  float *part = reinterpret_cast<float *>(src + n);
  const int lane = threadIdx.x & 31;
  float2 px[KPT], pz[KPT], pg[KPT], qx[KPT], qz[KPT];
#pragma unroll
  for (int p = 0; p < KPT; ++p) {
    px[p] = make_float2(-0.013f * (threadIdx.x + p), -0.017f * p);
    pz[p] = make_float2(-0.011f * p, -0.019f * (threadIdx.x & 3));
    pg[p] = make_float2(1e-3f * (p + 1), -1e-3f * (lane & 1));
    qx[p] = qz[p] = make_float2(0.f, 0.f);
  }
  const float2 rc = make_float2(rc4, rc4);
  const int nxt = (lane + 1) & 31;
  for (int rep = 0; rep < reps; ++rep) {
    for (int J0 = 0; J0 < n / 32; J0 += NPK) {
      float sx[NPK], sz[NPK], sg[NPK];
      float2 bx[NPK], bz[NPK];
      float bxs[NPK], bzs[NPK];
#pragma unroll
      for (int k = 0; k < NPK; ++k) {
        const float4 s = src[32 * (J0 + k) + lane];
        sx[k] = s.x;
        sz[k] = s.y;
        sg[k] = s.z;
        bx[k] = bz[k] = make_float2(0.f, 0.f);
        bxs[k] = bzs[k] = 0.f;
      }
#pragma unroll UNR
      for (int r = 0; r < 32; ++r) {
#pragma unroll
        for (int k = 0; k < NPK; ++k) {
          const float2 sx2 = make_float2(sx[k], sx[k]), sz2 = make_float2(sz[k], sz[k]),
                       sg2 = make_float2(sg[k], sg[k]);
          float2 tx = make_float2(0.f, 0.f), tz = make_float2(0.f, 0.f);
#pragma unroll
          for (int p = 0; p < KPT; ++p) {
            const float2 dx = __fadd2_rn(sx2, px[p]);
            const float2 dz = __fadd2_rn(sz2, pz[p]);
            const float2 r2 = __ffma2_rn(dx, dx, __fmul2_rn(dz, dz));
            const float2 q = __ffma2_rn(r2, r2, rc);
            const float2 rs = make_float2(rsq(q.x), rsq(q.y));
            const float2 cj = __fmul2_rn(sg2, rs);
            qx[p] = __ffma2_rn(cj, dz, qx[p]);
            qz[p] = __ffma2_rn(cj, dx, qz[p]);
            const float2 ci = __fmul2_rn(pg[p], rs);
            if (ACC2) {
              bx[k] = __ffma2_rn(ci, dz, bx[k]);
              bz[k] = __ffma2_rn(ci, dx, bz[k]);
            } else if (p == 0) {
              tx = __fmul2_rn(ci, dz);
              tz = __fmul2_rn(ci, dx);
            } else {
              tx = __ffma2_rn(ci, dz, tx);
              tz = __ffma2_rn(ci, dx, tz);
            }
          }
          if (!ACC2) {
            bxs[k] += tx.x + tx.y;
            bzs[k] += tz.x + tz.y;
          }
        }
#pragma unroll
        for (int k = 0; k < NPK; ++k) {
          sx[k] = __shfl_sync(0xffffffffu, sx[k], nxt);
          sz[k] = __shfl_sync(0xffffffffu, sz[k], nxt);
          sg[k] = __shfl_sync(0xffffffffu, sg[k], nxt);
          if (ACC2) {
            bx[k].x = __shfl_sync(0xffffffffu, bx[k].x, nxt);
            bx[k].y = __shfl_sync(0xffffffffu, bx[k].y, nxt);
            bz[k].x = __shfl_sync(0xffffffffu, bz[k].x, nxt);
            bz[k].y = __shfl_sync(0xffffffffu, bz[k].y, nxt);
          } else {
            bxs[k] = __shfl_sync(0xffffffffu, bxs[k], nxt);
            bzs[k] = __shfl_sync(0xffffffffu, bzs[k], nxt);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < NPK; ++k) {
        const int j = 32 * (J0 + k) + lane;
        part[2 * j] = ACC2 ? bx[k].x + bx[k].y : bxs[k];
        part[2 * j + 1] = ACC2 ? bz[k].x + bz[k].y : bzs[k];
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int p = 0; p < KPT; ++p) s += qx[p].x + qx[p].y + qz[p].x + qz[p].y;
  if (s == 1.2345f) out[blockIdx.x] = s;
}

// LDS-sourced rotation: the packet's coordinates are re-read from shared memory at the
// rotated index ((lane + r) & 31, a conflict-free 4-wavefront LDS.128) and only the
// reaction travels by shuffle: FOLD=0 two float2 partials (4 SHFL / step), FOLD=1
// folded to scalars every step (2 SHFL, 2 extra FADD).
template <int NPK, int FOLD, int MAXREG, int UNR>
__global__ void __maxnreg__(MAXREG) rotl_kernel(float *out, int n, int reps, float rc4) {
  extern __shared__ float4 src[];
  fill(src, n);
  float *part = reinterpret_cast<float *>(src + n);
  const int lane = threadIdx.x & 31;
  float2 px[2], pz[2], pg[2], qx[2], qz[2];
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    px[p] = make_float2(-0.013f * (threadIdx.x + p), -0.017f * p);
    pz[p] = make_float2(-0.011f * p, -0.019f * (threadIdx.x & 3));
    pg[p] = make_float2(1e-3f * (p + 1), -1e-3f * (lane & 1));
    qx[p] = qz[p] = make_float2(0.f, 0.f);
  }
  const float2 rc = make_float2(rc4, rc4);
  const int nxt = (lane + 1) & 31;
  for (int rep = 0; rep < reps; ++rep) {
    for (int J0 = 0; J0 < n / 32; J0 += NPK) {
      float2 bx[NPK], bz[NPK];
      float bxs[NPK], bzs[NPK];
#pragma unroll
      for (int k = 0; k < NPK; ++k) {
        bx[k] = bz[k] = make_float2(0.f, 0.f);
        bxs[k] = bzs[k] = 0.f;
      }
#pragma unroll UNR
      for (int r = 0; r < 32; ++r) {
#pragma unroll
        for (int k = 0; k < NPK; ++k) {
          const float4 s = src[32 * (J0 + k) + ((lane + r) & 31)];
          const float2 sx2 = make_float2(s.x, s.x), sz2 = make_float2(s.y, s.y), sg2 = make_float2(s.z, s.z);
          float2 tx = make_float2(0.f, 0.f), tz = make_float2(0.f, 0.f);
#pragma unroll
          for (int p = 0; p < 2; ++p) {
            const float2 dx = __fadd2_rn(sx2, px[p]);
            const float2 dz = __fadd2_rn(sz2, pz[p]);
            const float2 r2 = __ffma2_rn(dx, dx, __fmul2_rn(dz, dz));
            const float2 q = __ffma2_rn(r2, r2, rc);
            const float2 rs = make_float2(rsq(q.x), rsq(q.y));
            const float2 cj = __fmul2_rn(sg2, rs);
            qx[p] = __ffma2_rn(cj, dz, qx[p]);
            qz[p] = __ffma2_rn(cj, dx, qz[p]);
            const float2 ci = __fmul2_rn(pg[p], rs);
            if (!FOLD) {
              bx[k] = __ffma2_rn(ci, dz, bx[k]);
              bz[k] = __ffma2_rn(ci, dx, bz[k]);
            } else if (p == 0) {
              tx = __fmul2_rn(ci, dz);
              tz = __fmul2_rn(ci, dx);
            } else {
              tx = __ffma2_rn(ci, dz, tx);
              tz = __ffma2_rn(ci, dx, tz);
            }
          }
          if (FOLD) {
            bxs[k] += tx.x + tx.y;
            bzs[k] += tz.x + tz.y;
          }
        }
#pragma unroll
        for (int k = 0; k < NPK; ++k) {
          if (!FOLD) {
            bx[k].x = __shfl_sync(0xffffffffu, bx[k].x, nxt);
            bx[k].y = __shfl_sync(0xffffffffu, bx[k].y, nxt);
            bz[k].x = __shfl_sync(0xffffffffu, bz[k].x, nxt);
            bz[k].y = __shfl_sync(0xffffffffu, bz[k].y, nxt);
          } else {
            bxs[k] = __shfl_sync(0xffffffffu, bxs[k], nxt);
            bzs[k] = __shfl_sync(0xffffffffu, bzs[k], nxt);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < NPK; ++k) {
        const int j = 32 * (J0 + k) + lane;
        part[2 * j] = FOLD ? bxs[k] : bx[k].x + bx[k].y;
        part[2 * j + 1] = FOLD ? bzs[k] : bz[k].x + bz[k].y;
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int p = 0; p < 2; ++p) s += qx[p].x + qx[p].y + qz[p].x + qz[p].y;
  if (s == 1.2345f) out[blockIdx.x] = s;
}

// Source-packed rotation: each lane's packet holds two sources (float2), the four
// targets are scalar broadcasts: 10 shuffles per 8 pairs instead of 7 per 4.
template <int MAXREG, int UNR>
__global__ void __maxnreg__(MAXREG) rotsp_kernel(float *out, int n, int reps, float rc4) {
  extern __shared__ float4 src[];
  fill(src, n);
  float *part = reinterpret_cast<float *>(src + n);
  const int lane = threadIdx.x & 31;
  float tx[4], tz[4], tg[4];
  float2 ax[4], az[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    tx[i] = -0.013f * (threadIdx.x + i);
    tz[i] = -0.011f * i - 0.019f * (threadIdx.x & 3);
    tg[i] = 1e-3f * (i + 1) * ((lane & 1) ? -1.f : 1.f);
    ax[i] = az[i] = make_float2(0.f, 0.f);
  }
  const float2 rc = make_float2(rc4, rc4);
  const int nxt = (lane + 1) & 31;
  for (int rep = 0; rep < reps; ++rep) {
    for (int J0 = 0; J0 < n / 32; J0 += 2) {
      const float4 s0 = src[32 * J0 + lane], s1 = src[32 * J0 + 32 + lane];
      float2 sx = make_float2(s0.x, s1.x), sz = make_float2(s0.y, s1.y), sg = make_float2(s0.z, s1.z);
      float2 bx = make_float2(0.f, 0.f), bz = make_float2(0.f, 0.f);
#pragma unroll UNR
      for (int r = 0; r < 32; ++r) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 dx = __fadd2_rn(sx, make_float2(tx[i], tx[i]));
          const float2 dz = __fadd2_rn(sz, make_float2(tz[i], tz[i]));
          const float2 r2 = __ffma2_rn(dx, dx, __fmul2_rn(dz, dz));
          const float2 q = __ffma2_rn(r2, r2, rc);
          const float2 rs = make_float2(rsq(q.x), rsq(q.y));
          const float2 cj = __fmul2_rn(sg, rs);
          ax[i] = __ffma2_rn(cj, dz, ax[i]);
          az[i] = __ffma2_rn(cj, dx, az[i]);
          const float2 ci = __fmul2_rn(make_float2(tg[i], tg[i]), rs);
          bx = __ffma2_rn(ci, dz, bx);
          bz = __ffma2_rn(ci, dx, bz);
        }
        sx.x = __shfl_sync(0xffffffffu, sx.x, nxt);
        sx.y = __shfl_sync(0xffffffffu, sx.y, nxt);
        sz.x = __shfl_sync(0xffffffffu, sz.x, nxt);
        sz.y = __shfl_sync(0xffffffffu, sz.y, nxt);
        sg.x = __shfl_sync(0xffffffffu, sg.x, nxt);
        sg.y = __shfl_sync(0xffffffffu, sg.y, nxt);
        bx.x = __shfl_sync(0xffffffffu, bx.x, nxt);
        bx.y = __shfl_sync(0xffffffffu, bx.y, nxt);
        bz.x = __shfl_sync(0xffffffffu, bz.x, nxt);
        bz.y = __shfl_sync(0xffffffffu, bz.y, nxt);
      }
      part[2 * (32 * J0 + lane)] = bx.x;
      part[2 * (32 * J0 + lane) + 1] = bz.x;
      part[2 * (32 * J0 + 32 + lane)] = bx.y;
      part[2 * (32 * J0 + 32 + lane) + 1] = bz.y;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += ax[i].x + ax[i].y + az[i].x + az[i].y;
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

static void report(const char *name, int npk, int acc2, int unr, int maxreg, int ctas, double directed, float ms) {
  const double clk = ms * 1e-3 * g_clk_khz * 1e3;
  cudaError_t e = cudaGetLastError();
  printf("{\"probe\":\"%s\",\"packets\":%d,\"acc2\":%d,\"unroll\":%d,\"maxreg\":%d,\"ctas_per_sm\":%d,"
         "\"directed_per_clk_sm\":%.2f,\"err\":\"%s\"}\n",
         name, npk, acc2, unr, maxreg, ctas, directed / clk / g_sms, cudaGetErrorString(e));
}

template <int MAXREG>
static void run_direct(float *out, int n, int ctas) {
  const int reps = 20, threads = 128, grid = g_sms * ctas * 4;
  const size_t smem = n * 16 + n * 8;
  cudaFuncSetAttribute(direct_kernel<MAXREG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  float ms = time_ms([&] { direct_kernel<MAXREG><<<grid, threads, smem>>>(out, n, reps, 1e-4f); });
  report("direct", 0, 0, 8, MAXREG, ctas, (double)grid * threads * 4 * n * reps, ms);
}

template <int NPK, int ACC2, int MAXREG, int UNR, int KPT = 2>
static void run_rot(float *out, int n, int ctas) {
  const int reps = 20, threads = 128, grid = g_sms * ctas * 4;
  const size_t smem = n * 16 + n * 8;
  cudaFuncSetAttribute(rot_kernel<NPK, ACC2, MAXREG, UNR, KPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  float ms = time_ms([&] { rot_kernel<NPK, ACC2, MAXREG, UNR, KPT><<<grid, threads, smem>>>(out, n, reps, 1e-4f); });
  // per lane and step: 2 KPT targets x 1 source = 2 KPT pairs
  report(KPT == 2 ? "rot" : (KPT == 3 ? "rot_6targets" : "rot_8targets"), NPK, ACC2, UNR, MAXREG, ctas,
         2.0 * grid * threads * 2 * KPT * n * reps, ms);
}

template <int NPK, int FOLD, int MAXREG, int UNR>
static void run_rotl(float *out, int n, int ctas) {
  const int reps = 20, threads = 128, grid = g_sms * ctas * 4;
  const size_t smem = n * 16 + n * 8;
  cudaFuncSetAttribute(rotl_kernel<NPK, FOLD, MAXREG, UNR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  float ms = time_ms([&] { rotl_kernel<NPK, FOLD, MAXREG, UNR><<<grid, threads, smem>>>(out, n, reps, 1e-4f); });
  report(FOLD ? "rotl_fold" : "rotl", NPK, FOLD, UNR, MAXREG, ctas, 2.0 * grid * threads * 4 * n * reps, ms);
}

template <int MAXREG, int UNR>
static void run_rotsp(float *out, int n, int ctas) {
  const int reps = 20, threads = 128, grid = g_sms * ctas * 4;
  const size_t smem = n * 16 + n * 8;
  cudaFuncSetAttribute(rotsp_kernel<MAXREG, UNR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  float ms = time_ms([&] { rotsp_kernel<MAXREG, UNR><<<grid, threads, smem>>>(out, n, reps, 1e-4f); });
  report("rot_source_packed", 2, 1, UNR, MAXREG, ctas, 2.0 * grid * threads * 4 * n * reps, ms);
}

int main() {
  cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&g_clk_khz, cudaDevAttrClockRate, 0);
  float *out;
  cudaMalloc(&out, 1 << 24);
  const int n = 512;
  run_direct<72>(out, n, 7);
  run_rot<1, 1, 72, 4>(out, n, 7);
  run_rot<1, 1, 80, 4, 3>(out, n, 6);
  run_rot<1, 1, 88, 4, 3>(out, n, 5);
  run_rot<1, 1, 96, 4, 3>(out, n, 5);
  run_rot<1, 1, 96, 2, 4>(out, n, 5);
  run_rot<1, 1, 104, 2, 4>(out, n, 4);
  printf("{\"sms\":%d,\"clk_mhz\":%d}\n", g_sms, g_clk_khz / 1000);
  return 0;
}
