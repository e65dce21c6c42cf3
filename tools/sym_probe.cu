// Formulation probe for the wake-wake Biot-Savart sweep (tuning tool, not product).
//
//   direct   : the kernel's loop -- per (target pair, source) 8 packed FP32 ops +
//              2 MUFU.RSQ (8 lane-ops + 1 RSQ per directed interaction)
//   scaled   : direct, sources pre-scaled by a = 1/g: {a x, a z, -a, rc4 a^4}, so
//              d' = a (s - t) = fma(-a, t, a s), q' = a^4 q, rs' d' = g d / sqrt(q):
//              7 packed ops + 2 RSQ per target pair
//   sym<J>   : each unordered pair once.  A lane holds 4 targets (2 packed pairs,
//              raw coordinates + g); scaled sources are LDS.128 broadcasts; the
//              reaction on source j (sum_i g_i rs' d', times -a_j later) accumulates
//              in registers for a group of J sources and is reduced over the warp
//              with a transposing butterfly after every group, then stored.
//              10 packed ops + 2 RSQ per (target pair, source) = 4 directed.
// Prints directed interactions / clk / SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/sym_probe tools/sym_probe.cu
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
    const float a = 1.f / g;
    src[j] = make_float4(x, z, g, 0.f);
    src[n + j] = make_float4(a * x, a * z, -a, 1e-4f * a * a * a * a);
  }
  __syncthreads();
}

template <int KP, int MAXREG>
__global__ void __maxnreg__(MAXREG) direct_kernel(float *out, int n, int reps, float rc4) {
  extern __shared__ float4 src[];
  fill(src, n);
  float2 px[KP], pz[KP], qx[KP], qz[KP];
#pragma unroll
  for (int p = 0; p < KP; ++p) {
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
  }
  float s = 0.f;
#pragma unroll
  for (int p = 0; p < KP; ++p) s += qx[p].x + qx[p].y + qz[p].x + qz[p].y;
  if (s == 1.2345f) out[blockIdx.x] = s;
}

template <int KP, int MAXREG>
__global__ void __maxnreg__(MAXREG) scaled_kernel(float *out, int n, int reps) {
  extern __shared__ float4 src[];
  fill(src, n);
  const float4 *ssrc = src + n;
  float2 px[KP], pz[KP], qx[KP], qz[KP];
#pragma unroll
  for (int p = 0; p < KP; ++p) {
    px[p] = make_float2(0.013f * (threadIdx.x + p), 0.017f * p);
    pz[p] = make_float2(0.011f * p, 0.019f * (threadIdx.x & 3));
    qx[p] = qz[p] = make_float2(0.f, 0.f);
  }
  for (int r = 0; r < reps; ++r) {
#pragma unroll 8
    for (int j = 0; j < n; ++j) {
      const float4 s = ssrc[j];
      const float2 sx = make_float2(s.x, s.x), sz = make_float2(s.y, s.y), na = make_float2(s.z, s.z),
                   rc = make_float2(s.w, s.w);
#pragma unroll
      for (int p = 0; p < KP; ++p) {
        const float2 dx = __ffma2_rn(na, px[p], sx);
        const float2 dz = __ffma2_rn(na, pz[p], sz);
        const float2 r2 = __ffma2_rn(dx, dx, __fmul2_rn(dz, dz));
        const float2 q = __ffma2_rn(r2, r2, rc);
        const float2 rs = make_float2(rsq(q.x), rsq(q.y));
        qx[p] = __ffma2_rn(rs, dz, qx[p]);
        qz[p] = __ffma2_rn(rs, dx, qz[p]);
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int p = 0; p < KP; ++p) s += qx[p].x + qx[p].y + qz[p].x + qz[p].y;
  if (s == 1.2345f) out[blockIdx.x] = s;
}

// transposing butterfly: V = 2^k values per lane -> lane l holds the warp sum of
// value (l >> (5 - k)) (every lane of that group holds it after the final xors)
template <int V>
__device__ __forceinline__ float tsum(float *v, int lane) {
  int m = V;
  int off = 16;
#pragma unroll
  for (; m > 1; m >>= 1, off >>= 1) {
    const bool hi = lane & off;
#pragma unroll
    for (int i = 0; i < m / 2; ++i) {
      const float send = hi ? v[i] : v[i + m / 2];
      const float keep = hi ? v[i + m / 2] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
#pragma unroll
  for (; off >= 1; off >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
  return v[0];
}

template <int KP, int J, int MAXREG>
__global__ void __maxnreg__(MAXREG) sym_kernel(float *out, int n, int reps) {
  extern __shared__ float4 src[];
  fill(src, n);
  const float4 *ssrc = src + n;
  float *part = reinterpret_cast<float *>(src + 2 * n);
  const int lane = threadIdx.x & 31;
  float2 px[KP], pz[KP], pg[KP], qx[KP], qz[KP];
#pragma unroll
  for (int p = 0; p < KP; ++p) {
    px[p] = make_float2(0.013f * (threadIdx.x + p), 0.017f * p);
    pz[p] = make_float2(0.011f * p, 0.019f * (threadIdx.x & 3));
    pg[p] = make_float2(1e-3f * (p + 1), -1e-3f * (lane & 1));
    qx[p] = qz[p] = make_float2(0.f, 0.f);
  }
  for (int r = 0; r < reps; ++r) {
    for (int g0 = 0; g0 < n; g0 += J) {
      float2 bx[J], bz[J];
#pragma unroll
      for (int jj = 0; jj < J; ++jj) {
        const float4 s = ssrc[g0 + jj];
        const float2 sx = make_float2(s.x, s.x), sz = make_float2(s.y, s.y), na = make_float2(s.z, s.z),
                     rc = make_float2(s.w, s.w);
#pragma unroll
        for (int p = 0; p < KP; ++p) {
          const float2 dx = __ffma2_rn(na, px[p], sx);
          const float2 dz = __ffma2_rn(na, pz[p], sz);
          const float2 r2 = __ffma2_rn(dx, dx, __fmul2_rn(dz, dz));
          const float2 q = __ffma2_rn(r2, r2, rc);
          const float2 rs = make_float2(rsq(q.x), rsq(q.y));
          qx[p] = __ffma2_rn(rs, dz, qx[p]);
          qz[p] = __ffma2_rn(rs, dx, qz[p]);
          const float2 c = __fmul2_rn(pg[p], rs);
          if (p == 0) {
            bx[jj] = __fmul2_rn(c, dz);
            bz[jj] = __fmul2_rn(c, dx);
          } else {
            bx[jj] = __ffma2_rn(c, dz, bx[jj]);
            bz[jj] = __ffma2_rn(c, dx, bz[jj]);
          }
        }
      }
      float v[2 * J];
#pragma unroll
      for (int jj = 0; jj < J; ++jj) {
        v[jj] = bx[jj].x + bx[jj].y;
        v[J + jj] = bz[jj].x + bz[jj].y;
      }
      const float tot = tsum<2 * J>(v, lane);
      if ((lane & (32 / (2 * J) - 1)) == 0) part[g0 * 2 + lane / (32 / (2 * J))] = tot;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int p = 0; p < KP; ++p) s += qx[p].x + qx[p].y + qz[p].x + qz[p].y;
  if (s == 1.2345f) out[blockIdx.x] = s;
}


// Unscaled symmetric pairs (11 packed ops + 2 RSQ per target pair and source) as
// the kernel would run them: per group of J sources the reaction is reduced over
// the warp (transposing butterfly), quantised to int64 (2^-32) and added with a
// shared-memory atomic (order-free, hence deterministic); ATOM=0 stores instead.
template <int KP, int J, int MAXREG, int ATOM>
__global__ void __maxnreg__(MAXREG) symq_kernel(float *out, int n, int reps) {
  extern __shared__ float4 src[];
  fill(src, n);
  unsigned long long *acc = reinterpret_cast<unsigned long long *>(src + n);
  const int lane = threadIdx.x & 31;
  float2 px[KP], pz[KP], pg[KP], qx[KP], qz[KP];
#pragma unroll
  for (int p = 0; p < KP; ++p) {
    px[p] = make_float2(0.013f * (threadIdx.x + p), 0.017f * p);
    pz[p] = make_float2(0.011f * p, 0.019f * (threadIdx.x & 3));
    pg[p] = make_float2(1e-3f * (p + 1), -1e-3f * (lane & 1));
    qx[p] = qz[p] = make_float2(0.f, 0.f);
  }
  for (int r = 0; r < reps; ++r) {
    for (int g0 = 0; g0 < n; g0 += J) {
      float2 bx[J], bz[J];
#pragma unroll
      for (int jj = 0; jj < J; ++jj) {
        const float4 s = src[g0 + jj];
        const float2 sx = make_float2(s.x, s.x), sz = make_float2(s.y, s.y), sg = make_float2(s.z, s.z);
#pragma unroll
        for (int p = 0; p < KP; ++p) {
          const float2 dx = __fadd2_rn(sx, px[p]);
          const float2 dz = __fadd2_rn(sz, pz[p]);
          const float2 r2 = __ffma2_rn(dx, dx, __fmul2_rn(dz, dz));
          const float2 q = __ffma2_rn(r2, r2, make_float2(1e-4f, 1e-4f));
          const float2 rs = make_float2(rsq(q.x), rsq(q.y));
          const float2 cj = __fmul2_rn(sg, rs);
          qx[p] = __ffma2_rn(cj, dz, qx[p]);
          qz[p] = __ffma2_rn(cj, dx, qz[p]);
          const float2 ci = __fmul2_rn(pg[p], rs);
          if (p == 0) {
            bx[jj] = __fmul2_rn(ci, dz);
            bz[jj] = __fmul2_rn(ci, dx);
          } else {
            bx[jj] = __ffma2_rn(ci, dz, bx[jj]);
            bz[jj] = __ffma2_rn(ci, dx, bz[jj]);
          }
        }
      }
      float v[2 * J];
#pragma unroll
      for (int jj = 0; jj < J; ++jj) {
        v[jj] = bx[jj].x + bx[jj].y;
        v[J + jj] = bz[jj].x + bz[jj].y;
      }
      const float tot = tsum<2 * J>(v, lane);
      constexpr int G = 32 / (2 * J);
      if ((lane & (G - 1)) == 0) {
        const long long qv = __float2ll_rn(tot * 4294967296.f);
        unsigned long long *dst = acc + (g0 * 2 + lane / G) % (2 * n);
        if (ATOM) atomicAdd(dst, (unsigned long long)qv);
        else *dst = (unsigned long long)qv;
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int p = 0; p < KP; ++p) s += qx[p].x + qx[p].y + qz[p].x + qz[p].y;
  if (s == 1.2345f) out[blockIdx.x] = s;
}

// Direct loop reading sources packed as {x, z, g} triples: 3 LDS.128 per 4 sources
// instead of 4 (the float4 layout carries the age, which the sweep never reads).
template <int KP, int MAXREG>
__global__ void __maxnreg__(MAXREG) direct3_kernel(float *out, int n, int reps, float rc4) {
  extern __shared__ float4 src[];
  fill(src, n);
  float *tri = reinterpret_cast<float *>(src + n);  // overwrite the scaled copy with triples
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    tri[3 * j] = src[j].x;
    tri[3 * j + 1] = src[j].y;
    tri[3 * j + 2] = src[j].z;
  }
  __syncthreads();
  const float4 *t4 = reinterpret_cast<const float4 *>(tri);
  float2 px[KP], pz[KP], qx[KP], qz[KP];
#pragma unroll
  for (int p = 0; p < KP; ++p) {
    px[p] = make_float2(-0.013f * (threadIdx.x + p), -0.017f * p);
    pz[p] = make_float2(-0.011f * p, -0.019f * (threadIdx.x & 3));
    qx[p] = qz[p] = make_float2(0.f, 0.f);
  }
  const float2 rc = make_float2(rc4, rc4);
  for (int r = 0; r < reps; ++r) {
#pragma unroll 2
    for (int j4 = 0; j4 < n / 4; ++j4) {
      const float4 a = t4[3 * j4], b = t4[3 * j4 + 1], c = t4[3 * j4 + 2];
      const float sxs[4] = {a.x, a.w, b.z, c.y}, szs[4] = {a.y, b.x, b.w, c.z}, sgs[4] = {a.z, b.y, c.x, c.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 sx = make_float2(sxs[q], sxs[q]), sz = make_float2(szs[q], szs[q]),
                     sg = make_float2(sgs[q], sgs[q]);
#pragma unroll
        for (int p = 0; p < KP; ++p) {
          const float2 dx = __fadd2_rn(sx, px[p]);
          const float2 dz = __fadd2_rn(sz, pz[p]);
          const float2 r2 = __ffma2_rn(dx, dx, __fmul2_rn(dz, dz));
          const float2 qq = __ffma2_rn(r2, r2, rc);
          const float2 rs = make_float2(rsq(qq.x), rsq(qq.y));
          const float2 cc = __fmul2_rn(sg, rs);
          qx[p] = __ffma2_rn(cc, dz, qx[p]);
          qz[p] = __ffma2_rn(cc, dx, qz[p]);
        }
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int p = 0; p < KP; ++p) s += qx[p].x + qx[p].y + qz[p].x + qz[p].y;
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

static void report(const char *name, int kp, int j, int maxreg, int ctas, double directed, float ms) {
  const double clk = ms * 1e-3 * g_clk_khz * 1e3;
  cudaError_t e = cudaGetLastError();
  printf("{\"probe\":\"%s\",\"targets_per_lane\":%d,\"J\":%d,\"maxreg\":%d,\"ctas_per_sm\":%d,"
         "\"directed_per_clk_sm\":%.2f,\"err\":\"%s\"}\n",
         name, 2 * kp, j, maxreg, ctas, directed / clk / g_sms, cudaGetErrorString(e));
}

template <int KP, int MAXREG>
static void run_direct(float *out, int n, int ctas) {
  const int reps = 20, threads = 128, grid = g_sms * ctas * 4;
  const size_t smem = 2 * n * 16 + 2 * n * 4;
  cudaFuncSetAttribute(direct_kernel<KP, MAXREG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  float ms = time_ms([&] { direct_kernel<KP, MAXREG><<<grid, threads, smem>>>(out, n, reps, 1e-4f); });
  report("direct", KP, 0, MAXREG, ctas, (double)grid * threads * 2 * KP * n * reps, ms);
}

template <int KP, int MAXREG>
static void run_scaled(float *out, int n, int ctas) {
  const int reps = 20, threads = 128, grid = g_sms * ctas * 4;
  const size_t smem = 2 * n * 16 + 2 * n * 4;
  cudaFuncSetAttribute(scaled_kernel<KP, MAXREG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  float ms = time_ms([&] { scaled_kernel<KP, MAXREG><<<grid, threads, smem>>>(out, n, reps); });
  report("scaled", KP, 0, MAXREG, ctas, (double)grid * threads * 2 * KP * n * reps, ms);
}

template <int KP, int J, int MAXREG>
static void run_sym(float *out, int n, int ctas) {
  const int reps = 20, threads = 128, grid = g_sms * ctas * 4;
  const size_t smem = 2 * n * 16 + 2 * n * 4;
  cudaFuncSetAttribute(sym_kernel<KP, J, MAXREG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  float ms = time_ms([&] { sym_kernel<KP, J, MAXREG><<<grid, threads, smem>>>(out, n, reps); });
  // every (target, source) evaluation counts as 2 directed interactions
  report("sym", KP, J, MAXREG, ctas, 2.0 * grid * threads * 2 * KP * n * reps, ms);
}

template <int KP, int J, int MAXREG, int ATOM>
static void run_symq(float *out, int n, int ctas) {
  const int reps = 20, threads = 128, grid = g_sms * ctas * 4;
  const size_t smem = n * 16 + 2 * n * 8;
  cudaFuncSetAttribute(symq_kernel<KP, J, MAXREG, ATOM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  float ms = time_ms([&] { symq_kernel<KP, J, MAXREG, ATOM><<<grid, threads, smem>>>(out, n, reps); });
  report(ATOM ? "symq_atomic" : "symq_store", KP, J, MAXREG, ctas, 2.0 * grid * threads * 2 * KP * n * reps, ms);
}

template <int KP, int MAXREG>
static void run_direct3(float *out, int n, int ctas) {
  const int reps = 20, threads = 128, grid = g_sms * ctas * 4;
  const size_t smem = 2 * n * 16 + 2 * n * 4;
  cudaFuncSetAttribute(direct3_kernel<KP, MAXREG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  float ms = time_ms([&] { direct3_kernel<KP, MAXREG><<<grid, threads, smem>>>(out, n, reps, 1e-4f); });
  report("direct_triples", KP, 0, MAXREG, ctas, (double)grid * threads * 2 * KP * n * reps, ms);
}

int main() {
  cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&g_clk_khz, cudaDevAttrClockRate, 0);
  float *out;
  cudaMalloc(&out, 1 << 24);
  const int n = 512;
  run_direct<2, 64>(out, n, 8);
  run_direct3<2, 64>(out, n, 8);
  run_direct<2, 72>(out, n, 7);
  run_direct3<2, 72>(out, n, 7);
  run_direct<3, 72>(out, n, 7);
  run_direct3<3, 72>(out, n, 7);
  printf("{\"sms\":%d,\"clk_mhz\":%d}\n", g_sms, g_clk_khz / 1000);
  return 0;
}
