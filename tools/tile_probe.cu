// Tile-formulation probe for the wake-wake convection sweep (tuning tool, not product).
//
// One CTA = one rollout's wake of n particles in shared memory; every "rep" is one
// step's full wake-wake velocity evaluation, closed by a barrier (as in the kernel).
//
//   direct : the kernel's current loop -- every thread holds KP packed target pairs
//            (register tile) and runs over all n sources (8 lane-ops + 1 MUFU.RSQ
//            per directed interaction).
//   tile   : symmetric pairs on canonical 32-particle blocks.  Work units, taken by
//            warps from a shared-memory counter:
//              * off-diagonal: target blocks (I1, I2) (I1 < I2 < J, paired in
//                order down column J) x source block J: a lane holds targets
//                32 I1 + l and 32 I2 + l as one packed pair; per source 10 packed
//                ops + 2 RSQ give both targets' velocity and the reaction on the
//                source; reactions of G sources are reduced over the warp with a
//                transposing butterfly;
//              * diagonal: block I x block I directed (8 lane-ops + 1 RSQ).
//            Every unit result is quantised to int64 (2^-32) and added to the
//            particle's accumulator with a shared-memory atomic, so the sums are
//            exact and independent of which warp ran which unit.
// Prints directed interactions / clk / SM (each pair counts twice).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tile_probe tools/tile_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float rsq(float v) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

__device__ void fill(float4 *src, int n) {
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const float x = 0.01f * j + 0.001f * blockIdx.x, z = 0.02f * (j & 7), g = 1e-3f * ((j & 3) + 1);
    src[j] = make_float4(x, z, g, 0.f);
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
    __syncthreads();
  }
  float s = 0.f;
#pragma unroll
  for (int p = 0; p < KP; ++p) s += qx[p].x + qx[p].y + qz[p].x + qz[p].y;
  if (s == 1.2345f) out[blockIdx.x] = s;
}

// transposing butterfly over the warp: V = 2^k values per lane; afterwards lane l
// holds the warp sum of value (l >> (5 - k)) (replicated over 32/V lanes)
template <int V>
__device__ __forceinline__ float tsum(float *v, int lane) {
  int off = 16;
#pragma unroll
  for (int m = V; m > 1; m >>= 1, off >>= 1) {
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

__device__ __forceinline__ void acc_add(unsigned long long *a, float v) {
  atomicAdd(a, (unsigned long long)__float2ll_rn(v * 4294967296.f));
}

// units of a wake with nblk blocks: column J = 1..nblk-1 holds ceil(J/2) off-diagonal
// units; then nblk diagonal units
__device__ __forceinline__ void unit_decode(int u, int nblk, int &I1, int &I2, int &J) {
  int J_ = 1, base = 0;
  while (J_ < nblk && u >= base + (J_ + 1) / 2) { base += (J_ + 1) / 2; ++J_; }
  if (J_ < nblk) {
    const int k = u - base;
    I1 = 2 * k;
    I2 = (2 * k + 1 < J_) ? 2 * k + 1 : -1;
    J = J_;
  } else {
    I1 = u - base;
    I2 = -2;  // diagonal
    J = I1;
  }
}

template <int G, int MAXREG>
__global__ void __maxnreg__(MAXREG) tile_kernel(float *out, int n, int reps, float rc4) {
  extern __shared__ float4 src[];
  fill(src, n);
  unsigned long long *acc = reinterpret_cast<unsigned long long *>(src + n);
  __shared__ int ticket;
  const int lane = threadIdx.x & 31;
  const int nblk = n / 32;
  int nunits = nblk;  // diagonals
  for (int J = 1; J < nblk; ++J) nunits += (J + 1) / 2;
  const float2 rc = make_float2(rc4, rc4);
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x == 0) ticket = 0;
    for (int i = threadIdx.x; i < 2 * n; i += blockDim.x) acc[i] = 0ull;
    __syncthreads();
    for (;;) {
      int u = 0;
      if (lane == 0) u = atomicAdd(&ticket, 1);
      u = __shfl_sync(0xffffffffu, u, 0);
      if (u >= nunits) break;
      int I1, I2, J;
      unit_decode(u, nblk, I1, I2, J);
      if (I2 == -2) {
        // diagonal block, directed (self term is exactly 0)
        const float4 t = src[32 * I1 + lane];
        const float ntx = -t.x, ntz = -t.y;
        float ax = 0.f, az = 0.f;
#pragma unroll 8
        for (int j = 0; j < 32; ++j) {
          const float4 s = src[32 * I1 + j];
          const float dx = s.x + ntx, dz = s.y + ntz;
          const float r2 = fmaf(dx, dx, dz * dz);
          const float c = s.z * rsq(fmaf(r2, r2, rc4));
          ax = fmaf(c, dz, ax);
          az = fmaf(c, dx, az);
        }
        acc_add(acc + 2 * (32 * I1 + lane), ax);
        acc_add(acc + 2 * (32 * I1 + lane) + 1, az);
        continue;
      }
      const float4 t0 = src[32 * I1 + lane];
      const float4 t1 = I2 >= 0 ? src[32 * I2 + lane] : make_float4(1e4f, 1e4f, 0.f, 0.f);
      const float2 ntx = make_float2(-t0.x, -t1.x), ntz = make_float2(-t0.y, -t1.y), tg = make_float2(t0.z, t1.z);
      float2 ax = make_float2(0.f, 0.f), az = make_float2(0.f, 0.f);
      const float4 *sb = src + 32 * J;
#pragma unroll 1
      for (int g0 = 0; g0 < 32; g0 += G) {
        float v[2 * G];
#pragma unroll
        for (int jj = 0; jj < G; ++jj) {
          const float4 s = sb[g0 + jj];
          const float2 sx = make_float2(s.x, s.x), sz = make_float2(s.y, s.y), sg = make_float2(s.z, s.z);
          const float2 dx = __fadd2_rn(sx, ntx);
          const float2 dz = __fadd2_rn(sz, ntz);
          const float2 r2 = __ffma2_rn(dx, dx, __fmul2_rn(dz, dz));
          const float2 q = __ffma2_rn(r2, r2, rc);
          const float2 rs = make_float2(rsq(q.x), rsq(q.y));
          const float2 a = __fmul2_rn(sg, rs);
          ax = __ffma2_rn(a, dz, ax);
          az = __ffma2_rn(a, dx, az);
          const float2 b = __fmul2_rn(tg, rs);
          const float2 bx = __fmul2_rn(b, dz), bz = __fmul2_rn(b, dx);
          v[jj] = bx.x + bx.y;
          v[G + jj] = bz.x + bz.y;
        }
        const float tot = tsum<2 * G>(v, lane);
        constexpr int REP = 32 / (2 * G);
        if ((lane & (REP - 1)) == 0) {
          const int idx = lane / REP;  // value index: jj (x) or G + jj (z)
          const int jj = idx < G ? idx : idx - G;
          acc_add(acc + 2 * (32 * J + g0 + jj) + (idx < G ? 0 : 1), -tot);
        }
      }
      acc_add(acc + 2 * (32 * I1 + lane), ax.x);
      acc_add(acc + 2 * (32 * I1 + lane) + 1, az.x);
      if (I2 >= 0) {
        acc_add(acc + 2 * (32 * I2 + lane), ax.y);
        acc_add(acc + 2 * (32 * I2 + lane) + 1, az.y);
      }
    }
    __syncthreads();
  }
  if (acc[threadIdx.x] == 12345ull) out[blockIdx.x] = 1.f;
}

// Rotation variant of the off-diagonal unit: at sub-step k lane l pairs its two
// targets with source 32 J + ((l + k) & 31) (lane-varying LDS, conflict-free), and
// the reaction on that source is shuffled to the lane that owns it (source
// 32 J + l lives in lane l's accumulator) -- no butterflies, no selects.
template <int MAXREG, int UNROLL>
__global__ void __maxnreg__(MAXREG) rot_kernel(float *out, int n, int reps, float rc4) {
  extern __shared__ float4 src[];
  fill(src, n);
  unsigned long long *acc = reinterpret_cast<unsigned long long *>(src + n);
  __shared__ int ticket;
  const int lane = threadIdx.x & 31;
  const int nblk = n / 32;
  int nunits = nblk;
  for (int J = 1; J < nblk; ++J) nunits += (J + 1) / 2;
  const float2 rc = make_float2(rc4, rc4);
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x == 0) ticket = 0;
    for (int i = threadIdx.x; i < 2 * n; i += blockDim.x) acc[i] = 0ull;
    __syncthreads();
    for (;;) {
      int u = 0;
      if (lane == 0) u = atomicAdd(&ticket, 1);
      u = __shfl_sync(0xffffffffu, u, 0);
      if (u >= nunits) break;
      int I1, I2, J;
      unit_decode(u, nblk, I1, I2, J);
      if (I2 == -2) {
        const float4 t = src[32 * I1 + lane];
        const float ntx = -t.x, ntz = -t.y;
        float ax = 0.f, az = 0.f;
#pragma unroll 8
        for (int j = 0; j < 32; ++j) {
          const float4 s = src[32 * I1 + j];
          const float dx = s.x + ntx, dz = s.y + ntz;
          const float r2 = fmaf(dx, dx, dz * dz);
          const float c = s.z * rsq(fmaf(r2, r2, rc4));
          ax = fmaf(c, dz, ax);
          az = fmaf(c, dx, az);
        }
        acc_add(acc + 2 * (32 * I1 + lane), ax);
        acc_add(acc + 2 * (32 * I1 + lane) + 1, az);
        continue;
      }
      const float4 t0 = src[32 * I1 + lane];
      const float4 t1 = I2 >= 0 ? src[32 * I2 + lane] : make_float4(1e4f, 1e4f, 0.f, 0.f);
      const float2 ntx = make_float2(-t0.x, -t1.x), ntz = make_float2(-t0.y, -t1.y), tg = make_float2(t0.z, t1.z);
      float2 ax = make_float2(0.f, 0.f), az = make_float2(0.f, 0.f);
      float rx = 0.f, rz = 0.f;
      const float4 *sb = src + 32 * J;
#pragma unroll UNROLL
      for (int k = 0; k < 32; ++k) {
        const float4 s = sb[(lane + k) & 31];
        const float2 sx = make_float2(s.x, s.x), sz = make_float2(s.y, s.y), sg = make_float2(s.z, s.z);
        const float2 dx = __fadd2_rn(sx, ntx);
        const float2 dz = __fadd2_rn(sz, ntz);
        const float2 r2 = __ffma2_rn(dx, dx, __fmul2_rn(dz, dz));
        const float2 q = __ffma2_rn(r2, r2, rc);
        const float2 rs = make_float2(rsq(q.x), rsq(q.y));
        const float2 a = __fmul2_rn(sg, rs);
        ax = __ffma2_rn(a, dz, ax);
        az = __ffma2_rn(a, dx, az);
        const float2 b = __fmul2_rn(tg, rs);
        const float2 bx = __fmul2_rn(b, dz), bz = __fmul2_rn(b, dx);
        // reaction on source (lane + k) & 31 -> owned by that lane
        rx += __shfl_sync(0xffffffffu, bx.x + bx.y, (lane - k) & 31);
        rz += __shfl_sync(0xffffffffu, bz.x + bz.y, (lane - k) & 31);
      }
      acc_add(acc + 2 * (32 * J + lane), -rx);
      acc_add(acc + 2 * (32 * J + lane) + 1, -rz);
      acc_add(acc + 2 * (32 * I1 + lane), ax.x);
      acc_add(acc + 2 * (32 * I1 + lane) + 1, az.x);
      if (I2 >= 0) {
        acc_add(acc + 2 * (32 * I2 + lane), ax.y);
        acc_add(acc + 2 * (32 * I2 + lane) + 1, az.y);
      }
    }
    __syncthreads();
  }
  if (acc[threadIdx.x] == 12345ull) out[blockIdx.x] = 1.f;
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

static void report(const char *name, int threads, int g, int maxreg, int ctas, double directed, float ms) {
  const double clk = ms * 1e-3 * g_clk_khz * 1e3;
  cudaError_t e = cudaGetLastError();
  printf("{\"probe\":\"%s\",\"threads\":%d,\"G\":%d,\"maxreg\":%d,\"ctas_per_sm\":%d,"
         "\"directed_per_clk_sm\":%.2f,\"err\":\"%s\"}\n",
         name, threads, g, maxreg, ctas, directed / clk / g_sms, cudaGetErrorString(e));
}

template <int KP, int MAXREG>
static void run_direct(float *out, int n, int ctas) {
  const int reps = 20, threads = n / (2 * KP), grid = g_sms * ctas * 4;
  const size_t smem = n * 16 + n * 16;
  cudaFuncSetAttribute(direct_kernel<KP, MAXREG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  float ms = time_ms([&] { direct_kernel<KP, MAXREG><<<grid, threads, smem>>>(out, n, reps, 1e-4f); });
  report("direct", threads, 0, MAXREG, ctas, (double)grid * n * n * reps, ms);
}

template <int G, int MAXREG>
static void run_tile(float *out, int n, int ctas, int threads) {
  const int reps = 20, grid = g_sms * ctas * 4;
  const size_t smem = n * 16 + n * 16;
  cudaFuncSetAttribute(tile_kernel<G, MAXREG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  float ms = time_ms([&] { tile_kernel<G, MAXREG><<<grid, threads, smem>>>(out, n, reps, 1e-4f); });
  report("tile", threads, G, MAXREG, ctas, (double)grid * n * (n - 1) * reps, ms);
}

template <int MAXREG, int UNROLL>
static void run_rot(float *out, int n, int ctas, int threads) {
  const int reps = 20, grid = g_sms * ctas * 4;
  const size_t smem = n * 16 + n * 16;
  cudaFuncSetAttribute(rot_kernel<MAXREG, UNROLL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  float ms = time_ms([&] { rot_kernel<MAXREG, UNROLL><<<grid, threads, smem>>>(out, n, reps, 1e-4f); });
  report("rot", threads, UNROLL, MAXREG, ctas, (double)grid * n * (n - 1) * reps, ms);
}

int main() {
  cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&g_clk_khz, cudaDevAttrClockRate, 0);
  float *out;
  cudaMalloc(&out, 1 << 24);
  const int n = 512;
  run_direct<2, 64>(out, n, 8);
  run_direct<2, 72>(out, n, 7);
  run_tile<8, 72>(out, n, 7, 128);
  run_rot<64, 8>(out, n, 8, 128);
  run_rot<72, 8>(out, n, 7, 128);
  run_rot<64, 32>(out, n, 8, 128);
  run_rot<72, 32>(out, n, 7, 128);
  run_rot<64, 4>(out, n, 8, 128);
  run_rot<64, 8>(out, n, 4, 256);
  run_rot<64, 8>(out, n, 2, 512);
  printf("{\"sms\":%d,\"clk_mhz\":%d}\n", g_sms, g_clk_khz / 1000);
  return 0;
}
