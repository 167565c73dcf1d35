// Horner-step formulations for the correlation inner loop: FMA/clk/SM measured with clock64().
//   V1  pairs of components in FFMA2 (hr2, hi2), 4 FFMA2 per pair-step (the kernel's form)
//   V2  (re, im) of one component in one 64-bit register: 2 FFMA2 per component-step using broadcast
//       halves: h' = fma2((hr,hr), (wr,wi), fma2((hi,hi), (-wi,wr), (yr,yi)))
//   V3  scalar FFMA, 4 per component-step
//   V4  V1 with the y operands ordered first (t for all pairs, then u, then nr/ni)
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;
__device__ unsigned long long g_cycles[1024];
__device__ __forceinline__ u64 pk(float lo, float hi) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ void up(u64 v, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
__device__ __forceinline__ u64 f2(u64 a, u64 b, u64 c) { u64 d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ u64 bc_lo(u64 v) { float lo, hi; up(v, lo, hi); return pk(lo, lo); }
__device__ __forceinline__ u64 bc_hi(u64 v) { float lo, hi; up(v, lo, hi); return pk(hi, hi); }

constexpr int NK = 1024, REPS = 8;

template <int S>
__global__ void v1(float* out, const float4* __restrict__ ysrc) {
  __shared__ float4 ys[NK];
  for (int i = threadIdx.x; i < NK; i += blockDim.x) ys[i] = ysrc[i];
  constexpr int NP = S / 2;
  u64 hr[NP], hi[NP], wr[NP], wi[NP], nwi[NP];
  for (int q = 0; q < NP; ++q) {
    float a, b, c, d; __sincosf(0.01f * (threadIdx.x + 2 * q), &a, &b); __sincosf(0.013f * (threadIdx.x + q), &c, &d);
    hr[q] = hi[q] = 0; wr[q] = pk(b, d); wi[q] = pk(a, c); nwi[q] = pk(-a, -c);
  }
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int r = 0; r < REPS; ++r)
#pragma unroll 8
    for (int k = NK - 1; k >= 0; --k) {
      const float4 y = ys[k];
      const u64 yr = pk(y.x, y.y), yi = pk(y.z, y.w);
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        const u64 t = f2(hi[q], nwi[q], yr), u = f2(hi[q], wr[q], yi);
        const u64 nr = f2(hr[q], wr[q], t), ni = f2(hr[q], wi[q], u);
        hr[q] = nr; hi[q] = ni;
      }
    }
  __syncthreads();
  unsigned long long t1 = clock64();
  float acc = 0; for (int q = 0; q < NP; ++q) { float a, b; up(hr[q], a, b); acc += a + b; up(hi[q], a, b); acc += a - b; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

template <int S>
__global__ void v2(float* out, const float4* __restrict__ ysrc) {
  __shared__ float4 ys[NK];
  for (int i = threadIdx.x; i < NK; i += blockDim.x) ys[i] = ysrc[i];
  u64 h[S], W[S], Wp[S];
  for (int s = 0; s < S; ++s) {
    float a, b; __sincosf(0.01f * (threadIdx.x + s), &a, &b);
    h[s] = 0; W[s] = pk(b, a); Wp[s] = pk(-a, b);   // (wr, wi), (-wi, wr)
  }
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int r = 0; r < REPS; ++r)
#pragma unroll 8
    for (int k = NK - 1; k >= 0; --k) {
      const float4 y = ys[k];
      const u64 y2 = pk(y.x, y.z);   // (yr, yi)
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const u64 t = f2(bc_hi(h[s]), Wp[s], y2);
        h[s] = f2(bc_lo(h[s]), W[s], t);
      }
    }
  __syncthreads();
  unsigned long long t1 = clock64();
  float acc = 0; for (int s = 0; s < S; ++s) { float a, b; up(h[s], a, b); acc += a + b; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

template <int S>
__global__ void v3(float* out, const float4* __restrict__ ysrc) {
  __shared__ float4 ys[NK];
  for (int i = threadIdx.x; i < NK; i += blockDim.x) ys[i] = ysrc[i];
  float hr[S], hi[S], wr[S], wi[S];
  for (int s = 0; s < S; ++s) { hr[s] = hi[s] = 0; __sincosf(0.01f * (threadIdx.x + s), &wi[s], &wr[s]); }
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int r = 0; r < REPS; ++r)
#pragma unroll 8
    for (int k = NK - 1; k >= 0; --k) {
      const float4 y = ys[k];
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const float t = fmaf(-hi[s], wi[s], y.x), u = fmaf(hi[s], wr[s], y.z);
        const float nr = fmaf(hr[s], wr[s], t), ni = fmaf(hr[s], wi[s], u);
        hr[s] = nr; hi[s] = ni;
      }
    }
  __syncthreads();
  unsigned long long t1 = clock64();
  float acc = 0; for (int s = 0; s < S; ++s) acc += hr[s] + hi[s];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

// V5: two particles per thread, pairs over particles (p0, p1) for each component: same y operand in all
template <int S>
__global__ void v5(float* out, const float4* __restrict__ ysrc) {
  __shared__ float4 ys[NK];
  for (int i = threadIdx.x; i < NK; i += blockDim.x) ys[i] = ysrc[i];
  u64 hr[S], hi[S], wr[S], wi[S], nwi[S];
  for (int s = 0; s < S; ++s) {
    float a, b, c, d; __sincosf(0.01f * (threadIdx.x + s), &a, &b); __sincosf(0.017f * (threadIdx.x + s), &c, &d);
    hr[s] = hi[s] = 0; wr[s] = pk(b, d); wi[s] = pk(a, c); nwi[s] = pk(-a, -c);
  }
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int r = 0; r < REPS; ++r)
#pragma unroll 8
    for (int k = NK - 1; k >= 0; --k) {
      const float4 y = ys[k];
      const u64 yr = pk(y.x, y.y), yi = pk(y.z, y.w);
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const u64 t = f2(hi[s], nwi[s], yr), u = f2(hi[s], wr[s], yi);
        const u64 nr = f2(hr[s], wr[s], t), ni = f2(hr[s], wi[s], u);
        hr[s] = nr; hi[s] = ni;
      }
    }
  __syncthreads();
  unsigned long long t1 = clock64();
  float acc = 0; for (int s = 0; s < S; ++s) { float a, b; up(hr[s], a, b); acc += a + b; up(hi[s], a, b); acc += a - b; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

static double avg_cycles(int n) {
  static unsigned long long h[1024];
  cudaMemcpyFromSymbol(h, g_cycles, sizeof(unsigned long long) * n);
  double s = 0; for (int i = 0; i < n; ++i) s += h[i]; return s / n;
}

int main1() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, 1 << 26);
  float4* y; cudaMalloc(&y, NK * 16); cudaMemset(y, 0, NK * 16);
#define RUN(name, kern, comps_per_thread, thr, blocks_per_sm) { \
    kern<<<nsm * blocks_per_sm, thr>>>(out, y); cudaDeviceSynchronize(); \
    kern<<<nsm * blocks_per_sm, thr>>>(out, y); cudaDeviceSynchronize(); \
    double cyc = avg_cycles(nsm * blocks_per_sm); \
    double fma = 4.0 * NK * REPS * (comps_per_thread) * thr * blocks_per_sm; \
    printf("%-34s thr=%4d x%d  %7.2f FMA/clk/SM  (%s)\n", name, thr, blocks_per_sm, fma / cyc, cudaGetErrorString(cudaGetLastError())); }
  for (int b : {1, 2}) {
    RUN("V1 comp-pairs FFMA2 S=5(4+1)", v1<5>, 4, 256, b);
    RUN("V1 comp-pairs FFMA2 S=8", v1<8>, 8, 256, b);
    RUN("V2 re/im FFMA2 bcast S=5", v2<5>, 5, 256, b);
    RUN("V2 re/im FFMA2 bcast S=8", v2<8>, 8, 256, b);
    RUN("V3 scalar FFMA S=5", v3<5>, 5, 256, b);
    RUN("V3 scalar FFMA S=8", v3<8>, 8, 256, b);
    RUN("V5 particle-pairs FFMA2 S=5", v5<5>, 10, 256, b);
    RUN("V5 particle-pairs FFMA2 S=7", v5<7>, 14, 256, b);
  }
  return 0;
}

// V6: V1 (S=7 = 3 pairs + 1 scalar) + segment ends every SEGL steps: c += A*h (thread-private smem),
// A <- A*Z, h <- 0 -- the kernel's inner structure without TMA.
template <int SEGL>
__global__ void v6(float* out, const float4* __restrict__ ysrc) {
  constexpr int S = 7, NP = 3;
  __shared__ float4 ys[NK];
  __shared__ float cst[S * 256 * 2];
  for (int i = threadIdx.x; i < NK; i += blockDim.x) ys[i] = ysrc[i];
  u64 hr[NP], hi[NP], wr[NP], wi[NP], nwi[NP];
  float hrL = 0, hiL = 0, wrL, wiL, Ar[S], Ai[S], Zr[S], Zi[S];
  for (int q = 0; q < NP; ++q) {
    float a, b, c, d; __sincosf(0.01f * (threadIdx.x + 2 * q), &a, &b); __sincosf(0.013f * (threadIdx.x + q), &c, &d);
    hr[q] = hi[q] = 0; wr[q] = pk(b, d); wi[q] = pk(a, c); nwi[q] = pk(-a, -c);
  }
  __sincosf(0.02f * threadIdx.x, &wiL, &wrL);
  for (int s = 0; s < S; ++s) { __sincosf(0.03f * (threadIdx.x + s), &Ai[s], &Ar[s]); __sincosf(0.001f * s, &Zi[s], &Zr[s]);
    cst[(s * 256 + threadIdx.x) * 2] = 0; cst[(s * 256 + threadIdx.x) * 2 + 1] = 0; }
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int r = 0; r < REPS; ++r)
    for (int k0 = NK - SEGL; k0 >= 0; k0 -= SEGL) {
#pragma unroll
      for (int q = 0; q < NP; ++q) hr[q] = hi[q] = 0;
      hrL = hiL = 0;
#pragma unroll 8
      for (int i = SEGL - 1; i >= 0; --i) {
        const float4 y = ys[k0 + i];
        const u64 yr = pk(y.x, y.y), yi = pk(y.z, y.w);
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          const u64 t = f2(hi[q], nwi[q], yr), u = f2(hi[q], wr[q], yi);
          const u64 nr = f2(hr[q], wr[q], t), ni = f2(hr[q], wi[q], u);
          hr[q] = nr; hi[q] = ni;
        }
        const float t = fmaf(-hiL, wiL, y.x), u = fmaf(hiL, wrL, y.z);
        const float nr = fmaf(hrL, wrL, t), ni = fmaf(hrL, wiL, u);
        hrL = nr; hiL = ni;
      }
      float h_r[S], h_i[S];
      for (int q = 0; q < NP; ++q) { up(hr[q], h_r[2 * q], h_r[2 * q + 1]); up(hi[q], h_i[2 * q], h_i[2 * q + 1]); }
      h_r[6] = hrL; h_i[6] = hiL;
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int o = s * 256 + threadIdx.x;
        cst[2 * o] = fmaf(Ar[s], h_r[s], fmaf(-Ai[s], h_i[s], cst[2 * o]));
        cst[2 * o + 1] = fmaf(Ar[s], h_i[s], fmaf(Ai[s], h_r[s], cst[2 * o + 1]));
        const float nAr = Ar[s] * Zr[s] - Ai[s] * Zi[s], nAi = Ar[s] * Zi[s] + Ai[s] * Zr[s];
        Ar[s] = nAr; Ai[s] = nAi;
      }
    }
  __syncthreads();
  unsigned long long t1 = clock64();
  float acc = 0; for (int s = 0; s < S; ++s) acc += cst[(s * 256 + threadIdx.x) * 2];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, 1 << 26);
  float4* y; cudaMalloc(&y, NK * 16);
  float4 hy[NK];
  for (int i = 0; i < NK; ++i) { float a = 0.37f * i, b = 0.11f * i; hy[i] = make_float4(cosf(a), cosf(a), sinf(b), sinf(b)); }
  cudaMemcpy(y, hy, sizeof(hy), cudaMemcpyHostToDevice);
  for (int b : {2, 3}) {
    RUN("V1 S=8 nonzero y", v1<8>, 8, 256, b);
    RUN("V5 S=7 particle-pairs nonzero", v5<7>, 14, 256, b);
    RUN("V6 S=7 seg64", v6<64>, 7, 256, b);
    RUN("V6 S=7 seg128", v6<128>, 7, 256, b);
    RUN("V6 S=7 seg1024", v6<1024>, 7, 256, b);
  }
  return 0;
}
