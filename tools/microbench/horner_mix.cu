// Mixed-pipe Horner step: NP component pairs on the FP32 pipe (FFMA2), ODD scalar FP32 components and N64
// components on the FP64 pipe (DFMA, 64/clk/SM on B200, otherwise idle in the correlation loop).
// YM = 0: the fp64 components convert y from the float4 (yr, yr, yi, yi) tile (2 F2F per element)
// YM = 1: the fp64 components read y from a second double2 tile (one more LDS.128 per element)
// Reports complex-MAC*4 (FMA) per clk per SM, all pipes summed, with clock64().
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;
__device__ unsigned long long g_cycles[4096];
__device__ __forceinline__ u64 pk(float lo, float hi) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ void up(u64 v, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
__device__ __forceinline__ u64 f2(u64 a, u64 b, u64 c) { u64 d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }

constexpr int NK = 1024, REPS = 8;

template <int NP, int ODD, int N64, int YM>
__global__ void __launch_bounds__(256) mix(float* out, const float4* __restrict__ ysrc, const double2* __restrict__ ydsrc) {
  __shared__ float4 ys[NK];
  __shared__ double2 yd[YM ? NK : 1];
  for (int i = threadIdx.x; i < NK; i += blockDim.x) { ys[i] = ysrc[i]; if (YM) yd[i] = ydsrc[i]; }
  u64 hr[NP > 0 ? NP : 1], hi[NP > 0 ? NP : 1], wr[NP > 0 ? NP : 1], wi[NP > 0 ? NP : 1], nwi[NP > 0 ? NP : 1];
  float hrL = 0, hiL = 0, wrL = 1, wiL = 0;
  double dhr[N64 > 0 ? N64 : 1], dhi[N64 > 0 ? N64 : 1], dwr[N64 > 0 ? N64 : 1], dwi[N64 > 0 ? N64 : 1];
  for (int q = 0; q < NP; ++q) {
    float a, b, c, d; __sincosf(0.01f * (threadIdx.x + 2 * q), &a, &b); __sincosf(0.013f * (threadIdx.x + q), &c, &d);
    hr[q] = hi[q] = 0; wr[q] = pk(b, d); wi[q] = pk(a, c); nwi[q] = pk(-a, -c);
  }
  __sincosf(0.02f * threadIdx.x, &wiL, &wrL);
  for (int q = 0; q < N64; ++q) { dhr[q] = dhi[q] = 0; sincos(0.003 * (threadIdx.x + q), &dwi[q], &dwr[q]); }
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int r = 0; r < REPS; ++r)
#pragma unroll 8
    for (int k = NK - 1; k >= 0; --k) {
      const float4 y = ys[k];
      const u64 yr = pk(y.x, y.y), yi = pk(y.z, y.w);
      double ydr, ydi;
      if (YM) { const double2 t = yd[k]; ydr = t.x; ydi = t.y; }
      else { ydr = (double)y.x; ydi = (double)y.z; }
#pragma unroll
      for (int q = 0; q < N64; ++q) {
        const double t = fma(-dhi[q], dwi[q], ydr), u = fma(dhi[q], dwr[q], ydi);
        const double nr = fma(dhr[q], dwr[q], t), ni = fma(dhr[q], dwi[q], u);
        dhr[q] = nr; dhi[q] = ni;
      }
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        const u64 t = f2(hi[q], nwi[q], yr), u = f2(hi[q], wr[q], yi);
        const u64 nr = f2(hr[q], wr[q], t), ni = f2(hr[q], wi[q], u);
        hr[q] = nr; hi[q] = ni;
      }
      if (ODD) {
        const float t = fmaf(-hiL, wiL, y.x), u = fmaf(hiL, wrL, y.z);
        const float nr = fmaf(hrL, wrL, t), ni = fmaf(hrL, wiL, u);
        hrL = nr; hiL = ni;
      }
    }
  __syncthreads();
  unsigned long long t1 = clock64();
  float acc = hrL + hiL;
  for (int q = 0; q < NP; ++q) { float a, b; up(hr[q], a, b); acc += a + b; up(hi[q], a, b); acc += a - b; }
  for (int q = 0; q < N64; ++q) acc += (float)(dhr[q] + dhi[q]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

static double avg_cycles(int n) {
  static unsigned long long h[4096];
  cudaMemcpyFromSymbol(h, g_cycles, sizeof(unsigned long long) * n);
  double s = 0; for (int i = 0; i < n; ++i) s += h[i]; return s / n;
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, 1 << 26);
  float4* y; cudaMalloc(&y, NK * 16); cudaMemset(y, 0, NK * 16);
  double2* yd; cudaMalloc(&yd, NK * 16); cudaMemset(yd, 0, NK * 16);
#define RUN(NP, ODD, N64, YM, b) { \
    auto kern = mix<NP, ODD, N64, YM>; \
    kern<<<nsm * b, 256>>>(out, y, yd); cudaDeviceSynchronize(); \
    kern<<<nsm * b, 256>>>(out, y, yd); cudaDeviceSynchronize(); \
    double cyc = avg_cycles(nsm * b); \
    const int S = 2 * NP + ODD + N64; \
    double fma = 4.0 * NK * REPS * S * 256 * b; \
    double fp32_only = 4.0 * S; /* pipe clocks per element if all on FP32 */ \
    printf("S=%d  pairs32=%d odd32=%d fp64=%d ymode=%d  blocks/SM=%d  %7.2f FMA/clk/SM  (%.2fx of FP32 peak 128)  %s\n", \
           S, NP, ODD, N64, YM, b, fma / cyc, fma / cyc / 128.0, cudaGetErrorString(cudaGetLastError())); (void)fp32_only; }
  for (int b : {2, 3}) {
    RUN(2, 1, 0, 0, b);  // current S=5
    RUN(2, 0, 1, 0, b);
    RUN(2, 0, 1, 1, b);
    RUN(1, 1, 2, 1, b);
    RUN(1, 0, 1, 0, b);  // S=3
    RUN(1, 0, 1, 1, b);
    RUN(1, 1, 0, 0, b);
    RUN(3, 1, 0, 0, b);  // S=7
    RUN(3, 0, 1, 0, b);
    RUN(2, 0, 3, 1, b);
    RUN(2, 1, 2, 1, b);
    RUN(4, 1, 0, 0, b);  // S=9
    RUN(4, 0, 1, 1, b);
    RUN(3, 0, 3, 1, b);
    RUN(3, 0, 3, 0, b);
    RUN(2, 0, 2, 1, b);  // S=6
    RUN(3, 0, 0, 0, b);
  }
  return 0;
}
