// Microbenchmark: the kernel's inner structure -- FFMA2 Horner (S = 7: 3 pairs + 1 scalar), segment ends
// every 64 steps (c += A h in thread-private smem, A <- A Z), y fed per warp by 1-D bulk TMA chunks of 128
// (yr, yr, yi, yi) into a double buffer with mbarriers -- to isolate the cost of the TMA pipeline.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ unsigned long long g_cyc[2048];
__device__ __forceinline__ u64 pk(float lo, float hi) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ void up(u64 v, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
__device__ __forceinline__ u64 f2(u64 a, u64 b, u64 c) { u64 d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool trywait(uint64_t* b, uint32_t ph) { uint32_t ok; asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}" : "=r"(ok) : "r"(sa(b)), "r"(ph) : "memory"); return ok; }
constexpr int KC = 128, SEGL = 64, S = 7, NP = 3;

template <bool USE_TMA>
__global__ void __launch_bounds__(256, 2) k(float* out, const float4* __restrict__ yg, int nchunks) {
  __shared__ __align__(128) float4 yb[8][2][KC];
  __shared__ uint64_t bar[8][2];
  __shared__ float cst[S * 256 * 2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < 16) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bar[threadIdx.x / 2][threadIdx.x % 2])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  for (int i = threadIdx.x; i < 8 * 2 * KC; i += 256) (&yb[0][0][0])[i] = yg[i % (KC * 16)];
  u64 hr[NP], hi[NP], wr[NP], wi[NP], nwi[NP];
  float hrL, hiL, wrL, wiL, Ar[S], Ai[S], Zr[S], Zi[S];
  for (int q = 0; q < NP; ++q) {
    float a, b, c, d; __sincosf(0.01f * (threadIdx.x + 2 * q), &a, &b); __sincosf(0.013f * (threadIdx.x + q), &c, &d);
    wr[q] = pk(b, d); wi[q] = pk(a, c); nwi[q] = pk(-a, -c);
  }
  __sincosf(0.02f * threadIdx.x, &wiL, &wrL);
  for (int s = 0; s < S; ++s) { __sincosf(0.03f * (threadIdx.x + s), &Ai[s], &Ar[s]); __sincosf(0.001f * s, &Zi[s], &Zr[s]);
    cst[(s * 256 + threadIdx.x) * 2] = 0; cst[(s * 256 + threadIdx.x) * 2 + 1] = 0; }
  __syncthreads();
  auto issue = [&](int c) {
    uint64_t* b = &bar[warp][c & 1];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(b)), "r"(KC * 16) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                 "r"(sa(&yb[warp][c & 1][0])), "l"(yg + (size_t)((c * 8 + warp) % 64) * KC), "r"(KC * 16), "r"(sa(b)) : "memory");
  };
  if (USE_TMA && lane == 0) { issue(0); issue(1); }
  unsigned long long t0 = clock64();
  for (int c = 0; c < nchunks; ++c) {
    if (USE_TMA) while (!trywait(&bar[warp][c & 1], (c >> 1) & 1)) {}
    const float4* ys = &yb[warp][c & 1][0];
    for (int k0 = KC - SEGL; k0 >= 0; k0 -= SEGL) {
      const float4 yt = ys[k0 + SEGL - 1];
      for (int q = 0; q < NP; ++q) { hr[q] = pk(yt.x, yt.y); hi[q] = pk(yt.z, yt.w); }
      hrL = yt.x; hiL = yt.z;
#pragma unroll 7
      for (int i = SEGL - 2; i >= 0; --i) {
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
    if (USE_TMA) { __syncwarp(); if (lane == 0 && c + 2 < nchunks) issue(c + 2); }
  }
  unsigned long long t1 = clock64();
  float acc = 0; for (int s = 0; s < S; ++s) acc += cst[(s * 256 + threadIdx.x) * 2];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, 1 << 26);
  float4* y; cudaMalloc(&y, 64 * KC * 16);
  static float4 hy[64 * KC];
  for (int i = 0; i < 64 * KC; ++i) { float a = 0.37f * i, b = 0.11f * i; hy[i] = make_float4(cosf(a), cosf(a), sinf(b), sinf(b)); }
  cudaMemcpy(y, hy, sizeof(hy), cudaMemcpyHostToDevice);
  const int nch = 64;
  for (int tma = 0; tma < 2; ++tma) {
    for (int rep = 0; rep < 2; ++rep) {
      if (tma) k<true><<<nsm * 2, 256>>>(out, y, nch); else k<false><<<nsm * 2, 256>>>(out, y, nch);
      cudaDeviceSynchronize();
    }
    static unsigned long long h[2048];
    cudaMemcpyFromSymbol(h, g_cyc, sizeof(unsigned long long) * nsm * 2);
    double cyc = 0; for (int i = 0; i < nsm * 2; ++i) cyc += h[i]; cyc /= nsm * 2;
    double fma = 4.0 * (KC - 1) * nch * S * 256 * 2;  // per SM (2 blocks), first step of each segment has no FMA
    fma = 4.0 * (KC - 2) * nch * S * 256 * 2;
    printf("TMA=%d: %.2f FMA/clk/SM (%s)\n", tma, fma / cyc, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
