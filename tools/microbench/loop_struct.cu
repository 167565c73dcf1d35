// Microbenchmark of the K1 inner structure, to price each structural cost of the Horner phase:
//   S components (S/2 FFMA2 pairs + scalar odd), segments of SEGL steps ending in c += A h and A <- A Z,
//   c accumulated in thread-private shared memory (CSMEM = 1, the kernel's choice) or registers (0),
//   y fed per warp by 1-D bulk TMA chunks of KC (yr, yr, yi, yi) into a double buffer (TMA = 1) or re-read
//   from a resident buffer (0); MINB CTAs of 8 warps per SM.
// Reports algorithmic FMA (4 per complex MAC) per clock per SM; the FP32 peak is 128.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ unsigned long long g_cyc[4096];
__device__ unsigned long long g_ns[4096];
__device__ __forceinline__ u64 pk(float lo, float hi) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ void up(u64 v, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
__device__ __forceinline__ u64 f2(u64 a, u64 b, u64 c) { u64 d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool trywait(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}"
               : "=r"(ok) : "r"(sa(b)), "r"(ph) : "memory");
  return ok;
}

template <int S, int SEGL, int KC, bool CSMEM, bool TMA, int MINB>
__global__ void __launch_bounds__(256, MINB) k(float* out, const float4* __restrict__ yg, int nchunks) {
  constexpr int NP = S / 2;
  constexpr bool ODD = S & 1;
  extern __shared__ __align__(128) unsigned char smem[];
  float4* yb = reinterpret_cast<float4*>(smem);                 // [8][2][KC]
  uint64_t* bar = reinterpret_cast<uint64_t*>(yb + 8 * 2 * KC);  // [8][2]
  float* cst = reinterpret_cast<float*>(bar + 16);              // [S][256][2]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < 16) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[threadIdx.x])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  for (int i = threadIdx.x; i < 8 * 2 * KC; i += 256) yb[i] = yg[i % (KC * 16)];
  u64 hr[NP > 0 ? NP : 1], hi[NP > 0 ? NP : 1], wr[NP > 0 ? NP : 1], wi[NP > 0 ? NP : 1], nwi[NP > 0 ? NP : 1];
  float hrL = 0, hiL = 0, wrL = 1, wiL = 0, Ar[S], Ai[S], Zr[S], Zi[S], cr[S], ci[S];
  for (int q = 0; q < NP; ++q) {
    float a, b, c, d;
    __sincosf(0.01f * (threadIdx.x + 2 * q), &a, &b);
    __sincosf(0.013f * (threadIdx.x + q), &c, &d);
    wr[q] = pk(b, d); wi[q] = pk(a, c); nwi[q] = pk(-a, -c);
  }
  __sincosf(0.02f * threadIdx.x, &wiL, &wrL);
  for (int s = 0; s < S; ++s) {
    __sincosf(0.03f * (threadIdx.x + s), &Ai[s], &Ar[s]);
    __sincosf(0.001f * s, &Zi[s], &Zr[s]);
    cr[s] = ci[s] = 0.f;
    cst[(s * 256 + threadIdx.x) * 2] = 0.f;
    cst[(s * 256 + threadIdx.x) * 2 + 1] = 0.f;
  }
  __syncthreads();
  auto issue = [&](int c) {
    if (!TMA) return;
    uint64_t* b = &bar[warp * 2 + (c & 1)];
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(KC * 16) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sa(yb + (warp * 2 + (c & 1)) * KC)), "l"(yg + (size_t)((c * 8 + warp) % 1024) * KC), "r"(KC * 16),
                 "r"(sa(b)) : "memory");
  };
  if (lane == 0) { issue(0); issue(1); }
  unsigned long long g0, g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  unsigned long long t0 = clock64();
  for (int c = 0; c < nchunks; ++c) {
    if (TMA) while (!trywait(&bar[warp * 2 + (c & 1)], (c >> 1) & 1)) {}
    const float4* ys = yb + (warp * 2 + (c & 1)) * KC;
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
        if (ODD) {
          const float t = fmaf(-hiL, wiL, y.x), u = fmaf(hiL, wrL, y.z);
          const float nr = fmaf(hrL, wrL, t), ni = fmaf(hrL, wiL, u);
          hrL = nr; hiL = ni;
        }
      }
      float hrs[S], his[S];
      for (int q = 0; q < NP; ++q) { up(hr[q], hrs[2 * q], hrs[2 * q + 1]); up(hi[q], his[2 * q], his[2 * q + 1]); }
      if (ODD) { hrs[S - 1] = hrL; his[S - 1] = hiL; }
#pragma unroll
      for (int s = 0; s < S; ++s) {
        if (CSMEM) {
          float* cp = &cst[(s * 256 + threadIdx.x) * 2];
          cp[0] = fmaf(Ar[s], hrs[s], fmaf(-Ai[s], his[s], cp[0]));
          cp[1] = fmaf(Ar[s], his[s], fmaf(Ai[s], hrs[s], cp[1]));
        } else {
          cr[s] = fmaf(Ar[s], hrs[s], fmaf(-Ai[s], his[s], cr[s]));
          ci[s] = fmaf(Ar[s], his[s], fmaf(Ai[s], hrs[s], ci[s]));
        }
        const float nAr = Ar[s] * Zr[s] - Ai[s] * Zi[s], nAi = Ar[s] * Zi[s] + Ai[s] * Zr[s];
        Ar[s] = nAr; Ai[s] = nAi;
      }
    }
    __syncwarp();
    if (lane == 0 && c + 2 < nchunks) issue(c + 2);
  }
  unsigned long long t1 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  float acc = 0.f;
  for (int s = 0; s < S; ++s) acc += cr[s] + ci[s] + cst[(s * 256 + threadIdx.x) * 2] + Ar[s];
  out[blockIdx.x * 256 + threadIdx.x] = acc;
  if (threadIdx.x == 0) {
    g_cyc[blockIdx.x] = t1 - t0;
    g_ns[blockIdx.x] = g1 - g0;  // SM clock in MHz = cycles / ns * 1000
  }
}

template <int S, int SEGL, int KC, bool CSMEM, bool TMA, int MINB>
void run(float* out, const float4* yg, int nsm) {
  auto kern = k<S, SEGL, KC, CSMEM, TMA, MINB>;
  const int smem = 8 * 2 * KC * 16 + 16 * 8 + S * 256 * 2 * 4;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (getenv("CARVEOUT_MAX"))
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
  const int nchunks = 4096 / KC * 4;
  const int grid = nsm * MINB;
  kern<<<grid, 256, smem>>>(out, yg, nchunks);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 20;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) kern<<<grid, 256, smem>>>(out, yg, nchunks);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  static unsigned long long h[4096], hn[4096];
  cudaMemcpyFromSymbol(h, g_cyc, sizeof(unsigned long long) * grid);
  cudaMemcpyFromSymbol(hn, g_ns, sizeof(unsigned long long) * grid);
  double cyc = 0, ns = 0;
  for (int i = 0; i < grid; ++i) { cyc += h[i]; ns += hn[i]; }
  cyc /= grid;
  ns /= grid;
  const double fma = 4.0 * S * (double)nchunks * KC * 256.0 * MINB;
  const double tflops = 2.0 * fma * nsm * reps / (ms * 1e-3) / 1e12;  // wall clock, incl. launch gaps
  printf("S=%d SEG=%3d KC=%3d c_in_%s %s minb=%d : %6.1f FMA/clk/SM = %.3f of peak;  wall %.1f TFLOP/s = %.3f of "
         "74.45;  in-kernel SM clock %.0f MHz; occupancy %d CTAs/SM  (%s)\n", S, SEGL, KC, CSMEM ? "smem" : "regs", TMA ? "TMA     " : "resident",
         MINB, fma / cyc, fma / cyc / 128.0, tflops, tflops / 74.45, cyc / ns * 1e3, per_sm, cudaGetErrorString(cudaGetLastError()));
}

__global__ void fill_random(float4* y, int n) {  // (yr, yr, yi, yi) with yr, yi ~ U(-1, 1) (hash)
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t h = (uint32_t)i * 0x9E3779B1u;
  h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12;
  const float a = (float)(h & 0xFFFF) / 32768.f - 1.f, b = (float)(h >> 16) / 32768.f - 1.f;
  y[i] = make_float4(a, a, b, b);
}

int main(int argc, char** argv) {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 1 << 24);
  float4* y;
  cudaMalloc(&y, 1024 * 256 * 16);
  const bool rnd = argc > 1 && argv[1][0] == 'r';
  if (rnd) fill_random<<<1024, 256>>>(y, 1024 * 256);
  else cudaMemset(y, 0, 1024 * 256 * 16);
  cudaDeviceSynchronize();
  printf("y data: %s\n", rnd ? "random U(-1,1)" : "zeros");
  run<5, 64, 128, true, true, 3>(out, y, nsm);
  run<5, 64, 128, true, false, 3>(out, y, nsm);
  run<5, 64, 128, false, true, 3>(out, y, nsm);
  run<5, 128, 128, true, true, 3>(out, y, nsm);
  run<5, 128, 128, false, true, 3>(out, y, nsm);
  run<5, 64, 128, true, true, 2>(out, y, nsm);
  run<7, 64, 64, true, true, 3>(out, y, nsm);
  run<7, 64, 64, true, false, 3>(out, y, nsm);
  run<7, 64, 128, true, true, 2>(out, y, nsm);
  run<7, 64, 64, false, true, 3>(out, y, nsm);
  run<4, 64, 128, true, true, 3>(out, y, nsm);
  run<9, 64, 64, true, true, 2>(out, y, nsm);
  return 0;
}
