// Pipe-throughput microbenchmark for the B200 hot loop design (FFMA vs FFMA2 vs MUFU vs DFMA,
// and a Horner step fed from shared memory). Reports ops per SM per clock using clock64().
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
__device__ unsigned long long g_cycles[1024];

template <int NCHAIN>
__global__ void ffma_kernel(float* out, float a, float b) {
  float x[NCHAIN];
#pragma unroll
  for (int i = 0; i < NCHAIN; ++i) x[i] = threadIdx.x * 0.001f + i;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCHAIN; ++i) x[i] = fmaf(x[i], a, b);
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NCHAIN; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

// 3 distinct register operands per FMA (a, b vary per chain)
template <int NCHAIN>
__global__ void ffma3_kernel(float* out, float a0, float b0) {
  float x[NCHAIN], a[NCHAIN], b[NCHAIN];
#pragma unroll
  for (int i = 0; i < NCHAIN; ++i) { x[i] = threadIdx.x * 0.001f + i; a[i] = a0 + i * 1e-3f + threadIdx.x*1e-6f; b[i] = b0 - i * 1e-3f; }
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCHAIN; ++i) x[i] = fmaf(x[i], a[i], b[i]);
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NCHAIN; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

__device__ __forceinline__ unsigned long long f2fma(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long r;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ unsigned long long pk(float lo, float hi) {
  return (unsigned long long)__float_as_uint(lo) | ((unsigned long long)__float_as_uint(hi) << 32);
}

template <int NCHAIN>
__global__ void ffma2_kernel(float* out, float a0, float b0) {
  unsigned long long x[NCHAIN], a[NCHAIN], b[NCHAIN];
#pragma unroll
  for (int i = 0; i < NCHAIN; ++i) { x[i] = pk(threadIdx.x * 0.001f + i, i*0.5f); a[i] = pk(a0 + i*1e-3f, a0 - i*1e-3f + threadIdx.x*1e-6f); b[i] = pk(b0, b0 + i); }
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCHAIN; ++i) x[i] = f2fma(x[i], a[i], b[i]);
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NCHAIN; ++i) s += __uint_as_float((unsigned)x[i]) + __uint_as_float((unsigned)(x[i] >> 32));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

template <int NCHAIN>
__global__ void mufu_kernel(float* out, float a) {
  float x[NCHAIN];
#pragma unroll
  for (int i = 0; i < NCHAIN; ++i) x[i] = threadIdx.x * 0.001f + i;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
    for (int i = 0; i < NCHAIN; ++i) x[i] = __sinf(x[i]);
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NCHAIN; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

template <int NCHAIN>
__global__ void dfma_kernel(double* out, double a, double b) {
  double x[NCHAIN];
#pragma unroll
  for (int i = 0; i < NCHAIN; ++i) x[i] = threadIdx.x * 0.001 + i;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < NCHAIN; ++i) x[i] = fma(x[i], a, b);
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  double s = 0.;
#pragma unroll
  for (int i = 0; i < NCHAIN; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

// Horner step over S components, y from shared memory (broadcast), scalar FFMA form.
template <int S>
__global__ void horner_kernel(float* out, const float2* __restrict__ ysrc, int nk) {
  extern __shared__ float2 ys[];
  for (int i = threadIdx.x; i < nk; i += blockDim.x) ys[i] = ysrc[i];
  float ar[S], ai[S], zr[S], zi[S];
#pragma unroll
  for (int s = 0; s < S; ++s) { ar[s] = 0.f; ai[s] = 0.f; __sincosf(0.01f * (threadIdx.x + s), &zi[s], &zr[s]); }
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int rep = 0; rep < 8; ++rep)
  for (int k = nk - 1; k >= 0; --k) {
    float2 y = ys[k];
#pragma unroll
    for (int s = 0; s < S; ++s) {
      float t1 = fmaf(-ai[s], zi[s], y.x);
      float t2 = fmaf(ai[s], zr[s], y.y);
      float nr = fmaf(ar[s], zr[s], t1);
      float ni = fmaf(ar[s], zi[s], t2);
      ar[s] = nr; ai[s] = ni;
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int s = 0; s < S; ++s) acc += ar[s] + ai[s];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

// Horner step, FFMA2 form: pairs of components (s, s+1) vectorized; y stored as (yr,yr,yi,yi).
template <int S2>
__global__ void horner2_kernel(float* out, const float4* __restrict__ ysrc, int nk) {
  extern __shared__ float4 ys4[];
  for (int i = threadIdx.x; i < nk; i += blockDim.x) ys4[i] = ysrc[i];
  unsigned long long ar[S2], ai[S2], zr[S2], zi[S2], nzi[S2];
#pragma unroll
  for (int s = 0; s < S2; ++s) {
    float a, b, c, d;
    __sincosf(0.01f * (threadIdx.x + 2*s), &a, &b);
    __sincosf(0.01f * (threadIdx.x + 2*s + 1), &c, &d);
    ar[s] = 0; ai[s] = 0; zr[s] = pk(b, d); zi[s] = pk(a, c); nzi[s] = pk(-a, -c);
  }
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int rep = 0; rep < 8; ++rep)
  for (int k = nk - 1; k >= 0; --k) {
    float4 y = ys4[k];
    unsigned long long yr = pk(y.x, y.y), yi = pk(y.z, y.w);
#pragma unroll
    for (int s = 0; s < S2; ++s) {
      unsigned long long t1 = f2fma(ai[s], nzi[s], yr);
      unsigned long long t2 = f2fma(ai[s], zr[s], yi);
      unsigned long long nr = f2fma(ar[s], zr[s], t1);
      unsigned long long ni = f2fma(ar[s], zi[s], t2);
      ar[s] = nr; ai[s] = ni;
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int s = 0; s < S2; ++s) acc += __uint_as_float((unsigned)ar[s]) + __uint_as_float((unsigned)(ai[s] >> 32));
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

static double avg_cycles(int nblk) {
  static unsigned long long h[1024];
  cudaMemcpyFromSymbol(h, g_cycles, sizeof(unsigned long long) * nblk);
  double s = 0; for (int i = 0; i < nblk; ++i) s += h[i]; return s / nblk;
}

int main() {
  cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0);
  int nsm = prop.multiProcessorCount;
  printf("device %s SMs %d clockRate(kHz) %d\n", prop.name, nsm, prop.clockRate);
  float* out; cudaMalloc(&out, 1 << 24);
  double* dout; cudaMalloc(&dout, 1 << 24);
  int thr = 512;  // 16 warps per block, one block per SM
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
#define RUN(name, launch, ops_per_thread) { launch; cudaDeviceSynchronize(); cudaEventRecord(e0); launch; cudaEventRecord(e1); cudaEventSynchronize(e1); \
    float ms; cudaEventElapsedTime(&ms, e0, e1); double cyc = avg_cycles(nsm); double ops = (double)(ops_per_thread) * thr; \
    printf("%-28s %8.2f ops/clk/SM   (%.3f ms, eff clock %.0f MHz) err=%s\n", name, ops / cyc, ms, cyc / (ms * 1e3), cudaGetErrorString(cudaGetLastError())); }
  RUN("FFMA imm-ish (x*a+b) ch8", (ffma_kernel<8><<<nsm, thr>>>(out, 1.0001f, 0.5f)), 8.0 * ITERS);
  RUN("FFMA 3-reg ch8", (ffma3_kernel<8><<<nsm, thr>>>(out, 1.0001f, 0.5f)), 8.0 * ITERS);
  RUN("FFMA2 (x2 counted) ch8", (ffma2_kernel<8><<<nsm, thr>>>(out, 1.0001f, 0.5f)), 16.0 * ITERS);
  RUN("MUFU sin ch8", (mufu_kernel<8><<<nsm, thr>>>(out, 1.f)), 8.0 * ITERS / 8);
  RUN("DFMA ch8", (dfma_kernel<8><<<nsm, thr>>>(dout, 1.0001, 0.5)), 8.0 * ITERS / 4);
  int nk = 1024;
  float2* y2; cudaMalloc(&y2, nk * sizeof(float2)); cudaMemset(y2, 0, nk * sizeof(float2));
  float4* y4; cudaMalloc(&y4, nk * sizeof(float4)); cudaMemset(y4, 0, nk * sizeof(float4));
  for (int t : {256, 512}) {
    thr = t;
    char nm[64];
    snprintf(nm, 64, "Horner S=5 FFMA thr%d", t);
    RUN(nm, (horner_kernel<5><<<nsm, thr, nk * 8>>>(out, y2, nk)), 8.0 * nk * 5 * 4);
    snprintf(nm, 64, "Horner S=9 FFMA thr%d", t);
    RUN(nm, (horner_kernel<9><<<nsm, thr, nk * 8>>>(out, y2, nk)), 8.0 * nk * 9 * 4);
    snprintf(nm, 64, "Horner S=4(2x2) FFMA2 thr%d", t);
    RUN(nm, (horner2_kernel<2><<<nsm, thr, nk * 16>>>(out, y4, nk)), 8.0 * nk * 4 * 4);
    snprintf(nm, 64, "Horner S=8(4x2) FFMA2 thr%d", t);
    RUN(nm, (horner2_kernel<4><<<nsm, thr, nk * 16>>>(out, y4, nk)), 8.0 * nk * 8 * 4);
    snprintf(nm, 64, "Horner S=10(5x2) FFMA2 thr%d", t);
    RUN(nm, (horner2_kernel<5><<<nsm, thr, nk * 16>>>(out, y4, nk)), 8.0 * nk * 10 * 4);
  }
  return 0;
}
