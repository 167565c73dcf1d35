// Wall-clock FP32 throughput of FFMA2 vs FFMA with independent chains (CUDA events, whole GPU).
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float lo, float hi) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ u64 f2(u64 a, u64 b, u64 c) { u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
constexpr int IT = 8192;
template <int NC> __global__ void kf2(float* out, float a0) {
  u64 x[NC], w[NC], b[NC];
  for (int i = 0; i < NC; ++i) { x[i] = pk(threadIdx.x * 1e-3f + i, i * 0.5f); w[i] = pk(0.999f - 1e-4f * i, 1.0001f); b[i] = pk(a0, a0 * i); }
  for (int it = 0; it < IT; ++it)
#pragma unroll
    for (int i = 0; i < NC; ++i) x[i] = f2(x[i], w[i], b[i]);
  float s = 0; for (int i = 0; i < NC; ++i) s += __uint_as_float((unsigned)x[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NC> __global__ void kf1(float* out, float a0) {
  float x[NC], w[NC], b[NC];
  for (int i = 0; i < NC; ++i) { x[i] = threadIdx.x * 1e-3f + i; w[i] = 0.999f - 1e-4f * i; b[i] = a0 * i; }
  for (int it = 0; it < IT; ++it)
#pragma unroll
    for (int i = 0; i < NC; ++i) x[i] = fmaf(x[i], w[i], b[i]);
  float s = 0; for (int i = 0; i < NC; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int nsm, clk; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0); cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int bps : {1, 2, 4, 8}) {
    for (int kind = 0; kind < 2; ++kind) {
      int blocks = nsm * bps, thr = 256;
      for (int r = 0; r < 2; ++r) { if (kind) kf2<8><<<blocks, thr>>>(out, 0.5f); else kf1<8><<<blocks, thr>>>(out, 0.5f); }
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) { if (kind) kf2<8><<<blocks, thr>>>(out, 0.5f); else kf1<8><<<blocks, thr>>>(out, 0.5f); }
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fma = 5.0 * blocks * thr * 8.0 * IT * (kind ? 2 : 1);
      printf("%s %d blocks/SM: %.1f TFLOP/s (%.1f FMA/clk/SM at %d MHz) %s\n", kind ? "FFMA2" : "FFMA ", bps,
             2 * fma / (ms * 1e-3) / 1e12, fma / (ms * 1e-3) / (nsm * clk * 1e3), clk / 1000, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
