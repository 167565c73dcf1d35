// sort.cu -- locality order for the K1T likelihood kernels.
//
// The K1T correlation gathers one 64-byte table row per (particle, component, antenna) at the row of the element's
// delay; a warp of 32 random particles touches 32 unrelated rows per load (the kernel was L1-wavefront bound at large
// P).  Particles close in space have close delays to every anchor (R_s is 1-Lipschitz in the position), so processing
// them in a space-filling-curve order makes the warp's rows (nearly) coincide.  Per batch: a 30-bit Morton key of the
// position (10 bits per axis over a fixed 64 m cube, 6.25 cm cells), a radix sort of (key, index) pairs (CUB), and a
// gather of the positions (and per-particle SFVs) in that order.  The likelihood kernels then run on the sorted copy
// and the assembly writes every output back to its particle's index, so results are bit-identical to the unsorted
// evaluation (per-particle arithmetic does not depend on the processing order).
#include <cub/cub.cuh>

#include "cdms_internal.h"

namespace cdms {

__device__ __forceinline__ uint32_t spread10(uint32_t v) {  // 10 bits -> every third bit
  v &= 0x3FFu;
  v = (v | (v << 16)) & 0x030000FFu;
  v = (v | (v << 8)) & 0x0300F00Fu;
  v = (v | (v << 4)) & 0x030C30C3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}
__device__ __forceinline__ uint32_t cell10(double x) {
  const double c = floor((x + 32.0) * (1024.0 / 64.0));
  return (uint32_t)(c < 0.0 ? 0.0 : (c > 1023.0 ? 1023.0 : c));
}

__global__ void morton_kernel(const double* __restrict__ particles, int64_t P, int pstride, uint32_t* __restrict__ keys,
                              int* __restrict__ idx) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    const double* x = particles + i * pstride;
    keys[i] = spread10(cell10(x[0])) | (spread10(cell10(x[1])) << 1) | (spread10(cell10(x[2])) << 2);
    idx[i] = (int)i;
  }
}

// pos[i] = particles[perm[i]][0..2]; sfv_out[i] = sfv[perm[i]] (K x 3) when per-particle SFVs are given
__global__ void gather_sorted_kernel(const double* __restrict__ particles, int64_t P, int pstride,
                                     const double* __restrict__ sfv, int K, const int* __restrict__ perm,
                                     double* __restrict__ pos, double* __restrict__ sfv_out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = perm[i];
    const double* x = particles + p * pstride;
    pos[i * 3 + 0] = x[0];
    pos[i * 3 + 1] = x[1];
    pos[i * 3 + 2] = x[2];
    if (sfv_out)
      for (int k = 0; k < 3 * K; ++k) sfv_out[i * 3 * K + k] = sfv[p * 3 * K + k];
  }
}

size_t locality_sort_temp_bytes(int64_t P) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr, (const int*)nullptr,
                                  (int*)nullptr, (int)P, 0, 30);
  return bytes;
}

cudaError_t launch_locality_sort(const double* particles, int64_t P, int pstride, const double* sfv, int K, int sfv_pp,
                                 uint32_t* keys, uint32_t* keys_alt, int* idx, int* perm, void* temp, size_t temp_bytes,
                                 double* pos, double* sfv_out, cudaStream_t st) {
  if (P <= 0) return cudaSuccess;
  const unsigned g = (unsigned)((P + 255) / 256 < 65535 * 8 ? (P + 255) / 256 : 65535 * 8);
  morton_kernel<<<g, 256, 0, st>>>(particles, P, pstride, keys, idx);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys, keys_alt, idx, perm, (int)P, 0, 30, st);
  if (e != cudaSuccess) return e;
  gather_sorted_kernel<<<g, 256, 0, st>>>(particles, P, pstride, sfv, K, perm, pos, sfv_pp ? sfv_out : nullptr);
  return cudaGetLastError();
}

}  // namespace cdms
