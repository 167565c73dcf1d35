// F3: the efficient birth proposal of P:L3282-3346 for one new PF.
//
//   1. residual z~_j = Pi_perp_j z_j, Pi_perp_j = I - Psi_j Psi_j^dagger with Psi_j the steering vectors of the
//      LOS and the legacy PFs' MMSE SFVs at the predicted MMSE MT state: Psi from the fp64
//      response kernel, Psi^H Psi and Psi^H z as fixed-order fp64 block reductions (birth_dots_kernel), a
//      complex Cholesky solve per PA (birth_solve_kernel), z~ = z - Psi a rounded once to complex64
//      (birth_resid_kernel);
//   2. N_g candidates p_i uniform in the partition box (Philox (key; i, i >> 32, counter, 7)), padded to a multiple
//      of 8 with copies of the last one (birth_cand_kernel);
//      the coherent Bartlett correlations z~_j^H psi(x_hat, p_i) all share the MT position and differ only in the
//      wall, i.e. they are the components of pseudo-particles at x_hat whose SFVs are the candidates: the likelihood
//      engine (K1, or the tensor cores for PLANAR_NB) runs with K = 8 per-particle SFVs (8 candidates per
//      pseudo-particle, S = 9: the engine's efficient regime, where each snapshot element loaded from shared
//      memory feeds 9 components) and the residual as the snapshot (cdms.cpp); component 0 (LOS) is not used;
//   3. P_B,i = |sum_j c_ij|^2 / N_z^2, its sum, the first argmax (birth_pb_kernel, birth_mode_kernel) and the
//      weighted second moment about the mode (birth_cov_*), all fixed-partition fp64 reductions.
#include <math.h>

#include "cdms_internal.h"
#include "geometry.cuh"

namespace cdms {

namespace {
constexpr int BIRTH_BLOCK = 256;
constexpr int BIRTH_ITEMS = 2048;  // candidates per reduction block (fixed partition -> determinism)
constexpr int BIRTH_PACK = MAXS - 1;  // candidates per pseudo-particle (its walls)

__device__ __forceinline__ double2 cconj_mul(double2 a, double2 b) {  // conj(a) b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
template <typename T>
__device__ __forceinline__ T block_sum_d(T v, T* red) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int s = BIRTH_BLOCK / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) red[threadIdx.x] = red[threadIdx.x] + red[threadIdx.x + s];
    __syncthreads();
  }
  const T r = red[0];
  __syncthreads();
  return r;
}
__device__ __forceinline__ double2 operator+(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
}  // namespace

// (1a) dots[j][e]: e < n(n+1)/2 -> (Psi^H Psi)_{rc}, r >= c, row-major lower triangle; then (Psi^H z)_r.
// psi [J][n][Nz] (item j n + s), y [J][Nz] complex64.  Grid (entries, J).
__global__ void birth_dots_kernel(int nz, int n, const double2* __restrict__ psi, const float2* __restrict__ y,
                                  double2* __restrict__ dots) {
  __shared__ double2 red[BIRTH_BLOCK];
  const int j = blockIdx.y, e = blockIdx.x;
  const int ntri = n * (n + 1) / 2;
  const double2* pj = psi + (size_t)j * n * nz;
  double2 acc = make_double2(0.0, 0.0);
  if (e < ntri) {
    int r = 0, c = e;
    while (c > r) { c -= r + 1; ++r; }
    const double2* a = pj + (size_t)r * nz;
    const double2* b = pj + (size_t)c * nz;
    for (int k = threadIdx.x; k < nz; k += BIRTH_BLOCK) acc = acc + cconj_mul(a[k], b[k]);
  } else {
    const double2* a = pj + (size_t)(e - ntri) * nz;
    const float2* z = y + (size_t)j * nz;
    for (int k = threadIdx.x; k < nz; k += BIRTH_BLOCK) {
      const float2 v = z[k];
      acc = acc + cconj_mul(a[k], make_double2(v.x, v.y));
    }
  }
  const double2 s = block_sum_d(acc, red);
  if (threadIdx.x == 0) dots[(size_t)j * (ntri + n) + e] = s;
}

// (1b) per PA: Psi^H Psi = L L^H (complex Cholesky, fp64), a = (Psi^H Psi)^{-1} Psi^H z.  Singular -> FLAG_NAN.
__global__ void birth_solve_kernel(int J, int n, const double2* __restrict__ dots, double2* __restrict__ coef,
                                   int* flags) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= J) return;
  const int ntri = n * (n + 1) / 2;
  const double2* d = dots + (size_t)j * (ntri + n);
  double2 L[MAXS * MAXS], b[MAXS];
  for (int r = 0, e = 0; r < n; ++r)
    for (int c = 0; c <= r; ++c, ++e) L[r * n + c] = d[e];
  for (int r = 0; r < n; ++r) b[r] = d[ntri + r];
  for (int c = 0; c < n; ++c) {
    double dd = L[c * n + c].x;
    for (int k = 0; k < c; ++k) dd -= L[c * n + k].x * L[c * n + k].x + L[c * n + k].y * L[c * n + k].y;
    if (!(dd > 0.0)) {
      atomicOr(flags, FLAG_NAN);
      for (int r = 0; r < n; ++r) coef[(size_t)j * n + r] = make_double2(0.0, 0.0);
      return;
    }
    const double l = sqrt(dd);
    L[c * n + c] = make_double2(l, 0.0);
    for (int r = c + 1; r < n; ++r) {
      double2 acc = L[r * n + c];
      for (int k = 0; k < c; ++k) {  // acc -= L_rk conj(L_ck)
        const double2 x = L[r * n + k], y = L[c * n + k];
        acc.x -= x.x * y.x + x.y * y.y;
        acc.y -= x.y * y.x - x.x * y.y;
      }
      L[r * n + c] = make_double2(acc.x / l, acc.y / l);
    }
  }
  for (int r = 0; r < n; ++r) {  // L w = b
    double2 acc = b[r];
    for (int c = 0; c < r; ++c) {
      const double2 x = L[r * n + c], y = b[c];
      acc.x -= x.x * y.x - x.y * y.y;
      acc.y -= x.x * y.y + x.y * y.x;
    }
    b[r] = make_double2(acc.x / L[r * n + r].x, acc.y / L[r * n + r].x);
  }
  for (int r = n - 1; r >= 0; --r) {  // L^H a = w
    double2 acc = b[r];
    for (int c = r + 1; c < n; ++c) {  // acc -= conj(L_cr) a_c
      const double2 x = L[c * n + r], y = b[c];
      acc.x -= x.x * y.x + x.y * y.y;
      acc.y -= x.x * y.y - x.y * y.x;
    }
    b[r] = make_double2(acc.x / L[r * n + r].x, acc.y / L[r * n + r].x);
  }
  for (int r = 0; r < n; ++r) coef[(size_t)j * n + r] = b[r];
}

// (1c) z~ = z - Psi a (fp64), rounded once to complex64.  One thread per (j, element).
__global__ void birth_resid_kernel(int J, int nz, int n, const double2* __restrict__ psi, const float2* __restrict__ y,
                                   const double2* __restrict__ coef, float2* __restrict__ zr) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)J * nz) return;
  const int j = (int)(t / nz);
  const int k = (int)(t - (int64_t)j * nz);
  const float2 v = y[t];
  double re = v.x, im = v.y;
  for (int s = 0; s < n; ++s) {
    const double2 p = psi[((size_t)j * n + s) * nz + k], a = coef[(size_t)j * n + s];
    re -= p.x * a.x - p.y * a.y;
    im -= p.x * a.y + p.y * a.x;
  }
  zr[t] = make_float2((float)re, (float)im);
}

// (2) candidates, padded to n_pad with copies of the last (the pseudo-particles take BIRTH_PACK walls each)
__global__ void birth_cand_kernel(int64_t N_g, int64_t n_pad, uint64_t key, uint64_t counter, BirthBox box,
                                  double* __restrict__ cand) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_pad) return;
  const int64_t i = t < N_g ? t : N_g - 1;
  const uint4 x = philox_step(make_uint4((uint32_t)i, (uint32_t)((uint64_t)i >> 32), (uint32_t)counter, 7u),
                              make_uint2((uint32_t)key, (uint32_t)(key >> 32)));
  const uint32_t xs[3] = {x.x, x.y, x.z};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double u = ((double)xs[a] + 0.5) * 0x1p-32;  // exact
    cand[3 * t + a] = __dadd_rn(box.lo[a], __dmul_rn(u, box.hi[a] - box.lo[a]));  // uncontracted: bit-equal to the oracle
  }
}

// (3a) P_B,i = |sum_j c_ij|^2 / N_z^2 (c_ij = psi_ij^H z~_j; |sum conj| = |sum|), per-block (sum, max, argmax).
__global__ void birth_pb_kernel(int64_t N_g, int J, double inv_nz2, const double2* __restrict__ c, double* __restrict__ pb,
                                double4* __restrict__ part) {
  __shared__ double rs[BIRTH_BLOCK];
  __shared__ double rm[BIRTH_BLOCK];
  __shared__ int64_t ri[BIRTH_BLOCK];
  const int64_t i0 = (int64_t)blockIdx.x * BIRTH_ITEMS;
  double sum = 0.0, mx = -1.0;
  int64_t arg = -1;
  for (int t = threadIdx.x; t < BIRTH_ITEMS; t += BIRTH_BLOCK) {
    const int64_t i = i0 + t;
    if (i >= N_g) break;
    double re = 0.0, im = 0.0;
    const int64_t pp = i / BIRTH_PACK;
    const int comp = 1 + (int)(i - pp * BIRTH_PACK);
    for (int j = 0; j < J; ++j) {
      const double2 v = c[(pp * J + j) * (BIRTH_PACK + 1) + comp];
      re += v.x;
      im += v.y;
    }
    const double v = (re * re + im * im) * inv_nz2;
    pb[i] = v;
    sum += v;
    if (v > mx) { mx = v; arg = i; }  // per thread: increasing i -> first index kept on ties
  }
  rs[threadIdx.x] = sum;
  rm[threadIdx.x] = mx;
  ri[threadIdx.x] = arg;
  __syncthreads();
  for (int s = BIRTH_BLOCK / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) {
      rs[threadIdx.x] += rs[threadIdx.x + s];
      const double m2 = rm[threadIdx.x + s];
      const int64_t a2 = ri[threadIdx.x + s];
      if (m2 > rm[threadIdx.x] || (m2 == rm[threadIdx.x] && a2 >= 0 && (ri[threadIdx.x] < 0 || a2 < ri[threadIdx.x]))) {
        rm[threadIdx.x] = m2;
        ri[threadIdx.x] = a2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = make_double4(rs[0], rm[0], (double)ri[0], 0.0);
}

// (3b) combine the block partials: each thread folds a strided set of blocks in block order, then a fixed tree;
// ties keep the first index (thread t holds blocks t, t + 256, ... < those of thread t + 1 in each round, so the
// tree compares (value, index) pairs explicitly).  scratch = (sum P_B, i*, mu[3]); zero / non-finite sum -> flags.
__global__ void birth_mode_kernel(int64_t nblk, const double4* __restrict__ part, const double* __restrict__ cand,
                                  double* __restrict__ scratch, int* flags) {
  __shared__ double rs[BIRTH_BLOCK];
  __shared__ double rm[BIRTH_BLOCK];
  __shared__ int64_t ri[BIRTH_BLOCK];
  double sum = 0.0, mx = -1.0;
  int64_t arg = -1;
  for (int64_t b = threadIdx.x; b < nblk; b += BIRTH_BLOCK) {
    const double4 v = part[b];
    sum += v.x;
    const int64_t a2 = (int64_t)v.z;
    if (v.y > mx || (v.y == mx && a2 < arg)) { mx = v.y; arg = a2; }
  }
  rs[threadIdx.x] = sum;
  rm[threadIdx.x] = mx;
  ri[threadIdx.x] = arg;
  __syncthreads();
  for (int s = BIRTH_BLOCK / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) {
      rs[threadIdx.x] += rs[threadIdx.x + s];
      const double m2 = rm[threadIdx.x + s];
      const int64_t a2 = ri[threadIdx.x + s];
      if (m2 > rm[threadIdx.x] || (m2 == rm[threadIdx.x] && a2 >= 0 && (ri[threadIdx.x] < 0 || a2 < ri[threadIdx.x]))) {
        rm[threadIdx.x] = m2;
        ri[threadIdx.x] = a2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double tot = rs[0];
    int64_t a = ri[0];
    if (!isfinite(tot)) atomicOr(flags, FLAG_NAN);
    else if (!(tot > 0.0)) atomicOr(flags, FLAG_ZEROMASS);
    if (a < 0) a = 0;
    scratch[0] = tot;
    scratch[1] = (double)a;
    for (int q = 0; q < 3; ++q) scratch[2 + q] = cand[3 * a + q];
  }
}

// (3c) per block sum_i P_B,i (p_i - mu)(p_i - mu)^T, upper triangle (6 entries)
__global__ void birth_cov_partial_kernel(int64_t N_g, const double* __restrict__ pb, const double* __restrict__ cand,
                                         const double* __restrict__ scratch, double* __restrict__ part6) {
  __shared__ double red[BIRTH_BLOCK];
  const int64_t i0 = (int64_t)blockIdx.x * BIRTH_ITEMS;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  const double mu[3] = {scratch[2], scratch[3], scratch[4]};
  for (int t = threadIdx.x; t < BIRTH_ITEMS; t += BIRTH_BLOCK) {
    const int64_t i = i0 + t;
    if (i >= N_g) break;
    const double w = pb[i];
    const double d[3] = {cand[3 * i] - mu[0], cand[3 * i + 1] - mu[1], cand[3 * i + 2] - mu[2]};
    acc[0] += w * d[0] * d[0]; acc[1] += w * d[0] * d[1]; acc[2] += w * d[0] * d[2];
    acc[3] += w * d[1] * d[1]; acc[4] += w * d[1] * d[2]; acc[5] += w * d[2] * d[2];
  }
  for (int q = 0; q < 6; ++q) {
    const double s = block_sum_d(acc[q], red);
    if (threadIdx.x == 0) part6[(size_t)blockIdx.x * 6 + q] = s;
  }
}

// (3d) out[0..2] = mu, out[3..11] = C (row-major, symmetric), out[12] = i*; block-strided fixed-order sums
__global__ void birth_cov_final_kernel(int64_t nblk, const double* __restrict__ part6, const double* __restrict__ scratch,
                                       double* __restrict__ out) {
  __shared__ double red[BIRTH_BLOCK];
  double acc[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t b = threadIdx.x; b < nblk; b += BIRTH_BLOCK)
    for (int q = 0; q < 6; ++q) acc[q] += part6[b * 6 + q];
  double tot[6];
  for (int q = 0; q < 6; ++q) tot[q] = block_sum_d(acc[q], red);
  if (threadIdx.x == 0) {
    const double inv = scratch[0] > 0.0 ? 1.0 / scratch[0] : 0.0;
    const int map[9] = {0, 1, 2, 1, 3, 4, 2, 4, 5};
    for (int a = 0; a < 3; ++a) out[a] = scratch[2 + a];
    for (int q = 0; q < 9; ++q) out[3 + q] = tot[map[q]] * inv;
    out[12] = scratch[1];
  }
}

// (0) response items for Psi: item j n + s at x_hat, (j, s), and the legacy SFV list in device memory
__global__ void birth_items_kernel(BirthBox box, int J, double* __restrict__ pos, int32_t* __restrict__ js,
                                   double* __restrict__ sfv) {
  const int n = box.L + 1;
  const int t = threadIdx.x;
  if (t < J * n) {
    for (int a = 0; a < 3; ++a) pos[3 * t + a] = box.x_hat[a];
    js[2 * t] = t / n;
    js[2 * t + 1] = t % n;
  }
  if (t < box.L)
    for (int a = 0; a < 3; ++a) sfv[3 * t + a] = box.sfv[t][a];
}

// ---------------------------------------------------------------------------- launchers
cudaError_t launch_birth_items(const BirthBox& box, int J, double* pos, int32_t* js, double* sfv, cudaStream_t st) {
  birth_items_kernel<<<1, 128, 0, st>>>(box, J, pos, js, sfv);
  return cudaGetLastError();
}
int64_t birth_blocks(int64_t N_g) { return (N_g + BIRTH_ITEMS - 1) / BIRTH_ITEMS; }

cudaError_t launch_birth_residual(int J, int nz, int n, const double2* psi, const float2* y, double2* dots,
                                  double2* coef, float2* zr, int* flags, cudaStream_t st) {
  const int ntri = n * (n + 1) / 2;
  birth_dots_kernel<<<dim3(ntri + n, J), BIRTH_BLOCK, 0, st>>>(nz, n, psi, y, dots);
  birth_solve_kernel<<<1, 32, 0, st>>>(J, n, dots, coef, flags);
  const int64_t tot = (int64_t)J * nz;
  birth_resid_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(J, nz, n, psi, y, coef, zr);
  return cudaGetLastError();
}
int64_t birth_pseudo_particles(int64_t N_g) { return (N_g + BIRTH_PACK - 1) / BIRTH_PACK; }
cudaError_t launch_birth_candidates(int64_t N_g, uint64_t key, uint64_t counter, const BirthBox& box, double* cand,
                                    cudaStream_t st) {
  const int64_t n_pad = birth_pseudo_particles(N_g) * BIRTH_PACK;
  birth_cand_kernel<<<(unsigned)((n_pad + 255) / 256), 256, 0, st>>>(N_g, n_pad, key, counter, box, cand);
  return cudaGetLastError();
}
cudaError_t launch_birth_reduce(int64_t N_g, int J, int nz, const double2* c, const double* cand, double* pb,
                                double4* part, double* part6, double* scratch, double* out, int* flags,
                                cudaStream_t st) {
  const int64_t nblk = birth_blocks(N_g);
  const double inv_nz2 = 1.0 / ((double)nz * (double)nz);
  birth_pb_kernel<<<(unsigned)nblk, BIRTH_BLOCK, 0, st>>>(N_g, J, inv_nz2, c, pb, part);
  birth_mode_kernel<<<1, BIRTH_BLOCK, 0, st>>>(nblk, part, cand, scratch, flags);
  birth_cov_partial_kernel<<<(unsigned)nblk, BIRTH_BLOCK, 0, st>>>(N_g, pb, cand, scratch, part6);
  birth_cov_final_kernel<<<1, BIRTH_BLOCK, 0, st>>>(nblk, part6, scratch, out);
  return cudaGetLastError();
}

}  // namespace cdms
