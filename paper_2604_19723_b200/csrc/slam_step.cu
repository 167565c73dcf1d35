// slam_step.cu -- kernels of the F4 step driver (cdms_slam_step, cdms.cpp): the Gamma / Gaussian state transitions
// (P:L3757-3815), the birth message's particles, weighted sums for the MMSE estimates and existence
// probabilities (eq. existenceProb), the belief-averaged columns of the update messages (reading F4c;
// P:L686-698, eqs. musnj3/musnj4), the gathers of the driver's own arrays and the resampling gathers.
// The update messages themselves are the library's (cdms_loglik, cdms_noise_update, cdms_pf_update, cdms_ppr_update).
//
// Random numbers: Philox4x32-10 blocks (key; index, index >> 32, n, stream) with the stream map of DESIGN.md section
// 3 (F4-i): 0x100 + 16 j + a noise Gamma, 0x200 + 16 i SFV jitter, 0x201 + 16 i amplitude-mean jitter,
// 0x300 + 16 i + a amplitude-variance Gamma, 0x600 / 0x601 birth normals / uniforms, 0x700 + 16 i SFV
// regularization.
#include <math.h>

#include "cdms_internal.h"

namespace cdms {

namespace {

__device__ __forceinline__ uint4 philox_blk(uint64_t key, uint64_t index, uint64_t step, uint32_t stream) {
  return philox_step(make_uint4((uint32_t)index, (uint32_t)(index >> 32), (uint32_t)step, stream),
                     make_uint2((uint32_t)key, (uint32_t)(key >> 32)));
}
__device__ __forceinline__ double u01(uint32_t x) { return ((double)x + 0.5) * 0x1p-32; }

// four N(0, 1): Box-Muller on the block's word pairs (0, 1), (2, 3) (the MT prediction's generator, beliefs.cu)
__device__ __forceinline__ void normals4_slam(uint64_t key, uint64_t step, uint64_t index, uint32_t stream,
                                              double n[4]) {
  const uint4 x = philox_blk(key, index, step, stream);
  const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const double r = sqrt(-2.0 * log(u01(xs[2 * h])));
    n[2 * h] = r * cos(2.0 * PI * u01(xs[2 * h + 1]));
    n[2 * h + 1] = r * sin(2.0 * PI * u01(xs[2 * h + 1]));
  }
}

// Gamma(c, 1), c >= 1: Marsaglia-Tsang (d = c - 1/3, k = 1/sqrt(9 d); accept d v, v = (1 + k z)^3, if v > 0 and
// ln u < z^2/2 + d - d v + d ln v); attempt a uses block (index, step, stream + a): z from words 0, 1, u from word 2;
// d after 16 rejections (reading F4-g)
__device__ double gamma_draw(uint64_t key, uint64_t step, uint64_t index, uint32_t stream, double c) {
  const double d = c - 1.0 / 3.0, k = 1.0 / sqrt(9.0 * d);
  for (uint32_t a = 0; a < 16; ++a) {
    const uint4 x = philox_blk(key, index, step, stream + a);
    const double z = sqrt(-2.0 * log(u01(x.x))) * cos(2.0 * PI * u01(x.y));
    const double t = 1.0 + k * z;
    if (t <= 0.0) continue;
    const double v = t * t * t;
    if (log(u01(x.z)) < 0.5 * z * z + d - d * v + d * log(v)) return d * v;
  }
  return d;
}

constexpr int SB = 256;  // block of the single-block reductions

// fixed-order block tree (SB threads) of one double
__device__ double block_sum(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int o = SB / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

}  // namespace

// ---------------------------------------------------------------------------- transitions (phase (i))
// xi: eta_n = eta_{n-1} g / c_eta, g ~ Gamma(c_eta, 1) -- G(eta; c_eta, eta_{n-1}/c_eta) of P:L3783-3784
__global__ void slam_noise_predict_kernel(double* __restrict__ eta, int J, int64_t P, double c, uint64_t key,
                                          uint64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)J * P) return;
  const int j = (int)(i / P);
  const int64_t p = i - (int64_t)j * P;
  eta[i] *= gamma_draw(key, n, (uint64_t)p, 0x100u + 16u * (uint32_t)j, c) / c;
}
cudaError_t launch_slam_noise_predict(double* eta, int J, int64_t P, double c, uint64_t key, uint64_t n,
                                      cudaStream_t st) {
  const int64_t t = (int64_t)J * P;
  slam_noise_predict_kernel<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(eta, J, P, c, key, n);
  return cudaGetLastError();
}

// alpha (legacy PF, slot i): phi += sigma_sfv N(0, I3), mu += CN(0, sigma_mu^2), gamma <- gamma g /
// c_gamma, g ~ Gamma(c_gamma, 1), w <- p_s w; phi == NULL for the LOS
__global__ void slam_pf_predict_kernel(double* __restrict__ phi, double2* __restrict__ mu, double* __restrict__ gam,
                                       double* __restrict__ w, int64_t P, int slot, double sigma_sfv, double sigma_mu,
                                       double c_gamma, double p_s, uint64_t key, uint64_t n) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  double z[4];
  if (phi) {
    normals4_slam(key, n, (uint64_t)p, 0x200u + 16u * (uint32_t)slot, z);
    for (int a = 0; a < 3; ++a) phi[3 * p + a] += sigma_sfv * z[a];
  }
  normals4_slam(key, n, (uint64_t)p, 0x201u + 16u * (uint32_t)slot, z);
  const double s = sigma_mu / sqrt(2.0);
  double2 m = mu[p];
  m.x += s * z[0];
  m.y += s * z[1];
  mu[p] = m;
  gam[p] *= gamma_draw(key, n, (uint64_t)p, 0x300u + 16u * (uint32_t)slot, c_gamma) / c_gamma;
  w[p] *= p_s;
}
cudaError_t launch_slam_pf_predict(double* phi, double2* mu, double* gam, double* w, int64_t P, int slot,
                                   double sigma_sfv, double sigma_mu, double c_gamma, double p_s, uint64_t key,
                                   uint64_t n, cudaStream_t st) {
  slam_pf_predict_kernel<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(phi, mu, gam, w, P, slot, sigma_sfv, sigma_mu,
                                                                     c_gamma, p_s, key, n);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------- births (reading F4h)
// phi_p = mu_q + L_q z_p (z: stream 0x600 normals 0..2), mu_p = mu_max sqrt(u0) e^{j 2 pi u1}, gamma_p = gamma_max u2
// (stream 0x601 words 0..2); lw_p = log of the importance ratio f_B / f_B^p up to a constant: |z_p|^2 / 2 inside the
// box, -inf outside.  phi == NULL: the LOS at n = 0 (amplitudes only).  L9 row-major lower-triangular.
struct BirthArgs {
  double mu[3], L[9], lo[3], hi[3];
  double mu_max, gamma_max;
};
__global__ void slam_birth_sample_kernel(const BirthArgs a, double* __restrict__ phi, double2* __restrict__ mu,
                                         double* __restrict__ gam, double* __restrict__ lw, int64_t P, uint64_t key,
                                         uint64_t n) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const uint4 x = philox_blk(key, (uint64_t)p, n, 0x601u);
  const double u0 = u01(x.x), u1 = u01(x.y), u2 = u01(x.z);
  const double r = a.mu_max * sqrt(u0);
  mu[p] = make_double2(r * cos(2.0 * PI * u1), r * sin(2.0 * PI * u1));
  gam[p] = a.gamma_max * u2;
  if (!phi) return;
  double z[4];
  normals4_slam(key, n, (uint64_t)p, 0x600u, z);
  bool in = true;
  for (int c = 0; c < 3; ++c) {
    double v = a.mu[c];
    for (int b = 0; b <= c; ++b) v += a.L[3 * c + b] * z[b];
    phi[3 * p + c] = v;
    in = in && v >= a.lo[c] && v <= a.hi[c];
  }
  lw[p] = in ? 0.5 * (z[0] * z[0] + z[1] * z[1] + z[2] * z[2]) : -INFINITY;
}
// w_p = p_B e^{lw_p - M} / S from the two-level LSE (lse.cu); out[0] = S (0: no particle in the box)
__global__ void slam_birth_norm_kernel(const double* __restrict__ lw, int64_t P, double pB,
                                       const double* __restrict__ lse, double* __restrict__ w,
                                       double* __restrict__ out) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const double M = lse[0], S = lse[1];
  w[p] = S > 0.0 ? pB * exp(lw[p] - M) / S : 0.0;
  if (p == 0) out[0] = S;
}
cudaError_t launch_slam_birth(const double* mu_q, const double* Lq, const double* box, double mu_max, double gamma_max,
                              double pB, double* phi, double2* mu, double* gam, double* lw, double* w, double* out,
                              double* lse_part, int64_t P, uint64_t key, uint64_t n, cudaStream_t st) {
  BirthArgs a{};
  for (int c = 0; c < 3; ++c) {
    a.mu[c] = mu_q ? mu_q[c] : 0.0;
    a.lo[c] = box ? box[c] : 0.0;
    a.hi[c] = box ? box[3 + c] : 0.0;
  }
  for (int c = 0; c < 9; ++c) a.L[c] = Lq ? Lq[c] : 0.0;
  a.mu_max = mu_max;
  a.gamma_max = gamma_max;
  slam_birth_sample_kernel<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(a, phi, mu, gam, lw, P, key, n);
  if (phi) {
    double* lse = lse_part + 3 * lse_blocks(P);
    const cudaError_t e = launch_lse_rows(lw, P, 1, P, nullptr, 0, lse_part, lse, st);
    if (e != cudaSuccess) return e;
    slam_birth_norm_kernel<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(lw, P, pB, lse, w, out);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------- weighted sums
// out[4 job] = sum_p w_p (w == NULL: P), out[4 job + 1 + c] = sum_p w_p v[p vs + c], c < nc <= 3.  Two levels with a
// fixed grouping (NBW blocks per job over contiguous chunks, then one block per job over the chunks in order), so
// repeated calls give identical bits.
int slam_wsum_blocks(int64_t P) {
  int64_t nb = (P + 8191) / 8192;
  return (int)(nb < 1 ? 1 : (nb > 256 ? 256 : nb));
}
__global__ void __launch_bounds__(SB) slam_wsum_part_kernel(const __grid_constant__ SlamWsumJobs jobs, int NBW,
                                                            double* __restrict__ part) {
  __shared__ double sh[SB];
  const SlamWsumJob& jb = jobs.job[blockIdx.y];
  const int64_t C = (jb.P + NBW - 1) / NBW;
  const int64_t p0 = (int64_t)blockIdx.x * C, p1 = p0 + C < jb.P ? p0 + C : jb.P;
  double a[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t p = p0 + threadIdx.x; p < p1; p += SB) {
    const double w = jb.w ? jb.w[p] : 1.0;
    a[0] += w;
    for (int c = 0; c < jb.nc; ++c) a[1 + c] += w * jb.v[p * jb.vs + c];
  }
  for (int c = 0; c < 4; ++c) {
    const double r = block_sum(a[c], sh);
    if (threadIdx.x == 0) part[((int64_t)blockIdx.y * NBW + blockIdx.x) * 4 + c] = r;
  }
}
__global__ void __launch_bounds__(SB) slam_wsum_final_kernel(const double* __restrict__ part, int NBW,
                                                             double* __restrict__ out) {
  __shared__ double sh[SB];
  const double* pj = part + (int64_t)blockIdx.x * NBW * 4;
  for (int c = 0; c < 4; ++c) {
    double a = 0.0;
    for (int b = threadIdx.x; b < NBW; b += SB) a += pj[4 * b + c];
    const double r = block_sum(a, sh);
    if (threadIdx.x == 0) out[4 * blockIdx.x + c] = r;
  }
}
cudaError_t launch_slam_wsum(const SlamWsumJobs& jobs, double* part, double* out, cudaStream_t st) {
  if (jobs.n <= 0) return cudaSuccess;
  int64_t Pm = 1;
  for (int i = 0; i < jobs.n; ++i) Pm = jobs.job[i].P > Pm ? jobs.job[i].P : Pm;
  const int NBW = slam_wsum_blocks(Pm);
  slam_wsum_part_kernel<<<dim3(NBW, jobs.n), SB, 0, st>>>(jobs, NBW, part);
  slam_wsum_final_kernel<<<jobs.n, SB, 0, st>>>(part, NBW, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------- belief-averaged columns (reading F4c)
// Sample k < K of the paired particles: p_k = floor((2k + 1) P / (2K)).
__device__ __forceinline__ int64_t bv_index(int64_t k, int64_t K, int64_t P) { return ((2 * k + 1) * P) / (2 * K); }

// per slot s: sum_k w_s[p_k] (fixed order) -> wk[s]
__global__ void __launch_bounds__(SB) slam_bv_wsum_kernel(const double* __restrict__ w, int64_t P, int64_t K,
                                                          double* __restrict__ wk) {
  __shared__ double sh[SB];
  const int s = blockIdx.x;
  double a = 0.0;
  for (int64_t k = threadIdx.x; k < K; k += SB) a += w[(int64_t)s * P + bv_index(k, K, P)];
  a = block_sum(a, sh);
  if (threadIdx.x == 0) wk[s] = a;
}
// response items of samples [k0, k0 + B): item ((k - k0) J + j) S + s at the paired MT particle x_{p_k}; component 0
// (LOS) for slot 0, else component 1 with the item's own wall phi_s[p_k] (response_kernel with sfv_per_item)
__global__ void slam_bv_items_kernel(const double* __restrict__ x, const double* __restrict__ phi, int64_t P,
                                     int64_t K, int64_t k0, int B, int J, int S, double* __restrict__ pos,
                                     int32_t* __restrict__ js, double* __restrict__ sfv) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * J * S) return;
  const int s = (int)(i % S), j = (int)((i / S) % J);
  const int64_t k = k0 + i / ((int64_t)J * S);
  const int64_t p = bv_index(k < K ? k : K - 1, K, P);
  for (int c = 0; c < 3; ++c) {
    pos[3 * i + c] = x[6 * p + c];
    sfv[3 * i + c] = s ? phi[((int64_t)s * P + p) * 3 + c] : 0.0;
  }
  js[2 * i] = j;
  js[2 * i + 1] = s ? 1 : 0;
}
// thread per (j, s, element): the chunk's samples in order into the fp64 sums (eq. musnj4):
//   u += eps pi mu psi,  m += eps zeta pi sqrt(gamma + |mu|^2 (1 - zeta eps)) psi,
//   mw += eps pi sqrt(gamma + |mu|^2 (1 - zeta)) psi,   pi = w[p_k] / wk[s]
__global__ void slam_bv_accum_kernel(const double2* __restrict__ psi, const double2* __restrict__ mu,
                                     const double* __restrict__ gam, const double* __restrict__ w,
                                     const double* __restrict__ wk, const double* __restrict__ par, int64_t P,
                                     int64_t K, int64_t k0, int B, int J, int S, int64_t Nz, double2* __restrict__ au,
                                     double2* __restrict__ am, double2* __restrict__ aw) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)J * S * Nz) return;
  const int64_t e = i % Nz;
  const int s = (int)((i / Nz) % S), j = (int)(i / (Nz * S));
  const double eps = par[s], zeta = par[MAXS + s * MAXJ + j];
  const double wks = wk[s];
  if (!(eps > 0.0) || !(wks > 0.0)) return;
  double2 u = au[i], m = am[i], mw = aw[i];
  for (int b = 0; b < B && k0 + b < K; ++b) {
    const int64_t p = bv_index(k0 + b, K, P);
    const double pi = w[(int64_t)s * P + p] / wks;
    const double2 mp = mu[(int64_t)s * P + p];
    const double a2 = mp.x * mp.x + mp.y * mp.y, g = gam[(int64_t)s * P + p];
    const double2 v = psi[(((int64_t)b * J + j) * S + s) * Nz + e];
    const double cu_r = eps * pi * mp.x, cu_i = eps * pi * mp.y;
    u.x += cu_r * v.x - cu_i * v.y;
    u.y += cu_r * v.y + cu_i * v.x;
    const double cm = eps * zeta * pi * sqrt(g + a2 * (1.0 - zeta * eps));
    m.x += cm * v.x;
    m.y += cm * v.y;
    const double cw = eps * pi * sqrt(g + a2 * (1.0 - zeta));
    mw.x += cw * v.x;
    mw.y += cw * v.y;
  }
  au[i] = u;
  am[i] = m;
  aw[i] = mw;
}
cudaError_t launch_slam_bv_wsum(const double* w, int64_t P, int64_t K, int S, double* wk, cudaStream_t st) {
  slam_bv_wsum_kernel<<<S, SB, 0, st>>>(w, P, K, wk);
  return cudaGetLastError();
}
cudaError_t launch_slam_bv_items(const double* x, const double* phi, int64_t P, int64_t K, int64_t k0, int B, int J,
                                 int S, double* pos, int32_t* js, double* sfv, cudaStream_t st) {
  const int64_t n = (int64_t)B * J * S;
  slam_bv_items_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(x, phi, P, K, k0, B, J, S, pos, js, sfv);
  return cudaGetLastError();
}
cudaError_t launch_slam_bv_accum(const double2* psi, const double2* mu, const double* gam, const double* w,
                                 const double* wk, const double* par, int64_t P, int64_t K, int64_t k0, int B, int J,
                                 int S, int64_t Nz, double2* au, double2* am, double2* aw, cudaStream_t st) {
  const int64_t n = (int64_t)J * S * Nz;
  slam_bv_accum_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(psi, mu, gam, w, wk, par, P, K, k0, B, J, S, Nz,
                                                                   au, am, aw);
  return cudaGetLastError();
}

// complex64 columns for the update messages: m [J][S][Nz] (M of nu~), mu_nu [J][Nz] = sum_s zeta_s u_s
__global__ void slam_bv_final_kernel(const double2* __restrict__ am, const double2* __restrict__ au,
                                     const double* __restrict__ par, int J, int S, int64_t Nz, float2* __restrict__ m64,
                                     float2* __restrict__ munu) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)J * Nz) return;
  const int j = (int)(i / Nz);
  const int64_t e = i - (int64_t)j * Nz;
  double r = 0.0, im = 0.0;
  for (int s = 0; s < S; ++s) {
    const int64_t a = ((int64_t)j * S + s) * Nz + e;
    const double z = par[MAXS + s * MAXJ + j];
    r += z * au[a].x;
    im += z * au[a].y;
    m64[a] = make_float2((float)am[a].x, (float)am[a].y);
  }
  munu[i] = make_float2((float)r, (float)im);
}
cudaError_t launch_slam_bv_final(const double2* am, const double2* au, const double* par, int J, int S, int64_t Nz,
                                 float2* m64, float2* munu, cudaStream_t st) {
  const int64_t n = (int64_t)J * Nz;
  slam_bv_final_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(am, au, par, J, S, Nz, m64, munu);
  return cudaGetLastError();
}

// slot s's inputs of kappa~ and omega~: mu3 = sum_{s' != s} zeta_s' u_s', the other slots' columns M [J][S-1][Nz],
// m_omega,s and mu~_4 = u_s as [J][Nz] (complex64, from the fp64 sums)
__global__ void slam_others_kernel(const double2* __restrict__ au, const double2* __restrict__ am,
                                   const double2* __restrict__ aw, const double* __restrict__ par, int J, int S,
                                   int64_t Nz, int s, float2* __restrict__ mu3, float2* __restrict__ mo,
                                   float2* __restrict__ mws, float2* __restrict__ us) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)J * Nz) return;
  const int j = (int)(i / Nz);
  const int64_t e = i - (int64_t)j * Nz;
  double r = 0.0, im = 0.0;
  int l = 0;
  for (int t = 0; t < S; ++t) {
    const int64_t a = ((int64_t)j * S + t) * Nz + e;
    if (t == s) continue;
    const double z = par[MAXS + t * MAXJ + j];
    r += z * au[a].x;
    im += z * au[a].y;
    mo[((int64_t)j * (S - 1) + l) * Nz + e] = make_float2((float)am[a].x, (float)am[a].y);
    ++l;
  }
  mu3[i] = make_float2((float)r, (float)im);
  const int64_t a = ((int64_t)j * S + s) * Nz + e;
  mws[i] = make_float2((float)aw[a].x, (float)aw[a].y);
  us[i] = make_float2((float)au[a].x, (float)au[a].y);
}
cudaError_t launch_slam_others(const double2* au, const double2* am, const double2* aw, const double* par, int J, int S,
                               int64_t Nz, int s, float2* mu3, float2* mo, float2* mws, float2* us, cudaStream_t st) {
  const int64_t n = (int64_t)J * Nz;
  slam_others_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(au, am, aw, par, J, S, Nz, s, mu3, mo, mws, us);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------- gathers
// the MT likelihood's per-particle SFVs (C-amb-8): out [P][K][3] = phi_{k+1}[p]
__global__ void slam_sfv_pp_kernel(const double* __restrict__ phi, int64_t P, int K, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P * K) return;
  const int64_t p = i / K;
  const int k = (int)(i - p * K);
  for (int c = 0; c < 3; ++c) out[3 * i + c] = phi[((int64_t)(k + 1) * P + p) * 3 + c];
}
cudaError_t launch_slam_sfv_pp(const double* phi, int64_t P, int K, double* out, cudaStream_t st) {
  if (K <= 0) return cudaSuccess;
  slam_sfv_pp_kernel<<<(unsigned)((P * K + 255) / 256), 256, 0, st>>>(phi, P, K, out);
  return cudaGetLastError();
}
// resampled PF (slot src -> slot dst, dst <= src): phi, mu, gamma of the ancestors; w = exist / P
__global__ void slam_pf_gather_kernel(const double* __restrict__ phi, const double2* __restrict__ mu,
                                      const double* __restrict__ gam, const int64_t* __restrict__ anc, int64_t P,
                                      double* __restrict__ tphi, double2* __restrict__ tmu, double* __restrict__ tgam) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const int64_t a = anc[p];
  if (phi)
    for (int c = 0; c < 3; ++c) tphi[3 * p + c] = phi[3 * a + c];
  tmu[p] = mu[a];
  tgam[p] = gam[a];
}
__global__ void slam_fill_kernel(double* __restrict__ w, int64_t P, double v) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < P) w[p] = v;
}
__global__ void slam_gather1_kernel(const double* __restrict__ src, const int64_t* __restrict__ anc, int64_t P,
                                    double* __restrict__ dst) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < P) dst[p] = src[anc[p]];
}
cudaError_t launch_slam_pf_gather(const double* phi, const double2* mu, const double* gam, const int64_t* anc,
                                  int64_t P, double* tphi, double2* tmu, double* tgam, cudaStream_t st) {
  slam_pf_gather_kernel<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(phi, mu, gam, anc, P, tphi, tmu, tgam);
  return cudaGetLastError();
}
cudaError_t launch_slam_fill(double* w, int64_t P, double v, cudaStream_t st) {
  slam_fill_kernel<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(w, P, v);
  return cudaGetLastError();
}
cudaError_t launch_slam_gather1(const double* src, const int64_t* anc, int64_t P, double* dst, cudaStream_t st) {
  slam_gather1_kernel<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(src, anc, P, dst);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------- SFV regularization (reading F4k)
// Sigma = sum_p w_p (phi_p - m)(phi_p - m)^T / sum w in two fixed-order levels (as the weighted sums), then on
// thread 0 the Cholesky factor of Sigma + 1e-12 tr(Sigma) I (L = 0 when not positive definite: no move); L [9]
// row-major lower
__global__ void __launch_bounds__(SB) slam_cov3_part_kernel(const double* __restrict__ w, const double* __restrict__ phi,
                                                            int64_t P, double m0, double m1, double m2, int NBW,
                                                            double* __restrict__ part) {
  __shared__ double sh[SB];
  const int64_t C = (P + NBW - 1) / NBW;
  const int64_t p0 = (int64_t)blockIdx.x * C, p1 = p0 + C < P ? p0 + C : P;
  double a[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int64_t p = p0 + threadIdx.x; p < p1; p += SB) {
    const double wp = w[p];
    const double d0 = phi[3 * p] - m0, d1 = phi[3 * p + 1] - m1, d2 = phi[3 * p + 2] - m2;
    a[0] += wp;
    a[1] += wp * d0 * d0;
    a[2] += wp * d1 * d0;
    a[3] += wp * d1 * d1;
    a[4] += wp * d2 * d0;
    a[5] += wp * d2 * d1;
    a[6] += wp * d2 * d2;
  }
  for (int c = 0; c < 7; ++c) {
    const double r = block_sum(a[c], sh);
    if (threadIdx.x == 0) part[7 * blockIdx.x + c] = r;
  }
}
__global__ void __launch_bounds__(SB) slam_cov3_kernel(const double* __restrict__ part, int NBW,
                                                       double* __restrict__ L) {
  __shared__ double sh[SB];
  double r[7];
  for (int c = 0; c < 7; ++c) {
    double a = 0.0;
    for (int b = threadIdx.x; b < NBW; b += SB) a += part[7 * b + c];
    r[c] = block_sum(a, sh);
  }
  if (threadIdx.x != 0) return;
  double A[9];
  const double iw = r[0] > 0.0 ? 1.0 / r[0] : 0.0;
  A[0] = r[1] * iw; A[3] = A[1] = r[2] * iw; A[4] = r[3] * iw;
  A[6] = A[2] = r[4] * iw; A[7] = A[5] = r[5] * iw; A[8] = r[6] * iw;
  const double tr = A[0] + A[4] + A[8];
  for (int c = 0; c < 3; ++c) A[4 * c] += 1e-12 * tr;
  double Lq[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  bool ok = true;
  for (int j = 0; j < 3 && ok; ++j) {
    double d = A[4 * j];
    for (int k = 0; k < j; ++k) d -= Lq[3 * j + k] * Lq[3 * j + k];
    if (!(d > 0.0)) { ok = false; break; }
    Lq[4 * j] = sqrt(d);
    for (int i = j + 1; i < 3; ++i) {
      double x = A[3 * i + j];
      for (int k = 0; k < j; ++k) x -= Lq[3 * i + k] * Lq[3 * j + k];
      Lq[3 * i + j] = x / Lq[4 * j];
    }
  }
  for (int c = 0; c < 9; ++c) L[c] = ok ? Lq[c] : 0.0;
}
// phi_p += h L z_p, z_p: the first three of normals4(key, n, p, 0x700 + 16 slot)
__global__ void slam_reg3_kernel(double* __restrict__ phi, int64_t P, const double* __restrict__ L, double h,
                                 uint64_t key, uint64_t n, int slot) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  double z[4];
  normals4_slam(key, n, (uint64_t)p, 0x700u + 16u * (uint32_t)slot, z);
  for (int c = 0; c < 3; ++c) {
    double a = 0.0;
    for (int b = 0; b <= c; ++b) a += L[3 * c + b] * z[b];
    phi[3 * p + c] += h * a;
  }
}
cudaError_t launch_slam_sfv_reg(const double* w, const double* phi_src, double* phi_dst, int64_t P, const double* mean,
                                double h, double* L, double* part, uint64_t key, uint64_t n, int slot, cudaStream_t st) {
  const int NBW = slam_wsum_blocks(P);
  slam_cov3_part_kernel<<<NBW, SB, 0, st>>>(w, phi_src, P, mean[0], mean[1], mean[2], NBW, part);
  slam_cov3_kernel<<<1, SB, 0, st>>>(part, NBW, L);
  slam_reg3_kernel<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(phi_dst, P, L, h, key, n, slot);
  return cudaGetLastError();
}

}  // namespace cdms
