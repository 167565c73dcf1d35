// slam.cu -- F4 parts: the noise variance update message nu~ at the noise particles (Supplement S-V
// "Noise Variance Update Message"; weights P:L3398-3410) and the PPR update message omega~ with the PPR
// existence revival (S-V "PR State Update Message"; Supplement S-VI).
//
// Both are Woodbury forms over the features' columns M = [m_0 ...] (N_z x L) with a particle-independent Gram M^H M and
// projections M^H a of a few N_z-vectors, so the N_z-sized work is a handful of fp64 dot products per PA
// (vec_stack_kernel + vec_dots_kernel, pf.cu); the rest is O(L^3) per PA or O(L) per particle:
//  * nu~: log nu~(eta_p) = -N_z ln(pi eta_p) - ln det(I + G/eta_p) - |e|^2/eta_p + w^H (I + G/eta_p)^{-1} w / eta_p^2,
//    G = M^H M, w = M^H e, e = z - mu_nu.  Only eta_p varies per particle, so G = U diag(lambda) U^H is diagonalized
//    ONCE per PA (cyclic Jacobi on the real symmetric 2L x 2L embedding [[G_r, -G_i], [G_i, G_r]], fp64) and per particle
//    ln det(I + G/eta) = 1/2 sum_i ln(1 + lambda_i/eta), w^H (I + G/eta)^{-1} w = sum_i v_i^2 / (1 + lambda_i/eta),
//    v = Q^T [Re w; Im w] -- the same quantities as the paper's per-particle Cholesky (the oracle's order), O(L) per
//    (particle, PA) instead of O(L^3).
//  * omega~: per PA the rank-1 lemma log ratio of r = 1 against r = 0 (det A, pi^N_z cancel) from the dot products
//    of e0 = z - mu3, m_omega, mu4 and the columns, and the existence sigma(u), u = log(zeta/(1 - zeta)) + log ratio.
#include <math.h>

#include "cdms_internal.h"

namespace cdms {

constexpr int SL_MAXL = 9;   // feature columns (nu~: all S features, S <= 9)

// ---------------------------------------------------------------------------- nu~
// One warp per PA: cyclic Jacobi on the 2L x 2L real embedding in shared memory; every lane computes the same rotation
// (c, s) and lane k applies it to row / column element k (the serial order's arithmetic per element, so the result does
// not depend on the lane count; round 1 ran the sweeps on one thread, 2 ms per call at L = 9).
// out eig[j] = [lambda (2L), v (2L), |e|^2] (doubles).
__global__ void __launch_bounds__(32) noise_eig_kernel(int L, int T, const double2* __restrict__ dots,
                                                       double* __restrict__ eig) {
  __shared__ double A[2 * SL_MAXL][2 * SL_MAXL], Q[2 * SL_MAXL][2 * SL_MAXL];
  const int j = blockIdx.x, n = 2 * L, k = threadIdx.x;
  const double2* d = dots + (int64_t)j * T * T;
  auto D = [&](int a, int b) -> double2 {  // v_a^H v_b from the upper triangle
    if (a <= b) return d[a * T + b];
    const double2 x = d[b * T + a];
    return make_double2(x.x, -x.y);
  };
  auto wsum = [](double v) {  // butterfly: the same value on every lane
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  };
  if (k < L)
    for (int b = 0; b < L; ++b) {
      const double2 g = D(1 + k, 1 + b);  // G_kb = m_k^H m_b
      A[k][b] = g.x;
      A[L + k][L + b] = g.x;
      A[L + k][b] = g.y;
      A[k][L + b] = -g.y;
    }
  if (k < n)
    for (int b = 0; b < n; ++b) Q[k][b] = k == b ? 1.0 : 0.0;
  __syncwarp();
  double fr = 0.0;
  if (k < n)
    for (int b = 0; b < n; ++b) fr += A[k][b] * A[k][b];
  const double fro = wsum(fr);
  for (int sweep = 0; sweep < 60; ++sweep) {
    double of = 0.0;
    if (k < n)
      for (int q = k + 1; q < n; ++q) of += A[k][q] * A[k][q];
    const double off = wsum(of);
    if (!(off > 1e-32 * fro)) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A[p][q];
        if (apq == 0.0) continue;
        const double th = (A[q][q] - A[p][p]) / (2.0 * apq);
        const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        __syncwarp();
        if (k < n) {  // A <- A J (columns p, q)
          const double akp = A[k][p], akq = A[k][q];
          A[k][p] = c * akp - s * akq;
          A[k][q] = s * akp + c * akq;
        }
        __syncwarp();
        if (k < n) {  // A <- J^T A (rows p, q)
          const double apk = A[p][k], aqk = A[q][k];
          A[p][k] = c * apk - s * aqk;
          A[q][k] = s * apk + c * aqk;
          const double qkp = Q[k][p], qkq = Q[k][q];  // Q <- Q J
          Q[k][p] = c * qkp - s * qkq;
          Q[k][q] = s * qkp + c * qkq;
        }
        __syncwarp();
      }
  }
  double* o = eig + (int64_t)j * (4 * SL_MAXL + 1);
  if (k < n) {
    o[k] = fmax(A[k][k], 0.0);  // G is PSD; clamp rounding below zero
    double vi = 0.0;
    for (int a = 0; a < L; ++a) {
      const double2 w = D(1 + a, 0);  // w_a = m_a^H e
      vi += Q[a][k] * w.x + Q[L + a][k] * w.y;
    }
    o[n + k] = vi;
  }
  if (k == 0) o[4 * SL_MAXL] = D(0, 0).x;  // |e|^2
}

// logw[j][p] = log w_xi + log nu~(eta_p) for every (PA, particle)
__global__ void noise_particle_kernel(int J, int L, int64_t P, double Nz, const double* __restrict__ eig,
                                      const double* __restrict__ eta, const double* __restrict__ wxi,
                                      double* __restrict__ logw, int* flags) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)J * P) return;
  const int j = (int)(i / P);
  const double* o = eig + (int64_t)j * (4 * SL_MAXL + 1);
  const double et = eta[i];
  if (!(et > 0.0)) {
    atomicOr(flags, FLAG_NAN);
    logw[i] = -INFINITY;
    return;
  }
  const double inv = 1.0 / et;
  double ld = 0.0, q = 0.0;
  for (int k = 0; k < 2 * L; ++k) {
    const double mu = 1.0 + o[k] * inv;
    ld += log(mu);
    q += o[2 * L + k] * o[2 * L + k] / mu;
  }
  logw[i] = log(wxi[i]) - Nz * log(PI * et) - 0.5 * ld - o[4 * SL_MAXL] * inv + q * inv * inv;
}

// Per PA (one block, fixed order): lognorm[j] = log sum_p e^{logw}; w = e^{logw - lognorm}
// per PA: lognorm = M + ln S from the two-level LSE (lse.cu); w = e^{logw - lognorm} over every (PA, particle)
__global__ void noise_norm_kernel(int J, int64_t P, const double* __restrict__ lse, const double* __restrict__ logw,
                                  double* __restrict__ lognorm, double* __restrict__ w, int* flags) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)J * P) return;
  const int j = (int)(i / P);
  const double ln = lse[3 * j] + log(lse[3 * j + 1]);
  if (i - (int64_t)j * P == 0) {
    lognorm[j] = ln;
    if (!(ln > -INFINITY)) atomicOr(flags, FLAG_ZEROMASS);
  }
  if (w) w[i] = exp(logw[i] - ln);
}

// ---------------------------------------------------------------------------- omega~
// One thread per PA: vectors v_0 = e0 = z - mu3, v_{1..L} = m_l, v_{L+1} = m_omega, v_{L+2} = mu4 (T = L + 3).
__global__ void ppr_kernel(int J, int L, const double2* __restrict__ dots, const double* __restrict__ zeta,
                           const double* __restrict__ eta, double* __restrict__ out, int* flags) {
  const int j = threadIdx.x;
  if (j >= J) return;
  const int T = L + 3;
  const double2* d = dots + (int64_t)j * T * T;
  auto D = [&](int a, int b) -> double2 {
    if (a <= b) return d[a * T + b];
    const double2 x = d[b * T + a];
    return make_double2(x.x, -x.y);
  };
  const double e = eta[j];
  double2 K[SL_MAXL * SL_MAXL];
  for (int a = 0; a < L; ++a)
    for (int b = 0; b <= a; ++b) {
      const double2 g = D(1 + a, 1 + b);
      K[a * SL_MAXL + b] = make_double2((a == b ? 1.0 : 0.0) + g.x / e, g.y / e);
    }
  bool ok = true;
  for (int c = 0; c < L; ++c) {
    double dd = K[c * SL_MAXL + c].x;
    for (int k = 0; k < c; ++k) dd -= K[c * SL_MAXL + k].x * K[c * SL_MAXL + k].x + K[c * SL_MAXL + k].y * K[c * SL_MAXL + k].y;
    if (!(dd > 0.0)) {
      ok = false;
      dd = 1.0;
    }
    const double lc = sqrt(dd);
    K[c * SL_MAXL + c] = make_double2(lc, 0.0);
    for (int r = c + 1; r < L; ++r) {
      double ar = K[r * SL_MAXL + c].x, ai = K[r * SL_MAXL + c].y;
      for (int k = 0; k < c; ++k) {
        const double2 x = K[r * SL_MAXL + k], y = K[c * SL_MAXL + k];
        ar -= x.x * y.x + x.y * y.y;
        ai -= x.y * y.x - x.x * y.y;
      }
      K[r * SL_MAXL + c] = make_double2(ar / lc, ai / lc);
    }
  }
  if (!ok) atomicOr(flags, FLAG_NAN);
  // y_a = L^{-1} M^H a for a in {e0, m_omega, mu4}; maha(a, b) = a^H b/eta - y_a^H y_b/eta^2
  const int idx[3] = {0, L + 1, L + 2};
  double2 Y[3][SL_MAXL];
  for (int v = 0; v < 3; ++v)
    for (int a = 0; a < L; ++a) {
      const double2 w = D(1 + a, idx[v]);  // m_a^H v
      double yr = w.x, yi = w.y;
      for (int k = 0; k < a; ++k) {
        const double2 x = K[a * SL_MAXL + k], y = Y[v][k];
        yr -= x.x * y.x - x.y * y.y;
        yi -= x.x * y.y + x.y * y.x;
      }
      Y[v][a] = make_double2(yr / K[a * SL_MAXL + a].x, yi / K[a * SL_MAXL + a].x);
    }
  auto maha = [&](int u, int v) -> double2 {
    const double2 ab = D(idx[u], idx[v]);
    double qr = 0.0, qi = 0.0;
    for (int a = 0; a < L; ++a) {  // conj(Y_u) Y_v
      qr += Y[u][a].x * Y[v][a].x + Y[u][a].y * Y[v][a].y;
      qi += Y[u][a].x * Y[v][a].y - Y[u][a].y * Y[v][a].x;
    }
    return make_double2(ab.x / e - qr / (e * e), ab.y / e - qi / (e * e));
  };
  const double alpha = maha(1, 1).x;
  const double2 b0 = maha(1, 0), b4 = maha(1, 2);      // m_omega^H A^-1 e0, m_omega^H A^-1 mu4
  const double br = b0.x - b4.x, bi = b0.y - b4.y;      // m_omega^H A^-1 e1, e1 = e0 - mu4
  const double t0 = maha(0, 0).x;
  const double t1 = t0 - 2.0 * maha(0, 2).x + maha(2, 2).x;
  const double lr = (br * br + bi * bi) / (1.0 + alpha) - t1 + t0 - log(1.0 + alpha);
  const double u = log(zeta[j] / (1.0 - zeta[j])) + lr;
  out[3 * j + 0] = lr;
  out[3 * j + 1] = u;
  out[3 * j + 2] = 1.0 / (1.0 + exp(-u));
}

cudaError_t launch_noise_update(int J, int L, int64_t P, int64_t Nz, const double2* dots, double* eig, const double* eta,
                                const double* wxi, double* logw, double* lognorm, double* w, int* flags,
                                double* lse_part, cudaStream_t st) {
  if (L < 0 || L > SL_MAXL) return cudaErrorInvalidValue;
  noise_eig_kernel<<<J, 32, 0, st>>>(L, L + 1, dots, eig);
  const int64_t n = (int64_t)J * P;
  noise_particle_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(J, L, P, (double)Nz, eig, eta, wxi, logw, flags);
  double* lse = lse_part + (int64_t)3 * J * lse_blocks(P);
  cudaError_t e = launch_lse_rows(logw, P, J, P, nullptr, 0, lse_part, lse, st);
  if (e != cudaSuccess) return e;
  noise_norm_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(J, P, lse, logw, lognorm, w, flags);
  return cudaGetLastError();
}
int slam_eig_width() { return 4 * SL_MAXL + 1; }
int slam_max_columns() { return SL_MAXL; }

cudaError_t launch_ppr_update(int J, int L, const double2* dots, const double* zeta, const double* eta, double* out,
                              int* flags, cudaStream_t st) {
  if (L < 0 || L > SL_MAXL) return cudaErrorInvalidValue;
  ppr_kernel<<<1, 32, 0, st>>>(J, L, dots, zeta, eta, out, flags);
  return cudaGetLastError();
}

}  // namespace cdms
