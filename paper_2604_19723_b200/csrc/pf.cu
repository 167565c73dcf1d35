// pf.cu -- F1: the PF-particle update message kappa~ of one PF s evaluated at its particles, and the PF
// weights with the normalization constant M_{y,s,n} (Supplement S-V "PF State Update Message" P:L660-834; PF weights
// P:L3392-3432; Supplement S-IV P:L527-632).  Per PA j:
//   C^kappa(phi_p, r) = r q_p psi_p psi_p^H + A,  A = eta_j I + M M^H,
//   mu^kappa(phi_p, r) = r zeta_j mu_p psi_p + mu3_j,
// psi_p the response of PA j at the paired MT particle x_p through the wall of SFV phi_p (reading C-amb-F1a).  The
// inversion lemma reduces every quadratic form to a^H b / eta - (a^H M) K^{-1} (M^H b) / eta^2, K = I + M^H M / eta
// (eq. S-Maha-expression), and the determinant lemma the determinant to (1 + q psi^H A^{-1} psi) det A; det A
// and pi^Nz cancel against the H0 branch, so per particle
//   logr_p = log w_alpha,p + sum_j [ q |b|^2 / (1 + q beta) - (|c|^2 beta - 2 Re(conj(c) b0)) - ln(1 + q beta) ],
//   beta = psi^H A^-1 psi, b0 = psi^H A^-1 e0, c = zeta_j mu_p, b = b0 - c beta, e0 = z_j - mu3_j
// (e = e0 - c psi: e^H A^-1 e - e0^H A^-1 e0 = |c|^2 beta - 2 Re(conj(c) b0)).  Work per particle and PA: the T = L + 1
// correlations psi^H e0, psi^H m_l (taylor.cu pf_corr_kernel on K1T tables of the T snapshots), then O(L^2) fp64.
// The particle-independent part -- the dot products of the snapshots, the Cholesky factor of K, K^{-1} M^H e0 -- is
// formed once per PA in fp64 (pf_dots_kernel, pf_fixed_kernel).
#include <math.h>

#include "cdms_internal.h"

namespace cdms {

constexpr int PF_BLOCK = 256;
constexpr int PF_MAXT = 9;  // snapshots per PA: e0 and up to 8 columns of M

// snaps [J][T][Nz] complex64: t = 0 the H0 error vector e0 = z - mu3 (fp32 subtraction of the two complex64 inputs,
// as the MT engine reads its snapshot), t >= 1 the columns m_{t-1}
__global__ void pf_snap_kernel(int J, int T, int64_t Nz, const float2* __restrict__ y, const float2* __restrict__ mu3,
                               const float2* __restrict__ mcols, float2* __restrict__ snaps) {
  const int64_t n_all = (int64_t)J * T * Nz;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_all; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = i % Nz;
    const int64_t jt = i / Nz;
    const int t = (int)(jt % T), j = (int)(jt / T);
    float2 v;
    if (t == 0) {
      const float2 a = y[(int64_t)j * Nz + n], b = mu3[(int64_t)j * Nz + n];
      v = make_float2(a.x - b.x, a.y - b.y);
    } else {
      v = mcols[((int64_t)j * (T - 1) + (t - 1)) * Nz + n];
    }
    snaps[i] = v;
  }
}

// dots[j][a][b] = v_a^H v_b (a <= b) of PA j's snapshots in fp64, one block per (j, a, b), fixed-order reduction.
// Vector 0 (the error vector z - mu) is formed from the complex64 inputs y0, mu0 in fp64 here (exact difference), not
// read from the fp32 stack: its rounding would otherwise enter |e|^2 / eta, which the quadratic forms cancel by ~SNR.
__device__ __forceinline__ double2 dots_elem(const float2* v, const float2* y0, const float2* mu0, int64_t n) {
  if (y0 != nullptr) {
    const float2 a = y0[n], b = mu0[n];
    return make_double2((double)a.x - (double)b.x, (double)a.y - (double)b.y);
  }
  const float2 x = v[n];
  return make_double2((double)x.x, (double)x.y);
}
__global__ void __launch_bounds__(PF_BLOCK) pf_dots_kernel(int T, int64_t Nz, const float2* __restrict__ snaps,
                                                          const float2* __restrict__ y0, const float2* __restrict__ mu0,
                                                          double2* __restrict__ dots) {
  __shared__ double sr[PF_BLOCK], si[PF_BLOCK];
  const int np = T * (T + 1) / 2;
  const int j = blockIdx.x / np, q = blockIdx.x - j * np;
  int a = 0, rem = q;
  while (rem >= T - a) {
    rem -= T - a;
    ++a;
  }
  const int b = a + rem;
  const float2* va = snaps + ((int64_t)j * T + a) * Nz;
  const float2* vb = snaps + ((int64_t)j * T + b) * Nz;
  const float2* ya = (a == 0 && y0) ? y0 + (int64_t)j * Nz : nullptr;
  const float2* yb = (b == 0 && y0) ? y0 + (int64_t)j * Nz : nullptr;
  const float2* ma = mu0 ? mu0 + (int64_t)j * Nz : nullptr;
  double accr = 0.0, acci = 0.0;
  for (int64_t n = threadIdx.x; n < Nz; n += PF_BLOCK) {
    const double2 x = dots_elem(va, ya, ma, n), y = dots_elem(vb, yb, ma, n);
    accr += x.x * y.x + x.y * y.y;  // conj(x) y
    acci += x.x * y.y - x.y * y.x;
  }
  sr[threadIdx.x] = accr;
  si[threadIdx.x] = acci;
  __syncthreads();
  for (int o = PF_BLOCK / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      sr[threadIdx.x] += sr[threadIdx.x + o];
      si[threadIdx.x] += si[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) dots[((int64_t)j * T + a) * T + b] = make_double2(sr[0], si[0]);
}

// Per PA (one thread each): K = I + M^H M / eta = L L^H (complex Cholesky, fp64), w = M^H e0, kiw = K^{-1} w and
// t0 = e0^H A^{-1} e0 = |e0|^2 / eta - w^H K^{-1} w / eta^2.  fixed[j] = [Kc (Lm x Lm, lower, row-major; the
// diagonal entries hold (L_aa, 1 / L_aa)), kiw (Lm), (t0, 0)] with Lm = PF_MAXT - 1.  Non-positive pivot -> FLAG_NAN
// (M M^H not representable).
constexpr int PF_FIXED = (PF_MAXT - 1) * (PF_MAXT - 1) + (PF_MAXT - 1) + 1;  // double2 per PA
__global__ void pf_fixed_kernel(int J, int T, const double2* __restrict__ dots, const double* __restrict__ eta,
                                double2* __restrict__ fixed, int* flags) {
  const int j = threadIdx.x;
  if (j >= J) return;
  const int L = T - 1, Lm = PF_MAXT - 1;
  const double2* d = dots + (int64_t)j * T * T;
  const double e = eta[j];
  double2 K[(PF_MAXT - 1) * (PF_MAXT - 1)];
  for (int a = 0; a < L; ++a)
    for (int b = 0; b <= a; ++b) {
      // G_ab = m_a^H m_b = dots[1 + min][1 + max] (conjugated when a > b)
      const double2 g = d[(1 + b) * T + (1 + a)];  // m_b^H m_a
      const double gr = g.x, gi = -g.y;             // m_a^H m_b = conj(m_b^H m_a)
      K[a * Lm + b] = make_double2((a == b ? 1.0 : 0.0) + gr / e, gi / e);
    }
  bool ok = true;
  for (int c = 0; c < L; ++c) {  // K = L L^H in place (lower)
    double dd = K[c * Lm + c].x;
    for (int k = 0; k < c; ++k) dd -= K[c * Lm + k].x * K[c * Lm + k].x + K[c * Lm + k].y * K[c * Lm + k].y;
    if (!(dd > 0.0)) {
      ok = false;
      dd = 1.0;
    }
    const double l = sqrt(dd);
    K[c * Lm + c] = make_double2(l, 0.0);
    for (int r = c + 1; r < L; ++r) {
      double ar = K[r * Lm + c].x, ai = K[r * Lm + c].y;
      for (int k = 0; k < c; ++k) {  // - L_rk conj(L_ck)
        const double2 x = K[r * Lm + k], y = K[c * Lm + k];
        ar -= x.x * y.x + x.y * y.y;
        ai -= x.y * y.x - x.x * y.y;
      }
      K[r * Lm + c] = make_double2(ar / l, ai / l);
    }
  }
  if (!ok) atomicOr(flags, FLAG_NAN);
  // w_t = m_t^H e0 = conj(e0^H m_t) = conj(dots[0][1 + t]); forward then back substitution: kiw = K^{-1} w
  double2 y[PF_MAXT - 1];
  double wsq = 0.0;
  for (int a = 0; a < L; ++a) {
    const double2 w = d[0 * T + (1 + a)];
    double yr = w.x, yi = -w.y;
    for (int k = 0; k < a; ++k) {
      const double2 x = K[a * Lm + k];
      yr -= x.x * y[k].x - x.y * y[k].y;
      yi -= x.x * y[k].y + x.y * y[k].x;
    }
    y[a] = make_double2(yr / K[a * Lm + a].x, yi / K[a * Lm + a].x);
    wsq += y[a].x * y[a].x + y[a].y * y[a].y;  // w^H K^{-1} w = |L^{-1} w|^2
  }
  for (int a = L - 1; a >= 0; --a) {  // L^H kiw = y
    double xr = y[a].x, xi = y[a].y;
    for (int k = a + 1; k < L; ++k) {  // - conj(L_ka) kiw_k
      const double2 l = K[k * Lm + a], v = y[k];
      xr -= l.x * v.x + l.y * v.y;
      xi -= l.x * v.y - l.y * v.x;
    }
    y[a] = make_double2(xr / K[a * Lm + a].x, xi / K[a * Lm + a].x);
  }
  double2* f = fixed + (int64_t)j * PF_FIXED;
  for (int i = 0; i < Lm * Lm; ++i) f[i] = K[i];
  for (int a = 0; a < L; ++a) f[a * Lm + a].y = 1.0 / K[a * Lm + a].x;  // for the per-particle substitution
  for (int a = 0; a < Lm; ++a) f[Lm * Lm + a] = a < L ? y[a] : make_double2(0.0, 0.0);
  f[Lm * Lm + Lm] = make_double2(d[0].x / e - wsq / (e * e), 0.0);  // t0
}

// logr_p (one thread per particle): the per-PA terms of the header from the correlations cc [J][T][P] and fixed[j].
// T is a template parameter so the substitution loops unroll and y stays in registers (a runtime T put it in local
// memory: 128-byte stack frame)
template <int T>
__global__ void pf_asm_kernel(int J, double Nz, const double2* __restrict__ cc, const double2* __restrict__ fixed,
                              const double* __restrict__ eta, const double* __restrict__ zeta,
                              const double* __restrict__ gain2, const double* __restrict__ walpha,
                              const double2* __restrict__ mu, const double* __restrict__ gamma, int* __restrict__ pflag,
                              int64_t P, double* __restrict__ logr, int* flags) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const int L = T - 1, Lm = PF_MAXT - 1;
  const double2 mup = mu[p];
  const double mu2 = mup.x * mup.x + mup.y * mup.y;
  double acc = log(walpha[p]);
  const int fl = pflag[p];
  pflag[p] = 0;
  for (int j = 0; j < J; ++j) {
    double2 c[T];  // this particle's correlations for PA j (coalesced across the warp)
#pragma unroll
    for (int t = 0; t < T; ++t) c[t] = cc[((int64_t)j * T + t) * P + p];
    const double2* f = fixed + (int64_t)j * PF_FIXED;
    const double e = eta[j], z = zeta[j], ie = 1.0 / e, ie2 = ie * ie;  // the only divisions: 1 / eta, 1 / den
    // beta = N_z g^2 / eta - |L^{-1} u|^2 / eta^2, u_t = m_t^H psi = conj(c_{1+t});  b0 = c_0 / eta - sum_t c_{1+t}
    // (K^{-1} M^H e0)_t / eta^2
    double2 y[PF_MAXT - 1];
    double usq = 0.0, b0r = c[0].x * ie, b0i = c[0].y * ie;
#pragma unroll
    for (int a = 0; a < L; ++a) {
      double yr = c[1 + a].x, yi = -c[1 + a].y;
#pragma unroll
      for (int k = 0; k < a; ++k) {
        const double2 x = f[a * Lm + k];
        yr -= x.x * y[k].x - x.y * y[k].y;
        yi -= x.x * y[k].y + x.y * y[k].x;
      }
      const double il = f[a * Lm + a].y;  // 1 / L_aa (pf_fixed_kernel)
      y[a] = make_double2(yr * il, yi * il);
      usq += y[a].x * y[a].x + y[a].y * y[a].y;
      const double2 k = f[Lm * Lm + a];
      b0r -= (c[1 + a].x * k.x - c[1 + a].y * k.y) * ie2;
      b0i -= (c[1 + a].x * k.y + c[1 + a].y * k.x) * ie2;
    }
    const double beta = Nz * gain2[p * J + j] * ie - usq * ie2;
    const double cr = z * mup.x, ci = z * mup.y;                    // c = zeta mu_p
    const double br = b0r - cr * beta, bi = b0i - ci * beta;         // b = psi^H A^-1 e
    const double q = (gamma[p] + mu2 * (1.0 - z)) * z;
    const double den = 1.0 + q * beta;
    const double dquad = (cr * cr + ci * ci) * beta - 2.0 * (cr * b0r + ci * b0i);  // e^H A e - e0^H A e0
    acc += q * (br * br + bi * bi) / den - dquad - log(den);
  }
  if (fl) {
    acc = -INFINITY;
    atomicOr(flags, (fl & 1) ? FLAG_DEGENERATE : FLAG_NAN);
  }
  logr[p] = acc;
}

// |psi_p|^2 per element = g^2 (path-loss gain, 1 with unit modulus) for the analytic psi^H psi = N_z g^2
__global__ void pf_gain_kernel(const __grid_constant__ SceneDev sc, const double* __restrict__ particles, int64_t P,
                               int pstride, const double* __restrict__ phi, double* __restrict__ gain2) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P * sc.J) return;
  const int64_t p = i / sc.J;
  const int j = (int)(i - p * sc.J);
  double g2 = 1.0;
  if (sc.pathloss) {
    const double* x = particles + p * pstride;
    const double* pj = sc.pa_pos[j];
    double R = 1.0;
    if (!phi) {  // the LOS PF: p_VA = p_j
      const double r0 = x[0] - pj[0], r1 = x[1] - pj[1], r2 = x[2] - pj[2];
      R = sqrt(r0 * r0 + r1 * r1 + r2 * r2);
    }
    const double* s = phi ? phi + 3 * p : pj;
    const double n2 = phi ? s[0] * s[0] + s[1] * s[1] + s[2] * s[2] : 0.0;
    if (n2 > 0.0) {
      const double c = 2.0 * (pj[0] * s[0] + pj[1] * s[1] + pj[2] * s[2]) / n2 - 1.0;
      const double r0 = x[0] - (pj[0] - c * s[0]), r1 = x[1] - (pj[1] - c * s[1]), r2 = x[2] - (pj[2] - c * s[2]);
      R = sqrt(r0 * r0 + r1 * r1 + r2 * r2);
    }
    const double g = sc.lambda / (4.0 * PI * R);
    g2 = g * g;
  }
  gain2[i] = g2;
}

// M_y from the two-level LSE of logr (lse.cu: M = max logr, S = sum e^{logr - M}, A = sum w_alpha):
// h0 = max(0, 1 - A); out[0] = log M_y = log(S e^M + h0), out[1] = existence = S e^M / M_y (S-IV, eq. existenceProb)
__global__ void pf_norm_kernel(const double* __restrict__ lse, double* __restrict__ out, int* flags) {
  const double M = lse[0], S = lse[1], sa = lse[2];
  const double h0 = fmax(0.0, 1.0 - sa);
  double logM;
  if (M > -INFINITY) logM = M + log(S + h0 * exp(-M));
  else logM = log(h0);
  if (!(logM > -INFINITY)) atomicOr(flags, FLAG_ZEROMASS);
  out[0] = logM;
  out[1] = M > -INFINITY ? exp(M + log(S) - logM) : 0.0;
}

__global__ void pf_weights_kernel(const double* __restrict__ logr, int64_t P, const double* __restrict__ out,
                                  double* __restrict__ w) {
  const double logM = out[0];
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x)
    w[p] = exp(logr[p] - logM);
}

static unsigned pf_grid(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  return (unsigned)(g < 1 ? 1 : (g > 65535 * 4 ? 65535 * 4 : g));
}

cudaError_t launch_pf_prep(int J, int T, int64_t Nz, const float2* y, const float2* mu3, const float2* mcols,
                           float2* snaps, double2* dots, const double* d_eta, double2* fixed, int* flags,
                           cudaStream_t st) {
  if (T < 1 || T > PF_MAXT) return cudaErrorInvalidValue;
  pf_snap_kernel<<<pf_grid((int64_t)J * T * Nz, 256), 256, 0, st>>>(J, T, Nz, y, mu3, mcols, snaps);
  pf_dots_kernel<<<(unsigned)(J * T * (T + 1) / 2), PF_BLOCK, 0, st>>>(T, Nz, snaps, y, mu3, dots);
  pf_fixed_kernel<<<1, 32, 0, st>>>(J, T, dots, d_eta, fixed, flags);
  return cudaGetLastError();
}
// Generic stack of per-PA N_z-vectors for the F4 messages (slam.cu): t = 0 z - mu, t = 1..L the columns, then up to two
// extra vectors x1, x2 ([J][Nz] each, NULL to omit); and all their fp64 dot products (vec_dots = pf_dots_kernel)
__global__ void vec_stack_kernel(int J, int T, int L, int64_t Nz, const float2* __restrict__ y,
                                 const float2* __restrict__ mu, const float2* __restrict__ cols,
                                 const float2* __restrict__ x1, const float2* __restrict__ x2, float2* __restrict__ out) {
  const int64_t n_all = (int64_t)J * T * Nz;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_all; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = i % Nz;
    const int64_t jt = i / Nz;
    const int t = (int)(jt % T), j = (int)(jt / T);
    float2 v;
    if (t == 0) {
      const float2 a = y[(int64_t)j * Nz + n], b = mu[(int64_t)j * Nz + n];
      v = make_float2(a.x - b.x, a.y - b.y);
    } else if (t <= L) {
      v = cols[((int64_t)j * L + (t - 1)) * Nz + n];
    } else if (t == L + 1) {
      v = x1[(int64_t)j * Nz + n];
    } else {
      v = x2[(int64_t)j * Nz + n];
    }
    out[i] = v;
  }
}
cudaError_t launch_vec_stack_dots(int J, int T, int L, int64_t Nz, const float2* y, const float2* mu, const float2* cols,
                                  const float2* x1, const float2* x2, float2* stack, double2* dots, cudaStream_t st) {
  vec_stack_kernel<<<pf_grid((int64_t)J * T * Nz, 256), 256, 0, st>>>(J, T, L, Nz, y, mu, cols, x1, x2, stack);
  pf_dots_kernel<<<(unsigned)(J * T * (T + 1) / 2), PF_BLOCK, 0, st>>>(T, Nz, stack, y, mu, dots);
  return cudaGetLastError();
}
int pf_fixed_width() { return PF_FIXED; }
int pf_max_snapshots() { return PF_MAXT; }

cudaError_t launch_pf_finish(const SceneDev& sc, int T, const double2* cc, const double2* fixed, const double* d_eta,
                             const double* d_zeta, double* gain2, const double* particles, int pstride,
                             const double* phi, const double* walpha, const double2* mu, const double* gamma,
                             int* pflag, int64_t P, double* logr, double* w, double* out, int* flags,
                             double* lse_part, cudaStream_t st) {
  const int64_t n = P * sc.J;
  pf_gain_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(sc, particles, P, pstride, phi, gain2);
  switch (T) {
#define PF_ASM(n)                                                                                                   \
  case n:                                                                                                           \
    pf_asm_kernel<n><<<(unsigned)((P + 127) / 128), 128, 0, st>>>(sc.J, (double)sc.nf * sc.Na, cc, fixed, d_eta, \
                                                                  d_zeta, gain2, walpha, mu, gamma, pflag, P, logr, \
                                                                  flags);                                          \
    break;
    PF_ASM(1) PF_ASM(2) PF_ASM(3) PF_ASM(4) PF_ASM(5) PF_ASM(6) PF_ASM(7) PF_ASM(8) PF_ASM(9)
#undef PF_ASM
    default: return cudaErrorInvalidValue;
  }
  cudaError_t e = launch_lse_rows(logr, P, 1, P, walpha, P, lse_part, lse_part + 3 * lse_blocks(P), st);
  if (e != cudaSuccess) return e;
  pf_norm_kernel<<<1, 1, 0, st>>>(lse_part + 3 * lse_blocks(P), out, flags);
  if (w) pf_weights_kernel<<<pf_grid(P, 256), 256, 0, st>>>(logr, P, out, w);
  return cudaGetLastError();
}

}  // namespace cdms
