// K1T: the spherical / planar-WB correlation of row A3 from per-PA spectral Taylor tables (FP32 mode).
//
// The correlation of component s with the snapshot, c_s = psi_s^H z, is, per antenna m, a
// trigonometric polynomial of the element's delay evaluated at one point:
//   c_s = sum_m e^{j2pi f_c d_m/c} Y_m(phi_m),   Y_m(phi) = sum_k y[m,k] e^{j2pi (k - k0) phi},  phi_m = df d_m / c,
// (f_k = f_c + (k - k0) df, k0 = (N_f - 1)/2; d_m the spherical distance or the planar projection of the element,
// P:L108-143).  Y_m is 1-periodic up to the sign (-1)^(N_f - 1) (k - k0 is a half-integer for even N_f) and
// band-limited to |k - k0| <= N_f/2, so on G = 4 N_f centres phi_g = g/G its
// Taylor expansion in delta' = (phi - phi_g) G, |delta'| <= 1/2,
//   Y_m(phi_g + delta'/G) = sum_l C_l(m, g) delta'^l,  C_l = sum_k y[m,k] e^{j2pi (k-k0) g/G} (j2pi (k-k0)/G)^l / l!,
// truncated after TAY_L = 8 terms has a relative error below (pi/8)^8/8! = 1.4e-8 of sum_k |y[m,k]| (|2pi (k-k0)
// delta'/G| <= pi/8): far below fp32 rounding, so K1T evaluates the same correlation as the Horner recurrence of
// K1 to fp32 accuracy with one 64-byte table row and 8 real-coefficient steps per (particle, component, antenna)
// instead of N_f complex multiply-adds.  The tables (fp64 sums rounded once to complex64, tay_prep_kernel) cost
// O(J N_a G N_f) per call and stay L2-resident (N_a G 64 bytes per PA).  The Gram is K1's closed form (K1 runs in
// its Horner-free variant first, K1T then writes c).
#include <math.h>

#include "cdms_internal.h"
#include "geometry.cuh"

namespace cdms {

namespace {
constexpr int TAY_L = 8;
constexpr int TAY_BLOCK = 128;
}  // namespace

int tay_centres(int nf) { return 4 * nf; }
size_t tay_table_bytes(const SceneDev& sc) { return (size_t)sc.J * sc.Na * tay_centres(sc.nf) * TAY_L * sizeof(float2); }

// tab[j][m][g][l] (complex64, l fastest: one 64-byte row per (j, m, g)).  TAY_KS lanes per row split the subcarrier
// sum (each from an exact anchor e^{j2pi (k - k0) g / G}, fp64 phasor recurrence inside its segment), combined by a
// fixed shuffle tree: row count alone (J N_a G) would leave most SMs idle at small N_a G.
constexpr int TAY_KS = 8;
__global__ void tay_prep_kernel(const __grid_constant__ SceneDev sc, int G, const float2* __restrict__ y,
                                float2* __restrict__ tab) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t t = tid / TAY_KS;
  const int seg = (int)(tid - t * TAY_KS);
  const int64_t per_j = (int64_t)sc.Na * G;
  const bool live = t < per_j * sc.J;
  const int64_t tt = live ? t : 0;
  const int j = (int)(tt / per_j);
  const int64_t r = tt - (int64_t)j * per_j;
  const int m = (int)(r / G), g = (int)(r - (int64_t)m * G);
  const double k0 = 0.5 * (sc.nf - 1);
  double cr[TAY_L], ci[TAY_L];
#pragma unroll
  for (int l = 0; l < TAY_L; ++l) cr[l] = ci[l] = 0.0;
  const int kseg = (sc.nf + TAY_KS - 1) / TAY_KS;
  const int kb = seg * kseg, ke = min(kb + kseg, sc.nf);
  if (live && kb < ke) {
    double sw, cw;
    sincospi(2.0 * (double)g / (double)G, &sw, &cw);  // step e^{j2pi g/G}
    double pr = 1.0, pi = 0.0;
    const float2* ym = y + (int64_t)j * sc.nf * sc.Na + m;
    for (int k = kb; k < ke; ++k) {
      if (((k - kb) & 63) == 0) {  // anchor e^{j2pi (k - k0) g / G}: exact argument reduction of 2 (k - k0) g mod 2G
        const double num = fmod(2.0 * ((double)k - k0) * (double)g, 2.0 * (double)G);
        sincospi(num / (double)G, &pi, &pr);
      }
      const float2 v = ym[(int64_t)k * sc.Na];
      double br = v.x * pr - v.y * pi, bi = v.x * pi + v.y * pr;  // y_k e^{j2pi (k-k0) g/G}
      const double tk = 2.0 * PI * ((double)k - k0) / (double)G;
#pragma unroll
      for (int l = 0; l < TAY_L; ++l) {
        cr[l] += br;
        ci[l] += bi;
        const double nr = -bi * tk / (double)(l + 1), ni = br * tk / (double)(l + 1);  // * (j tk)/(l+1)
        br = nr;
        bi = ni;
      }
      const double npr = pr * cw - pi * sw;
      pi = pr * sw + pi * cw;
      pr = npr;
    }
  }
#pragma unroll
  for (int o = TAY_KS / 2; o > 0; o >>= 1) {
#pragma unroll
    for (int l = 0; l < TAY_L; ++l) {
      cr[l] += __shfl_xor_sync(0xffffffffu, cr[l], o);
      ci[l] += __shfl_xor_sync(0xffffffffu, ci[l], o);
    }
  }
  if (live && seg == 0) {
    float2* out = tab + t * TAY_L;
#pragma unroll
    for (int l = 0; l < TAY_L; ++l) out[l] = make_float2((float)cr[l], (float)ci[l]);
  }
}

// c_s for one particle per thread and one PA per blockIdx.y: per component the fp64 geometry (VA, H r, R), the
// fp64-reduced phase bases e^{j2pi f_c R/c} and frac(df R/c); per antenna the fp32 offset Delta_m (cancellation-free,
// as K1), the phasor e^{j2pi f_c Delta_m/c}, the table centre and delta', one table row and the Taylor sum.
__global__ void __launch_bounds__(TAY_BLOCK)
    tay_corr_kernel(const __grid_constant__ SceneDev sc, int G, const float2* __restrict__ tab,
                    const float4* __restrict__ tmpl, const double* __restrict__ particles, int64_t P, int pstride,
                    const double* __restrict__ sfv, int sfv_pp, double2* __restrict__ terms, int* __restrict__ pflag,
                    int gram_diag) {
  const int64_t p = (int64_t)blockIdx.x * TAY_BLOCK + threadIdx.x;
  const int j = blockIdx.y;
  if (p >= P) return;
  const int J = sc.J, S = sc.S, Na = sc.Na, T = S + S * (S + 1) / 2;
  const int Na_pad = sc.n_mb * NWARP;
  const double* pos = particles + p * pstride;
  const float2* tj = tab + (int64_t)j * Na * G * TAY_L;
  const float4* tm = tmpl + (int64_t)j * Na_pad;
  const bool sph = sc.wavefront == CDMS_SPHERICAL;
  int fl = 0;
  for (int s = 0; s < S; ++s) {
    const double* sfv_s = nullptr;
    if (s > 0) sfv_s = sfv_pp ? sfv + (p * sc.K + (s - 1)) * 3 : sfv + (int64_t)(s - 1) * 3;
    double va[3], sh[3];
    if (!anchor_va(sc, j, sfv_s, va, sh)) {
      fl |= 2;
      continue;
    }
    const double r0 = pos[0] - va[0], r1 = pos[1] - va[1], r2 = pos[2] - va[2];
    const double rs2 = 2.0 * (r0 * sh[0] + r1 * sh[1] + r2 * sh[2]);
    const float hx = (float)(r0 - rs2 * sh[0]), hy = (float)(r1 - rs2 * sh[1]), hz = (float)(r2 - rs2 * sh[2]);
    const double R64 = sqrt(r0 * r0 + r1 * r1 + r2 * r2);
    if (!(R64 > 0.0)) {
      fl |= 1;
      continue;
    }
    const float R = (float)R64;
    const double phib = R64 * sc.df_c;  // delay phase base (cycles), fp64, not reduced (see the parity below)
    double sb, cb;
    sincospi(2.0 * frac_c(R64 * sc.fc_c), &sb, &cb);
    const float Ebr = (float)cb, Ebi = (float)sb;  // e^{j2pi f_c R/c}
    double accr = 0.0, acci = 0.0;
    for (int m0 = 0; m0 < Na; m0 += 16) {
      float pr = 0.f, pi = 0.f;
      const int m1 = min(m0 + 16, Na);
      for (int m = m0; m < m1; ++m) {
        const float4 v = __ldg(&tm[m]);
        const float rq = hx * v.x + hy * v.y + hz * v.z;
        float delta;
        if (sph) {
          const float n = v.w - 2.f * rq;
          const float d = sqrtf(R * R + n);
          if (!(d > 0.f)) fl |= 1;
          delta = n / (d + R);
        } else {
          delta = -rq / R;
        }
        float er, ei;
        cis2pi_fast<float>(delta * sc.fc_cf, er, ei);
        const float Er = Ebr * er - Ebi * ei, Ei = Ebr * ei + Ebi * er;  // e^{j2pi f_c d_m/c}
        // phi = n + phi_r, |phi_r| <= 1/2; centre g = rint(phi_r G) wrapped into [0, G).  Y(phi + 1) =
        // (-1)^(N_f - 1) Y(phi) (k - k0 is a half-integer for even N_f), so the table value at the wrapped centre
        // is multiplied by (-1)^((n - w)(N_f - 1)), w = 1 when the centre was moved up by one period.
        const double xx = phib + (double)(delta * sc.df_cf);
        const double nper = rint(xx);
        const double x = (xx - nper) * (double)G;
        const double gi = rint(x);
        const float dp = (float)(x - gi);
        int g = (int)gi;
        int wper = 0;
        if (g < 0) { g += G; wper = 1; }
        if (g >= G) { g -= G; wper = -1; }
        const bool flip = (sc.nf & 1) == 0 && (((long long)nper - wper) & 1);
        const float4* row = reinterpret_cast<const float4*>(tj + ((int64_t)m * G + g) * TAY_L);
        const float4 c01 = __ldg(row), c23 = __ldg(row + 1), c45 = __ldg(row + 2), c67 = __ldg(row + 3);
        float yr = c67.z, yi = c67.w;  // Horner in delta', l = 7 .. 0
        yr = fmaf(yr, dp, c67.x); yi = fmaf(yi, dp, c67.y);
        yr = fmaf(yr, dp, c45.z); yi = fmaf(yi, dp, c45.w);
        yr = fmaf(yr, dp, c45.x); yi = fmaf(yi, dp, c45.y);
        yr = fmaf(yr, dp, c23.z); yi = fmaf(yi, dp, c23.w);
        yr = fmaf(yr, dp, c23.x); yi = fmaf(yi, dp, c23.y);
        yr = fmaf(yr, dp, c01.z); yi = fmaf(yi, dp, c01.w);
        yr = fmaf(yr, dp, c01.x); yi = fmaf(yi, dp, c01.y);
        if (flip) { yr = -yr; yi = -yi; }
        pr = fmaf(Er, yr, fmaf(-Ei, yi, pr));
        pi = fmaf(Er, yi, fmaf(Ei, yr, pi));
      }
      accr += (double)pr;
      acci += (double)pi;
    }
    const double gn = sc.pathloss ? sc.lambda / (4.0 * PI * R64) : 1.0;
    terms[(p * J + j) * T + s] = make_double2(accr * gn, acci * gn);
    double2* gr = terms + (p * J + j) * T + S + s * (s + 1) / 2;  // row s of the lower triangle of G
    gr[s] = make_double2((double)sc.nf * (double)Na * gn * gn, 0.0);  // G_ss = g^2 N_z
    if (gram_diag)  // callers that use c only: no off-diagonal Gram
      for (int c = 0; c < s; ++c) gr[c] = make_double2(0.0, 0.0);
  }
  if (fl) atomicOr(&pflag[p], fl);
}

// Off-diagonal Gram (row A4) next to K1T: one thread per (particle, PA), antennas in the outer loop; per antenna the
// S fp32 offsets Delta_s (as K1T / K1) and phasors E_s = e^{j2pi f_c Delta_s/c} once, then all S(S-1)/2 pair terms:
// carrier E_a conj(E_b) and K1's closed-form Dirichlet factor (gram_dirichlet_f) (fp32 over
// blocks of 8 antennas, fp64 totals per thread in shared memory: no barriers).  The pair's delay base
// x_ab = (R_a - R_b) df/c comes from per-component fp64 fractions split hi + lo in fp32 (K1 rounds the fp64
// difference once; the hi + lo difference is as accurate).  At the end the shared base carrier
// e^{j2pi (R_a - R_b) f_c/c} and the gains in fp64 (K1's hand-off convention, lower-triangle entry G_ba).
__device__ __forceinline__ bool tay_component(const SceneDev& sc, int j, const double* pos, const double* sfv_s,
                                              float& hx, float& hy, float& hz, double& R64) {
  double va[3], sh[3];
  if (!anchor_va(sc, j, sfv_s, va, sh)) return false;
  const double r0 = pos[0] - va[0], r1 = pos[1] - va[1], r2 = pos[2] - va[2];
  const double rs2 = 2.0 * (r0 * sh[0] + r1 * sh[1] + r2 * sh[2]);
  hx = (float)(r0 - rs2 * sh[0]); hy = (float)(r1 - rs2 * sh[1]); hz = (float)(r2 - rs2 * sh[2]);
  R64 = sqrt(r0 * r0 + r1 * r1 + r2 * r2);
  return R64 > 0.0;
}
template <int S>
__global__ void __launch_bounds__(TAY_BLOCK)
    tay_gram_kernel(const __grid_constant__ SceneDev sc, const float4* __restrict__ tmpl,
                    const double* __restrict__ particles, int64_t P, int pstride, const double* __restrict__ sfv,
                    int sfv_pp, double2* __restrict__ terms) {
  constexpr int NP = S * (S - 1) / 2;
  extern __shared__ double2 gsum[];  // [NP][TAY_BLOCK]
  const int64_t p = (int64_t)blockIdx.x * TAY_BLOCK + threadIdx.x;
  const int j = blockIdx.y;
  if (p >= P) return;
  const int J = sc.J, Na = sc.Na, T = S + S * (S + 1) / 2;
  const double* pos = particles + p * pstride;
  float hx[S], hy[S], hz[S], Rf[S], iR[S], uh[S], ul[S];
  double R64[S];
  int npar[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const double* sfv_s = s == 0 ? nullptr : (sfv_pp ? sfv + (p * sc.K + (s - 1)) * 3 : sfv + (int64_t)(s - 1) * 3);
    if (!tay_component(sc, j, pos, sfv_s, hx[s], hy[s], hz[s], R64[s])) return;  // flagged by K1T
    Rf[s] = (float)R64[s];
    iR[s] = 1.f / Rf[s];
    const double xs = R64[s] * sc.df_c, ns = rint(xs), us = xs - ns;
    uh[s] = (float)us;
    ul[s] = (float)(us - (double)uh[s]);
    npar[s] = (int)((long long)ns & 1);
  }
#pragma unroll
  for (int q = 0; q < NP; ++q) gsum[q * TAY_BLOCK + threadIdx.x] = make_double2(0.0, 0.0);
  const bool sph = sc.wavefront == CDMS_SPHERICAL;
  const float4* tm = tmpl + (int64_t)j * sc.n_mb * NWARP;
  for (int m0 = 0; m0 < Na; m0 += 8) {
    float gr[NP], gi[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) gr[q] = gi[q] = 0.f;
    const int m1 = min(m0 + 8, Na);
    for (int m = m0; m < m1; ++m) {
      const float4 v = __ldg(&tm[m]);
      float dl[S], er[S], ei[S];
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const float rq = hx[s] * v.x + hy[s] * v.y + hz[s] * v.z;
        if (sph) {
          const float n = v.w - 2.f * rq;
          dl[s] = n / (sqrtf(Rf[s] * Rf[s] + n) + Rf[s]);
        } else {
          dl[s] = -rq * iR[s];
        }
        cis2pi_fast<float>(dl[s] * sc.fc_cf, er[s], ei[s]);  // e^{j2pi f_c Delta_s/c}: the pairs' carriers as products
      }
      int q = 0;
#pragma unroll
      for (int a = 0; a < S; ++a) {
#pragma unroll
        for (int b = a + 1; b < S; ++b, ++q) {
          GramPairF gp;
          gp.xbr = (uh[a] - uh[b]) + (ul[a] - ul[b]);
          gp.nbpar = (uint32_t)((npar[a] ^ npar[b]) & 1) << 31;
          const float D = gram_dirichlet_f(sc, dl[a] - dl[b], gp);
          const float cr = fmaf(er[a], er[b], ei[a] * ei[b]), ci = fmaf(ei[a], er[b], -er[a] * ei[b]);  // E_a conj(E_b)
          gr[q] = fmaf(D, cr, gr[q]);
          gi[q] = fmaf(D, ci, gi[q]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      double2 t = gsum[q * TAY_BLOCK + threadIdx.x];
      gsum[q * TAY_BLOCK + threadIdx.x] = make_double2(t.x + (double)gr[q], t.y + (double)gi[q]);
    }
  }
  int q = 0;
#pragma unroll
  for (int a = 0; a < S; ++a) {
#pragma unroll
    for (int b = a + 1; b < S; ++b, ++q) {
      const double2 acc = gsum[q * TAY_BLOCK + threadIdx.x];
      double sn, cs;
      sincospi(2.0 * frac_c((R64[a] - R64[b]) * sc.fc_c), &sn, &cs);
      const double vr = cs * acc.x - sn * acc.y, vi = cs * acc.y + sn * acc.x;
      const double g2 = sc.pathloss ? (sc.lambda / (4.0 * PI * R64[a])) * (sc.lambda / (4.0 * PI * R64[b])) : 1.0;
      terms[(p * J + j) * T + S + b * (b + 1) / 2 + a] = make_double2(vr * g2, -vi * g2);
    }
  }
}
template <int S>
static cudaError_t launch_tay_gram_t(const SceneDev& sc, const float4* tmpl, const double* particles, int64_t P,
                                     int pstride, const double* sfv, int sfv_pp, double2* terms, cudaStream_t st) {
  constexpr int NP = S * (S - 1) / 2;
  const size_t smem = (size_t)NP * TAY_BLOCK * sizeof(double2);
  cudaError_t e = cudaFuncSetAttribute(tay_gram_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((P + TAY_BLOCK - 1) / TAY_BLOCK), sc.J);
  tay_gram_kernel<S><<<grid, TAY_BLOCK, smem, st>>>(sc, tmpl, particles, P, pstride, sfv, sfv_pp, terms);
  return cudaGetLastError();
}
cudaError_t launch_tay_gram(const SceneDev& sc, const float4* tmpl, const double* particles, int64_t P, int pstride,
                            const double* sfv, int sfv_pp, double2* terms, cudaStream_t st) {
  if (P <= 0) return cudaSuccess;
  switch (sc.S) {
    case 1: return cudaSuccess;
#define CASE_S(n) \
  case n: return launch_tay_gram_t<n>(sc, tmpl, particles, P, pstride, sfv, sfv_pp, terms, st);
    CASE_S(2) CASE_S(3) CASE_S(4) CASE_S(5) CASE_S(6) CASE_S(7) CASE_S(8) CASE_S(9)
#undef CASE_S
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_tay_prep(const SceneDev& sc, const float2* y, float2* tab, cudaStream_t st) {
  const int G = tay_centres(sc.nf);
  const int64_t n = (int64_t)sc.J * sc.Na * G * TAY_KS;
  tay_prep_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(sc, G, y, tab);
  return cudaGetLastError();
}
cudaError_t launch_tay_corr(const SceneDev& sc, const float2* tab, const float4* tmpl, const double* particles,
                            int64_t P, int pstride, const double* sfv, int sfv_pp, double2* terms, int* pflag,
                            int gram_diag, cudaStream_t st) {
  if (P <= 0) return cudaSuccess;
  dim3 grid((unsigned)((P + TAY_BLOCK - 1) / TAY_BLOCK), sc.J);
  tay_corr_kernel<<<grid, TAY_BLOCK, 0, st>>>(sc, tay_centres(sc.nf), tab, tmpl, particles, P, pstride, sfv, sfv_pp,
                                              terms, pflag, gram_diag);
  return cudaGetLastError();
}

}  // namespace cdms
