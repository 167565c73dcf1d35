// geometry.cuh -- device functions shared by every kernel that touches the array responses
// (loglik.cu, response.cu): anchor geometry (row A1), per-(particle, component) fp64 set-up and per-antenna
// offsets / phasors (row A2), and the Dirichlet kernel of the closed-form Gram (row A4).  The same
// functions serve the hot kernel, the test entry cdms_response and cdms_layout, so the parity checks of
// the latter two exercise the arithmetic of the former.
#pragma once
#include <math.h>

#include "cdms_internal.h"

namespace cdms {

// ---------------------------------------------------------------------------- numeric traits
template <typename RT>
struct Num;
template <>
struct Num<float> {
  static __device__ __forceinline__ void sincospi_(float x, float* s, float* c) { sincospif(x, s, c); }
  static __device__ __forceinline__ float sinpi_(float x) { return sinpif(x); }
  static __device__ __forceinline__ float rint_(float x) { return rintf(x); }
  static __device__ __forceinline__ float sqrt_(float x) { return sqrtf(x); }
  // ~2 ulp approximations without denormal fix-ups (arguments are metres, far from the denormal range)
  static __device__ __forceinline__ float fsqrt_(float x) {  // x > 0
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return x * r;
  }
  static __device__ __forceinline__ float fdiv_(float a, float b) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(b));
    return a * r;
  }
  static constexpr float tiny_x = 1e-6f;  // |xr| below which D_N uses its 2nd-order series
};
template <>
struct Num<double> {
  static __device__ __forceinline__ void sincospi_(double x, double* s, double* c) { sincospi(x, s, c); }
  static __device__ __forceinline__ double sinpi_(double x) { return sinpi(x); }
  static __device__ __forceinline__ double rint_(double x) { return rint(x); }
  static __device__ __forceinline__ double sqrt_(double x) { return sqrt(x); }
  static __device__ __forceinline__ double fsqrt_(double x) { return sqrt(x); }
  static __device__ __forceinline__ double fdiv_(double a, double b) { return a / b; }
  static constexpr double tiny_x = 1e-12;
};

// e^{j 2 pi x}, x in cycles (argument range-reduced to [-1/2, 1/2] first)
template <typename RT>
__device__ __forceinline__ void cis2pi(RT x, RT& re, RT& im) {
  x = x - Num<RT>::rint_(x);
  Num<RT>::sincospi_(RT(2) * x, &im, &re);
}

__device__ __forceinline__ double frac_c(double x) { return x - rint(x); }  // centred fraction

// e^{j 2 pi x} for per-antenna phase terms whose error only needs to be small and independent across
// antennas: fp32 uses the MUFU sin/cos (|abs error| <= 2^-21.4 on the reduced argument), fp64 stays exact.
template <typename RT>
__device__ __forceinline__ void cis2pi_fast(RT x, RT& re, RT& im);
template <>
__device__ __forceinline__ void cis2pi_fast<float>(float x, float& re, float& im) {
  x = x - ((x + 12582912.f) - 12582912.f);  // rint (|x| < 2^22) on the FMA pipe, bit-identical to rintf
  __sincosf(6.28318530717958647692f * x, &im, &re);
}
template <>
__device__ __forceinline__ void cis2pi_fast<double>(double x, double& re, double& im) {
  x = x - rint(x);
  sincospi(2.0 * x, &im, &re);
}

// e^{j 2 pi f_c Delta / c} from fp32 Delta (metres) and w = fp32(2 pi f_c / c): no centred reduction -- MUFU.SIN/COS
// take the argument in revolutions and drop the integer part themselves, so the only cost of |w Delta| > pi is the
// rounding of the revolutions (|err| <= |Delta f_c/c| 2^-23 cycles; tools/microbench/sincos_range.cu measures it
// against fp64, profiles/r02_sincos_range.txt).  Three FMA-pipe instructions fewer than cis2pi_fast per call.
__device__ __forceinline__ void carrier_f(float delta, float w, float& re, float& im) { __sincosf(delta * w, &im, &re); }

// ---------------------------------------------------------------------------- row A1 (geometry)
// VA phase centre p_VA = p_j - (2 p_j^T s/||s||^2 - 1) s and the unit wall normal
// shat = s/||s|| that defines H = I - 2 shat shat^T.  LOS (sfv == nullptr): p_VA = p_j,
// shat = 0, H = I.  Returns false for ||s|| = 0.
__device__ __forceinline__ bool anchor_va(const SceneDev& sc, int j, const double* sfv, double va[3],
                                          double sh[3]) {
  const double* pj = sc.pa_pos[j];
  if (sfv == nullptr) {
    va[0] = pj[0]; va[1] = pj[1]; va[2] = pj[2];
    sh[0] = sh[1] = sh[2] = 0.0;
    return true;
  }
  const double s0 = sfv[0], s1 = sfv[1], s2 = sfv[2];
  const double n2 = s0 * s0 + s1 * s1 + s2 * s2;
  if (!(n2 > 0.0)) return false;
  const double c = 2.0 * (pj[0] * s0 + pj[1] * s1 + pj[2] * s2) / n2 - 1.0;
  va[0] = pj[0] - c * s0; va[1] = pj[1] - c * s1; va[2] = pj[2] - c * s2;
  const double inv = 1.0 / sqrt(n2);
  sh[0] = s0 * inv; sh[1] = s1 * inv; sh[2] = s2 * inv;
  return true;
}

// R_j p~_m for template column m = iy*nv + iv: p~ = (0, p_y[iy], p_z[iv])
__device__ __forceinline__ void template_col(const SceneDev& sc, int j, int m, double v[3], double& q2) {
  const int iy = m / sc.nv, iv = m - iy * sc.nv;
  const double py = (iy - 0.5 * (sc.ny - 1)) * sc.dy;
  const double pz = (iv - 0.5 * (sc.nv - 1)) * sc.dv;
  const double* R = sc.pa_rot[j];
  v[0] = R[1] * py + R[2] * pz;
  v[1] = R[4] * py + R[5] * pz;
  v[2] = R[7] * py + R[8] * pz;
  q2 = py * py + pz * pz;  // ||H R p~||^2 = ||p~||^2
}

// Per (particle, PA j, component s) set-up (fp64), kept in shared memory as RT fields:
//   h = H r with r = p - p_VA (so that r.q_m = r.(H v_m) = h.v_m, H symmetric: one dot product per antenna),
//   R = ||r|| (fp64 and RT), and the phase-centre phasors
//   E0 = e^{j2pi R f0/c}, W = e^{j2pi R df/c}, Zp = e^{j2pi SEG R df/c}, evaluated in fp64 from fp64
//   range-reduced phases and only then rounded (a fp32 phase in cycles would carry a ~1e-7 cycle error
//   that w^k repeats coherently on every antenna), gain = lambda/(4 pi R) with path loss
//   (C-amb-6) else 1.
// W and Zp stay in fp64: the per-antenna step w = fp32(W * s_m) must be rounded independently on every
// antenna, otherwise the fp32 rounding of a shared W (|W| - 1 ~ 3e-8) is raised to the k-th power
// identically on all antennas and the Horner correlation drifts coherently away from the exact
// closed-form Gram.
// With exactly two Horner segments (SEG < N_f <= 2 SEG, sc.two_seg) the second segment's start phasor is
// formed directly like the first, E1 = e^{j2pi R (f0 + SEG df)/c} (fp64) times its per-antenna correction, instead
// of A0 Z: one MUFU pair instead of the accurate Z polynomial and the product.
template <typename RT>
struct PSField {
  RT hx, hy, hz, R, E0r, E0i, gain;
  RT Whr, Whi, Wlr, Wli, Zhr, Zhi, Zlr, Zli;  // W, Zp as unevaluated sums hi + lo (fp32: ~48-bit mantissa)
  RT E1r, E1i;                                // second-segment phase-centre phasor (two_seg only)
};
constexpr int NPSF = 17;       // RT fields of PSField
// shared-memory stride per (component, particle): 80 B (fp32), 4 x LDS.128; a stride of 4 x odd words keeps the
// per-lane 128-bit loads of a quarter warp on distinct banks (64 B would be 4-way conflicted)
constexpr int NPSF_PAD = 20;
constexpr int PSF_GAIN = 6;    // index of .gain

// Load the NPSF fields of one (component, particle) record with 128-bit shared-memory loads.
template <typename RT>
__device__ __forceinline__ void load_psf(const RT* src, RT* fv) {
  const float4* s4 = reinterpret_cast<const float4*>(src);
  float4* d4 = reinterpret_cast<float4*>(fv);
  constexpr int N4 = (NPSF * (int)sizeof(RT) + 15) / 16;
  float4 tmp[(NPSF_PAD * sizeof(RT)) / 16];
#pragma unroll
  for (int i = 0; i < N4; ++i) tmp[i] = s4[i];
  const RT* t = reinterpret_cast<const RT*>(tmp);
#pragma unroll
  for (int q = 0; q < NPSF; ++q) fv[q] = t[q];
  (void)d4;
}

// Returns PS_OK, PS_DEGENERATE (MT on the phase centre, r' = 0 excluded by P:L2137) or PS_BADSFV
// (||sfv|| = 0).  On failure the fields hold a harmless finite placeholder.
enum { PS_OK = 0, PS_DEGENERATE = 1, PS_BADSFV = 2 };
// PH = false (K1's Gram-only variant): geometry and gain only, no phase-centre phasors.
template <typename RT, bool PH = true>
__device__ __forceinline__ int setup_ps(const SceneDev& sc, int j, const double* pos, const double* sfv_s,
                                        PSField<RT>& f, double& R64) {
  double va[3], sh[3];
  const bool sfv_ok = anchor_va(sc, j, sfv_s, va, sh);
  if (!sfv_ok) {
    va[0] = pos[0] - 1.0; va[1] = pos[1]; va[2] = pos[2];
    sh[0] = sh[1] = sh[2] = 0.0;
  }
  const double r0 = pos[0] - va[0], r1 = pos[1] - va[1], r2 = pos[2] - va[2];
  const double R = sqrt(r0 * r0 + r1 * r1 + r2 * r2);
  R64 = R;
  const double rs2 = 2.0 * (r0 * sh[0] + r1 * sh[1] + r2 * sh[2]);
  f.hx = (RT)(r0 - rs2 * sh[0]); f.hy = (RT)(r1 - rs2 * sh[1]); f.hz = (RT)(r2 - rs2 * sh[2]);
  f.R = (RT)R;
  if (PH) {
    double s_, c_;
    sincospi(2.0 * frac_c(R * sc.f0_c), &s_, &c_);
    f.E0r = (RT)c_; f.E0i = (RT)s_;
    sincospi(2.0 * frac_c(R * sc.df_c), &s_, &c_);
    f.Whr = (RT)c_; f.Whi = (RT)s_;
    f.Wlr = (RT)(c_ - (double)f.Whr); f.Wli = (RT)(s_ - (double)f.Whi);
    sincospi(2.0 * frac_c(R * sc.segdf_c), &s_, &c_);
    f.Zhr = (RT)c_; f.Zhi = (RT)s_;
    f.Zlr = (RT)(c_ - (double)f.Zhr); f.Zli = (RT)(s_ - (double)f.Zhi);
    if (sc.two_seg) {
      sincospi(2.0 * frac_c(R * sc.f1_c), &s_, &c_);
      f.E1r = (RT)c_; f.E1i = (RT)s_;
    } else {
      f.E1r = RT(1); f.E1i = RT(0);
    }
  } else {
    f.E0r = f.Whr = f.Zhr = f.E1r = RT(1);
    f.E0i = f.Whi = f.Zhi = f.E1i = f.Wlr = f.Wli = f.Zlr = f.Zli = RT(0);
  }
  f.gain = (RT)(sc.pathloss ? sc.lambda / (4.0 * PI * R) : 1.0);
  if (!sfv_ok) return PS_BADSFV;
  if (!(R > 0.0)) {  // also catches NaN positions
    f.R = RT(1); f.hx = RT(1); f.hy = RT(0); f.hz = RT(0); f.gain = RT(1);
    R64 = 1.0;
    return PS_DEGENERATE;
  }
  return PS_OK;
}

// Per (particle, component, antenna) offset Delta_m of the element distance from R and the three
// phasors of the recurrence (all conjugate-response phases, e^{+j 2 pi d f / c}):
//   spherical: d_m = ||r - q_m||, q_m = H R p~_m, Delta = (||q||^2 - 2 r.q)/(d_m + R)
//   planar WB / NB: Delta = -q.u = -(r.q)/R
//   A = E0 e^{j2pi Delta f0/c}, w = W e^{j2pi Delta df/c}, Z = Zp e^{j2pi SEG Delta df/c}
//   NB: the spatial term uses f_c: A = E0 e^{j2pi Delta fc/c}, w = W, Z = Zp.
// The per-antenna step correction Delta df/c is tiny (|Delta| <= half the aperture): when the scene
// guarantees |2 pi Delta df/c| <= 0.2 (sc.small_step) it is a degree-7 Taylor polynomial (error < 3e-10).
template <typename RT>
__device__ __forceinline__ void cis_small(RT x_cycles, RT& re, RT& im) {
  const RT t = RT(2.0 * PI) * x_cycles, t2 = t * t;
  re = RT(1) + t2 * (RT(-0.5) + t2 * (RT(1.0 / 24) + t2 * RT(-1.0 / 720)));
  im = t * (RT(1) + t2 * (RT(-1.0 / 6) + t2 * (RT(1.0 / 120) + t2 * RT(-1.0 / 5040))));
}
// |2 pi Delta df/c| <= 0.02 (sc.small_step == 2, e.g. every BASELINE config): degree 4 / 3 (error < 3e-11)
template <typename RT>
__device__ __forceinline__ void cis_tiny(RT x_cycles, RT& re, RT& im) {
  const RT t = RT(2.0 * PI) * x_cycles, t2 = t * t;
  re = RT(1) + t2 * (RT(-0.5) + t2 * RT(1.0 / 24));
  im = t * (RT(1) + t2 * RT(-1.0 / 6));
}
// e^{j 2 pi x} for |2 pi x| <= 1 (sc.small_z): degree-12/13 Taylor polynomials (error < 1.1e-11)
template <typename RT>
__device__ __forceinline__ void cis_med(RT x_cycles, RT& re, RT& im) {
  const RT t = RT(2.0 * PI) * x_cycles, t2 = t * t;
  re = RT(1) + t2 * (RT(-1.0 / 2) + t2 * (RT(1.0 / 24) + t2 * (RT(-1.0 / 720) + t2 * (RT(1.0 / 40320) +
       t2 * (RT(-1.0 / 3628800) + t2 * RT(1.0 / 479001600))))));
  im = t * (RT(1) + t2 * (RT(-1.0 / 6) + t2 * (RT(1.0 / 120) + t2 * (RT(-1.0 / 5040) + t2 * (RT(1.0 / 362880) +
       t2 * (RT(-1.0 / 39916800) + t2 * RT(1.0 / 6227020800.0)))))));
}
template <typename RT>
__device__ __forceinline__ void cmul(RT ar, RT ai, RT br, RT bi, RT& cr, RT& ci) {
  cr = ar * br - ai * bi;
  ci = ar * bi + ai * br;
}
// (W_hi + W_lo) * s with the small products first and one final rounding per component: the result's
// rounding depends on the antenna's s, so it is independent across antennas (fp32 FMAs only)
template <typename RT>
__device__ __forceinline__ void cmul_df(RT Whr, RT Whi, RT Wlr, RT Wli, RT sr, RT si, RT& cr, RT& ci) {
  const RT lr = fma(Wlr, sr, -Wli * si), li = fma(Wlr, si, Wli * sr);
  cr = fma(Whr, sr, fma(-Whi, si, lr));
  ci = fma(Whr, si, fma(Whi, sr, li));
}
// deterministic per-(antenna, component) rotation in (-2^-24, 2^-24) rad: decorrelates the fp32 rounding of
// an otherwise shared step phasor across antennas (NB, where the per-antenna step correction is 1)
__device__ __forceinline__ double dither_angle(int m, int s) {
  uint32_t h = (uint32_t)m * 0x9E3779B1u ^ ((uint32_t)s + 0x7F4A7C15u) * 0x85EBCA77u;
  h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12;
  return ((double)(h >> 8) * 0x1p-24 - 0.5) * 0x1p-23;
}
template <typename RT>
struct SMPhasors {
  RT Ar, Ai, wr, wi, Zr, Zi, delta;
};

template <typename RT>
__device__ __forceinline__ void setup_sm(const SceneDev& sc, const PSField<RT>& f, const RT v[3], RT q2, int m,
                                         int s, SMPhasors<RT>& o, bool& degenerate) {
  const RT rq = f.hx * v[0] + f.hy * v[1] + f.hz * v[2];  // r.q_m = (H r).v_m
  RT delta;
  if (sc.wavefront == CDMS_SPHERICAL) {
    const RT n = q2 - RT(2) * rq;
    const RT d = Num<RT>::fsqrt_(f.R * f.R + n);
    degenerate = !(d > RT(0));
    delta = Num<RT>::fdiv_(n, d + f.R);  // |delta| <= aperture: ~1 ulp relative error is ample
  } else {
    delta = Num<RT>::fdiv_(-rq, f.R);
    degenerate = false;
  }
  o.delta = delta;
  // frequency constants in RT (fp32: the host-rounded copies, constant-bank operands, no per-use F2F)
  constexpr bool F32 = sizeof(RT) == 4;
  const RT fc_c = F32 ? (RT)sc.fc_cf : (RT)sc.fc_c, f0_c = F32 ? (RT)sc.f0_cf : (RT)sc.f0_c;
  const RT df_c = F32 ? (RT)sc.df_cf : (RT)sc.df_c, segdf_c = F32 ? (RT)sc.segdf_cf : (RT)sc.segdf_c;
  RT er, ei;
  if (sc.wavefront == CDMS_PLANAR_NB) {
    cis2pi_fast<RT>(delta * fc_c, er, ei);
    cmul<RT>(f.E0r, f.E0i, er, ei, o.Ar, o.Ai);
    const RT t = (sizeof(RT) == 4) ? (RT)dither_angle(m, s) : RT(0);
    cmul_df<RT>(f.Whr, f.Whi, f.Wlr, f.Wli, RT(1), t, o.wr, o.wi);
    const RT tz = (sizeof(RT) == 4) ? (RT)dither_angle(m, s + 16) : RT(0);
    cmul_df<RT>(f.Zhr, f.Zhi, f.Zlr, f.Zli, RT(1), tz, o.Zr, o.Zi);
  } else {
    // A: one rounding per antenna, independent across antennas -> MUFU accuracy suffices
    cis2pi_fast<RT>(delta * f0_c, er, ei);
    cmul<RT>(f.E0r, f.E0i, er, ei, o.Ar, o.Ai);
    // w, Z are raised to powers: accurate small-angle polynomials / sincospi, products rounded once in fp64
    if (sc.small_step == 2) cis_tiny<RT>(delta * df_c, er, ei);
    else if (sc.small_step) cis_small<RT>(delta * df_c, er, ei);
    else cis2pi<RT>(delta * df_c, er, ei);
    cmul_df<RT>(f.Whr, f.Whi, f.Wlr, f.Wli, er, ei, o.wr, o.wi);
    if (sc.two_seg) {  // the (Zr, Zi) slot carries A1 itself: the second segment starts at A1, not A0 Z
      const RT f1_c = F32 ? (RT)sc.f1_cf : (RT)sc.f1_c;
      cis2pi_fast<RT>(delta * f1_c, er, ei);
      cmul<RT>(f.E1r, f.E1i, er, ei, o.Zr, o.Zi);
    } else if (sc.nf > SEG) {  // Z only advances A between segments
      if (sc.small_z) cis_med<RT>(delta * segdf_c, er, ei);
      else cis2pi<RT>(delta * segdf_c, er, ei);
      cmul_df<RT>(f.Zhr, f.Zhi, f.Zlr, f.Zli, er, ei, o.Zr, o.Zi);
    } else {
      o.Zr = RT(1);
      o.Zi = RT(0);
    }
  }
}

// Dirichlet kernel D_N(x) = sin(pi N x)/sin(pi x) for x = n + xr, |xr| <= 1/2:
// D_N(x) = (-1)^{n (N-1)} D_N(xr), D_N(0) = N (C-amb-13).
template <typename RT>
__device__ __forceinline__ RT dirichlet(RT xr, long long n, int N) {
  RT d;
  if (xr < Num<RT>::tiny_x && xr > -Num<RT>::tiny_x) {
    const RT N2 = (RT)N * (RT)N;
    d = (RT)N * (RT(1) - RT(PI * PI / 6.0) * (N2 - RT(1)) * xr * xr);
  } else {
    d = Num<RT>::sinpi_((RT)N * xr) / Num<RT>::sinpi_(xr);
  }
  if (((N - 1) & 1) && (n & 1)) d = -d;
  return d;
}

// ---------------------------------------------------------------------------- Gram term per (pair, antenna)
// sum_k e^{j 2 pi dd_m f_k / c} relative to the pair's base carrier, for one antenna (row A4):
//   e^{j 2 pi dd fc/c} D_N(x), x = dR df/c + dd df/c = nb + xbr + dd df/c, dd = Delta_a,m - Delta_b,m
//   D_N(n + xr) = (-1)^{n (N-1)} sin(pi N xr) / sin(pi xr), D_N(0) = N (C-amb-13)
// fp32: MUFU carrier and numerator (after exact mod-2 reduction of N xr), polynomial sin(pi xr), one
// approximate reciprocal, branch-free small-|xr| series and sign; fp64: exact library functions.
struct GramPairF {
  float xbr;        // centred fraction of dR df/c (from fp64)
  uint32_t nbpar;   // parity of the integer part nb, shifted to bit 31 when N is even (sign flips), else 0
};
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// sin(pi t) for the Dirichlet numerator, t = N xr reduced mod 2 to [-1, 1]: MUFU (absolute error <= 2^-21.4) when
// |t| > 1/4, where that is <= 5e-7 of the value; for |t| <= 1/4 (near-equal delays of the pair, N |xr| small) the
// relative accuracy matters -- D_N ~ N there and every antenna of the pair sees about the same x, so a relative
// numerator error adds coherently into G_ab (tests/test_k1t_terms_gpu.py, equal-delay particles) -- and the odd
// Taylor polynomial pi t S(pi t), S(z) = 1 - z^2/6 + z^4/120 - z^6/5040 + z^8/362880 (relative error < 3e-9 at
// pi/4) replaces it.  The branch is taken with probability ~1/(2N) per (pair, antenna).
__device__ __forceinline__ float dirichlet_num(float t) {
  // selects, not a branch: the callers' pair loops are fully unrolled and a branch per term would serialize them
  const float z = 3.14159265358979f * t, z2 = z * z;
  const float ps = z * fmaf(z2, fmaf(z2, fmaf(z2, fmaf(z2, 1.f / 362880, -1.f / 5040), 1.f / 120), -1.f / 6), 1.f);
  return fabsf(t) <= 0.25f ? ps : __sinf(z);
}
// The Dirichlet factor of gram_term_f alone (the caller supplies the carrier e^{j2pi dd f_c/c}).
__device__ __forceinline__ float gram_dirichlet_f(const SceneDev& sc, float dd, const GramPairF& gp) {
  const float df_c = sc.df_cf, Nf = sc.nf_f;
  // rint by the 1.5 * 2^23 magic constant (FADDs, |x| << 2^22) rather than FRND: the Gram kernels that call this
  // per (pair, antenna) are XU-bound (profiles/r01_k1t_lanes.txt); the sum's low mantissa bit is n2's parity
  constexpr float M = 12582912.f;
  const float x = fmaf(dd, df_c, gp.xbr);
  const float xm = x + M;
  const float xr = x - (xm - M);
  float t = Nf * xr;
  t = fmaf(-2.f, (fmaf(0.5f, t, M) - M), t);
  const float num = dirichlet_num(t);
  const float u = 3.14159265358979f * xr, u2 = u * u;
  const float den = u * fmaf(u2, fmaf(u2, fmaf(u2, fmaf(u2, fmaf(u2, -1.f / 39916800, 1.f / 362880), -1.f / 5040),
                                                1.f / 120), -1.f / 6), 1.f);
  float D = num * rcp_approx(den);
  D = (fabsf(xr) < 1e-30f) ? Nf : D;  // D_N(0) = N (C-amb-13); num and den are relatively accurate down to tiny xr
  const uint32_t par = ((uint32_t)__float_as_int(xm) << 31) ^ gp.nbpar;
  return __int_as_float(__float_as_int(D) ^ (int)(par & sc.evenN_mask));
}
__device__ __forceinline__ void gram_term_f(const SceneDev& sc, float dd, const GramPairF& gp, float& gr,
                                            float& gi) {
  const float fc_c = sc.fc_cf;
  float ph = dd * fc_c;
  ph -= rintf(ph);
  float sn, cs;
  __sincosf(6.28318530717958647692f * ph, &sn, &cs);
  const float D = gram_dirichlet_f(sc, dd, gp);
  gr = fmaf(D, cs, gr);
  gi = fmaf(D, sn, gi);
}


}  // namespace cdms
