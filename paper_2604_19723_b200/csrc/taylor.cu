// K1T: the spherical / planar-WB correlation of row A3 from per-PA spectral Taylor tables (FP32 mode).
//
// The correlation of component s with the snapshot, c_s = psi_s^H z, is, per antenna m, a
// trigonometric polynomial of the element's delay evaluated at one point:
//   c_s = sum_m e^{j2pi f_c d_m/c} Y_m(phi_m),   Y_m(phi) = sum_k y[m,k] e^{j2pi (k - k0) phi},  phi_m = df d_m / c,
// (f_k = f_c + (k - k0) df, k0 = (N_f - 1)/2; d_m the spherical distance or the planar projection of the element,
// P:L108-143).  Y_m is 1-periodic up to the sign (-1)^(N_f - 1) (k - k0 is a half-integer for even N_f) and
// band-limited to |k - k0| <= N_f/2, so on centres phi_g = (g - G/2)/G of one period [-1/2, 1/2] (and a few beyond
// each end: the reduction needs no wrap) its Taylor expansion in delta' = (phi - phi_g) G,
//   Y_m(phi_g + delta'/G) = sum_l C_l(m, g) delta'^l,  C_l = sum_k y[m,k] e^{j2pi (k-k0) phi_g} (j2pi (k-k0)/G)^l / l!,
// truncated after L terms has a relative error below (pi N_f/(2G))^L/L! of sum_k |y[m,k]|: L = 8 at G = 4 N_f (1.4e-8,
// the lane-group kernel's table) or L = 6 at G = 8 N_f (8.2e-8, the thread-per-particle kernels'), at or below fp32
// rounding, so K1T evaluates the same correlation as the Horner recurrence of K1 to fp32 accuracy with one 64- or
// 48-byte table row and a short Horner per (particle, component, antenna) instead of N_f complex multiply-adds.  The
// tables (fp64 sums rounded once to complex64, tay_prep_fft_kernel / tay_prep_kernel) cost O(J N_a G log G) per call
// and stay L2-resident.  The Gram is the closed form with a Taylor table of the Dirichlet kernel (tay_gram_kernel).
#include <math.h>

#include <algorithm>

#include "cdms_internal.h"
#include "geometry.cuh"

namespace cdms {

namespace {
constexpr int TAY_L = 8;
constexpr int TAY_BLOCK = 128;
}  // namespace

// 32 bytes (4 complex64 coefficients) in one 256-bit load (LDG.E.ENL2.256, sm_100): the table gathers are
// L1-wavefront / issue bound, and a 64-byte row then takes 2 loads instead of 4.  p must be 32-byte aligned.
__device__ __forceinline__ void ldg256(const float4* p, float4& a, float4& b) {
  asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
      : "l"(p));
}

// Two table forms.  Lane-group kernel ([j][g][h][m] layout): G = 4 N_f centres per period and TAY_L = 8 coefficients
// (truncation (pi/8)^8/8! = 1.4e-8).  Thread-per-particle kernels ([j][m][g], split in two arrays): G = 8 N_f and
// TAY_L6 = 6 coefficients (truncation (pi/16)^6/6! = 8.2e-8 of sum_k |y[m,k]|, at fp32 rounding) -- 48 instead of
// 64 bytes per element through the L1 data path that bounds that kernel, as one 32-byte row (C_0..C_3) in array A and
// one 16-byte row (C_4, C_5) in array B (48-byte rows in one array would break the 32-byte alignment of the
// 256-bit loads).  Measured (c5 4M, correlation kernel): 64-byte rows 20.5 ms, 48-byte rows 16.7 ms with the same
// table size (profiles/r02_gram_onechunk.txt); 1.5x the table bytes.
constexpr int TAY_L6 = 6;
int tay_centres(int nf, int lanes) { return lanes ? 4 * nf : 8 * nf; }
// The table holds TAY_EXT centres beyond each end of the period as well (phi_g = (g - TAY_EXT - G/2)/G, g = 0 ..
// G + 2 TAY_EXT): evaluated from the definition, they carry Y's (-1)^(N_f - 1) per period themselves, so the
// correlation kernel's fast locate (tay_corr_kernel, FL) needs neither a wrap nor a per-element sign.
constexpr int TAY_EXT = 4;
__host__ __device__ constexpr int tay_rows(int G) { return G + 1 + 2 * TAY_EXT; }
size_t tay_table_bytes(const SceneDev& sc, int lanes) {
  return (size_t)sc.J * sc.Na * tay_rows(tay_centres(sc.nf, lanes)) * (lanes ? TAY_L : TAY_L6) * sizeof(float2);
}
// thread layout: coefficient l of row (j, m, g) -- A [J][N_a][rows][4] for l < 4, then B [J][N_a][rows][2]
__host__ __device__ __forceinline__ int64_t tay_t6_index(int J, int Na, int G, int j, int m, int g, int l) {
  const int64_t row = ((int64_t)j * Na + m) * tay_rows(G) + g;
  return l < 4 ? row * 4 + l : (int64_t)J * Na * tay_rows(G) * 4 + row * 2 + (l - 4);
}

// tab[j][m][g][l] (complex64, l fastest: one 64-byte row per (j, m, g), g = 0..G) or, with lanes, [j][g][h][m] of
// 32-byte entries (coefficients 4h .. 4h+3).  TAY_KS lanes per row split the subcarrier sum (each from an exact anchor
// e^{j2pi (k - k0) phi_g}, fp64 phasor recurrence inside its segment), combined by a
// fixed shuffle tree: row count alone (J N_a G) would leave most SMs idle at small N_a G.
constexpr int TAY_KS = 8;
template <int L>  // coefficients per row: TAY_L (lanes layout) or TAY_L6 (thread layout)
__global__ void tay_prep_kernel(const __grid_constant__ SceneDev sc, int G, const float2* __restrict__ y,
                                float2* __restrict__ tab, int lanes) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t t = tid / TAY_KS;
  const int seg = (int)(tid - t * TAY_KS);
  const int64_t per_j = (int64_t)sc.Na * tay_rows(G);
  const bool live = t < per_j * sc.J;
  const int64_t tt = live ? t : 0;
  const int j = (int)(tt / per_j);
  const int64_t r = tt - (int64_t)j * per_j;
  const int m = (int)(r / tay_rows(G)), g = (int)(r - (int64_t)m * tay_rows(G));
  const int gs = g - TAY_EXT - G / 2;  // phi_g = gs / G
  const double k0 = 0.5 * (sc.nf - 1);
  double cr[L], ci[L];
#pragma unroll
  for (int l = 0; l < L; ++l) cr[l] = ci[l] = 0.0;
  const int kseg = (sc.nf + TAY_KS - 1) / TAY_KS;
  const int kb = seg * kseg, ke = min(kb + kseg, sc.nf);
  if (live && kb < ke) {
    double sw, cw;
    sincospi(2.0 * (double)gs / (double)G, &sw, &cw);  // step e^{j2pi phi_g}
    double pr = 1.0, pi = 0.0;
    const float2* ym = y + (int64_t)j * sc.nf * sc.Na + m;
    for (int k = kb; k < ke; ++k) {
      if (((k - kb) & 63) == 0) {  // anchor e^{j2pi (k - k0) gs/G}: exact reduction of 2 (k - k0) gs mod 2G
        const double num = fmod(2.0 * ((double)k - k0) * (double)gs, 2.0 * (double)G);
        sincospi(num / (double)G, &pi, &pr);
      }
      const float2 v = ym[(int64_t)k * sc.Na];
      double br = v.x * pr - v.y * pi, bi = v.x * pi + v.y * pr;  // y_k e^{j2pi (k-k0) g/G}
      const double tk = 2.0 * PI * ((double)k - k0) / (double)G;
#pragma unroll
      for (int l = 0; l < L; ++l) {
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
    for (int l = 0; l < L; ++l) {
      cr[l] += __shfl_xor_sync(0xffffffffu, cr[l], o);
      ci[l] += __shfl_xor_sync(0xffffffffu, ci[l], o);
    }
  }
  if (live && seg == 0) {
    if (lanes) {  // [j][g][h][m][4]
      float2* out = tab + ((((int64_t)j * tay_rows(G) + g) * 2) * sc.Na + m) * 4;
#pragma unroll
      for (int l = 0; l < L; ++l) out[(int64_t)(l >> 2) * sc.Na * 4 + (l & 3)] = make_float2((float)cr[l], (float)ci[l]);
    } else {  // thread layout (arrays A, B)
#pragma unroll
      for (int l = 0; l < L; ++l) tab[tay_t6_index(sc.J, sc.Na, G, j, m, g, l)] = make_float2((float)cr[l], (float)ci[l]);
    }
  }
}

// The same table by FFT when G is a power of two: for each l, c_l(g) = e^{-j2pi k0 g/G} sum_k a_k e^{j2pi k g/G}
// with a_k = y_k (j t_k)^l / l!, the zero-padded length-G DFT (positive exponent) of a.  One block per (j, m, l):
// fp64 radix-2 decimation in time in shared memory (bit-reversed load, log2 G stages, twiddle table e^{j2pi i/G}
// from sincospi), G/2 log2 G butterflies instead of the direct sum's G N_f terms; the centring phase uses the exact
// integer reduction (N_f - 1) gs mod 2G; centre g = 0..G reads bin (g - G/2) mod G.
constexpr int TAY_FFT_THREADS = 256;
__global__ void __launch_bounds__(TAY_FFT_THREADS)
    tay_prep_fft_kernel(const __grid_constant__ SceneDev sc, int G, int lgG, const float2* __restrict__ y,
                        float2* __restrict__ tab, int lanes) {
  extern __shared__ double2 fsm[];
  double2* a = fsm;      // [G]
  double2* w = fsm + G;  // [G/2]
  const int L = lanes ? TAY_L : TAY_L6;
  const int l = blockIdx.x % L;
  const int jm = blockIdx.x / L;
  const int j = jm / sc.Na, m = jm - j * sc.Na;
  const int nf = sc.nf;
  const double k0 = 0.5 * (nf - 1);
  for (int i = threadIdx.x; i < G / 2; i += TAY_FFT_THREADS) {
    double s, c;
    sincospi(2.0 * (double)i / (double)G, &s, &c);
    w[i] = make_double2(c, s);
  }
  for (int i = threadIdx.x; i < G; i += TAY_FFT_THREADS) {
    double2 v = make_double2(0.0, 0.0);
    if (i < nf) {
      const float2 yy = y[((int64_t)j * nf + i) * sc.Na + m];
      const double tk = 2.0 * PI * ((double)i - k0) / (double)G;
      double f = 1.0;
      for (int q = 1; q <= l; ++q) f *= tk / (double)q;  // t_k^l / l!
      const double vr = (double)yy.x * f, vi = (double)yy.y * f;
      switch (l & 3) {  // times j^l
        case 0: v = make_double2(vr, vi); break;
        case 1: v = make_double2(-vi, vr); break;
        case 2: v = make_double2(-vr, -vi); break;
        default: v = make_double2(vi, -vr); break;
      }
    }
    a[__brev((unsigned)i) >> (32 - lgG)] = v;
  }
  __syncthreads();
  for (int lh = 0; lh < lgG; ++lh) {  // butterflies of span h = 2^lh
    const int h = 1 << lh;
    for (int b = threadIdx.x; b < G / 2; b += TAY_FFT_THREADS) {
      const int pos = b & (h - 1);
      const int i0 = ((b >> lh) << (lh + 1)) + pos, i1 = i0 + h;
      const double2 tw = w[pos << (lgG - 1 - lh)];  // e^{j2pi pos/(2h)}
      const double2 u = a[i0], x = a[i1];
      const double vr = x.x * tw.x - x.y * tw.y, vi = x.x * tw.y + x.y * tw.x;
      a[i0] = make_double2(u.x + vr, u.y + vi);
      a[i1] = make_double2(u.x - vr, u.y - vi);
    }
    __syncthreads();
  }
  for (int g = threadIdx.x; g < tay_rows(G); g += TAY_FFT_THREADS) {
    const int gs = g - TAY_EXT - G / 2;  // phi_g = gs / G
    int64_t num = ((int64_t)(nf - 1) * gs) % (2 * (int64_t)G);  // e^{-j2pi k0 phi_g} = e^{-j pi num/G}
    if (num < 0) num += 2 * (int64_t)G;
    double s, c;
    sincospi(-(double)num / (double)G, &s, &c);
    const double2 v = a[gs & (G - 1)];
    const float2 o = make_float2((float)(v.x * c - v.y * s), (float)(v.x * s + v.y * c));
    if (lanes)  // [j][g][h][m][4] (coefficients 4h .. 4h+3)
      tab[((((int64_t)j * tay_rows(G) + g) * 2 + (l >> 2)) * sc.Na + m) * 4 + (l & 3)] = o;
    else  // thread layout (arrays A, B)
      tab[tay_t6_index(sc.J, sc.Na, G, j, m, g, l)] = o;
  }
}

// Delay phase base of one (particle, component), phib = R df/c cycles, reduced once in fp64 to n0 + hi + lo
// (|hi| <= 1/2, lo the fp32 remainder, par = n0 mod 2); per antenna tay_locate then needs fp32 only.
struct TayBase {
  float hi, lo;
  int par;
};
__device__ __forceinline__ TayBase tay_base(double phib) {
  const double n0 = rint(phib), r0 = phib - n0;
  TayBase b;
  b.hi = (float)r0;
  b.lo = (float)(r0 - (double)b.hi);
  b.par = (int)((long long)n0 & 1);
  return b;
}
constexpr float TAY_MAGIC = 12582912.f;  // 1.5 * 2^23: (x + M) - M = rint(x) for |x| < 2^22, int bits of x + M - bits(M) = rint(x)
// phi = phib + t (t = Delta_m df/c) = n + r, |r| <= 1/2 (TwoSum keeps hi + t exact as s + e); centre
// g = rint(r G) + G/2 in [0, G] (phi_g = r rounded to the grid: no wrap, the table stores both ends), delta' =
// r G - rint(r G) (one fma, then the e + lo correction).  Y(phi + 1) = (-1)^(N_f - 1) Y(phi) (k - k0 is a
// half-integer for even N_f), so the table value is multiplied by (-1)^((n0 + n)(N_f - 1)).  No conversions or MUFU:
// the fp64 version of this reduction (F2F, F2I, DFRND per antenna) held the XU pipe.
__device__ __forceinline__ void tay_locate(float t, float hi, float lo, int par, int Gh, float Gf, bool evenN,
                                           uint32_t& g, float& dp, bool& flip) {
  const float s = hi + t;
  const float bb = s - hi;
  const float e = (hi - (s - bb)) + (t - bb);
  const float sm = s + TAY_MAGIC;
  const float r = s - (sm - TAY_MAGIC);     // exact
  const float gm = fmaf(r, Gf, TAY_MAGIC);  // rint(r G) + M
  const float gi = gm - TAY_MAGIC;
  dp = fmaf(r, Gf, -gi) + (e + lo) * Gf;
  g = (uint32_t)(__float_as_int(gm) - __float_as_int(TAY_MAGIC) + Gh + TAY_EXT);  // the extended table's row
  const int nn = __float_as_int(sm) - __float_as_int(TAY_MAGIC);
  flip = evenN && ((par + nn) & 1);
}

// c_s for one particle per thread and one PA per blockIdx.y ([j][m][g][l] table; used when P J fills the SMs,
// else tay_corr_lanes_kernel below): per component the fp64 geometry (VA, H r, R), the
// fp64-reduced phase bases e^{j2pi f_c R/c} and frac(df R/c); per antenna the fp32 offset Delta_m (cancellation-free,
// as K1), the phasor e^{j2pi f_c Delta_m/c}, the table centre and delta', one table row and the Taylor sum.
// SPH: spherical (else planar WB), a template so the antenna loop carries no predicated other path.  TC: the template
// columns from the constant bank (TmplC kernel parameter): the per-element column read then leaves the L1 data path
// to the 64-byte table rows, which saturate it.  FL (fast locate, when the aperture's delay spread is within TAY_EXT
// centres, |Delta| df/c G <= TAY_EXT - 0.6: every BASELINE config): per component the fp64 phase base R df/c in
// centres, x G = B_i + B_f (B_i integer, |B_f| <= 1/2 in fp32) and the sign (-1)^(n0 (N_f - 1)) once; per element
// u = B_f + Delta (df/c) G in one fma, its rounding k by the magic constant, the row B_i + k on the extended table and
// delta' = u - k -- 5 instructions instead of tay_locate's TwoSum reduction, wrap and per-element sign (|u| < 3 keeps
// u's rounding below 1.2e-7 centres).
#ifndef CDMS_CORR_UNROLL
#define CDMS_CORR_UNROLL 8  // antennas per unrolled step (measured c5 4M corr 4: 17.25, 8: 16.91, 16: 17.01 ms)
#endif
constexpr int CORR_UNROLL = CDMS_CORR_UNROLL;
template <bool SPH, bool TC, bool FL>
__global__ void __launch_bounds__(TAY_BLOCK)
    tay_corr_kernel(const __grid_constant__ SceneDev sc, int G, const float2* __restrict__ tab,
                    const float4* __restrict__ tmpl, const double* __restrict__ particles, int64_t P, int pstride,
                    const double* __restrict__ sfv, int sfv_pp, float2* __restrict__ terms, int* __restrict__ pflag,
                    int gram_diag, const __grid_constant__ TmplC tc) {
  const int J = sc.J, S = sc.S, Na = sc.Na, T = S + S * (S + 1) / 2;
  const int64_t p = (int64_t)blockIdx.x * TAY_BLOCK + threadIdx.x;
  const int j = blockIdx.y;
  if (p >= P) return;
  const int Na_pad = sc.n_mb * NWARP;
  const double* pos = particles + p * pstride;
  // thread layout: 32-byte rows of C_0..C_3 (2 float4) in A, 16-byte rows of C_4, C_5 (1 float4) in B
  const float4* tA = reinterpret_cast<const float4*>(tab) + (int64_t)j * Na * tay_rows(G) * 2;
  const float4* tB = reinterpret_cast<const float4*>(tab) + (int64_t)J * Na * tay_rows(G) * 2 + (int64_t)j * Na * tay_rows(G);
  const float4* tm = tmpl + (int64_t)j * Na_pad;
  constexpr bool sph = SPH;
  const float dfG = (float)(sc.df_c * (double)G);  // FL: centres per metre of delay offset
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
    const TayBase tb = tay_base(R64 * sc.df_c);  // delay phase base
    float Bf = 0.f;  // FL: the base in centres, B_i + B_f, and its period's sign
    uint32_t gbase = 0;
    bool cflip = false;
    if (FL) {
      const double phib = R64 * sc.df_c, n0 = rint(phib), X = (phib - n0) * (double)G, Bi = rint(X);
      Bf = (float)(X - Bi);
      gbase = (uint32_t)((int)Bi + G / 2 + TAY_EXT);
      cflip = (sc.nf & 1) == 0 && ((long long)n0 & 1);
    }
    double sb, cb;
    sincospi(2.0 * frac_c(R64 * sc.fc_c), &sb, &cb);
    // an antenna distance can vanish only within the aperture (R <= ap_r): that rare case is checked apart
    if (sph && !(R64 > sc.ap_r))
      for (int m = 0; m < Na; ++m) {
        const float4 v = __ldg(&tm[m]);
        if (!(Num<float>::fsqrt_(R * R + v.w - 2.f * (hx * v.x + hy * v.y + hz * v.z)) > 0.f)) fl |= 1;
      }
    double accr = 0.0, acci = 0.0;  // sum_m e^{j2pi f_c Delta_m/c} Y_m; times e^{j2pi f_c R/c} (cb, sb) at the end
    for (int m0 = 0; m0 < Na; m0 += 16) {
      float pr = 0.f, pi = 0.f;
      const int m1 = min(m0 + 16, Na);
#pragma unroll CORR_UNROLL
      for (int m = m0; m < m1; ++m) {
        const float4 v = TC ? tc.v[j * Na_pad + m] : __ldg(&tm[m]);
        const float rq = hx * v.x + hy * v.y + hz * v.z;
        float delta;
        if (sph) {
          const float n = v.w - 2.f * rq;
          const float d = Num<float>::fsqrt_(R * R + n);  // approximate: no IEEE slow-path call in the loop
          delta = Num<float>::fdiv_(n, d + R);
        } else {
          delta = Num<float>::fdiv_(-rq, R);
        }
        float er, ei;
        carrier_f(delta, sc.fc2pi_f, er, ei);
        uint32_t g;
        float dp;
        bool flip = false;
        if (FL) {
          const float u = fmaf(delta, dfG, Bf), um = u + TAY_MAGIC;
          g = gbase + (uint32_t)(__float_as_int(um) - __float_as_int(TAY_MAGIC));
          dp = u - (um - TAY_MAGIC);
        } else {
          tay_locate(delta * sc.df_cf, tb.hi, tb.lo, tb.par, G / 2, (float)G, (sc.nf & 1) == 0, g, dp, flip);
        }
        const uint32_t row = (uint32_t)m * (uint32_t)tay_rows(G) + g;
        float4 c01, c23;
        ldg256(tA + 2u * row, c01, c23);
        const float4 c45 = __ldg(tB + row);
        float yr = c45.z, yi = c45.w;  // Horner in delta', l = 5 .. 0
        yr = fmaf(yr, dp, c45.x); yi = fmaf(yi, dp, c45.y);
        yr = fmaf(yr, dp, c23.z); yi = fmaf(yi, dp, c23.w);
        yr = fmaf(yr, dp, c23.x); yi = fmaf(yi, dp, c23.y);
        yr = fmaf(yr, dp, c01.z); yi = fmaf(yi, dp, c01.w);
        yr = fmaf(yr, dp, c01.x); yi = fmaf(yi, dp, c01.y);
        if (!FL && flip) { yr = -yr; yi = -yi; }
        pr = fmaf(er, yr, fmaf(-ei, yi, pr));
        pi = fmaf(er, yi, fmaf(ei, yr, pi));
      }
      accr += (double)pr;
      acci += (double)pi;
    }
    if (cflip) {
      accr = -accr;
      acci = -acci;
    }
    const double gn = sc.pathloss ? sc.lambda / (4.0 * PI * R64) : 1.0;
    terms[term_idx(p, j, s, T, P)] = term_f2((accr * cb - acci * sb) * gn, (accr * sb + acci * cb) * gn);
    const int grow = S + s * (s + 1) / 2;  // row s of the lower triangle of G
    terms[term_idx(p, j, grow + s, T, P)] = term_f2((double)sc.nf * (double)Na * gn * gn, 0.0);  // G_ss = g^2 N_z
    if (gram_diag)  // callers that use c only: no off-diagonal Gram
      for (int c = 0; c < s; ++c) terms[term_idx(p, j, grow + c, T, P)] = term_f2(0.0, 0.0);
  }
  if (fl) atomicOr(&pflag[p], fl);
}

// c_s with antennas across groups of LP = 2^lg lanes: for one component the phases of all antennas lie within a few
// table centres, so with the [g][h][m] layout (32-byte entries) a group's gathers are (nearly) contiguous.  A warp owns npw = floor(32/S)
// particles; lane i < npw S runs the fp64 set-up of pair i = (particle i / S, component i % S); the 32/LP groups then
// take pairs i0 + group, each lane a strided subset of the antennas, and a fixed-order tree inside the group sums them.
template <int EPL, bool FL>  // FL: fast locate as tay_corr_kernel  // antennas per lane (ceil(N_a / LP)), 0: runtime loop
__global__ void __launch_bounds__(TAY_BLOCK)
    tay_corr_lanes_kernel(const __grid_constant__ SceneDev sc, int G, const float2* __restrict__ tab,
                          const float4* __restrict__ tmpl, const double* __restrict__ particles, int64_t P,
                          int pstride, const double* __restrict__ sfv, int sfv_pp, float2* __restrict__ terms,
                          int* __restrict__ pflag, int gram_diag, int lg) {
  const int lane = threadIdx.x & 31;
  const int S = sc.S, Na = sc.Na, T = S + S * (S + 1) / 2;
  const int npw = 32 / S, LP = 1 << lg, ng = 32 >> lg;
  const int grp = lane >> lg, gl = lane & (LP - 1);
  const int64_t p0 = ((int64_t)blockIdx.x * (TAY_BLOCK / 32) + (threadIdx.x >> 5)) * npw;
  const int j = blockIdx.y;
  if (p0 >= P) return;  // warp-uniform
  const int npairs = (int)min((int64_t)npw, P - p0) * S;
  const float4* tj = reinterpret_cast<const float4*>(tab) + (int64_t)j * tay_rows(G) * (TAY_L / 2) * Na;
  const uint32_t rstride = (uint32_t)(TAY_L / 2) * (uint32_t)Na;  // float4s per centre ([h][m] of 32-byte entries)
  const float4* tm = tmpl + (int64_t)j * sc.n_mb * NWARP;
  const bool sph = sc.wavefront == CDMS_SPHERICAL;
  float hx = 1.f, hy = 0.f, hz = 0.f, R = 1.f;
  double Ebr = 1.0, Ebi = 0.0;  // e^{j2pi f_c R/c}, applied to the antenna sum at the end
  float bhi = 0.f, blo = 0.f;
  int bpar = 0;
  float Bf = 0.f;      // FL: base in centres (fraction) and its row, the period sign; near: R <= ap_r
  int gbase = 0;
  bool cflip = false, near = false;
  const float dfG = (float)(sc.df_c * (double)G);
  double gn = 1.0;
  int ok = 0;
  if (lane < npairs) {
    const int64_t p = p0 + lane / S;
    const int s = lane % S;
    const double* pos = particles + p * pstride;
    const double* sfv_s = s == 0 ? nullptr : (sfv_pp ? sfv + (p * sc.K + (s - 1)) * 3 : sfv + (int64_t)(s - 1) * 3);
    double va[3], sh[3];
    int fl = 0;
    if (!anchor_va(sc, j, sfv_s, va, sh)) {
      fl = 2;
    } else {
      const double r0 = pos[0] - va[0], r1 = pos[1] - va[1], r2 = pos[2] - va[2];
      const double rs2 = 2.0 * (r0 * sh[0] + r1 * sh[1] + r2 * sh[2]);
      const double R64 = sqrt(r0 * r0 + r1 * r1 + r2 * r2);
      if (!(R64 > 0.0)) {
        fl = 1;
      } else {
        hx = (float)(r0 - rs2 * sh[0]); hy = (float)(r1 - rs2 * sh[1]); hz = (float)(r2 - rs2 * sh[2]);
        R = (float)R64;
        const TayBase tb = tay_base(R64 * sc.df_c);
        bhi = tb.hi; blo = tb.lo; bpar = tb.par;
        if (FL) {
          const double phib = R64 * sc.df_c, n0 = rint(phib), X = (phib - n0) * (double)G, Bi = rint(X);
          Bf = (float)(X - Bi);
          gbase = (int)Bi + G / 2 + TAY_EXT;
          cflip = (sc.nf & 1) == 0 && ((long long)n0 & 1);
          near = !(R64 > sc.ap_r);
        }
        double sb, cb;
        sincospi(2.0 * frac_c(R64 * sc.fc_c), &sb, &cb);
        Ebr = cb; Ebi = sb;
        gn = sc.pathloss ? sc.lambda / (4.0 * PI * R64) : 1.0;
        ok = 1;
      }
    }
    if (fl) atomicOr(&pflag[p], fl);
  }
  float4 vt[EPL > 0 ? EPL : 1];  // this lane's antenna templates, loaded once for all pairs
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    const int m = gl + (e << lg);
    vt[e] = m < Na ? __ldg(&tm[m]) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float cr = 0.f, ci = 0.f;  // lane i: pair i's correlation once reduced
  for (int i0 = 0; i0 < npairs; i0 += ng) {
    const int i = i0 + grp;  // this group's pair
    const int src = min(i, 31);
    const int pok = __shfl_sync(0xffffffffu, ok, src) && i < npairs;
    const float shx = __shfl_sync(0xffffffffu, hx, src), shy = __shfl_sync(0xffffffffu, hy, src);
    const float shz = __shfl_sync(0xffffffffu, hz, src), sR = __shfl_sync(0xffffffffu, R, src);
    float shi = 0.f, slo = 0.f, sBf = 0.f;
    int spar = 0, sgb = 0, snear = 1;
    if (FL) {
      sBf = __shfl_sync(0xffffffffu, Bf, src);
      sgb = __shfl_sync(0xffffffffu, gbase, src);
      snear = __shfl_sync(0xffffffffu, (int)near, src);
    } else {
      shi = __shfl_sync(0xffffffffu, bhi, src);
      slo = __shfl_sync(0xffffffffu, blo, src);
      spar = __shfl_sync(0xffffffffu, bpar, src);
    }
    float pr = 0.f, pi = 0.f;
    int efl = 0;
    auto element = [&](int m, const float4 v) {
      const float rq = shx * v.x + shy * v.y + shz * v.z;
      float delta;
      if (sph) {
        const float n = v.w - 2.f * rq;
        const float d = Num<float>::fsqrt_(sR * sR + n);
        if (snear && !(d > 0.f)) efl = 1;  // FL: only pairs within the aperture can hit an antenna
        delta = Num<float>::fdiv_(n, d + sR);
      } else {
        delta = Num<float>::fdiv_(-rq, sR);
      }
      float er, ei;
      carrier_f(delta, sc.fc2pi_f, er, ei);
      uint32_t g;
      float dp;
      bool flip = false;
      if (FL) {
        const float u = fmaf(delta, dfG, sBf), um = u + TAY_MAGIC;
        g = (uint32_t)(sgb + (__float_as_int(um) - __float_as_int(TAY_MAGIC)));
        dp = u - (um - TAY_MAGIC);
      } else {
        tay_locate(delta * sc.df_cf, shi, slo, spar, G / 2, (float)G, (sc.nf & 1) == 0, g, dp, flip);
      }
      const float4* row = tj + (g * rstride + 2u * (uint32_t)m);
      float4 c01, c23, c45, c67;
      ldg256(row, c01, c23);
      ldg256(row + 2 * Na, c45, c67);
      float yr = c67.z, yi = c67.w;
      yr = fmaf(yr, dp, c67.x); yi = fmaf(yi, dp, c67.y);
      yr = fmaf(yr, dp, c45.z); yi = fmaf(yi, dp, c45.w);
      yr = fmaf(yr, dp, c45.x); yi = fmaf(yi, dp, c45.y);
      yr = fmaf(yr, dp, c23.z); yi = fmaf(yi, dp, c23.w);
      yr = fmaf(yr, dp, c23.x); yi = fmaf(yi, dp, c23.y);
      yr = fmaf(yr, dp, c01.z); yi = fmaf(yi, dp, c01.w);
      yr = fmaf(yr, dp, c01.x); yi = fmaf(yi, dp, c01.y);
      if (!FL && flip) { yr = -yr; yi = -yi; }
      pr = fmaf(er, yr, fmaf(-ei, yi, pr));
      pi = fmaf(er, yi, fmaf(ei, yr, pi));
    };
    if (EPL > 0) {
#pragma unroll
      for (int e = 0; e < (EPL > 0 ? EPL : 1); ++e)
        if (pok && gl + (e << lg) < Na) element(gl + (e << lg), vt[e]);
    } else {
      for (int m = pok ? gl : Na; m < Na; m += LP) element(m, __ldg(&tm[m]));
    }
    for (int o = LP >> 1; o > 0; o >>= 1) {  // fixed-order tree inside the group
      pr += __shfl_xor_sync(0xffffffffu, pr, o);
      pi += __shfl_xor_sync(0xffffffffu, pi, o);
    }
    // pair i0 + k's sum sits in group k: lane i0 + k, which holds that pair's set-up, takes it
    const int from = min(max(lane - i0, 0), ng - 1) << lg;
    const float tr = __shfl_sync(0xffffffffu, pr, from), ti = __shfl_sync(0xffffffffu, pi, from);
    if (lane >= i0 && lane < i0 + ng) {
      cr = tr;
      ci = ti;
    }
    if (efl) atomicOr(&pflag[p0 + i / S], efl);
  }
  if (lane < npairs && ok) {  // one store round per warp: lane i writes pair i's c_s, G_ss (and zero off-diagonals)
    const int64_t p = p0 + lane / S;
    const int s = lane % S;
    if (cflip) {  // FL: the period's sign, once per pair
      cr = -cr;
      ci = -ci;
    }
    terms[term_idx(p, j, s, T, P)] =
        term_f2(((double)cr * Ebr - (double)ci * Ebi) * gn, ((double)cr * Ebi + (double)ci * Ebr) * gn);
    const int r0 = S + s * (s + 1) / 2;
    terms[term_idx(p, j, r0 + s, T, P)] = term_f2((double)sc.nf * (double)Na * gn * gn, 0.0);
    if (gram_diag)
      for (int c = 0; c < s; ++c) terms[term_idx(p, j, r0 + c, T, P)] = term_f2(0.0, 0.0);
  }
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
// D_N(x) for |x| <= ~0.56 without reducing x (FAST Gram path): the pair's integer part nb is taken out once per pair
// in fp64 (its sign (-1)^{nb (N - 1)} applied to the pair total) and the per-antenna offset e = dd df/c is small
// (sc.small_step >= 1: |e| <= 0.064), so x = xb + e stays inside the validity range of the denominator polynomial
// sin(pi x) = u S(u^2), u = pi x, S to u^10 (relative error < 1e-6 at 0.56, < 6e-8 at 0.52).  Numerator sin(pi t),
// t = N x reduced mod 2: MUFU, or for |t| <= 1/4 the odd polynomial (dirichlet_num's reasoning); at x = 0 D = N.
__device__ __forceinline__ float dirichlet_fast(float x, float Nf) {
  constexpr float M = 12582912.f;
  float t = Nf * x;
  t = fmaf(-2.f, (fmaf(0.5f, t, M) - M), t);
  const float u = 3.14159265358979f * x, u2 = u * u;
  const float den = u * fmaf(u2, fmaf(u2, fmaf(u2, fmaf(u2, fmaf(u2, -1.f / 39916800, 1.f / 362880), -1.f / 5040),
                                                1.f / 120), -1.f / 6), 1.f);
  // branch-free (selects): a divergent branch per (pair, antenna) fences the fully unrolled pair loop into serial
  // pieces and costs its ILP (measured: c5 Gram 280 -> 310 ms with the branch)
  const float z = 3.14159265358979f * t, z2 = z * z;
  const float ps = z * fmaf(z2, fmaf(z2, fmaf(z2, fmaf(z2, 1.f / 362880, -1.f / 5040), 1.f / 120), -1.f / 6), 1.f);
  const float num = fabsf(t) <= 0.25f ? ps : __sinf(z);
  const float D = num * rcp_approx(den);
  return fabsf(x) < 1e-30f ? Nf : D;
}
// Pairs q in [Q0, Q1) (row order (0,1), (0,2), ..., (1,2), ...): large S splits the pairs over blockIdx.z so each
// thread holds only its part's accumulators (S = 9: 255 registers and 73 KB of totals per block for all 36 pairs).
// FAST (sc.small_step >= 1, every BASELINE config): per pair the fp64 delay base (R_a - R_b) df/c = nb + xb is reduced
// once (xb in registers, nb's sign at the end) and per antenna D = dirichlet_fast(xb + dd df/c): no per-antenna
// range reduction or parity bookkeeping.  Else per antenna gram_dirichlet_f (reduction and parity per term).
// TAB (FAST with the scene's Dirichlet table, dn_table_kernel): D_N from per-centre Taylor coefficients instead of the
// sine quotient -- one table row and a short Horner per (pair, antenna), no MUFU, no reciprocal, and the function is
// entire, so near-equal delays need no special case.  Centres x_r = r / G_D; per pair the fp64 base x_b G_D = g_b + r_b
// (|r_b| <= 1/2), per antenna d' = r_b + dd (df/c) G_D, its rounding g2 and the offset d = d' - g2 (|d| <= 1/2; with
// CDMS_GRAM_UCOMP 2, the default, the rounding is per component and |d| <= 1), all fp32-exact enough.  The row is kept
// at 16 bytes: degree 3 at G_D = 64 N (truncation below N (pi N |d|max / G_D)^4 / 4! = N (pi/64)^4/24 = 2.4e-7 N per
// term at |d| <= 1; round 2's per-pair rounding ran 32 N at |d| <= 1/2, the same bound), |x| <= 0.6 (FAST:
// |x| <= 0.564), both signs stored (1.26 MB at N_f = 1024, L2-resident;
// the even-symmetric half-table, -DCDMS_DN_SYM, costs a mirror per term: measured c5 Gram 49.3 vs 46.8 ms,
// profiles/r02_dn_table.txt).  Against round 2's first table (degree 7 at 8 N, 32-byte rows, -DCDMS_DN_DEG7 for A/B)
// the 4 Horner steps fewer per (pair, antenna) took the c5 Gram from 55.9 to 49.3 ms.
struct GramTab {
  const float4* dn;  // [rows][DN_L / 4] float4 of real coefficients per centre
  float G;           // centres per unit x
  int R0;            // row of x = 0
};
#ifdef CDMS_DN_DEG7
constexpr int DN_L = 8, DN_DENS = 8;
constexpr bool DN_SYM = false;
#else
#ifndef CDMS_DN_DENS
#define CDMS_DN_DENS 64
#endif
constexpr int DN_L = 4, DN_DENS = CDMS_DN_DENS;
#ifdef CDMS_DN_SYM
constexpr bool DN_SYM = true;
#else
constexpr bool DN_SYM = false;
#endif
#endif
int dn_centres(int nf) { return DN_DENS * nf; }
int dn_rows(int nf) {
  const int h = (int)ceil(0.6 * dn_centres(nf));
  return DN_SYM ? h + 2 : 2 * h + 1;
}
int dn_r0(int nf) { return DN_SYM ? 0 : (dn_rows(nf) - 1) / 2; }
// C_l(r) = D_N^{(l)}(x_r) / l! / G_D^l = sum_kappa cos(2 pi kappa x_r + l pi/2) (2 pi kappa / G_D)^l / l!, kappa = k - k0
// (D_N(x) = sum_k e^{j2pi (k - k0) x} is real and even); fp64, exact integer reduction of 2 kappa (r - R0) mod 2 G_D.
__global__ void dn_table_kernel(int N, int GD, int R0, int rows, float* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * DN_L) return;
  const int r = i / DN_L, l = i - r * DN_L;
  const int64_t rs = r - R0;
  double f = 1.0;
  double acc = 0.0;
  for (int k = 0; k < N; ++k) {
    const int twok = 2 * k - (N - 1);  // 2 kappa, an integer
    int64_t num = ((int64_t)twok * rs) % (2 * (int64_t)GD);  // 2 kappa x_r = num / G_D (mod 2)
    double s, c;
    sincospi((double)num / (double)GD, &s, &c);
    const double w = PI * (double)twok / (double)GD;  // 2 pi kappa / G_D
    f = 1.0;
    for (int q = 1; q <= l; ++q) f *= w / (double)q;
    const double tr = (l & 3) == 0 ? c : (l & 3) == 1 ? -s : (l & 3) == 2 ? -c : s;  // cos(theta + l pi/2)
    acc += tr * f;
  }
  out[i] = (float)acc;
}
size_t dn_table_floats(int nf) { return (size_t)dn_rows(nf) * DN_L; }
cudaError_t launch_dn_table(int nf, float* out, cudaStream_t st) {
  const int GD = dn_centres(nf), rows = dn_rows(nf), R0 = dn_r0(nf);
  const int n = rows * DN_L;
  dn_table_kernel<<<(n + 127) / 128, 128, 0, st>>>(nf, GD, R0, rows, out);
  return cudaGetLastError();
}

// TAB per-antenna offsets (A/B: -DCDMS_GRAM_UCOMP=1 or 0): 2 rounds u_s = k_s + r_s once per (component, antenna), so a
// pair needs r_a - r_b (|.| <= 1 centre) and k_a - k_b; 1 rounds d' = u_a - u_b per pair (|d| <= 1/2); 0 holds one
// fractional base per pair.  The |d| <= 1 of 2 is why the table is at G_D = 64 N (the truncation bound of 32 N at
// |d| <= 1/2); measured c5 4M Gram 44.7 -> 43.6 ms, c4 3.09 -> 2.67 ms with 2 (profiles/r02_gram_onechunk.txt)
#ifndef CDMS_GRAM_UCOMP
#define CDMS_GRAM_UCOMP 2
#endif
#ifndef CDMS_GRAM_CHUNK
#define CDMS_GRAM_CHUNK 16  // antennas per fp32 partial sum (measured 4 / 8 / 16: c5 4M Gram 49.1 / 46.8 / 45.5 ms, G parity 5.5e-7 of N_z at 16)
#endif
#ifndef CDMS_GRAM_ONE_MAX
#define CDMS_GRAM_ONE_MAX 64  // lanes with at most this many antennas sum them in one fp32 pass (no fp64 totals)
#endif
// ONE (TAB, at most CDMS_GRAM_ONE_MAX antennas per lane): the pair sums stay in fp32 registers over all the lane's
// antennas (a single chunk) and the block needs no fp64 totals in shared memory -- with (hx, hy, hz, R) parked there
// too, 128 registers and 4 blocks (16 warps) per SM at S >= 7.  Measured c5 4M Gram 43.6 -> 38.4 ms, c3 2.84 ->
// 2.53 ms; one fp32 sum of 64 terms against 4 of 16 moved the K1T terms' worst G error within the parity bounds
// (profiles/r02_gram_onechunk.txt).
// W0 (TAB and ONE only): every pair's base has W = rint((R_a - R_b) df/c) = 0 (path differences below half of c/df:
// 300 m at c5), so a pair's table row is R0 + (k_a + I_a) - (k_b + I_b) from per-component integers and no per-pair
// base row is held (36 registers at S = 9: its main-loop spills 116 -> 48 bytes, c5 4M Gram 33.1 -> 32.0 ms).  A
// particle with some W != 0 sets *wflag, and the W0 = false kernel launched after it then recomputes the batch (it
// returns at once while *wflag is 0).
template <int S, int Q0, int Q1, bool FAST, bool TAB, bool ONE, bool W0>
__device__ __forceinline__ void tay_gram_part(const SceneDev& sc, const float4* __restrict__ tmpl,
                                              const double* __restrict__ particles, int64_t P, int pstride,
                                              const double* __restrict__ sfv, int sfv_pp, float2* __restrict__ terms,
                                              int lsplit, double2* gsum, double* rsh, float4* csh,
                                              const GramTab tb, int* __restrict__ wflag, int64_t bx) {
  constexpr int NP = Q1 - Q0;  // this part's pairs; gsum [NP][TAY_BLOCK] (not ONE)
  // A = 2^lsplit adjacent lanes per particle, lane a takes antennas a, a + A, ... (A > 1 when P J threads alone would
  // leave the SMs latency-bound); no early exit: the group's fp64 totals are combined by shuffles below
  const int A = 1 << lsplit;
  const int64_t t = bx * TAY_BLOCK + threadIdx.x;  // bx: the block's tile (blockIdx.x, or the fallback's loop)
  const int64_t p = t >> lsplit;
  const int a0 = (int)(t & (A - 1));
  const int j = blockIdx.y;
  const int Na = sc.Na, T = S + S * (S + 1) / 2;
  bool live = p < P;
  const double* pos = particles + (live ? p : 0) * pstride;
  float hx[S], hy[S], hz[S], Rf[S], uh[S], ul[S];
  double R64[S];
  int npar[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const double* sfv_s = s == 0 ? nullptr : (sfv_pp ? sfv + ((live ? p : 0) * sc.K + (s - 1)) * 3 : sfv + (int64_t)(s - 1) * 3);
    if (!tay_component(sc, j, pos, sfv_s, hx[s], hy[s], hz[s], R64[s])) live = false;  // flagged by K1T
    if (!live) R64[s] = 1.0;
    Rf[s] = (float)R64[s];
    if (!FAST) {
      const double xs = R64[s] * sc.df_c, ns = rint(xs), us = xs - ns;
      uh[s] = (float)us;
      ul[s] = (float)(us - (double)uh[s]);
      npar[s] = (int)((long long)ns & 1);
    }
  }
  // FAST: per pair the centred fraction of (R_a - R_b) df/c (fp64 difference, one rounding).  TAB with UCOMP: per
  // component C_s = R_s (df/c) G_D = I_s + f_s (fp64, |f_s| <= 1/2 in fp32) and per pair only the integer row
  // gb = I_a - I_b - W G_D + R0 (W = rint((R_a - R_b) df/c) periods); per antenna u_s = f_s + Delta_s (df/c) G_D once
  // per component and d' = u_a - u_b per pair -- one float per component instead of one per pair held in registers
  float xb[(FAST && !(TAB && CDMS_GRAM_UCOMP)) ? NP : 1];
  float fc_[(TAB && CDMS_GRAM_UCOMP) ? S : 1];
  int gb[(TAB && !W0) ? NP : 1];  // TAB: the centre row of x_b G_D (offset by R0)
  int Iq[W0 ? S : 1];             // W0: I_s, added to the per-antenna row k_s
  if (W0) {
    bool wz = true;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const double C = R64[s] * sc.df_c * (double)tb.G, I = rint(C);
      fc_[s] = (float)(C - I);
      Iq[W0 ? s : 0] = (int)I;
    }
#pragma unroll
    for (int a = 0; a < S; ++a)
#pragma unroll
      for (int b = 0; b < S; ++b)
        if (b > a) wz &= rint((R64[a] - R64[b]) * sc.df_c) == 0.0;
    if (!wz && live) atomicOr(wflag, 1);  // this batch is recomputed by the W0 = false kernel
  } else if (TAB && CDMS_GRAM_UCOMP) {
    double Ic[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const double C = R64[s] * sc.df_c * (double)tb.G;
      Ic[s] = rint(C);
      fc_[s] = (float)(C - Ic[s]);
    }
#pragma unroll
    for (int a = 0; a < S; ++a)
#pragma unroll
      for (int b = 0; b < S; ++b) {
        if (b <= a) continue;
        const int q = a * (2 * S - a - 1) / 2 + (b - a - 1) - Q0;
        if (q < 0 || q >= NP) continue;
        const double W = rint((R64[a] - R64[b]) * sc.df_c);
        gb[(TAB && !W0) ? q : 0] = (int)(Ic[a] - Ic[b] - W * (double)tb.G) + tb.R0;
      }
  } else if (FAST) {
#pragma unroll
    for (int a = 0; a < S; ++a)
#pragma unroll
      for (int b = 0; b < S; ++b) {
        if (b <= a) continue;
        const int q = a * (2 * S - a - 1) / 2 + (b - a - 1) - Q0;
        if (q < 0 || q >= NP) continue;
        const double x = frac_c((R64[a] - R64[b]) * sc.df_c);
        if (TAB) {
          const double xg = x * (double)tb.G, g = rint(xg);
          gb[(TAB && !W0) ? q : 0] = (int)g + tb.R0;
          xb[q] = (float)(xg - g);
        } else {
          xb[q] = (float)x;
        }
      }
  }
  // R_s (fp64) are needed again only in the epilogue: parked in shared memory, not in registers through the loop
  // (18 registers at S = 9, which removed the kernel's spills under its 168-register cap)
  // TAB: per component (h'_y, h'_z, R, f_s) parked in shared memory, h' = R_j^T h, so that h.v_m = h'_y p~_y +
  // h'_z p~_z against the PA-independent template row (p~ = (0, p~_y, p~_z)): two products per
  // (component, antenna) instead of three, and f_s out of the registers
  const double* Rj = sc.pa_rot[j];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    rsh[s * TAY_BLOCK + threadIdx.x] = R64[s];
    if (TAB) {
      const float hyp = (float)((double)hx[s] * Rj[1] + (double)hy[s] * Rj[4] + (double)hz[s] * Rj[7]);
      const float hzp = (float)((double)hx[s] * Rj[2] + (double)hy[s] * Rj[5] + (double)hz[s] * Rj[8]);
      csh[s * TAY_BLOCK + threadIdx.x] = make_float4(hyp, hzp, Rf[s], fc_[(TAB && CDMS_GRAM_UCOMP) ? s : 0]);
    }
  }
  const float dfG = sc.df_cf * tb.G;  // TAB: d' per unit of the element offset difference
#pragma unroll
  for (int q = 0; q < NP; ++q)
    if (!ONE) gsum[q * TAY_BLOCK + threadIdx.x] = make_double2(0.0, 0.0);
  const bool sph = sc.wavefront == CDMS_SPHERICAL;
  const float4* tm = tmpl + (TAB ? (int64_t)sc.J : (int64_t)j) * sc.n_mb * NWARP;  // TAB: (p~_y, p~_z, ||p~||^2)
  const int Nl = live ? (Na - a0 + A - 1) >> lsplit : 0;  // this lane's antennas m = a0 + A i, i < Nl
  float gr[NP], gi[NP];
#pragma unroll
  for (int q = 0; q < NP; ++q) gr[q] = gi[q] = 0.f;
  const int chunk = ONE ? Nl : CDMS_GRAM_CHUNK;
  for (int i0 = 0; i0 < Nl; i0 += chunk) {  // fp32 partial sums over a chunk, then fp64
    if (!ONE && i0 > 0) {
#pragma unroll
      for (int q = 0; q < NP; ++q) gr[q] = gi[q] = 0.f;
    }
    const int i1 = min(i0 + chunk, Nl);
    for (int i = i0; i < i1; ++i) {
      const int m = a0 + (i << lsplit);
      const float4 v = __ldg(&tm[m]);
      float dl[S], er[S], ei[S];
      int ik[(TAB && CDMS_GRAM_UCOMP == 2) ? S : 1];  // UCOMP 2: u_s = k_s + r_s, k_s as the bits of k_s + M
#pragma unroll
      for (int s = 0; s < S; ++s) {
        float rq, Rs, q2;
        if (TAB) {
          const float4 h = csh[s * TAY_BLOCK + threadIdx.x];
          rq = fmaf(h.x, v.x, h.y * v.y);
          Rs = h.z;
          q2 = v.z;
        } else {
          rq = hx[s] * v.x + hy[s] * v.y + hz[s] * v.z;
          Rs = Rf[s];
          q2 = v.w;
        }
        if (sph) {
          const float n = q2 - 2.f * rq;
          dl[s] = Num<float>::fdiv_(n, Num<float>::fsqrt_(Rs * Rs + n) + Rs);
        } else {
          dl[s] = Num<float>::fdiv_(-rq, Rs);  // planar WB only: no 1/R array held through the loop
        }
        carrier_f(dl[s], sc.fc2pi_f, er[s], ei[s]);  // e^{j2pi f_c Delta_s/c}: the pairs' carriers as products
        if (TAB && CDMS_GRAM_UCOMP) dl[s] = fmaf(dl[s], dfG, csh[s * TAY_BLOCK + threadIdx.x].w);  // u_s, in centres
        if (TAB && CDMS_GRAM_UCOMP == 2) {  // rounded per component: per pair r_a - r_b (|.| <= 1) and k_a - k_b
          constexpr float M = 12582912.f;
          const float um = dl[s] + M;
          ik[(TAB && CDMS_GRAM_UCOMP == 2) ? s : 0] = __float_as_int(um) + (W0 ? Iq[W0 ? s : 0] : 0);
          dl[s] = dl[s] - (um - M);
        }
      }
#pragma unroll
      for (int a = 0; a < S; ++a) {  // constant trip counts: both loops unroll fully, the arrays stay in registers
#pragma unroll
        for (int b = 0; b < S; ++b) {
          if (b <= a) continue;
          const int q = a * (2 * S - a - 1) / 2 + (b - a - 1) - Q0;
          if (q < 0 || q >= NP) continue;
          float D;
          if (TAB) {
            constexpr float M = 12582912.f;
            const float d1 = (TAB && CDMS_GRAM_UCOMP) ? dl[a] - dl[b]  // offset from the pair's base row, in centres
                                                      : fmaf(dl[a] - dl[b], dfG, xb[(FAST && !(TAB && CDMS_GRAM_UCOMP)) ? q : 0]);
            const float dm = d1 + M;
            float d = d1 - (dm - M);
            int g2 = gb[(TAB && !W0) ? q : 0] + (__float_as_int(dm) - __float_as_int(M));
            if (CDMS_GRAM_UCOMP == 2) {
              d = d1;
              g2 = (W0 ? tb.R0 : gb[(TAB && !W0) ? q : 0]) + ik[(TAB && CDMS_GRAM_UCOMP == 2) ? a : 0] -
                   ik[(TAB && CDMS_GRAM_UCOMP == 2) ? b : 0];
            }
            if (DN_SYM) {  // D_N even: the row of |x|, the offset mirrored (selects, no branch)
              const bool neg = g2 < 0;
              g2 = neg ? -g2 : g2;
              d = neg ? -d : d;
            }
            if (DN_L == 4) {
              const float4 c = __ldg(tb.dn + g2);
              D = fmaf(fmaf(fmaf(c.w, d, c.z), d, c.y), d, c.x);
            } else {
              float4 c03, c47;
              ldg256(tb.dn + 2 * g2, c03, c47);
              D = fmaf(fmaf(fmaf(fmaf(fmaf(fmaf(fmaf(c47.w, d, c47.z), d, c47.y), d, c47.x), d, c03.w), d, c03.z), d,
                            c03.y), d, c03.x);
            }
          } else if (FAST) {
            D = dirichlet_fast(fmaf(dl[a] - dl[b], sc.df_cf, xb[q]), sc.nf_f);
          } else {
            GramPairF gp;
            gp.xbr = (uh[a] - uh[b]) + (ul[a] - ul[b]);
            gp.nbpar = (uint32_t)((npar[a] ^ npar[b]) & 1) << 31;
            D = gram_dirichlet_f(sc, dl[a] - dl[b], gp);
          }
          const float cr = fmaf(er[a], er[b], ei[a] * ei[b]), ci = fmaf(ei[a], er[b], -er[a] * ei[b]);  // E_a conj(E_b)
          gr[q] = fmaf(D, cr, gr[q]);
          gi[q] = fmaf(D, ci, gi[q]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      if (ONE) continue;
      double2 t = gsum[q * TAY_BLOCK + threadIdx.x];
      gsum[q * TAY_BLOCK + threadIdx.x] = make_double2(t.x + (double)gr[q], t.y + (double)gi[q]);
    }
  }
  // TAB: the pair base carriers e^{j2pi (R_a - R_b) f_c/c} as E_a conj(E_b) from the S component phasors (fp64, each
  // from its exactly reduced phase), kept in this thread's now unused (h', R, f) slots: S sincospi instead of one per
  // pair.  Not for the one-part S = 9 kernel: the epilogue's extra live values spilled in its main loop (measured c5 4M
  // Gram 33.1 -> 34.8 ms; c3 2.386 -> 2.341 ms)
  constexpr bool CPH = TAB && !(ONE && S >= 9);
  double2* cph = reinterpret_cast<double2*>(csh);
  if (CPH && live && a0 == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      double sn, cs;
      sincospi(2.0 * frac_c(rsh[s * TAY_BLOCK + threadIdx.x] * sc.fc_c), &sn, &cs);
      cph[s * TAY_BLOCK + threadIdx.x] = make_double2(cs, sn);
    }
  }
#pragma unroll
  for (int a = 0; a < S; ++a) {
#pragma unroll
    for (int b = 0; b < S; ++b) {
      if (b <= a) continue;
      const int q = a * (2 * S - a - 1) / 2 + (b - a - 1) - Q0;
      if (q < 0 || q >= NP) continue;
      double2 acc = ONE ? make_double2((double)gr[q], (double)gi[q]) : gsum[q * TAY_BLOCK + threadIdx.x];
      for (int o = 1; o < A; o <<= 1) {  // fixed-order tree over the group's lanes
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
      }
      if (!live || a0 != 0) continue;
      double sn, cs;
      const double Ra = rsh[a * TAY_BLOCK + threadIdx.x], Rb = rsh[b * TAY_BLOCK + threadIdx.x];
      if (CPH) {
        const double2 ea = cph[a * TAY_BLOCK + threadIdx.x], eb = cph[b * TAY_BLOCK + threadIdx.x];
        cs = ea.x * eb.x + ea.y * eb.y;
        sn = ea.y * eb.x - ea.x * eb.y;
      } else {
        sincospi(2.0 * frac_c((Ra - Rb) * sc.fc_c), &sn, &cs);
      }
      double g2 = sc.pathloss ? (sc.lambda / (4.0 * PI * Ra)) * (sc.lambda / (4.0 * PI * Rb)) : 1.0;
      if (FAST && ((sc.nf - 1) & 1)) {  // D_N(nb + x) = (-1)^{nb (N - 1)} D_N(x) (C-amb-13)
        const double d = (Ra - Rb) * sc.df_c;
        if ((long long)rint(d) & 1) g2 = -g2;
      }
      const double vr = cs * acc.x - sn * acc.y, vi = cs * acc.y + sn * acc.x;
      terms[term_idx(p, j, S + b * (b + 1) / 2 + a, T, P)] = term_f2(vr * g2, -vi * g2);
    }
  }
}
// measured: S = 9 in 3 parts 58.8 vs 59.8 ms (c5 shard); S = 7 in 2 parts 9.16 vs 8.87 ms (c3: one part already fits
// 168 registers, splitting only repeats the per-component work)
// S = 9 pair parts over blockIdx.z (A/B: -DCDMS_GRAM_PARTS9=3): with the FAST path's smaller per-component state two
// parts of 18 pairs fit 168 registers; measured (4M c5 particles) Gram 64.1 ms in 2 parts vs 70.7 ms in 3 (each part
// repeats the per-(component, antenna) offsets and carriers)
#ifndef CDMS_GRAM_PARTS9
#define CDMS_GRAM_PARTS9 2
#endif
#ifndef CDMS_GRAM_MINB
#define CDMS_GRAM_MINB 3
#endif
#ifndef CDMS_GRAM_PARTS9_ONE
#define CDMS_GRAM_PARTS9_ONE 1
#endif
// ONE at S = 9: all 36 pairs in one part at 3 blocks per SM (168 registers, a few spilled per antenna) -- the 9
// components' offsets and carriers computed once instead of per part; measured c5 4M Gram 38.0 (2 parts, 4 blocks per
// SM) vs 34.5 ms (1 part, 3 blocks; 2 blocks: 41.2 ms), profiles/r02_gram_onechunk.txt
template <int S, bool ONE>
__host__ __device__ constexpr int tay_gram_parts() {
  return S >= 9 ? (ONE ? CDMS_GRAM_PARTS9_ONE : CDMS_GRAM_PARTS9) : (S == 8 ? 2 : 1);
}
template <int S, bool ONE>
__host__ __device__ constexpr int tay_gram_minb() {
  return S < 7 ? 1 : !ONE ? CDMS_GRAM_MINB : tay_gram_parts<S, ONE>() == 1 && S >= 9 ? 3 : 4;
}
// MODE 0: one tile per block; 1: W0 (see tay_gram_part); 2: the fallback of a W0 launch -- returns at once unless a
// particle had W != 0 (*wflag), else strides over all tiles with a one-wave grid (a separate instantiation: the loop
// costs registers, W0 S = 9 spilled 104 instead of 32 bytes with it)
template <int S, bool FAST, bool TAB, bool ONE, int MODE>
__global__ void __launch_bounds__(TAY_BLOCK, (tay_gram_minb<S, ONE>()))  // S >= 7: 12 or 16 (ONE) warps per SM
    tay_gram_kernel(const __grid_constant__ SceneDev sc, const float4* __restrict__ tmpl,
                    const double* __restrict__ particles, int64_t P, int pstride, const double* __restrict__ sfv,
                    int sfv_pp, float2* __restrict__ terms, int lsplit, const GramTab tb, int* __restrict__ wflag,
                    int64_t ntiles) {
  constexpr bool W0 = MODE == 1;
  if (MODE == 2 && !*(volatile int*)wflag) return;
  constexpr int NP = S * (S - 1) / 2, NPART = tay_gram_parts<S, ONE>(), H = NP / NPART;
  constexpr int NPMAX = NP - NP / NPART * (NPART - 1);  // the larger part
  extern __shared__ double2 smem_g[];
  double* rsh = reinterpret_cast<double*>(smem_g);        // [S][TAY_BLOCK] R_s
  double2* gsum = smem_g + (S * TAY_BLOCK + 1) / 2;       // not ONE: [NPMAX][TAY_BLOCK] fp64 pair totals
  float4* csh = reinterpret_cast<float4*>(gsum + (ONE ? 0 : NPMAX * TAY_BLOCK));  // TAB: [S][TAY_BLOCK]
  for (int64_t bx = blockIdx.x; bx < ntiles; bx += (MODE == 2 ? gridDim.x : ntiles)) {
    if constexpr (NPART == 1) {
      tay_gram_part<S, 0, NP, FAST, TAB, ONE, W0>(sc, tmpl, particles, P, pstride, sfv, sfv_pp, terms, lsplit, gsum, rsh, csh, tb, wflag, bx);
    } else if constexpr (NPART == 2) {
      if (blockIdx.z == 0)
        tay_gram_part<S, 0, H, FAST, TAB, ONE, W0>(sc, tmpl, particles, P, pstride, sfv, sfv_pp, terms, lsplit, gsum, rsh, csh, tb, wflag, bx);
      else
        tay_gram_part<S, H, NP, FAST, TAB, ONE, W0>(sc, tmpl, particles, P, pstride, sfv, sfv_pp, terms, lsplit, gsum, rsh, csh, tb, wflag, bx);
    } else {
      static_assert(NPART == 3, "");
      if (blockIdx.z == 0)
        tay_gram_part<S, 0, H, FAST, TAB, ONE, W0>(sc, tmpl, particles, P, pstride, sfv, sfv_pp, terms, lsplit, gsum, rsh, csh, tb, wflag, bx);
      else if (blockIdx.z == 1)
        tay_gram_part<S, H, 2 * H, FAST, TAB, ONE, W0>(sc, tmpl, particles, P, pstride, sfv, sfv_pp, terms, lsplit, gsum, rsh, csh, tb, wflag, bx);
      else
        tay_gram_part<S, 2 * H, NP, FAST, TAB, ONE, W0>(sc, tmpl, particles, P, pstride, sfv, sfv_pp, terms, lsplit, gsum, rsh, csh, tb, wflag, bx);
    }
  }
}
template <int S, bool FAST, bool TAB, bool ONE, int MODE>
static cudaError_t launch_tay_gram_v(const SceneDev& sc, const float4* tmpl, const double* particles, int64_t P,
                                     int pstride, const double* sfv, int sfv_pp, float2* terms, const GramTab& tb,
                                     int lsplit, int* wflag, cudaStream_t st) {
  constexpr int NP = S * (S - 1) / 2, NPART = tay_gram_parts<S, ONE>();
  const size_t smem = (size_t)(S * TAY_BLOCK + 1) / 2 * sizeof(double2) +                                   // R_s
                      (ONE ? 0 : (size_t)(NP - NP / NPART * (NPART - 1)) * TAY_BLOCK * sizeof(double2)) +  // totals
                      (TAB ? (size_t)S * TAY_BLOCK * sizeof(float4) : 0);                                   // h_s, R_s
  cudaError_t e = cudaFuncSetAttribute(tay_gram_kernel<S, FAST, TAB, ONE, MODE>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t ntiles = ((P << lsplit) + TAY_BLOCK - 1) / TAY_BLOCK;
  int64_t gx = ntiles;
  if (MODE == 2) {  // the fallback: one resident wave
    int per_sm = 1, dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tay_gram_kernel<S, FAST, TAB, ONE, MODE>, TAY_BLOCK, smem);
    gx = std::min<int64_t>(ntiles, (int64_t)std::max(per_sm, 1) * nsm / (sc.J * NPART) + 1);
  }
  dim3 grid((unsigned)gx, sc.J, NPART);
  tay_gram_kernel<S, FAST, TAB, ONE, MODE><<<grid, TAY_BLOCK, smem, st>>>(sc, tmpl, particles, P, pstride, sfv,
                                                                        sfv_pp, terms, lsplit, tb, wflag, ntiles);
  return cudaGetLastError();
}
#ifndef CDMS_GRAM_FAST
#define CDMS_GRAM_FAST 1
#endif
template <int S>
static cudaError_t launch_tay_gram_t(const SceneDev& sc, const float4* tmpl, const double* particles, int64_t P,
                                     int pstride, const double* sfv, int sfv_pp, float2* terms, const float* dn,
                                     int* wflag, cudaStream_t st) {
  const bool fast = CDMS_GRAM_FAST && sc.small_step >= 1;
  GramTab tb;
  tb.dn = reinterpret_cast<const float4*>(dn);
  tb.G = (float)dn_centres(sc.nf);
  tb.R0 = dn_r0(sc.nf);
  // antennas over 2 lanes per particle when P J threads are fewer than ~2 resident waves (measured at c2: 1 lane
  // 0.391, 2 lanes 0.388, 4 lanes 0.405, 8 lanes 0.448 ms per step; at P = 1.4e5 2 lanes 0.494 vs 4 lanes 0.517)
  const int lsplit = (double)P * sc.J < 2.0 * 148 * 1024 ? 1 : 0;
  const bool one = ((sc.Na + (1 << lsplit) - 1) >> lsplit) <= CDMS_GRAM_ONE_MAX;
  // W0 (S = 9, the one-part kernel whose registers it relieves; measured slower at S = 7 and 5 with its fallback
  // launch): the W0 kernel, then its fallback
  if constexpr (S >= 9) {
    if (fast && dn && one && wflag) {
      cudaError_t e = cudaMemsetAsync(wflag, 0, sizeof(int), st);
      if (e == cudaSuccess)
        e = launch_tay_gram_v<S, true, true, true, 1>(sc, tmpl, particles, P, pstride, sfv, sfv_pp, terms, tb, lsplit,
                                                      wflag, st);
      if (e != cudaSuccess) return e;
#ifdef CDMS_GRAM_NO_FALLBACK  // test aid only: shows that a parity case reaches the fallback (it must then fail)
      return cudaSuccess;
#endif
      return launch_tay_gram_v<S, true, true, true, 2>(sc, tmpl, particles, P, pstride, sfv, sfv_pp, terms, tb, lsplit,
                                                       wflag, st);
    }
  }
  if (fast && dn && one)
    return launch_tay_gram_v<S, true, true, true, 0>(sc, tmpl, particles, P, pstride, sfv, sfv_pp, terms, tb, lsplit,
                                                     nullptr, st);
  if (fast && dn)
    return launch_tay_gram_v<S, true, true, false, 0>(sc, tmpl, particles, P, pstride, sfv, sfv_pp, terms, tb, lsplit,
                                                      nullptr, st);
  if (fast)
    return launch_tay_gram_v<S, true, false, false, 0>(sc, tmpl, particles, P, pstride, sfv, sfv_pp, terms, tb, lsplit,
                                                       nullptr, st);
  return launch_tay_gram_v<S, false, false, false, 0>(sc, tmpl, particles, P, pstride, sfv, sfv_pp, terms, tb, lsplit,
                                                      nullptr, st);
}
// kernel launches one launch_tay_gram call makes (the W0 kernel and its fallback at S = 9 with the table)
int tay_gram_launches(const SceneDev& sc, int64_t P, bool tab) {
  if (P <= 0 || sc.S < 2) return 0;
  const int lsplit = (double)P * sc.J < 2.0 * 148 * 1024 ? 1 : 0;
  const bool one = ((sc.Na + (1 << lsplit) - 1) >> lsplit) <= CDMS_GRAM_ONE_MAX;
  return (tab && one && sc.S >= 9 && sc.small_step >= 1 && CDMS_GRAM_FAST) ? 2 : 1;
}
cudaError_t launch_tay_gram(const SceneDev& sc, const float4* tmpl, const double* particles, int64_t P, int pstride,
                            const double* sfv, int sfv_pp, float2* terms, const float* dn, int* wflag,
                            cudaStream_t st) {
  if (P <= 0) return cudaSuccess;
  switch (sc.S) {
    case 1: return cudaSuccess;
#define CASE_S(n) \
  case n: return launch_tay_gram_t<n>(sc, tmpl, particles, P, pstride, sfv, sfv_pp, terms, dn, wflag, st);
    CASE_S(2) CASE_S(3) CASE_S(4) CASE_S(5) CASE_S(6) CASE_S(7) CASE_S(8) CASE_S(9)
#undef CASE_S
    default: return cudaErrorInvalidValue;
  }
}

// Layout / kernel choice (measured, profiles/r01_k1t_lanes.txt, CDMS_TAY_LANES=0/1 A/B): at small P J the
// thread-per-particle kernel is latency-bound on its uncoalesced row gathers and the lane-group kernel with the
// [g][h][m] table wins; with enough particles the thread kernel hides them and wins (c2 scene, ms per step, thread
// vs lanes: P = 1e5 0.58 vs 0.50 (v22), 2e5 0.701 vs 0.660, 3e5 0.896 vs 0.925, 4e5 1.167 vs 1.183 (v55); c4 8.36
// vs 9.02).  Decided once per loglik call (from its particle count) for the table build and every batch.
bool tay_lanes(const SceneDev& sc, int64_t P) { return (double)P * sc.J < 2.5e5; }
// FFT when G is a power of two in [64, 4096] (N_f a power of two up to 1024), unless direct = 1 (A/B); else the
// direct sum.  Both fp64, rounded once to complex64.
cudaError_t launch_tay_prep(const SceneDev& sc, const float2* y, float2* tab, int lanes, int direct, cudaStream_t st) {
  const int G = tay_centres(sc.nf, lanes);
  if (!direct && (G & (G - 1)) == 0 && G >= 64 && G <= 8192) {  // G = 8192: 192 KB of shared memory
    int lgG = 0;
    while ((1 << lgG) < G) ++lgG;
    const size_t smem = (size_t)G * sizeof(double2) * 3 / 2;
    cudaError_t e = cudaFuncSetAttribute(tay_prep_fft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    tay_prep_fft_kernel<<<(unsigned)(sc.J * sc.Na * (lanes ? TAY_L : TAY_L6)), TAY_FFT_THREADS, smem, st>>>(
        sc, G, lgG, y, tab, lanes);
    return cudaGetLastError();
  }
  const int64_t n = (int64_t)sc.J * sc.Na * tay_rows(G) * TAY_KS;
  if (lanes)
    tay_prep_kernel<TAY_L><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(sc, G, y, tab, lanes);
  else
    tay_prep_kernel<TAY_L6><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(sc, G, y, tab, lanes);
  return cudaGetLastError();
}
cudaError_t launch_tay_corr(const SceneDev& sc, const float2* tab, const float4* tmpl, const double* particles,
                            int64_t P, int pstride, const double* sfv, int sfv_pp, float2* terms, int* pflag,
                            int gram_diag, int lanes, cudaStream_t st) {
  if (P <= 0) return cudaSuccess;
  if (lanes) {
    int lg = 2;
    while ((1 << lg) < 32 && (4 << lg) < sc.Na) ++lg;  // ~4 antennas per lane
    const int epl = (sc.Na + (1 << lg) - 1) >> lg;
    const int64_t per_block = (int64_t)(TAY_BLOCK / 32) * (32 / sc.S);
    dim3 grid((unsigned)((P + per_block - 1) / per_block), sc.J);
    const int G = tay_centres(sc.nf, 1);
    const bool fast = (sc.ap_r / 1.5) * sc.df_c * (double)G <= TAY_EXT - 0.6;
#define TAY_LANES(E)                                                                                              \
  if (fast)                                                                                                       \
    tay_corr_lanes_kernel<E, true><<<grid, TAY_BLOCK, 0, st>>>(sc, G, tab, tmpl, particles, P, pstride, sfv, sfv_pp, \
                                                               terms, pflag, gram_diag, lg);                      \
  else                                                                                                            \
    tay_corr_lanes_kernel<E, false><<<grid, TAY_BLOCK, 0, st>>>(sc, G, tab, tmpl, particles, P, pstride, sfv,      \
                                                                sfv_pp, terms, pflag, gram_diag, lg)
    if (epl == 1) {
      TAY_LANES(1);
    } else if (epl == 2) {
      TAY_LANES(2);
    } else if (epl <= 4) {
      TAY_LANES(4);
    } else if (epl <= 8) {
      TAY_LANES(8);
    } else {
      TAY_LANES(0);
    }
#undef TAY_LANES
    return cudaGetLastError();
  }
  dim3 grid((unsigned)((P + TAY_BLOCK - 1) / TAY_BLOCK), sc.J);
  static thread_local TmplC tc;  // 8 KB: not on the stack
  make_tmplc(sc, &tc);
  const int G = tay_centres(sc.nf, 0);
  const bool fast = (sc.ap_r / 1.5) * sc.df_c * (double)G <= TAY_EXT - 0.6;  // the aperture within the extension
#define TAY_CORR(SPH, TC, FL) \
  tay_corr_kernel<SPH, TC, FL><<<grid, TAY_BLOCK, 0, st>>>(sc, G, tab, tmpl, particles, P, pstride, sfv, sfv_pp, \
                                                           terms, pflag, gram_diag, tc)
#define TAY_CORR_FL(SPH, TC) \
  if (fast) TAY_CORR(SPH, TC, true); \
  else TAY_CORR(SPH, TC, false);
  if (sc.wavefront == CDMS_SPHERICAL) {
    if (tc.n) { TAY_CORR_FL(true, true) }
    else { TAY_CORR_FL(true, false) }
  } else {
    if (tc.n) { TAY_CORR_FL(false, true) }
    else { TAY_CORR_FL(false, false) }
  }
#undef TAY_CORR_FL
#undef TAY_CORR
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------- F1: one component, T snapshots
// The correlations psi_p^H v_t of the F1 update (pf.cu, Supplement S-V P:L780-834): ONE component per particle -- the
// wall of PF particle p's SFV phi_p seen from the paired MT particle x_p (reading C-amb-F1a) -- against T snapshots
// per PA (K1T tables of snapshot t of PA j at table index j T + t, [m][g][l] layout).  Per antenna the fp32 offset,
// carrier and table centre are formed once (as tay_corr_kernel) and reused for every snapshot: one 64-byte row and one
// Taylor sum per (antenna, snapshot).  out [J][T][P] complex128 (consecutive particles contiguous: coalesced stores
// here and loads in pf_asm_kernel), path-loss gain applied; pflag as K1T.
template <int T>
__global__ void __launch_bounds__(TAY_BLOCK)
    pf_corr_kernel(const __grid_constant__ SceneDev sc, int G, const float2* __restrict__ tab,
                   const float4* __restrict__ tmpl, const double* __restrict__ particles, int64_t P, int pstride,
                   const double* __restrict__ phi, double2* __restrict__ out, int* __restrict__ pflag) {
  const int Na = sc.Na;
  const int64_t p = (int64_t)blockIdx.x * TAY_BLOCK + threadIdx.x;
  const int j = blockIdx.y;
  if (p >= P) return;
  const double* pos = particles + p * pstride;
  double2* o = out + (int64_t)j * T * P + p;  // o[t * P]
  double va[3], sh[3];
  if (!anchor_va(sc, j, phi ? phi + 3 * p : nullptr, va, sh)) {  // phi == NULL: the LOS PF (sh = 0, H = I)
    atomicOr(&pflag[p], 2);
#pragma unroll
    for (int t = 0; t < T; ++t) o[t * P] = make_double2(0.0, 0.0);
    return;
  }
  const double r0 = pos[0] - va[0], r1 = pos[1] - va[1], r2 = pos[2] - va[2];
  const double rs2 = 2.0 * (r0 * sh[0] + r1 * sh[1] + r2 * sh[2]);
  const float hx = (float)(r0 - rs2 * sh[0]), hy = (float)(r1 - rs2 * sh[1]), hz = (float)(r2 - rs2 * sh[2]);
  const double R64 = sqrt(r0 * r0 + r1 * r1 + r2 * r2);
  if (!(R64 > 0.0)) {
    atomicOr(&pflag[p], 1);
#pragma unroll
    for (int t = 0; t < T; ++t) o[t * P] = make_double2(0.0, 0.0);
    return;
  }
  const float R = (float)R64;
  const TayBase tb = tay_base(R64 * sc.df_c);
  double sb, cb;
  sincospi(2.0 * frac_c(R64 * sc.fc_c), &sb, &cb);
  const int Na_pad = sc.n_mb * NWARP;
  const float4* tm = tmpl + (int64_t)j * Na_pad;
  const size_t tstride = (size_t)Na * tay_rows(G);  // rows per (PA, snapshot) table (thread layout: A 2, B 1 float4)
  const float4* tA = reinterpret_cast<const float4*>(tab) + (size_t)j * T * tstride * 2;
  const float4* tB = reinterpret_cast<const float4*>(tab) + (size_t)sc.J * T * tstride * 2 + (size_t)j * T * tstride;
  const bool sph = sc.wavefront == CDMS_SPHERICAL;
  double accr[T], acci[T];
#pragma unroll
  for (int t = 0; t < T; ++t) accr[t] = acci[t] = 0.0;
  int fl = 0;
  for (int m0 = 0; m0 < Na; m0 += 16) {
    float pr[T], pi[T];
#pragma unroll
    for (int t = 0; t < T; ++t) pr[t] = pi[t] = 0.f;
    const int m1 = min(m0 + 16, Na);
    for (int m = m0; m < m1; ++m) {
      const float4 v = __ldg(&tm[m]);
      const float rq = hx * v.x + hy * v.y + hz * v.z;
      float delta;
      if (sph) {
        const float n = v.w - 2.f * rq;
        const float d = Num<float>::fsqrt_(R * R + n);
        if (!(d > 0.f)) fl |= 1;
        delta = Num<float>::fdiv_(n, d + R);
      } else {
        delta = Num<float>::fdiv_(-rq, R);
      }
      float er, ei;
      carrier_f(delta, sc.fc2pi_f, er, ei);
      uint32_t g;
      float dp;
      bool flip;
      tay_locate(delta * sc.df_cf, tb.hi, tb.lo, tb.par, G / 2, (float)G, (sc.nf & 1) == 0, g, dp, flip);
      if (flip) { er = -er; ei = -ei; }
      const size_t roff = (size_t)m * (uint32_t)tay_rows(G) + g;
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const size_t row = (size_t)t * tstride + roff;
        float4 c01, c23;
        ldg256(tA + 2 * row, c01, c23);
        const float4 c45 = __ldg(tB + row);
        float yr = c45.z, yi = c45.w;
        yr = fmaf(yr, dp, c45.x); yi = fmaf(yi, dp, c45.y);
        yr = fmaf(yr, dp, c23.z); yi = fmaf(yi, dp, c23.w);
        yr = fmaf(yr, dp, c23.x); yi = fmaf(yi, dp, c23.y);
        yr = fmaf(yr, dp, c01.z); yi = fmaf(yi, dp, c01.w);
        yr = fmaf(yr, dp, c01.x); yi = fmaf(yi, dp, c01.y);
        pr[t] = fmaf(er, yr, fmaf(-ei, yi, pr[t]));
        pi[t] = fmaf(er, yi, fmaf(ei, yr, pi[t]));
      }
    }
#pragma unroll
    for (int t = 0; t < T; ++t) {
      accr[t] += (double)pr[t];
      acci[t] += (double)pi[t];
    }
  }
  if (fl) atomicOr(&pflag[p], fl);
  const double gn = sc.pathloss ? sc.lambda / (4.0 * PI * R64) : 1.0;
#pragma unroll
  for (int t = 0; t < T; ++t)
    o[t * P] = make_double2((accr[t] * cb - acci[t] * sb) * gn, (accr[t] * sb + acci[t] * cb) * gn);
}
cudaError_t launch_pf_corr(const SceneDev& sc, int T, const float2* tab, const float4* tmpl, const double* particles,
                           int64_t P, int pstride, const double* phi, double2* out, int* pflag, cudaStream_t st) {
  if (P <= 0) return cudaSuccess;
  dim3 grid((unsigned)((P + TAY_BLOCK - 1) / TAY_BLOCK), sc.J);
  const int G = tay_centres(sc.nf, 0);
  switch (T) {
#define CASE_T(n) \
  case n: pf_corr_kernel<n><<<grid, TAY_BLOCK, 0, st>>>(sc, G, tab, tmpl, particles, P, pstride, phi, out, pflag); break;
    CASE_T(1) CASE_T(2) CASE_T(3) CASE_T(4) CASE_T(5) CASE_T(6) CASE_T(7) CASE_T(8) CASE_T(9)
#undef CASE_T
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace cdms
