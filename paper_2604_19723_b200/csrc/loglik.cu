// loglik.cu -- rows A2-A5 of the hot path on sm_100a.
//
// K1 corr_kernel<S, RT>: for a batch of particles and every PA j, the correlation c = Psi^H z^(j) by
// segmented Horner recurrences over the (never materialized) spherical / planar responses, and the Gram
// G = Psi^H Psi in closed form; writes the S + S(S+1)/2 sufficient statistics per
// (particle, PA) to HBM.
// K1b assemble_kernel<S>: one thread per particle, fp64: the S x S low-rank evaluation of the MT update
// message iota~ (Supplement S-V-C), summed over the PAs.
//
// K1 work decomposition: CTA = 32 particles (lanes) x 8 antennas (warps), persistent grid; CTAs claim
// (tile, PA) groups dynamically (see corr_kernel).  For each PA and
// each block of 8 antennas, y^(j) streams through shared memory in chunks of <= 128 subcarriers x 8 antennas
// by 1-D bulk TMA (cp.async.bulk, mbarrier, double buffered), stored as (yr, yr, yi, yi) so one broadcast
// LDS.128 feeds FFMA2 (fma.rn.f32x2) Horner steps that advance two components per instruction.  Per
// (particle, component) geometry and phase bases are fp64.
#include <math.h>

#include "cdms_internal.h"
#include "geometry.cuh"

namespace cdms {

// ---------------------------------------------------------------------------- y re-layout
// y [J][nf][Na] (paper vec order) -> ytiles [J][Na_pad][n_kc][kc_len] of (yr, yr, yi, yi), Na_pad = 8 n_mb
// (zero padded): each warp streams its own antenna's chunks; ||z^(j)||^2 in fp64 (block 0 of each PA,
// fixed reduction order); and the template columns tmpl[j][m] = (R_j p~_m, ||p~_m||^2) evaluated in fp64 and
// rounded once to fp32 (padded antennas repeat m = 0); after the J PAs' columns, the PA-independent row
// tmpl[J][m] = (p~_y, p~_z, ||p~||^2, 0) of the template itself (the Gram folds R_j into its per-component h).
// Host copy of template_col (same formula; fp64 rounded once to fp32) for TmplC.
void make_tmplc(const SceneDev& sc, TmplC* out) {
  const int npad = sc.n_mb * NWARP;
  out->n = sc.J * npad <= TMPLC_MAX ? sc.J * npad : 0;
  if (!out->n) return;
  for (int j = 0; j < sc.J; ++j)
    for (int m = 0; m < npad; ++m) {
      const int mm = m < sc.Na ? m : 0, iy = mm / sc.nv, iv = mm - iy * sc.nv;
      const double py = (iy - 0.5 * (sc.ny - 1)) * sc.dy, pz = (iv - 0.5 * (sc.nv - 1)) * sc.dv;
      const double* R = sc.pa_rot[j];
      out->v[j * npad + m] = make_float4((float)(R[1] * py + R[2] * pz), (float)(R[4] * py + R[5] * pz),
                                         (float)(R[7] * py + R[8] * pz), (float)(py * py + pz * pz));
    }
}

__global__ void prep_y_kernel(const __grid_constant__ SceneDev sc, const float2* __restrict__ y,
                              float4* __restrict__ yt, double* __restrict__ ynorm2, float4* __restrict__ tmpl,
                              const __grid_constant__ TmplC tc) {
  const int j = blockIdx.y;
  const int64_t per_j = (int64_t)sc.n_mb * sc.n_kc * sc.kc_len * NWARP;
  if (blockIdx.x == gridDim.x - 1) {
    if (j == 0)
      for (int m = threadIdx.x; m < sc.n_mb * NWARP; m += blockDim.x) {
        const int mm = m < sc.Na ? m : 0, iy = mm / sc.nv, iv = mm - iy * sc.nv;
        const double py = (iy - 0.5 * (sc.ny - 1)) * sc.dy, pz = (iv - 0.5 * (sc.nv - 1)) * sc.dv;
        tmpl[(int64_t)sc.J * sc.n_mb * NWARP + m] = make_float4((float)py, (float)pz, (float)(py * py + pz * pz), 0.f);
      }
    for (int m = threadIdx.x; m < sc.n_mb * NWARP; m += blockDim.x) {
      if (tc.n) {  // the host's columns (identical to the correlation kernel's constant-bank copy)
        tmpl[(int64_t)j * sc.n_mb * NWARP + m] = tc.v[j * sc.n_mb * NWARP + m];
        continue;
      }
      double v[3], q2;
      template_col(sc, j, m < sc.Na ? m : 0, v, q2);
      tmpl[(int64_t)j * sc.n_mb * NWARP + m] = make_float4((float)v[0], (float)v[1], (float)v[2], (float)q2);
    }
  }
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < per_j;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int kl = (int)(t % sc.kc_len);
    int64_t rest = t / sc.kc_len;
    const int kc = (int)(rest % sc.n_kc);
    const int m = (int)(rest / sc.n_kc);
    const int k = kc * sc.kc_len + kl;
    float2 v = make_float2(0.f, 0.f);
    if (m < sc.Na && k < sc.nf) v = y[((int64_t)j * sc.nf + k) * sc.Na + m];
    yt[(int64_t)j * per_j + t] = make_float4(v.x, v.x, v.y, v.y);
  }
  if (blockIdx.x == 0) {
    __shared__ double red[256];
    double acc = 0.0;
    const int64_t nz = (int64_t)sc.nf * sc.Na;
    for (int64_t n = threadIdx.x; n < nz; n += blockDim.x) {
      const float2 v = y[(int64_t)j * nz + n];
      acc += (double)v.x * v.x + (double)v.y * v.y;
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
      if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
      __syncthreads();
    }
    if (threadIdx.x == 0) ynorm2[j] = red[0];
  }
}

cudaError_t launch_prep_y(const SceneDev& sc, const float2* y, float4* ytiles, double* ynorm2, float4* tmpl,
                          cudaStream_t st) {
  const int64_t per_j = (int64_t)sc.n_mb * sc.n_kc * sc.kc_len * NWARP;
  int gx = (int)((per_j + 255) / 256);
  if (gx > 1024) gx = 1024;
  if (gx < 2) gx = 2;
  dim3 grid(gx, sc.J);
  static thread_local TmplC tc;  // 8 KB: not on the stack
  make_tmplc(sc, &tc);
  prep_y_kernel<<<grid, 256, 0, st>>>(sc, y, ytiles, ynorm2, tmpl, tc);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------- index helpers
__host__ __device__ constexpr int tri(int r, int c) { return r * (r + 1) / 2 + c; }  // r >= c
// pair q -> (a, b), a < b, row by row: (0,1), (0,2), ..., (1,2), ...
__device__ __forceinline__ void pair_ab(int q, int S, int& a, int& b) {
  int aa = 0, rem = q;
  while (rem >= S - 1 - aa) {
    rem -= S - 1 - aa;
    ++aa;
  }
  a = aa;
  b = aa + 1 + rem;
}
__device__ __forceinline__ int pair_index(int a, int b, int S) { return a * S - a * (a + 1) / 2 + (b - a - 1); }

// ---------------------------------------------------------------------------- Horner state
// acc <- acc * w + y for S components (row A3).  fp32: components paired in 64-bit registers and
// advanced by fma.rn.f32x2 (FFMA2): t = hi*(-wi) + yr, u = hi*wr + yi, hr' = hr*wr + t, hi' = hr*wi + u.

template <int S, typename RT>
struct Horner;

template <int S>
struct Horner<S, float> {
  static constexpr int NP = S / 2;
  static constexpr bool ODD = (S & 1) != 0;
  u64 wr2[NP > 0 ? NP : 1], wi2[NP > 0 ? NP : 1], nwi2[NP > 0 ? NP : 1], hr2[NP > 0 ? NP : 1],
      hi2[NP > 0 ? NP : 1];
  float wrL, wiL, hrL, hiL;
  __device__ __forceinline__ void init(const float* wr, const float* wi) {
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      wr2[q] = pk2(wr[2 * q], wr[2 * q + 1]);
      wi2[q] = pk2(wi[2 * q], wi[2 * q + 1]);
      nwi2[q] = pk2(-wi[2 * q], -wi[2 * q + 1]);
    }
    if (ODD) {
      wrL = wr[S - 1];
      wiL = wi[S - 1];
    }
  }
  __device__ __forceinline__ void reset_to(const float4 y) {
    const u64 yr2 = pk2(y.x, y.y), yi2 = pk2(y.z, y.w);
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      hr2[q] = yr2;
      hi2[q] = yi2;
    }
    hrL = y.x;
    hiL = y.z;
  }
  __device__ __forceinline__ void step(const float4 y) {
    const u64 yr2 = pk2(y.x, y.y), yi2 = pk2(y.z, y.w);
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const u64 t = ffma2(hi2[q], nwi2[q], yr2);
      const u64 u = ffma2(hi2[q], wr2[q], yi2);
      const u64 nr = ffma2(hr2[q], wr2[q], t);
      const u64 ni = ffma2(hr2[q], wi2[q], u);
      hr2[q] = nr;
      hi2[q] = ni;
    }
    if (ODD) {
      const float t = fmaf(-hiL, wiL, y.x);
      const float u = fmaf(hiL, wrL, y.z);
      const float nr = fmaf(hrL, wrL, t);
      const float ni = fmaf(hrL, wiL, u);
      hrL = nr;
      hiL = ni;
    }
  }
  __device__ __forceinline__ void get(float* hr, float* hi) const {
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      up2(hr2[q], hr[2 * q], hr[2 * q + 1]);
      up2(hi2[q], hi[2 * q], hi[2 * q + 1]);
    }
    if (ODD) {
      hr[S - 1] = hrL;
      hi[S - 1] = hiL;
    }
  }
};

template <int S>
struct Horner<S, double> {
  double wr[S], wi[S], hr[S], hi[S];
  __device__ __forceinline__ void init(const double* wr_, const double* wi_) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      wr[s] = wr_[s];
      wi[s] = wi_[s];
    }
  }
  __device__ __forceinline__ void reset_to(const float4 y) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      hr[s] = (double)y.x;
      hi[s] = (double)y.z;
    }
  }
  __device__ __forceinline__ void step(const float4 y) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const double t = fma(-hi[s], wi[s], (double)y.x);
      const double u = fma(hi[s], wr[s], (double)y.z);
      const double nr = fma(hr[s], wr[s], t);
      const double ni = fma(hr[s], wi[s], u);
      hr[s] = nr;
      hi[s] = ni;
    }
  }
  __device__ __forceinline__ void get(double* hr_, double* hi_) const {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      hr_[s] = hr[s];
      hi_[s] = hi[s];
    }
  }
};

// ---------------------------------------------------------------------------- shared memory plan
// y chunk length (subcarriers per TMA chunk and warp).  With 128 the plan gives 3 CTAs (24 warps) per SM for
// S <= 5 and 2 CTAs (128 registers, no spills) for S >= 6; 64 would fit 3 CTAs for S = 6, 7 but at 80
// registers with spills, measured ~1% slower on c3 / c5.
__host__ __device__ constexpr int kchunk_for(int S) {
#ifdef CDMS_KCHUNK_ALL
  return CDMS_KCHUNK_ALL + 0 * S;
#else
  return 128 + 0 * S;  // measured: S = 6, 7 run better at 2 CTAs x 128 registers than at 3 CTAs with spills
#endif
}

template <int S, typename RT>
struct Plan {
  static constexpr int NPAIR = S * (S - 1) / 2;
  static constexpr int NTRI = S * (S + 1) / 2;
  static constexpr int T = S + NTRI;
  static constexpr int KC = kchunk_for(S);
  static constexpr size_t ybuf = 2ull * KC * NWARP * sizeof(float4);
  static constexpr size_t ps =
      (size_t)NPSF_PAD * S * TILE_P * sizeof(RT) + (size_t)S * TILE_P * sizeof(double);
  static constexpr size_t dlt = (size_t)S * NWARP * TILE_P * sizeof(RT);            // Delta [S][8][32]
  static constexpr size_t cst = (size_t)S * NWARP * TILE_P * 2 * sizeof(RT);        // c per antenna
  static constexpr size_t acc = (size_t)(S + NPAIR) * TILE_P * sizeof(double2);     // fp64 sums [item][32]
  // mbarriers, positions, per-particle flags, claimed-group ring
  static constexpr size_t misc =
      2 * NWARP * sizeof(uint64_t) + TILE_P * 3 * sizeof(double) + TILE_P * sizeof(int) + 4 * sizeof(unsigned);
  static constexpr size_t total = ybuf + ps + dlt + cst + acc + misc;
  // resident CTAs per SM the kernel is compiled for (fp32): as many as (smem + 1 KB reserve) fits in 228 KB,
  // capped so that each thread keeps >= 80 registers (the Horner state + phasors of S <= 7 without spills)
  static constexpr int smem_fit = (int)((228 * 1024) / (total + 1024));
  static constexpr int reg_fit = 65536 / (NTHREADS * 80);
#if defined(CDMS_XP_MINB_ALL)  // experiment builds: force the CTAs per SM (registers follow)
  static constexpr int min_blocks = (sizeof(RT) == 8) ? 1 : CDMS_XP_MINB_ALL;
#elif defined(CDMS_XP_MINB_BIG_S)  // experiment builds: force the CTAs per SM of S >= 6
  static constexpr int min_blocks = (sizeof(RT) == 8) ? 1 : (S >= 6 ? CDMS_XP_MINB_BIG_S
                                                                   : (smem_fit < reg_fit ? smem_fit : reg_fit));
#else
  static constexpr int min_blocks =
      (sizeof(RT) == 8) ? 1 : (smem_fit < reg_fit ? (smem_fit < 1 ? 1 : smem_fit) : reg_fit);
#endif
};

size_t corr_smem_bytes(int S, int precision) {
  switch (S) {
#define CASE_S(n) \
  case n: return precision == CDMS_FP64 ? Plan<n, double>::total : Plan<n, float>::total;
    CASE_S(1) CASE_S(2) CASE_S(3) CASE_S(4) CASE_S(5) CASE_S(6) CASE_S(7) CASE_S(8) CASE_S(9)
#undef CASE_S
    default: return 0;
  }
}

// ---------------------------------------------------------------------------- phase timing (debug build)
// -DCDMS_PHASE_TIMING: per-warp clock64 cycles per phase of K1, summed into g_phase (tools/phase_timing.py).
#ifdef CDMS_PHASE_TIMING
__device__ unsigned long long g_phase[8];
#define PT_DECL unsigned long long pt_t = clock64(), pt_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define PT(i) { const unsigned long long n_ = clock64(); pt_acc[i] += n_ - pt_t; pt_t = n_; }
#define PT_FLUSH if (lane == 0) { for (int i_ = 0; i_ < 8; ++i_) atomicAdd(&g_phase[i_], pt_acc[i_]); }
}  // namespace cdms
extern "C" int cdms_debug_phase_read(double* out8, int reset) {
  unsigned long long h[8];
  if (cudaMemcpyFromSymbol(h, cdms::g_phase, sizeof(h)) != cudaSuccess) return 1;
  for (int i = 0; i < 8; ++i) out8[i] = (double)h[i];
  if (reset) {
    const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(cdms::g_phase, z, sizeof(z));
  }
  return 0;
}
namespace cdms {
#else
#define PT_DECL
#define PT(i)
#define PT_FLUSH
#endif

// ---------------------------------------------------------------------------- K1
// Work distribution: dynamic.  A group is (tile of 32 particles, PA j), g = tile J + j; thread 0 of each
// persistent CTA claims groups from a global counter one or two groups ahead (ring in shared memory) so the per-warp
// TMA streams run across group boundaries without a stall.  Co-resident CTAs progress at different rates under
// the warp scheduler's age priority; static partitions left ~17% of the warp slots idle (ncu warps_active 20
// of 24), dynamic claiming keeps every slot busy until the queue drains.  Each group is computed entirely by
// one CTA: results do not depend on the schedule.  The last CTA to finish resets the counters.
// TWO: compile-time sc.two_seg (the segment end either moves A1 in or multiplies by Z; two instantiations keep
// both Horner loops free of the other's register pressure).
// NOH: Gram-only variant (no phasors, no Horner steps; the y chunks still stream so the per-warp TMA ring keeps its
// protocol) -- it served the K1T A/B option CDMS_TAYLOR_GRAM=k1 (profiles/r01_k1t_gram_select.txt), removed in round
// 2; no launcher instantiates it now.
template <int S, typename RT, bool TWO, bool NOH = false>
__global__ void __launch_bounds__(NTHREADS, (Plan<S, RT>::min_blocks))
    corr_kernel(const __grid_constant__ SceneDev sc, const CorrArgs a) {
  using PL = Plan<S, RT>;
  constexpr int NPAIR = PL::NPAIR;
  constexpr int T = PL::T;
  constexpr int KC = PL::KC;
  constexpr bool F32 = sizeof(RT) == 4;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* sp = smem;
  float4* ybuf = reinterpret_cast<float4*>(sp);                         sp += PL::ybuf;
  RT* psf = reinterpret_cast<RT*>(sp);                                  // [S][32][NPSF_PAD]
  double* R64s = reinterpret_cast<double*>(sp + (size_t)NPSF_PAD * S * TILE_P * sizeof(RT));  // [S][32]
  sp += PL::ps;
  RT* dlt = reinterpret_cast<RT*>(sp);                                  sp += PL::dlt;
  RT* cst = reinterpret_cast<RT*>(sp);                                  sp += PL::cst;
  double2* acc = reinterpret_cast<double2*>(sp);                        sp += PL::acc;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sp);                     // [NWARP][2]
  double* pos_s = reinterpret_cast<double*>(sp + 2 * NWARP * sizeof(uint64_t));  // [3][32]
  int* pfl = reinterpret_cast<int*>(sp + 2 * NWARP * sizeof(uint64_t) + TILE_P * 3 * sizeof(double));

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int J = sc.J, Na = sc.Na, nf = sc.nf, kcl = sc.kc_len;
  const int n_mb = sc.n_mb, n_kc = sc.n_kc, Na_pad = sc.n_mb * NWARP;
  const bool nb_mode = sc.wavefront == CDMS_PLANAR_NB;
  const uint32_t n_groups = (uint32_t)a.n_groups;
  unsigned int* gring = reinterpret_cast<unsigned int*>(pfl + TILE_P);  // [4] claimed group indices

  // Every warp streams its own antenna's y chunks (no CTA-wide barrier per chunk): lane 0 issues a 1-D bulk
  // TMA of kc_len (yr, yr, yi, yi) into the warp's double buffer, completion on the warp's mbarrier.  The
  // stream walks the CTA's claimed groups in order; chunk (mb, kc) of group g sits at element offset
  // (((j n_mb + mb) 8 + warp) n_kc + kc) kc_len of ytiles [J][Na_pad][n_kc][kc_len], j = g mod J: a running
  // offset, re-based when the stream enters the next claimed group (published in gring one group earlier).
  int is_gi = 0, is_mb = 0, is_kc = 0, is_c = 0;
  uint32_t is_g = 0;
  int64_t is_off = 0;
  auto rebase = [&]() {
    is_g = gring[is_gi & 3];
    is_off = (((int64_t)(is_g % (uint32_t)sc.J) * sc.n_mb * NWARP + warp) * sc.n_kc) * sc.kc_len;
  };
  auto issue = [&]() {
    if (is_g >= n_groups) return;
    // No proxy fence: the buffer is only read by the generic proxy (LDS, completed before the __syncwarp that
    // precedes every reissue) and only written by the async proxy.
    if (!NOH) {  // the Gram-only variant keeps the stream's counters (group claims) but moves no data
      uint64_t* bar = &mbar[warp * 2 + (is_c & 1)];
      const uint32_t chunk_bytes = (uint32_t)(sc.kc_len * sizeof(float4));
      mbar_expect_tx(bar, chunk_bytes);
      tma_load_1d(ybuf + (warp * 2 + (is_c & 1)) * KC, a.ytiles + is_off, chunk_bytes, bar);
    }
    ++is_c;
    is_off += sc.kc_len;
    if (++is_kc == sc.n_kc) {
      is_kc = 0;
      is_off += sc.y_mb_step;
      if (++is_mb == sc.n_mb) {
        is_mb = 0;
        ++is_gi;
        rebase();
      }
    }
  };

  if (tid < 2 * NWARP) mbar_init(&mbar[tid], 1);
  // Claims run L groups ahead of the consumer, as few as the TMA stream needs (it runs <= 2 chunks ahead, so it
  // enters group gi + 1 during group gi when groups hold >= 2 chunks, gi + 2 otherwise): claimed-but-unstarted
  // groups are exactly what the last CTAs still hold when the queue drains (c2: ~7 groups per CTA).
  const int L = (sc.n_mb * sc.n_kc >= 2) ? 1 : 2;
  if (tid == 0) {
    fence_mbar_init();
    for (int i = 0; i < L; ++i) gring[i] = atomicAdd(a.sched, 1u);
  }
  if (tid < TILE_P) pfl[tid] = 0;
  __syncthreads();
  if (lane == 0) {
    rebase();
    issue();
    issue();
  }

  int64_t ci = 0;            // flat chunk counter (the same sequence in every warp)
  for (int ring_i = 0;; ++ring_i) {
    const uint32_t g = gring[ring_i & 3];
    if (g >= n_groups) break;
    const int64_t tile = g / (uint32_t)J;
    const int j = (int)(g - (uint32_t)tile * (uint32_t)J);
    const int64_t p = tile * TILE_P + lane;
    const bool pvalid = p < a.P;
    if (warp == 0) {
#pragma unroll
      for (int c = 0; c < 3; ++c) pos_s[c * TILE_P + lane] = pvalid ? a.particles[p * a.pstride + c] : 1.0;
    }
    if (tid == 0) gring[(ring_i + L) & 3] = atomicAdd(a.sched, 1u);
    __syncthreads();
    PT_DECL

    // ---- (1) per (component, particle) set-up in fp64 (rows A1/A2); zero the fp64 accumulators
    for (int it = tid; it < S * TILE_P; it += NTHREADS) {
      const int s = it / TILE_P, pl = it - s * TILE_P;
      const int64_t pp = tile * TILE_P + pl;
      const double pos[3] = {pos_s[pl], pos_s[TILE_P + pl], pos_s[2 * TILE_P + pl]};
      const double* sfv_s = nullptr;
      if (s > 0) sfv_s = a.sfv + ((a.sfv_pp && pp < a.P) ? pp * 3 * sc.K : 0) + 3 * (s - 1);
      PSField<RT> f;
      double R64 = 1.0;
      const int st = setup_ps<RT, !NOH>(sc, j, pos, sfv_s, f, R64);
      if (st != PS_OK && pp < a.P) {
        const bool bad = st == PS_BADSFV || !(pos[0] == pos[0] && pos[1] == pos[1] && pos[2] == pos[2]);
        atomicOr(&pfl[pl], bad ? 3 : 1);
      }
      const RT* fv = reinterpret_cast<const RT*>(&f);
#pragma unroll
      for (int q = 0; q < NPSF; ++q) psf[(s * TILE_P + pl) * NPSF_PAD + q] = fv[q];
      R64s[s * TILE_P + pl] = R64;
    }
    for (int it = tid; it < (S + NPAIR) * TILE_P; it += NTHREADS) acc[it] = make_double2(0.0, 0.0);
    __syncthreads();
    PT(0)

    // ---- (1b) planar NB Gram, separable closed form in fp64 (P:L2160-2184 with the template P:L29-39):
    //   G_ab = e^{j 2 pi dR fc/c} D_Nf(dR df/c) D_ny(dy du'_y fc/c) D_nv(dv du'_z fc/c),
    //   dR = R_a - R_b, du' = u'_b - u'_a, u'_s = R_j^T H_s r_s / R_s (local directions).
    if (nb_mode && NPAIR > 0 && !a.no_gram) {
      for (int it = tid; it < NPAIR * TILE_P; it += NTHREADS) {
        const int q = it / TILE_P, pl = it - q * TILE_P;
        int ca, cb;
        pair_ab(q, S, ca, cb);
        const int64_t pp = tile * TILE_P + pl;
        const double pos[3] = {pos_s[pl], pos_s[TILE_P + pl], pos_s[2 * TILE_P + pl]};
        double ul[2][3];
        const int comp[2] = {ca, cb};
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int s = comp[e];
          const double* sfv_s = s ? a.sfv + ((a.sfv_pp && pp < a.P) ? pp * 3 * sc.K : 0) + 3 * (s - 1) : nullptr;
          double va[3], sh[3];
          if (!anchor_va(sc, j, sfv_s, va, sh)) { va[0] = pos[0] - 1.0; va[1] = pos[1]; va[2] = pos[2]; sh[0] = sh[1] = sh[2] = 0.0; }
          double r[3] = {pos[0] - va[0], pos[1] - va[1], pos[2] - va[2]};
          const double R = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
          const double rs = r[0] * sh[0] + r[1] * sh[1] + r[2] * sh[2];
          double h[3] = {r[0] - 2.0 * rs * sh[0], r[1] - 2.0 * rs * sh[1], r[2] - 2.0 * rs * sh[2]};
          const double* Rj = sc.pa_rot[j];
          const double inv = R > 0.0 ? 1.0 / R : 0.0;
#pragma unroll
          for (int c = 0; c < 3; ++c) ul[e][c] = (Rj[0 * 3 + c] * h[0] + Rj[1 * 3 + c] * h[1] + Rj[2 * 3 + c] * h[2]) * inv;
        }
        const double dR = R64s[ca * TILE_P + pl] - R64s[cb * TILE_P + pl];
        double sb, cbv;
        sincospi(2.0 * frac_c(dR * sc.fc_c), &sb, &cbv);
        const double xb = dR * sc.df_c, nbr = rint(xb);
        double D = dirichlet<double>(xb - nbr, (long long)nbr, nf);
        const double xy = sc.dy * (ul[1][1] - ul[0][1]) * sc.fc_c, xv = sc.dv * (ul[1][2] - ul[0][2]) * sc.fc_c;
        const double ny_ = rint(xy), nv_ = rint(xv);
        D *= dirichlet<double>(xy - ny_, (long long)ny_, sc.ny) * dirichlet<double>(xv - nv_, (long long)nv_, sc.nv);
        acc[(S + q) * TILE_P + pl] = make_double2(D * cbv, D * sb);
      }
    }

    for (int mb = 0; mb < n_mb; ++mb) {
      const int m = mb * NWARP + warp;
      const bool mvalid = m < Na;
      // ---- (2) per (component, antenna) offsets and phasors (row A2)
      RT Ar[S], Ai[S], Zr[S], Zi[S];
      Horner<S, RT> H;
      {
        RT wr[S], wi[S];
        RT v[3], q2;
        if (F32) {
          // template column R_j p~_m: fp64, rounded once (table from prep_y, L1-resident)
          const float4 tv = __ldg(&a.tmpl[j * Na_pad + m]);
          v[0] = (RT)tv.x; v[1] = (RT)tv.y; v[2] = (RT)tv.z; q2 = (RT)tv.w;
        } else {
          double v64[3], q264;
          template_col(sc, j, mvalid ? m : 0, v64, q264);
          v[0] = (RT)v64[0]; v[1] = (RT)v64[1]; v[2] = (RT)v64[2]; q2 = (RT)q264;
        }
        bool deg_any = false;
#pragma unroll
        for (int s = 0; s < S; ++s) {
          PSField<RT> f;
          RT* fv = reinterpret_cast<RT*>(&f);
          load_psf<RT>(psf + (s * TILE_P + lane) * NPSF_PAD, fv);  // 128-bit loads
          SMPhasors<RT> o;
          bool dg;
#ifdef CDMS_XP_CHEAP_SETUP  // experiment build only: trivial phasors (wrong results) to price the set-up
          o.Ar = f.E0r; o.Ai = f.E0i; o.wr = f.Whr; o.wi = f.Whi; o.Zr = f.Zhr; o.Zi = f.Zhi; o.delta = f.hx * v[0];
          dg = false;
#else
          if (NOH) {  // Delta only (the Gram's input)
            const RT rq = f.hx * v[0] + f.hy * v[1] + f.hz * v[2];
            if (sc.wavefront == CDMS_SPHERICAL) {
              const RT n = q2 - RT(2) * rq;
              const RT d = Num<RT>::fsqrt_(f.R * f.R + n);
              dg = !(d > RT(0));
              o.delta = Num<RT>::fdiv_(n, d + f.R);
            } else {
              o.delta = Num<RT>::fdiv_(-rq, f.R);
              dg = false;
            }
            o.Ar = o.Ai = o.wr = o.wi = o.Zr = o.Zi = RT(0);
          } else {
            setup_sm<RT>(sc, f, v, q2, m, s, o, dg);
          }
#endif
          deg_any |= dg;
          Ar[s] = o.Ar; Ai[s] = o.Ai; wr[s] = o.wr; wi[s] = o.wi; Zr[s] = o.Zr; Zi[s] = o.Zi;
          const int o_ = (s * NWARP + warp) * TILE_P + lane;
          dlt[o_] = o.delta;
          cst[2 * o_] = RT(0);
          cst[2 * o_ + 1] = RT(0);
        }
        if (deg_any && mvalid && pvalid) atomicOr(&pfl[lane], 1);
        H.init(wr, wi);
        PT(2)
      }
      // ---- (3) correlation over all subcarriers (row A3): segmented Horner on TMA-staged y chunks
      for (int kc = 0; kc < n_kc; ++kc, ++ci) {
        if (!NOH) mbar_wait(&mbar[warp * 2 + (ci & 1)], (uint32_t)((ci >> 1) & 1));
        const float4* yb = ybuf + (warp * 2 + (ci & 1)) * KC;
        const int k_begin = kc * kcl;
        const int k_end = NOH ? k_begin : min(k_begin + kcl, nf);  // Gram-only: no correlation
        for (int k0 = k_begin; k0 < k_end; k0 += SEG) {
          const int k1 = min(k0 + SEG, k_end);
          const float4* yk = yb + (k1 - 1 - k_begin);  // Horner runs from the top subcarrier down
          H.reset_to(yk[0]);                            // acc = y_top (= 0 * w + y_top)
#ifdef CDMS_XP_SKIP_HORNER  // experiment build only (wrong results): price everything but the Horner steps
          if (false) {
#else
          if (!NOH && k1 - k0 == SEG) {
#endif
#pragma unroll 7
            for (int i = 1; i < SEG; ++i) H.step(yk[-i]);
          } else if (!NOH) {
#ifndef CDMS_XP_SKIP_HORNER
            for (int i = 1; i < k1 - k0; ++i) H.step(yk[-i]);
#endif
          }
          // c += A_seg H_seg (thread-private slot), A_seg <- A_seg Z (two_seg: A_1 itself sits in Z)
          RT hr[S], hi[S];
          H.get(hr, hi);
          constexpr bool two_seg = TWO;
#pragma unroll
          for (int s = 0; s < S; ++s) {
            const int o_ = (s * NWARP + warp) * TILE_P + lane;
            cst[2 * o_] = fma(Ar[s], hr[s], fma(-Ai[s], hi[s], cst[2 * o_]));
            cst[2 * o_ + 1] = fma(Ar[s], hi[s], fma(Ai[s], hr[s], cst[2 * o_ + 1]));
            if (two_seg) {
              Ar[s] = Zr[s];
              Ai[s] = Zi[s];
            } else {
              const RT nAr = Ar[s] * Zr[s] - Ai[s] * Zi[s];
              const RT nAi = Ar[s] * Zi[s] + Ai[s] * Zr[s];
              Ar[s] = nAr;
              Ai[s] = nAi;
            }
          }
        }
        __syncwarp();  // every lane of this warp is done with the buffer
        if (lane == 0) issue();
      }
      PT(3)
      __syncthreads();  // publish this block's cst / dlt
      PT(4)
      const int nw_valid = min(NWARP, Na - mb * NWARP);
      // ---- (4a) c_s += sum over the block's antennas, ascending m; owner warp rotates with mb
      for (int s = (warp - mb) & (NWARP - 1); s < S; s += NWARP) {
        double sr = 0.0, si = 0.0;
        for (int w2 = 0; w2 < nw_valid; ++w2) {
          const int o_ = (s * NWARP + w2) * TILE_P + lane;
          sr += (double)cst[2 * o_];
          si += (double)cst[2 * o_ + 1];
        }
        double2 v = acc[s * TILE_P + lane];
        acc[s * TILE_P + lane] = make_double2(v.x + sr, v.y + si);
      }
      // ---- (4b) spherical / planar WB Gram terms (row A4) over the block's antennas:
      //   sum_m e^{j 2 pi (D_a,m - D_b,m) fc/c} D_N((d_a,m - d_b,m) df/c); the base carrier e^{j 2 pi dR fc/c}
      //   is applied in fp64 at the hand-off (shared by all antennas: its rounding must not repeat)
#ifdef CDMS_XP_SKIP_GRAM  // experiment build only (wrong results): price the per-antenna Gram terms
      if (false) {
#else
      if (!nb_mode && !a.no_gram) {
#endif
        for (int q = (warp - mb - S) & (NWARP - 1); q < NPAIR; q += NWARP) {
          int pa, pb;
          pair_ab(q, S, pa, pb);
          const double dR = R64s[pa * TILE_P + lane] - R64s[pb * TILE_P + lane];
          const double xb = dR * sc.df_c;
          const double nbd = rint(xb);
          RT gr = RT(0), gi = RT(0);
          if (F32) {
            GramPairF gp;
            gp.xbr = (float)(xb - nbd);
            gp.nbpar = (uint32_t)((long long)nbd & 1) << 31;
            for (int w2 = 0; w2 < nw_valid; ++w2) {
              const float dd = (float)(dlt[(pa * NWARP + w2) * TILE_P + lane] - dlt[(pb * NWARP + w2) * TILE_P + lane]);
              float fr = (float)gr, fi = (float)gi;
              gram_term_f(sc, dd, gp, fr, fi);
              gr = (RT)fr; gi = (RT)fi;
            }
          } else {
            const long long nbi = (long long)nbd;
            const RT xbr = (RT)(xb - nbd);
            for (int w2 = 0; w2 < nw_valid; ++w2) {
              const RT dd = dlt[(pa * NWARP + w2) * TILE_P + lane] - dlt[(pb * NWARP + w2) * TILE_P + lane];
              RT er, ei;
              cis2pi_fast<RT>(dd * (RT)sc.fc_c, er, ei);
              const RT x = xbr + dd * (RT)sc.df_c;
              const RT n2 = Num<RT>::rint_(x);
              const RT D = dirichlet<RT>(x - n2, nbi + (long long)n2, nf);
              gr = fma(D, er, gr);
              gi = fma(D, ei, gi);
            }
          }
          double2 v = acc[(S + q) * TILE_P + lane];
          acc[(S + q) * TILE_P + lane] = make_double2(v.x + (double)gr, v.y + (double)gi);
        }
      }
      PT(5)
      __syncthreads();  // before the next block's set-up rewrites dlt / cst
      PT(6)
    }

    // ---- (5) hand-off: c (with gains) and the lower triangle of G (with gains) -> terms [P][J][T]
    const double nz = (double)nf * (double)Na;
    for (int it = tid; it < T * TILE_P; it += NTHREADS) {
      const int t = it / TILE_P, pl = it - t * TILE_P;  // consecutive threads: consecutive particles (term_idx)
      const int64_t pp = tile * TILE_P + pl;
      if (pp >= a.P) continue;
      double2 out;
      if (t < S) {
        const double gn = (double)psf[(t * TILE_P + pl) * NPSF_PAD + PSF_GAIN];
        const double2 v = acc[t * TILE_P + pl];
        out = make_double2(v.x * gn, v.y * gn);
      } else {
        int r = 0, e = t - S;
        while (e >= r + 1) { e -= r + 1; ++r; }
        const int c = e;  // (r, c), r >= c
        const double gr_ = (double)psf[(r * TILE_P + pl) * NPSF_PAD + PSF_GAIN];
        const double gc_ = (double)psf[(c * TILE_P + pl) * NPSF_PAD + PSF_GAIN];
        if (r == c) {
          out = make_double2(nz * gr_ * gc_, 0.0);
        } else {
          // G_cr (c < r) accumulated; lower entry G_rc = conj(G_cr)
          const int q = pair_index(c, r, S);
          double2 v = acc[(S + q) * TILE_P + pl];
          if (!nb_mode) {
            const double dR = R64s[c * TILE_P + pl] - R64s[r * TILE_P + pl];
            double sb, cb;
            sincospi(2.0 * frac_c(dR * sc.fc_c), &sb, &cb);
            v = make_double2(cb * v.x - sb * v.y, cb * v.y + sb * v.x);
          }
          const double g2 = gr_ * gc_;
          out = make_double2(v.x * g2, -v.y * g2);
        }
      }
      a.terms[term_idx(pp, j, t, T, a.P)] = out;
    }
    if (warp == 0 && pfl[lane]) {  // per-particle flags: OR over the group's CTAs (K1b reads and clears them)
      if (pvalid) atomicOr(&a.pflag[p], pfl[lane]);
      pfl[lane] = 0;
    }
    __syncthreads();  // the next group's set-up rewrites psf / R64s / acc / pos_s / pfl
    PT(7)
    PT_FLUSH
  }
  // the last CTA to finish resets the claim counter for the next launch (all claims precede every increment)
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(a.sched + 1, 1u) == gridDim.x - 1) {
      a.sched[0] = 0u;
      a.sched[1] = 0u;
      __threadfence();
    }
  }
}

// ---------------------------------------------------------------------------- K1b assembly (row A5)
// One thread per particle, fp64, everything in registers (S is a compile-time constant and every loop is
// unrolled, so the Hermitian S x S matrix lives in NTRI complex registers):
//   g = c - G m; ||e||^2 = ||z||^2 - 2 Re(m^H c) + m^H G m; K = I + V^1/2 G V^1/2 / eta = L L^H;
//   x = L^-1 V^1/2 g; l_j = -Nz ln(pi eta) - 2 sum ln L_ii - ||e||^2/eta + ||x||^2/eta^2;
//   amplitudes: m + V^1/2 L^-H x / eta (LMMSE).
#ifndef CDMS_ASM_T
#define CDMS_ASM_T 64  // threads per block (measured c3 assembly 64: 0.218, 128: 0.234, 256: 0.253 ms; c5 4M 2.53 / 2.54 / 2.68)
#endif
constexpr int ASM_T = CDMS_ASM_T;

template <bool F32>
struct TermT {  // a term as stored: complex64 from K1T, else complex128
  using type = double2;
};
template <>
struct TermT<true> {
  using type = float2;
};
template <bool F32>
__device__ __forceinline__ typename TermT<F32>::type ld_term(const void* terms, int64_t i) {  // streaming, read once
  return __ldcs(static_cast<const typename TermT<F32>::type*>(terms) + i);
}
__device__ __forceinline__ double2 to_d2(float2 v) { return make_double2((double)v.x, (double)v.y); }
__device__ __forceinline__ double2 to_d2(double2 v) { return v; }
// Per-call constants (scene, not particle, quantities) are formed once per block in shared memory: w_js =
// sqrt(v_js / eta_j) (K = I + W G W), sv_js = sqrt(v_js), 1/eta_j and N_z ln(pi eta_j); each pivot takes one fp64
// rsqrt (L_qq = d rsqrt(d), its reciprocal kept in the diagonal's unused imaginary slot for the substitutions) and
// ln det K = ln prod_q d_q is one log per (particle, PA).  Measured c5 4M: 6.13 -> 2.60 ms, c3 0.434 -> 0.235 ms (the per-element divisions
// by eta, the per-pivot sqrt, division and log were most of the kernel's instructions).
template <int S, bool F32>
__global__ void __launch_bounds__(ASM_T) assemble_kernel(const __grid_constant__ SceneDev sc, const AsmArgs a) {
  constexpr int NTRI = S * (S + 1) / 2;
  constexpr int T = S + NTRI;
  __shared__ double s_w[MAXJ][S], s_sv[MAXJ][S], s_ieta[MAXJ], s_lz[MAXJ];
  const int J = sc.J;
  const double nz = (double)sc.nf * (double)sc.Na;
  for (int i = threadIdx.x; i < J * S; i += ASM_T) {
    const int j = i / S, s = i - j * S;
    s_w[j][s] = sqrt(sc.v[j][s] / sc.eta[j]);
    s_sv[j][s] = sqrt(sc.v[j][s]);
    if (s == 0) {
      s_ieta[j] = 1.0 / sc.eta[j];
      s_lz[j] = -nz * log(PI * sc.eta[j]);
    }
  }
  __syncthreads();
  const int64_t p = (int64_t)blockIdx.x * ASM_T + threadIdx.x;  // processing index (terms, pflag)
  if (p >= a.P) return;
  const int64_t po = a.perm ? (int64_t)a.perm[p] : p;             // particle index (outputs)
  double l = a.logw_prior ? a.logw_prior[po] : 0.0;
  for (int j = 0; j < J; ++j) {
    const double ieta = s_ieta[j];
    // one pass over the terms: c_s gives m^H c and b = V^1/2 c; each G_rq (r >= q) as it arrives updates
    // b -= V^1/2 G m (both triangle halves) and m^H G m, and is then scaled in place to K_rq = delta_rq + w_r w_q G_rq,
    // so neither c nor a second copy of G stays live into the factorization (S = 9: no register spills)
    // (all loads first, in the stored precision: the optional output stores below could alias them)
    typename TermT<F32>::type craw[S], graw[NTRI];
#pragma unroll
    for (int s = 0; s < S; ++s) craw[s] = ld_term<F32>(a.terms, term_idx(p, j, s, T, a.P));
#pragma unroll
    for (int t = 0; t < NTRI; ++t) graw[t] = ld_term<F32>(a.terms, term_idx(p, j, S + t, T, a.P));
    double mhc = 0.0, mGm = 0.0;
    double2 b[S], k[NTRI];
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const double2 cs = to_d2(craw[s]);
      if (a.term_c != nullptr) a.term_c[(po * J + j) * S + s] = cs;
      mhc += sc.m_re[j][s] * cs.x + sc.m_im[j][s] * cs.y;
      b[s] = make_double2(s_sv[j][s] * cs.x, s_sv[j][s] * cs.y);
    }
#pragma unroll
    for (int r = 0; r < S; ++r) {
      const double mr = sc.m_re[j][r], mi = sc.m_im[j][r], svr = s_sv[j][r], wr = s_w[j][r];
#pragma unroll
      for (int q = 0; q <= r; ++q) {
        const double2 G = to_d2(graw[tri(r, q)]);  // G_rq, r >= q
        if (a.term_G != nullptr) {  // (c and G are independent outputs: the birth proposal reads c only)
          a.term_G[((po * J + j) * S + r) * S + q] = G;
          if (q < r) a.term_G[((po * J + j) * S + q) * S + r] = make_double2(G.x, -G.y);
        }
        const double nr = sc.m_re[j][q], ni = sc.m_im[j][q];
        const double gr = G.x * nr - G.y * ni, gi = G.x * ni + G.y * nr;  // G_rq m_q
        b[r].x -= svr * gr;
        b[r].y -= svr * gi;
        const double mg = mr * gr + mi * gi;  // Re(conj(m_r) G_rq m_q)
        if (q < r) {
          const double hr = G.x * mr + G.y * mi, hi = G.x * mi - G.y * mr;  // conj(G_rq) m_r
          b[q].x -= s_sv[j][q] * hr;
          b[q].y -= s_sv[j][q] * hi;
          mGm += 2.0 * mg;
        } else {
          mGm += mg;
        }
        const double f = wr * s_w[j][q];
        k[tri(r, q)] = make_double2((r == q ? 1.0 : 0.0) + G.x * f, G.y * f);
      }
    }
    const double e2 = a.ynorm2[j] - 2.0 * mhc + mGm;
    // Cholesky factor L of K (lower, in place)
    double det = 1.0;
    bool okc = true;
#pragma unroll
    for (int q = 0; q < S; ++q) {
      double d = k[tri(q, q)].x;
#pragma unroll
      for (int t = 0; t < S; ++t)
        if (t < q) d -= k[tri(q, t)].x * k[tri(q, t)].x + k[tri(q, t)].y * k[tri(q, t)].y;
      okc &= d > 0.0;
      d = fmax(d, 1e-300);
      det *= d;
      const double inv = rsqrt(d);
      k[tri(q, q)] = make_double2(d * inv, inv);  // (L_qq, 1 / L_qq)
#pragma unroll
      for (int i = 0; i < S; ++i) {
        if (i <= q) continue;
        double2 ac = k[tri(i, q)];
#pragma unroll
        for (int t = 0; t < S; ++t) {
          if (t >= q) continue;
          const double2 li = k[tri(i, t)], lk = k[tri(q, t)];
          ac.x -= li.x * lk.x + li.y * lk.y;  // ac -= L_it conj(L_qt)
          ac.y -= li.y * lk.x - li.x * lk.y;
        }
        k[tri(i, q)] = make_double2(ac.x * inv, ac.y * inv);
      }
    }
    // x = L^-1 b (forward substitution), ||x||^2
    double x2 = 0.0;
#pragma unroll
    for (int r = 0; r < S; ++r) {
      double2 t = b[r];
#pragma unroll
      for (int q = 0; q < S; ++q) {
        if (q >= r) continue;
        const double2 lr = k[tri(r, q)];
        t.x -= lr.x * b[q].x - lr.y * b[q].y;
        t.y -= lr.x * b[q].y + lr.y * b[q].x;
      }
      const double li = k[tri(r, r)].y;
      b[r] = make_double2(t.x * li, t.y * li);
      x2 += b[r].x * b[r].x + b[r].y * b[r].y;
    }
    double lj = s_lz[j] - log(det) - e2 * ieta + x2 * (ieta * ieta);
    if (!okc || !(lj == lj)) lj = -INFINITY;
    l += lj;
    if (a.amp != nullptr) {
      // L^H u = x (back substitution), amplitudes m + V^1/2 u / eta
#pragma unroll
      for (int r = S - 1; r >= 0; --r) {
        double2 t = b[r];
#pragma unroll
        for (int q = 0; q < S; ++q) {
          if (q <= r) continue;
          const double2 lk = k[tri(q, r)];  // (L^H)_rq = conj(L_qr)
          t.x -= lk.x * b[q].x + lk.y * b[q].y;
          t.y -= lk.x * b[q].y - lk.y * b[q].x;
        }
        const double li = k[tri(r, r)].y;
        b[r] = make_double2(t.x * li, t.y * li);
      }
#pragma unroll
      for (int s = 0; s < S; ++s)
        a.amp[(po * J + j) * S + s] = make_double2(sc.m_re[j][s] + s_sv[j][s] * b[s].x * ieta,
                                                   sc.m_im[j][s] + s_sv[j][s] * b[s].y * ieta);
    }
  }
  const int pf = a.pflag[p];
  if (pf) a.pflag[p] = 0;  // K1 ORs into a zeroed buffer
  if (pf) {
    l = -INFINITY;
    atomicOr(a.flags, (pf & 2) ? (FLAG_NAN | FLAG_DEGENERATE) : FLAG_DEGENERATE);
  } else if (!(l == l)) {
    atomicOr(a.flags, FLAG_NAN);
  }
  a.loglik[po] = l;
}

// ---------------------------------------------------------------------------- launch
int corr_kchunk(int S) { return kchunk_for(S); }

// Persistent grid: every resident CTA (latency hiding), at most one CTA per (tile, PA) group.  0 on error.
template <typename K>
static int64_t grid_for_kernel(K kern, int threads, size_t smem, int64_t n_groups, int num_sms) {
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
  // the persistent grid assumes every CTA resident at once: ask for the full shared-memory carveout (a smaller
  // driver-chosen one would run the excess CTAs as a second wave)
  if (cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared) !=
      cudaSuccess)
    return 0;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) != cudaSuccess) return 0;
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)per_sm * num_sms;
  if (grid > n_groups) grid = n_groups;
  return grid < 1 ? 1 : grid;
}

template <int S, typename RT>
static int64_t corr_grid_t(const SceneDev& sc, int64_t n_tiles, int num_sms) {
  if (sc.two_seg) return grid_for_kernel(corr_kernel<S, RT, true>, NTHREADS, Plan<S, RT>::total, n_tiles * sc.J, num_sms);
  return grid_for_kernel(corr_kernel<S, RT, false>, NTHREADS, Plan<S, RT>::total, n_tiles * sc.J, num_sms);
}

template <int S, typename RT>
static cudaError_t launch_corr_t(const SceneDev& sc, const CorrArgs& a, cudaStream_t st) {
  if (a.grid < 1 || a.n_groups < 1) return cudaSuccess;
  if (sc.two_seg)
    corr_kernel<S, RT, true><<<(unsigned)a.grid, NTHREADS, Plan<S, RT>::total, st>>>(sc, a);
  else
    corr_kernel<S, RT, false><<<(unsigned)a.grid, NTHREADS, Plan<S, RT>::total, st>>>(sc, a);
  return cudaGetLastError();
}

int64_t corr_grid(const SceneDev& sc, int64_t n_tiles, int precision, int num_sms) {
  switch (sc.S) {
#define CASE_S(n) \
  case n: return precision == CDMS_FP64 ? corr_grid_t<n, double>(sc, n_tiles, num_sms) \
                                        : corr_grid_t<n, float>(sc, n_tiles, num_sms);
    CASE_S(1) CASE_S(2) CASE_S(3) CASE_S(4) CASE_S(5) CASE_S(6) CASE_S(7) CASE_S(8) CASE_S(9)
#undef CASE_S
    default: return 0;
  }
}

cudaError_t launch_corr(const SceneDev& sc, const CorrArgs& a, int precision, cudaStream_t st) {
  switch (sc.S) {
#define CASE_S(n) \
  case n: return precision == CDMS_FP64 ? launch_corr_t<n, double>(sc, a, st) \
                                        : launch_corr_t<n, float>(sc, a, st);
    CASE_S(1) CASE_S(2) CASE_S(3) CASE_S(4) CASE_S(5) CASE_S(6) CASE_S(7) CASE_S(8) CASE_S(9)
#undef CASE_S
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_assemble(const SceneDev& sc, const AsmArgs& a, cudaStream_t st) {
  if (a.P <= 0) return cudaSuccess;
  const unsigned grid = (unsigned)((a.P + ASM_T - 1) / ASM_T);
  switch (sc.S) {
#define CASE_S(n)                                                \
  case n:                                                        \
    if (a.terms_f32) assemble_kernel<n, true><<<grid, ASM_T, 0, st>>>(sc, a); \
    else assemble_kernel<n, false><<<grid, ASM_T, 0, st>>>(sc, a);           \
    break;
    CASE_S(1) CASE_S(2) CASE_S(3) CASE_S(4) CASE_S(5) CASE_S(6) CASE_S(7) CASE_S(8) CASE_S(9)
#undef CASE_S
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace cdms
