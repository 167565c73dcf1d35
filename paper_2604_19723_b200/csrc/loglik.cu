// loglik.cu -- rows A2-A5 of the hot path on sm_100a: correlation c = Psi^H z by segmented Horner
// recurrences over the (never materialized) spherical/planar wideband responses, the closed-form Gram
// G = Psi^H Psi, and the S x S low-rank assembly of the coherent log-likelihood of the MT update message
// iota~ (Supplement S-V-C).  DESIGN.md "Kernels" describes the work decomposition.
//
// CTA = 32 particles (lanes) x 8 antennas (warps).  For each PA j and each block of 8 antennas the CTA
// streams y^(j) through shared memory in chunks of <= 256 subcarriers x 8 antennas with 1-D bulk TMA
// (cp.async.bulk + mbarrier, double buffered); every lane keeps the S Horner accumulators of its
// (particle, antenna) pair in registers and reads y by a broadcast LDS.  Per (particle, component) the
// geometry and the phase bases are fp64; the per-element loop is FP32 (or FP64 in CDMS_FP64 mode).
#include <math.h>

#include "cdms_internal.h"
#include "geometry.cuh"

namespace cdms {

// ---------------------------------------------------------------------------- y re-layout
// y [J][nf][Na] (paper vec order) -> ytiles [J][n_mb][n_kc][kc_len][NWARP] (zero padded), and
// ||z^(j)||^2 in fp64 (one block per PA, fixed reduction order).
__global__ void prep_y_kernel(const SceneDev sc, const float2* __restrict__ y, float2* __restrict__ yt,
                              double* __restrict__ ynorm2) {
  const int j = blockIdx.y;
  const int64_t per_j = (int64_t)sc.n_mb * sc.n_kc * sc.kc_len * NWARP;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < per_j;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int w = (int)(t % NWARP);
    int64_t rest = t / NWARP;
    const int kl = (int)(rest % sc.kc_len);
    rest /= sc.kc_len;
    const int kc = (int)(rest % sc.n_kc);
    const int mb = (int)(rest / sc.n_kc);
    const int m = mb * NWARP + w, k = kc * sc.kc_len + kl;
    float2 v = make_float2(0.f, 0.f);
    if (m < sc.Na && k < sc.nf) v = y[((int64_t)j * sc.nf + k) * sc.Na + m];
    yt[(int64_t)j * per_j + t] = v;
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

cudaError_t launch_prep_y(const SceneDev& sc, const float2* y, float2* ytiles, double* ynorm2, cudaStream_t st) {
  const int64_t per_j = (int64_t)sc.n_mb * sc.n_kc * sc.kc_len * NWARP;
  int gx = (int)((per_j + 255) / 256);
  if (gx > 1024) gx = 1024;
  dim3 grid(gx, sc.J);
  prep_y_kernel<<<grid, 256, 0, st>>>(sc, y, ytiles, ynorm2);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------- shared memory plan
template <int S, typename RT>
struct SmemPlan {
  static constexpr int NPAIR = S * (S - 1) / 2;
  static constexpr int NTRI = S * (S + 1) / 2;
  static constexpr int PPW = NPAIR > 0 ? (NPAIR + NWARP - 1) / NWARP : 1;  // Gram pairs per warp
  static constexpr int CPW = (S + NWARP - 1) / NWARP;                      // components per warp
  // TMA y buffers: 2 x KCHUNK x NWARP complex64
  static constexpr size_t ybuf = 2ull * KCHUNK * NWARP * sizeof(float2);
  // per (s, particle) set-up fields [12][S][32] and fp64 ranges [S][32]
  static constexpr size_t ps =
      (size_t)NPSF * S * TILE_P * sizeof(RT) + (size_t)(NPSD + 1) * S * TILE_P * sizeof(double);
  // offsets Delta of the current and previous antenna block [2][S][8][32]
  static constexpr size_t dlt = 2ull * S * NWARP * TILE_P * sizeof(RT);
  // thread-private running sums of c (CPW) and G (PPW) over the antennas, complex fp64 [(CPW+PPW)][256]
  static constexpr size_t acc = (size_t)(CPW + PPW) * NTHREADS * 2 * sizeof(double);
  // staging of one block's per-antenna correlations [S][8][32] complex RT, aliased by the fp64
  // assembly workspace: c [S][32], vector [S][32], lower-tri K [NTRI][32] (complex)
  static constexpr size_t stage_c = (size_t)S * NWARP * TILE_P * 2 * sizeof(RT);
  static constexpr size_t work = (size_t)(2 * S + NTRI) * TILE_P * sizeof(double2);
  static constexpr size_t stage = stage_c > work ? stage_c : work;
  static constexpr size_t misc = 64 + TILE_P * 4 * sizeof(double) + TILE_P * sizeof(int);
  static constexpr size_t total = ybuf + ps + dlt + acc + stage + misc;
};

// lower-triangle index of (r, c), r >= c
__host__ __device__ constexpr int tri(int r, int c) { return r * (r + 1) / 2 + c; }

// pair q -> (a, b), a < b, enumerated row by row: (0,1), (0,2), ..., (1,2), ...
__device__ __forceinline__ void pair_ab(int q, int S, int& a, int& b) {
  int aa = 0, rem = q;
  while (rem >= S - 1 - aa) {
    rem -= S - 1 - aa;
    ++aa;
  }
  a = aa;
  b = aa + 1 + rem;
}

// ---------------------------------------------------------------------------- row A5 (assembly)
// One lane = one particle, fp64, vectors and the S x S matrix in shared memory columns [item][32]:
//   c_s, G_ab with path-loss gains; g = c - G m; ||e||^2 = ||z||^2 - 2 Re(m^H c) + m^H G m;
//   K = I + V^1/2 G V^1/2 / eta = L L^H; x = L^-1 V^1/2 g;
//   l_j = -Nz ln(pi eta) - 2 sum ln L_ii - ||e||^2/eta + ||x||^2/eta^2
//   amplitudes (optional): m + V^1/2 L^-H x / eta  (LMMSE).
// wc: c [S][32]; wv: path-loss gains (.x) on entry, then scratch [S][32]; wk: lower-tri G on entry,
// L on exit [NTRI][32].
template <int S>
__device__ __noinline__ double assemble_lane(const SceneDev& sc, int j, int lane, double2* wc, double2* wv,
                                             double2* wk, double ynorm2, double2* amp_out) {
  const double eta = sc.eta[j];
#pragma unroll 1
  for (int s = 0; s < S; ++s) {
    const double gs = wv[s * TILE_P + lane].x;
    double2 c = wc[s * TILE_P + lane];
    wc[s * TILE_P + lane] = make_double2(c.x * gs, c.y * gs);
#pragma unroll 1
    for (int t = 0; t <= s; ++t) {
      const double gg = gs * wv[t * TILE_P + lane].x;
      double2 G = wk[tri(s, t) * TILE_P + lane];
      wk[tri(s, t) * TILE_P + lane] = make_double2(G.x * gg, G.y * gg);
    }
  }
  // g = c - G m (G Hermitian from its lower triangle), Re(m^H c), Re(m^H G m)
  double mhc = 0.0, mGm = 0.0;
#pragma unroll 1
  for (int r = 0; r < S; ++r) {
    const double2 c = wc[r * TILE_P + lane];
    double gmr = 0.0, gmi = 0.0;
#pragma unroll 1
    for (int t = 0; t < S; ++t) {
      double2 G = (r >= t) ? wk[tri(r, t) * TILE_P + lane] : wk[tri(t, r) * TILE_P + lane];
      if (r < t) G.y = -G.y;
      const double mr = sc.m_re[j][t], mi = sc.m_im[j][t];
      gmr += G.x * mr - G.y * mi;
      gmi += G.x * mi + G.y * mr;
    }
    const double mr = sc.m_re[j][r], mi = sc.m_im[j][r];
    mhc += mr * c.x + mi * c.y;
    mGm += mr * gmr + mi * gmi;
    const double sv = sqrt(sc.v[j][r]);
    wv[r * TILE_P + lane] = make_double2(sv * (c.x - gmr), sv * (c.y - gmi));  // b = V^1/2 g
  }
  const double e2 = ynorm2 - 2.0 * mhc + mGm;
  // K = I + V^1/2 G V^1/2 / eta (lower triangle, in place)
#pragma unroll 1
  for (int r = 0; r < S; ++r)
#pragma unroll 1
    for (int t = 0; t <= r; ++t) {
      const double f = sqrt(sc.v[j][r]) * sqrt(sc.v[j][t]) / eta;
      const double2 G = wk[tri(r, t) * TILE_P + lane];
      wk[tri(r, t) * TILE_P + lane] = make_double2((r == t ? 1.0 : 0.0) + G.x * f, G.y * f);
    }
  // Cholesky K = L L^H
  double logdet = 0.0;
  bool okc = true;
#pragma unroll 1
  for (int q = 0; q < S; ++q) {
    double d = wk[tri(q, q) * TILE_P + lane].x;
#pragma unroll 1
    for (int k = 0; k < q; ++k) {
      const double2 l = wk[tri(q, k) * TILE_P + lane];
      d -= l.x * l.x + l.y * l.y;
    }
    okc &= d > 0.0;
    const double lqq = sqrt(fmax(d, 1e-300));
    logdet += 2.0 * log(lqq);
    wk[tri(q, q) * TILE_P + lane] = make_double2(lqq, 0.0);
#pragma unroll 1
    for (int i = q + 1; i < S; ++i) {
      double2 acc = wk[tri(i, q) * TILE_P + lane];
#pragma unroll 1
      for (int k = 0; k < q; ++k) {
        const double2 li = wk[tri(i, k) * TILE_P + lane], lq = wk[tri(q, k) * TILE_P + lane];
        acc.x -= li.x * lq.x + li.y * lq.y;  // acc -= L_ik conj(L_qk)
        acc.y -= li.y * lq.x - li.x * lq.y;
      }
      wk[tri(i, q) * TILE_P + lane] = make_double2(acc.x / lqq, acc.y / lqq);
    }
  }
  // forward solve L x = b (x overwrites wv)
  double x2 = 0.0;
#pragma unroll 1
  for (int r = 0; r < S; ++r) {
    double2 b = wv[r * TILE_P + lane];
#pragma unroll 1
    for (int k = 0; k < r; ++k) {
      const double2 l = wk[tri(r, k) * TILE_P + lane], xk = wv[k * TILE_P + lane];
      b.x -= l.x * xk.x - l.y * xk.y;
      b.y -= l.x * xk.y + l.y * xk.x;
    }
    const double ld = wk[tri(r, r) * TILE_P + lane].x;
    const double2 xr = make_double2(b.x / ld, b.y / ld);
    wv[r * TILE_P + lane] = xr;
    x2 += xr.x * xr.x + xr.y * xr.y;
  }
  const double nz = (double)sc.nf * (double)sc.Na;
  double l = -nz * log(PI * eta) - logdet - e2 / eta + x2 / (eta * eta);
  if (!okc || !(l == l)) l = -INFINITY;
  if (amp_out != nullptr) {
    // back solve L^H t = x, amp = m + V^1/2 t / eta
#pragma unroll 1
    for (int r = S - 1; r >= 0; --r) {
      double2 t = wv[r * TILE_P + lane];
#pragma unroll 1
      for (int k = r + 1; k < S; ++k) {
        const double2 lk = wk[tri(k, r) * TILE_P + lane], xk = wv[k * TILE_P + lane];  // (L^H)_rk = conj(L_kr)
        t.x -= lk.x * xk.x + lk.y * xk.y;
        t.y -= lk.x * xk.y - lk.y * xk.x;
      }
      const double ld = wk[tri(r, r) * TILE_P + lane].x;
      wv[r * TILE_P + lane] = make_double2(t.x / ld, t.y / ld);
    }
#pragma unroll 1
    for (int s = 0; s < S; ++s) {
      const double sv = sqrt(sc.v[j][s]);
      const double2 t = wv[s * TILE_P + lane];
      amp_out[s] = make_double2(sc.m_re[j][s] + sv * t.x / eta, sc.m_im[j][s] + sv * t.y / eta);
    }
  }
  return l;
}

// ---------------------------------------------------------------------------- the hot kernel
template <int S, typename RT>
__global__ void __launch_bounds__(NTHREADS, (sizeof(RT) == 4) ? 2 : 1)
    loglik_kernel(const __grid_constant__ SceneDev sc, const LoglikArgs a) {
  using Plan = SmemPlan<S, RT>;
  constexpr int NPAIR = Plan::NPAIR;
  constexpr int PPW = Plan::PPW;
  constexpr int CPW = Plan::CPW;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* sp = smem;
  float2* ybuf = reinterpret_cast<float2*>(sp);                        sp += Plan::ybuf;
  RT* psf = reinterpret_cast<RT*>(sp);                                 // [NPSF][S][32]
  double* psd = reinterpret_cast<double*>(sp + (size_t)NPSF * S * TILE_P * sizeof(RT));  // [NPSD][S][32]
  double* R64s = psd + NPSD * S * TILE_P;                              // [S][32]
  sp += Plan::ps;
  RT* dlt = reinterpret_cast<RT*>(sp);                                 sp += Plan::dlt;   // [2][S][8][32]
  double* accs = reinterpret_cast<double*>(sp);                        sp += Plan::acc;   // [CPW+PPW][256][2]
  RT* cst = reinterpret_cast<RT*>(sp);                                 // [S][8][32][2]
  double2* wc = reinterpret_cast<double2*>(sp);                        // [S][32]  (aliases cst)
  double2* wv = wc + S * TILE_P;                                       // [S][32]
  double2* wk = wv + S * TILE_P;                                       // [NTRI][32]
  sp += Plan::stage;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sp);
  double* pos_s = reinterpret_cast<double*>(sp + 64);                  // [3][32]
  int* degen = reinterpret_cast<int*>(sp + 64 + TILE_P * 4 * sizeof(double));

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int J = sc.J, Na = sc.Na, nf = sc.nf, kcl = sc.kc_len;
  const int n_mb = sc.n_mb, n_kc = sc.n_kc;
  const int64_t chunks_per_tile = (int64_t)J * n_mb * n_kc;
  const uint32_t chunk_bytes = (uint32_t)(kcl * NWARP * sizeof(float2));
  const int64_t my_tiles =
      (a.n_tiles > (int64_t)blockIdx.x) ? (a.n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total_chunks = my_tiles * chunks_per_tile;

  auto issue = [&](int64_t c) {
    const int64_t f = c % chunks_per_tile;  // (j, mb, kc) flattened: the same sequence for every tile
    uint64_t* bar = &mbar[c & 1];
    fence_proxy_async();
    mbar_expect_tx(bar, chunk_bytes);
    tma_load_1d(ybuf + (c & 1) * (KCHUNK * NWARP), a.ytiles + f * (int64_t)kcl * NWARP, chunk_bytes, bar);
  };

  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    if (total_chunks > 0) issue(0);
    if (total_chunks > 1) issue(1);
  }

  int64_t ci = 0;  // flat chunk counter of this CTA
  for (int64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
    const int64_t p = tile * TILE_P + lane;
    const bool pvalid = p < a.P;
    if (warp == 0) {
      for (int c = 0; c < 3; ++c) pos_s[c * TILE_P + lane] = pvalid ? a.particles[p * a.pstride + c] : 1.0;
      degen[lane] = 0;
    }
    double lsum = 0.0;  // warp 0: l_p accumulated over the PAs
    if (warp == 0 && pvalid) lsum = a.logw_prior ? a.logw_prior[p] : 0.0;
    __syncthreads();

    for (int j = 0; j < J; ++j) {
      // ---- per (s, particle) set-up in fp64 (rows A1/A2)
      for (int it = tid; it < S * TILE_P; it += NTHREADS) {
        const int s = it / TILE_P, pl = it - s * TILE_P;
        const int64_t pp = tile * TILE_P + pl;
        const double pos[3] = {pos_s[pl], pos_s[TILE_P + pl], pos_s[2 * TILE_P + pl]};
        const double* sfv_s = nullptr;
        if (s > 0) sfv_s = a.sfv + ((a.sfv_pp && pp < a.P) ? pp * 3 * sc.K : 0) + 3 * (s - 1);
        PSField<RT> f;
        double R64 = 1.0;
        const int st = setup_ps<RT>(sc, j, pos, sfv_s, f, R64);
        if (st != PS_OK && pp < a.P) {
          atomicOr(&degen[pl], 1);
          if (st == PS_BADSFV || !(pos[0] == pos[0] && pos[1] == pos[1] && pos[2] == pos[2]))
            atomicOr(a.flags, FLAG_NAN);  // invalid input -> CDMS_EINVAL at sync
        }
        const RT* fv = reinterpret_cast<const RT*>(&f);
#pragma unroll
        for (int q = 0; q < NPSF; ++q) psf[(q * S + s) * TILE_P + pl] = fv[q];
        psd[(0 * S + s) * TILE_P + pl] = f.Wr;
        psd[(1 * S + s) * TILE_P + pl] = f.Wi;
        psd[(2 * S + s) * TILE_P + pl] = f.Zr;
        psd[(3 * S + s) * TILE_P + pl] = f.Zi;
        R64s[s * TILE_P + pl] = R64;
      }
#pragma unroll
      for (int u = 0; u < CPW + PPW; ++u) {
        accs[(u * NTHREADS + tid) * 2] = 0.0;
        accs[(u * NTHREADS + tid) * 2 + 1] = 0.0;
      }
      __syncthreads();

      for (int mb = 0; mb < n_mb; ++mb) {
        const int m = mb * NWARP + warp;
        const bool mvalid = m < Na;
        RT* dcur = dlt + (mb & 1) * (S * NWARP * TILE_P);
        // ---- per (s, antenna) offsets and phasors (row A2)
        RT Ar[S], Ai[S], wr[S], wi[S], Zr[S], Zi[S], cr[S], cm[S];
        {
          double v64[3], q264;
          template_col(sc, j, mvalid ? m : 0, v64, q264);
          const RT v[3] = {(RT)v64[0], (RT)v64[1], (RT)v64[2]};
          const RT q2 = (RT)q264;
          bool deg_any = false;
#pragma unroll
          for (int s = 0; s < S; ++s) {
            PSField<RT> f;
            RT* fv = reinterpret_cast<RT*>(&f);
#pragma unroll
            for (int q = 0; q < NPSF; ++q) fv[q] = psf[(q * S + s) * TILE_P + lane];
            f.Wr = psd[(0 * S + s) * TILE_P + lane];
            f.Wi = psd[(1 * S + s) * TILE_P + lane];
            f.Zr = psd[(2 * S + s) * TILE_P + lane];
            f.Zi = psd[(3 * S + s) * TILE_P + lane];
            SMPhasors<RT> o;
            bool dg;
            setup_sm<RT>(sc, f, v, q2, m, s, o, dg);
            deg_any |= dg;
            Ar[s] = o.Ar; Ai[s] = o.Ai; wr[s] = o.wr; wi[s] = o.wi; Zr[s] = o.Zr; Zi[s] = o.Zi;
            cr[s] = RT(0); cm[s] = RT(0);
            dcur[(s * NWARP + warp) * TILE_P + lane] = o.delta;
          }
          if (deg_any && mvalid && pvalid) atomicOr(&degen[lane], 1);
        }
        // ---- correlation over all subcarriers (row A3): segmented Horner on TMA-staged y chunks
        for (int kc = 0; kc < n_kc; ++kc, ++ci) {
          mbar_wait(&mbar[ci & 1], (uint32_t)((ci >> 1) & 1));
          const float2* yb = ybuf + (ci & 1) * (KCHUNK * NWARP) + warp;
          const int k_begin = kc * kcl;
          const int k_end = min(k_begin + kcl, nf);
          for (int k0 = k_begin; k0 < k_end; k0 += SEG) {
            const int k1 = min(k0 + SEG, k_end);
            RT hr[S], hi[S];
#pragma unroll
            for (int s = 0; s < S; ++s) { hr[s] = RT(0); hi[s] = RT(0); }
            const float2* yk = yb + (k1 - 1 - k_begin) * NWARP;  // Horner runs from the top subcarrier down
            auto step = [&](const float2 yv) {
              const RT yr = (RT)yv.x, yi = (RT)yv.y;
#pragma unroll
              for (int s = 0; s < S; ++s) {
                const RT t = fma(-hi[s], wi[s], yr);
                const RT u = fma(hi[s], wr[s], yi);
                const RT nr = fma(hr[s], wr[s], t);
                const RT ni = fma(hr[s], wi[s], u);
                hr[s] = nr;
                hi[s] = ni;
              }
            };
            if (k1 - k0 == SEG) {
#pragma unroll 8
              for (int i = 0; i < SEG; ++i) step(yk[-i * NWARP]);
            } else {
              for (int i = 0; i < k1 - k0; ++i) step(yk[-i * NWARP]);
            }
            // c += A_seg H_seg ; A_seg <- A_seg Z
#pragma unroll
            for (int s = 0; s < S; ++s) {
              cr[s] = fma(Ar[s], hr[s], fma(-Ai[s], hi[s], cr[s]));
              cm[s] = fma(Ar[s], hi[s], fma(Ai[s], hr[s], cm[s]));
              const RT nAr = Ar[s] * Zr[s] - Ai[s] * Zi[s];
              const RT nAi = Ar[s] * Zi[s] + Ai[s] * Zr[s];
              Ar[s] = nAr;
              Ai[s] = nAi;
            }
          }
          __syncthreads();  // every warp is done with this buffer (and, at kc = 0, with the previous
                            // block's staging reads)
          if (tid == 0 && ci + 2 < total_chunks) issue(ci + 2);
        }
        // ---- stage this antenna block's correlations
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const int o = (s * NWARP + warp) * TILE_P + lane;
          cst[2 * o] = mvalid ? cr[s] : RT(0);
          cst[2 * o + 1] = mvalid ? cm[s] : RT(0);
        }
        __syncthreads();
        const int nw_valid = min(NWARP, Na - mb * NWARP);
        // c_s += sum over the block's antennas in ascending m (this thread owns s = warp + 8u)
#pragma unroll
        for (int u = 0; u < CPW; ++u) {
          const int s = warp + u * NWARP;
          if (s < S) {
            double sr = accs[(u * NTHREADS + tid) * 2], si = accs[(u * NTHREADS + tid) * 2 + 1];
            for (int w2 = 0; w2 < nw_valid; ++w2) {
              const int o = (s * NWARP + w2) * TILE_P + lane;
              sr += (double)cst[2 * o];
              si += (double)cst[2 * o + 1];
            }
            accs[(u * NTHREADS + tid) * 2] = sr;
            accs[(u * NTHREADS + tid) * 2 + 1] = si;
          }
        }
        // ---- Gram (row A4), closed form on the uniform grid (this thread owns pairs q = warp + 8u):
        //   G_ab = e^{j 2 pi (R_a - R_b) fc/c} sum_m e^{j 2 pi (D_a,m - D_b,m) fc/c} D_N((d_a,m - d_b,m) df/c)
        //   [NB: D_N((R_a - R_b) df/c) e^{j 2 pi (R_a - R_b) fc/c} sum_m e^{j 2 pi (D_a,m - D_b,m) fc/c}].
        // The factors shared by every antenna (base carrier; NB's Dirichlet) are applied once, in fp64, at
        // the hand-off below, so that their rounding does not repeat coherently over the antennas.
#pragma unroll
        for (int u = 0; u < PPW; ++u) {
          const int q = warp + u * NWARP;
          if (q < NPAIR) {
            int pa, pb;
            pair_ab(q, S, pa, pb);
            double gr = accs[((CPW + u) * NTHREADS + tid) * 2], gi = accs[((CPW + u) * NTHREADS + tid) * 2 + 1];
            if (sc.wavefront == CDMS_PLANAR_NB) {
              for (int w2 = 0; w2 < nw_valid; ++w2) {
                const RT dd = dcur[(pa * NWARP + w2) * TILE_P + lane] - dcur[(pb * NWARP + w2) * TILE_P + lane];
                RT er, ei;
                cis2pi<RT>(dd * (RT)sc.fc_c, er, ei);
                gr += (double)er;
                gi += (double)ei;
              }
            } else {
              const double dR = R64s[pa * TILE_P + lane] - R64s[pb * TILE_P + lane];
              const double xb = dR * sc.df_c;
              const double nb = rint(xb);
              const RT xbr = (RT)(xb - nb);
              const long long nbi = (long long)nb;
              for (int w2 = 0; w2 < nw_valid; ++w2) {
                const RT dd = dcur[(pa * NWARP + w2) * TILE_P + lane] - dcur[(pb * NWARP + w2) * TILE_P + lane];
                RT er, ei;
                cis2pi<RT>(dd * (RT)sc.fc_c, er, ei);
                const RT x = xbr + dd * (RT)sc.df_c;
                const RT n2 = Num<RT>::rint_(x);
                const RT D = dirichlet<RT>(x - n2, nbi + (long long)n2, nf);
                gr += (double)(D * er);
                gi += (double)(D * ei);
              }
            }
            accs[((CPW + u) * NTHREADS + tid) * 2] = gr;
            accs[((CPW + u) * NTHREADS + tid) * 2 + 1] = gi;
          }
        }
      }
      __syncthreads();  // all staging reads done: the assembly workspace aliases the staging area
      // ---- hand the per-thread sums to the fp64 assembly workspace
#pragma unroll
      for (int u = 0; u < CPW; ++u) {
        const int s = warp + u * NWARP;
        if (s < S)
          wc[s * TILE_P + lane] = make_double2(accs[(u * NTHREADS + tid) * 2], accs[(u * NTHREADS + tid) * 2 + 1]);
      }
#pragma unroll
      for (int u = 0; u < PPW; ++u) {
        const int q = warp + u * NWARP;
        if (q < NPAIR) {
          int pa, pb;
          pair_ab(q, S, pa, pb);
          // shared factors in fp64: base carrier e^{j 2 pi (R_a - R_b) fc/c}, NB Dirichlet D_N((R_a - R_b) df/c)
          const double dR = R64s[pa * TILE_P + lane] - R64s[pb * TILE_P + lane];
          double sb, cb;
          sincospi(2.0 * frac_c(dR * sc.fc_c), &sb, &cb);
          double D = 1.0;
          if (sc.wavefront == CDMS_PLANAR_NB) {
            const double xb = dR * sc.df_c, nb = rint(xb);
            D = dirichlet<double>(xb - nb, (long long)nb, nf);
          }
          const double ar = accs[((CPW + u) * NTHREADS + tid) * 2], ai = accs[((CPW + u) * NTHREADS + tid) * 2 + 1];
          const double Gr = D * (cb * ar - sb * ai), Gi = D * (cb * ai + sb * ar);
          // lower-triangle entry (b, a) = G_ba = conj(G_ab)
          wk[tri(pb, pa) * TILE_P + lane] = make_double2(Gr, -Gi);
        }
      }
      if (warp == 0) {
        const double nz = (double)nf * (double)Na;  // G_ss = Nz (unit modulus)
        for (int s = 0; s < S; ++s) {
          wk[tri(s, s) * TILE_P + lane] = make_double2(nz, 0.0);
          // the gains travel in wv: the next PA's set-up may overwrite psf while warp 0 assembles
          wv[s * TILE_P + lane] = make_double2((double)psf[(PSF_GAIN * S + s) * TILE_P + lane], 0.0);
        }
      }
      __syncthreads();
      if (warp == 0 && a.term_c != nullptr && pvalid) {  // cdms_loglik_terms: c and full G, gains applied
        for (int r = 0; r < S; ++r) {
          const double gr_ = wv[r * TILE_P + lane].x;
          const double2 cc = wc[r * TILE_P + lane];
          a.term_c[(p * J + j) * S + r] = make_double2(cc.x * gr_, cc.y * gr_);
          for (int t = 0; t < S; ++t) {
            const double g2 = gr_ * wv[t * TILE_P + lane].x;
            double2 G = (r >= t) ? wk[tri(r, t) * TILE_P + lane] : wk[tri(t, r) * TILE_P + lane];
            if (r < t) G.y = -G.y;
            a.term_G[((p * J + j) * S + r) * S + t] = make_double2(G.x * g2, G.y * g2);
          }
        }
      }
      if (warp == 0) {
        double2* amp = (a.amp != nullptr && pvalid) ? a.amp + (p * J + j) * S : nullptr;
        lsum += assemble_lane<S>(sc, j, lane, wc, wv, wk, a.ynorm2[j], amp);
      }
      // the next PA's set-up barrier orders warp 0's use of the workspace before any reuse
    }
    if (warp == 0 && pvalid) {
      if (degen[lane]) {
        lsum = -INFINITY;
        atomicOr(a.flags, FLAG_DEGENERATE);
      } else if (!(lsum == lsum)) {
        atomicOr(a.flags, FLAG_NAN);
      }
      a.loglik[p] = lsum;
    }
    __syncthreads();  // pos_s / degen reuse by the next tile
  }
}

// ---------------------------------------------------------------------------- launch
template <int S, typename RT>
static cudaError_t launch_loglik_t(const SceneDev& sc, const LoglikArgs& a, cudaStream_t st, int num_sms) {
  const size_t smem = SmemPlan<S, RT>::total;
  auto kern = loglik_kernel<S, RT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NTHREADS, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)per_sm * num_sms;
  if (grid > a.n_tiles) grid = a.n_tiles;
  if (grid < 1) return cudaSuccess;
  kern<<<(unsigned)grid, NTHREADS, smem, st>>>(sc, a);
  return cudaGetLastError();
}

template <typename RT>
static cudaError_t dispatch_loglik(const SceneDev& sc, const LoglikArgs& a, cudaStream_t st, int num_sms) {
  switch (sc.S) {
    case 1: return launch_loglik_t<1, RT>(sc, a, st, num_sms);
    case 2: return launch_loglik_t<2, RT>(sc, a, st, num_sms);
    case 3: return launch_loglik_t<3, RT>(sc, a, st, num_sms);
    case 4: return launch_loglik_t<4, RT>(sc, a, st, num_sms);
    case 5: return launch_loglik_t<5, RT>(sc, a, st, num_sms);
    case 6: return launch_loglik_t<6, RT>(sc, a, st, num_sms);
    case 7: return launch_loglik_t<7, RT>(sc, a, st, num_sms);
    case 8: return launch_loglik_t<8, RT>(sc, a, st, num_sms);
    case 9: return launch_loglik_t<9, RT>(sc, a, st, num_sms);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_loglik(const SceneDev& sc, const LoglikArgs& a, int precision, cudaStream_t st, int num_sms) {
  return precision == CDMS_FP64 ? dispatch_loglik<double>(sc, a, st, num_sms)
                                : dispatch_loglik<float>(sc, a, st, num_sms);
}

size_t loglik_smem_bytes(int S, int precision) {
  switch (S) {
#define CASE_S(n) \
  case n: return precision == CDMS_FP64 ? SmemPlan<n, double>::total : SmemPlan<n, float>::total;
    CASE_S(1) CASE_S(2) CASE_S(3) CASE_S(4) CASE_S(5) CASE_S(6) CASE_S(7) CASE_S(8) CASE_S(9)
#undef CASE_S
    default: return 0;
  }
}

}  // namespace cdms
