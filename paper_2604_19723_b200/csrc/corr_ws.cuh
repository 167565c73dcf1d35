// corr_ws.cuh -- K1 with warp specialization (rows A2-A4), included by loglik.cu after the shared device code.
//
// In the plain corr_kernel every warp runs the same phases in lockstep with its CTA (per-antenna set-up,
// Horner, then the Gram terms and antenna sums behind a CTA barrier).  Here each CTA has
//   * 8 Horner warps (warp w = antenna w of every 8-antenna block): the per-(component, antenna) phasors and
//     Delta of their own antenna (A2), the FFMA2 Horner over their own TMA-streamed y chunks (A3), c and
//     Delta to shared memory (double-buffered by block parity) -- no CTA-wide barrier;
//   * 4 auxiliary warps: per group the fp64 set-up records (double-buffered by group parity, prepared one group
//     ahead), per block the Gram terms (A4) and the fp64 antenna sums of c, per group the hand-off.
// Hand-offs use named barriers, each ID used strictly alternately by one producer arrival and one consumer
// wait: PSF_READY / STARTED per group, C_READY_b / C_FREE_b per block parity b.  The arithmetic and the orders
// of summation are the plain kernel's, so the results are identical.  fp32, S <= 5, spherical / planar WB;
// 2 CTAs (24 warps) per SM.  Opt-in (CDMS_WS=1): measured slower than the plain kernel so far.

constexpr int WS_NH = NWARP;                 // Horner warps
constexpr int WS_NA = 4;                     // auxiliary warps
constexpr int WS_THREADS = (WS_NH + WS_NA) * 32;
constexpr int WS_KC = 128;                   // subcarriers per TMA chunk
enum { WSB_PSF_READY = 1, WSB_STARTED = 2, WSB_C_READY0 = 3, WSB_C_FREE0 = 5, WSB_AUX = 7 };

__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int S>
struct WSPlan {
  static constexpr int NPAIR = S * (S - 1) / 2;
  static constexpr int T = S + S * (S + 1) / 2;
  static constexpr size_t ybuf = 2ull * WS_KC * WS_NH * sizeof(float4);
  static constexpr size_t psf1 = (size_t)NPSF_PAD * S * TILE_P * sizeof(float) + (size_t)S * TILE_P * sizeof(double);
  static constexpr size_t psf = 2 * psf1;                                            // by group parity
  static constexpr size_t dlt1 = (size_t)S * WS_NH * TILE_P * sizeof(float);
  static constexpr size_t cst1 = (size_t)S * WS_NH * TILE_P * 2 * sizeof(float);
  static constexpr size_t dlt = 2 * dlt1;                                            // by block parity
  static constexpr size_t cst = 2 * cst1;                                            // by block parity
  static constexpr size_t acc = (size_t)(S + NPAIR) * TILE_P * sizeof(double2);
  static constexpr size_t misc = 2 * WS_NH * sizeof(uint64_t) + 2 * 3 * TILE_P * sizeof(double) +
                                 2 * TILE_P * sizeof(int) + 8 * sizeof(unsigned);
  static constexpr size_t total = ybuf + psf + dlt + cst + acc + misc;
};

template <int S>
__global__ void __launch_bounds__(WS_THREADS, 2) corr_ws_kernel(const __grid_constant__ SceneDev sc, const CorrArgs a) {
  using PL = WSPlan<S>;
  constexpr int NPAIR = PL::NPAIR;
  constexpr int T = PL::T;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* sp = smem;
  float4* ybuf = reinterpret_cast<float4*>(sp);                  sp += PL::ybuf;
  unsigned char* psf_base = sp;                                  sp += PL::psf;
  float* dlt2 = reinterpret_cast<float*>(sp);                    sp += PL::dlt;
  float* cst2 = reinterpret_cast<float*>(sp);                    sp += PL::cst;
  double2* acc = reinterpret_cast<double2*>(sp);                 sp += PL::acc;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sp);              // [8][2]
  double* pos2 = reinterpret_cast<double*>(sp + 2 * WS_NH * sizeof(uint64_t));             // [2][3][32]
  int* pfl2 = reinterpret_cast<int*>(pos2 + 2 * 3 * TILE_P);                               // [2][32]
  unsigned* gring = reinterpret_cast<unsigned*>(pfl2 + 2 * TILE_P);                        // [8]
  auto psf_of = [&](int par) { return reinterpret_cast<float*>(psf_base + par * PL::psf1); };
  auto r64_of = [&](int par) {
    return reinterpret_cast<double*>(psf_base + par * PL::psf1 + (size_t)NPSF_PAD * S * TILE_P * sizeof(float));
  };
  auto dlt_of = [&](int64_t B) { return dlt2 + (size_t)(B & 1) * S * WS_NH * TILE_P; };
  auto cst_of = [&](int64_t B) { return cst2 + (size_t)(B & 1) * S * WS_NH * TILE_P * 2; };

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int J = sc.J, Na = sc.Na, nf = sc.nf, n_mb = sc.n_mb, n_kc = sc.n_kc, kcl = sc.kc_len;
  const int Na_pad = n_mb * NWARP;
  const uint32_t n_groups = (uint32_t)a.n_groups;

  if (tid < 2 * WS_NH) mbar_init(&mbar[tid], 1);
  if (tid == 0) {
    fence_mbar_init();
    gring[0] = atomicAdd(a.sched, 1u);
    gring[1] = atomicAdd(a.sched, 1u);
    gring[2] = atomicAdd(a.sched, 1u);
  }
  if (tid < 2 * TILE_P) pfl2[tid] = 0;
  __syncthreads();

  if (warp < WS_NH) {
    // ================================================================== Horner warps
    int is_gi = 0, is_mb = 0, is_kc = 0, is_c = 0;
    uint32_t is_g = 0;
    int64_t is_off = 0;
    auto rebase = [&]() {
      is_g = gring[is_gi & 7];
      is_off = (((int64_t)(is_g % (uint32_t)sc.J) * sc.n_mb * NWARP + warp) * sc.n_kc) * sc.kc_len;
    };
    auto issue = [&]() {
      if (is_g >= n_groups) return;
      uint64_t* bar = &mbar[warp * 2 + (is_c & 1)];
      const uint32_t chunk_bytes = (uint32_t)(sc.kc_len * sizeof(float4));
      mbar_expect_tx(bar, chunk_bytes);
      tma_load_1d(ybuf + (warp * 2 + (is_c & 1)) * WS_KC, a.ytiles + is_off, chunk_bytes, bar);
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
    if (lane == 0) {
      rebase();
      issue();
      issue();
    }
    int64_t ci = 0;
    int64_t B = 0;  // global block counter (same sequence as the auxiliary warps)
    for (int gi = 0;; ++gi) {
      const uint32_t g = gring[gi & 7];
      if (g >= n_groups) break;
      const int64_t tile = g / (uint32_t)J;
      const int j = (int)(g - (uint32_t)tile * (uint32_t)J);
      const int par = gi & 1;
      nbar_sync(WSB_PSF_READY, WS_THREADS);   // this group's set-up records
      nbar_arrive(WSB_STARTED, WS_THREADS);   // the auxiliary warps may now prepare group gi + 1
      const float* psf = psf_of(par);
      int* pfl = pfl2 + par * TILE_P;
      const bool pvalid = tile * TILE_P + lane < a.P;
      for (int mb = 0; mb < n_mb; ++mb, ++B) {
        const int m = mb * WS_NH + warp;
        const bool mvalid = m < Na;
        if (B >= 2) nbar_sync(WSB_C_FREE0 + (int)(B & 1), WS_THREADS);  // block B-2's c / Delta consumed
        float* dlt = dlt_of(B);
        float* cst = cst_of(B);
        // ---- (2) phasors and Delta of this antenna (row A2)
        float Ar[S], Ai[S], Zr[S], Zi[S];
        Horner<S, float> H;
        {
          float wr[S], wi[S];
          const float4 tv = __ldg(&a.tmpl[j * Na_pad + m]);
          const float v[3] = {tv.x, tv.y, tv.z};
          bool deg_any = false;
#pragma unroll
          for (int s = 0; s < S; ++s) {
            PSField<float> f;
            load_psf<float>(psf + (s * TILE_P + lane) * NPSF_PAD, reinterpret_cast<float*>(&f));
            SMPhasors<float> o;
            bool dg;
            setup_sm<float>(sc, f, v, tv.w, m, s, o, dg);
            deg_any |= dg;
            Ar[s] = o.Ar; Ai[s] = o.Ai; wr[s] = o.wr; wi[s] = o.wi; Zr[s] = o.Zr; Zi[s] = o.Zi;
            const int o_ = (s * WS_NH + warp) * TILE_P + lane;
            dlt[o_] = o.delta;
            cst[2 * o_] = 0.f;
            cst[2 * o_ + 1] = 0.f;
          }
          if (deg_any && mvalid && pvalid) atomicOr(&pfl[lane], 1);
          H.init(wr, wi);
        }
        // ---- (3) correlation (row A3)
        for (int kc = 0; kc < n_kc; ++kc, ++ci) {
          mbar_wait(&mbar[warp * 2 + (ci & 1)], (uint32_t)((ci >> 1) & 1));
          const float4* yb = ybuf + (warp * 2 + (ci & 1)) * WS_KC;
          const int k_begin = kc * kcl;
          const int k_end = min(k_begin + kcl, nf);
          for (int k0 = k_begin; k0 < k_end; k0 += SEG) {
            const int k1 = min(k0 + SEG, k_end);
            const float4* yk = yb + (k1 - 1 - k_begin);
            H.reset_to(yk[0]);
            if (k1 - k0 == SEG) {
#pragma unroll 7
              for (int i = 1; i < SEG; ++i) H.step(yk[-i]);
            } else {
              for (int i = 1; i < k1 - k0; ++i) H.step(yk[-i]);
            }
            float hr[S], hi[S];
            H.get(hr, hi);
#pragma unroll
            for (int s = 0; s < S; ++s) {
              const int o_ = (s * WS_NH + warp) * TILE_P + lane;
              cst[2 * o_] = fmaf(Ar[s], hr[s], fmaf(-Ai[s], hi[s], cst[2 * o_]));
              cst[2 * o_ + 1] = fmaf(Ar[s], hi[s], fmaf(Ai[s], hr[s], cst[2 * o_ + 1]));
              const float nAr = Ar[s] * Zr[s] - Ai[s] * Zi[s];
              const float nAi = Ar[s] * Zi[s] + Ai[s] * Zr[s];
              Ar[s] = nAr;
              Ai[s] = nAi;
            }
          }
          __syncwarp();
          if (lane == 0) issue();
        }
        nbar_arrive(WSB_C_READY0 + (int)(B & 1), WS_THREADS);  // this block's c and Delta are complete
      }
    }
    return;
  }

  // ==================================================================== auxiliary warps
  const int at = tid - WS_NH * 32;          // 0..127
  const int aw = at >> 5;                   // auxiliary warp 0..3
  auto aux_sync = [&]() { nbar_sync(WSB_AUX, WS_NA * 32); };

  // per-group fp64 set-up (rows A1/A2) of group g into the records of parity par
  auto setup_group = [&](uint32_t g, int par) {
    const int64_t tile = g / (uint32_t)J;
    const int j = (int)(g - (uint32_t)tile * (uint32_t)J);
    float* psf = psf_of(par);
    double* R64s = r64_of(par);
    double* pos_s = pos2 + par * 3 * TILE_P;
    int* pfl = pfl2 + par * TILE_P;
    if (at < TILE_P) {
      const int64_t p = tile * TILE_P + at;
      const bool pvalid = p < a.P;
#pragma unroll
      for (int c = 0; c < 3; ++c) pos_s[c * TILE_P + at] = pvalid ? a.particles[p * a.pstride + c] : 1.0;
    }
    aux_sync();
    for (int it = at; it < S * TILE_P; it += WS_NA * 32) {
      const int s = it / TILE_P, pl = it - s * TILE_P;
      const int64_t pp = tile * TILE_P + pl;
      const double pos[3] = {pos_s[pl], pos_s[TILE_P + pl], pos_s[2 * TILE_P + pl]};
      const double* sfv_s = nullptr;
      if (s > 0) sfv_s = a.sfv + ((a.sfv_pp && pp < a.P) ? pp * 3 * sc.K : 0) + 3 * (s - 1);
      PSField<float> f;
      double R64 = 1.0;
      const int st = setup_ps<float>(sc, j, pos, sfv_s, f, R64);
      if (st != PS_OK && pp < a.P) {
        const bool bad = st == PS_BADSFV || !(pos[0] == pos[0] && pos[1] == pos[1] && pos[2] == pos[2]);
        atomicOr(&pfl[pl], bad ? 3 : 1);
      }
      const float* fv = reinterpret_cast<const float*>(&f);
#pragma unroll
      for (int q = 0; q < NPSF; ++q) psf[(s * TILE_P + pl) * NPSF_PAD + q] = fv[q];
      R64s[s * TILE_P + pl] = R64;
    }
    aux_sync();
  };

  // block B (group parity par, antenna block mb): Gram terms and fp64 antenna sums of c into acc
  auto finish_block = [&](int64_t B, int par, int mb) {
    nbar_sync(WSB_C_READY0 + (int)(B & 1), WS_THREADS);
    const float* dlt = dlt_of(B);
    const float* cst = cst_of(B);
    const double* R64s = r64_of(par);
    const int nw_valid = min(WS_NH, Na - mb * WS_NH);
    for (int s = (aw - mb) & (WS_NA - 1); s < S; s += WS_NA) {
      double sr = 0.0, si = 0.0;
      for (int w2 = 0; w2 < nw_valid; ++w2) {
        const int o_ = (s * WS_NH + w2) * TILE_P + lane;
        sr += (double)cst[2 * o_];
        si += (double)cst[2 * o_ + 1];
      }
      double2 v = acc[s * TILE_P + lane];
      acc[s * TILE_P + lane] = make_double2(v.x + sr, v.y + si);
    }
    for (int q = (aw - mb) & (WS_NA - 1); q < NPAIR; q += WS_NA) {
      int pa, pb;
      pair_ab(q, S, pa, pb);
      const double dR = R64s[pa * TILE_P + lane] - R64s[pb * TILE_P + lane];
      const double xb = dR * sc.df_c;
      const double nbd = rint(xb);
      GramPairF gp;
      gp.xbr = (float)(xb - nbd);
      gp.nbpar = (uint32_t)((long long)nbd & 1) << 31;
      float fr = 0.f, fi = 0.f;
      for (int w2 = 0; w2 < nw_valid; ++w2) {
        const float dd = dlt[(pa * WS_NH + w2) * TILE_P + lane] - dlt[(pb * WS_NH + w2) * TILE_P + lane];
        gram_term_f(sc, dd, gp, fr, fi);
      }
      double2 v = acc[(S + q) * TILE_P + lane];
      acc[(S + q) * TILE_P + lane] = make_double2(v.x + (double)fr, v.y + (double)fi);
    }
    aux_sync();  // every auxiliary read of this block's c / Delta is done
    nbar_arrive(WSB_C_FREE0 + (int)(B & 1), WS_THREADS);
  };

  // hand-off of group (tile, j) with set-up parity par: c (with gains) and the lower triangle of G -> terms
  auto handoff = [&](uint32_t g, int par) {
    const int64_t tile = g / (uint32_t)J;
    const int j = (int)(g - (uint32_t)tile * (uint32_t)J);
    const float* psf = psf_of(par);
    const double* R64s = r64_of(par);
    const double nz = (double)nf * (double)Na;
    for (int it = at; it < T * TILE_P; it += WS_NA * 32) {
      const int pl = it / T, t = it - pl * T;
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
        const int c = e;
        const double gr_ = (double)psf[(r * TILE_P + pl) * NPSF_PAD + PSF_GAIN];
        const double gc_ = (double)psf[(c * TILE_P + pl) * NPSF_PAD + PSF_GAIN];
        if (r == c) {
          out = make_double2(nz * gr_ * gc_, 0.0);
        } else {
          const int q = pair_index(c, r, S);
          double2 v = acc[(S + q) * TILE_P + pl];
          const double dR = R64s[c * TILE_P + pl] - R64s[r * TILE_P + pl];
          double sb, cb;
          sincospi(2.0 * frac_c(dR * sc.fc_c), &sb, &cb);
          v = make_double2(cb * v.x - sb * v.y, cb * v.y + sb * v.x);
          const double g2 = gr_ * gc_;
          out = make_double2(v.x * g2, -v.y * g2);
        }
      }
      a.terms[(pp * J + j) * T + t] = out;
    }
    if (at < TILE_P) {
      int* pfl = pfl2 + par * TILE_P;
      const int64_t pp = tile * TILE_P + at;
      if (pfl[at]) {
        if (pp < a.P) atomicOr(&a.pflag[pp], pfl[at]);
        pfl[at] = 0;
      }
    }
    aux_sync();  // acc / pfl reads done before the next group's accumulation
    for (int it = at; it < (S + NPAIR) * TILE_P; it += WS_NA * 32) acc[it] = make_double2(0.0, 0.0);
    aux_sync();
  };

  for (int it = at; it < (S + NPAIR) * TILE_P; it += WS_NA * 32) acc[it] = make_double2(0.0, 0.0);
  int64_t B = 0;
  if (gring[0] < n_groups) {
    setup_group(gring[0], 0);
    nbar_arrive(WSB_PSF_READY, WS_THREADS);
  }
  for (int gi = 0;; ++gi) {
    const uint32_t g = gring[gi & 7];
    if (g >= n_groups) break;
    if (at == 0) gring[(gi + 3) & 7] = atomicAdd(a.sched, 1u);  // ring of 8: readers lag <= 2 groups
    // prepare group gi + 1 while the Horner warps work on group gi (its buffers were last read in group gi - 1)
    nbar_sync(WSB_STARTED, WS_THREADS);
    aux_sync();  // the claim above is visible to every auxiliary warp
    const uint32_t gn = gring[(gi + 1) & 7];
    if (gn < n_groups) {
      setup_group(gn, (gi + 1) & 1);
      nbar_arrive(WSB_PSF_READY, WS_THREADS);
    }
    for (int mb = 0; mb < n_mb; ++mb, ++B) finish_block(B, gi & 1, mb);
    handoff(g, gi & 1);
  }
  // the last CTA to finish resets the claim counter for the next launch
  if (at == 0) {
    __threadfence();
    if (atomicAdd(a.sched + 1, 1u) == gridDim.x - 1) {
      a.sched[0] = 0u;
      a.sched[1] = 0u;
      __threadfence();
    }
  }
}
