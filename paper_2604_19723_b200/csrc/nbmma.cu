// F2: the PLANAR_NB correlation as a complex GEMM on the 5th-generation tensor cores.
//
// PLANAR_NB responses are rank one as an N_f x N_a matrix:
//   psi_s[k, m] = g_s e^{-j2pi f_c R_s/c} b_s[k] a_s[m],   b_s[k] = e^{-j2pi (k - (N_f-1)/2) df R_s/c},
//   a_s[m] = a_y[iy] a_v[iv] = e^{j2pi (p~_y[iy] u'_y + p~_z[iv] u'_z)/lambda}       (m = iy N_v + iv)
// with R_s = ||r'||, u' = r'/R_s the local ray.  Hence
//   c_s = psi_s^H z = g_s e^{+j2pi f_c R_s/c} sum_m conj(a_s[m]) W_s[m],   W_s[m] = sum_k conj(b_s[k]) y[m, k],
// and W for every hypothesis (particle, component) of a PA is ONE real GEMM shared by all of them:
//   D[h, n] = sum_kk A[h, kk] B[n, kk],   A[h, 2k + {0,1}] = (Re b_h[k], Im b_h[k])          (generated on chip)
//   B[m, .] = (Re y[m,k], Im y[m,k]),  B[Nh + m, .] = (Im y[m,k], -Re y[m,k])               (one per PA)
// so D[h, m] = Re W_h[m] and D[h, Nh + m] = Im W_h[m].  The Gram matrix of the same hypotheses factors into
// three Dirichlet kernels (closed form: fp64 set-up and range reduction, fp32 sines; nb_gram_kernel).
//
// Precision (tools/f2_precision.py).  Two measured properties of the tensor core shape the split:
//  (1) fp16 subnormal operands read as zero -> both operands are scaled by powers of two into fp16's upper
//      range (A by 2^8, y per PA to max |Re|, |Im| in [2^7, 2^8));
//  (2) fp32 accumulation into TMEM is biased toward zero (measured: a coherent |c| shrink of ~2e-8 per
//      accumulation, -1e-6 after 48, rel-l 2e-4 near the true position).
// Hence an error-free split of the dominant term: x = x_hi + x_lo with x_hi on an integer grid (A: 2^-p of
// |b| = 1, y: 2^-q of its max) chosen so that K 2^(p+q) <= 2^24 -- every partial sum of A_hi B_hi is an exactly
// representable fp32 integer multiple of the grid product, so D1 = A_hi B_hi accumulates WITHOUT rounding --
// and D2 = A_hi B_lo + A_lo B_hi + A_lo B_lo (lo in fp16) in a second accumulator.  D2's partial sums are
// random walks (rounding residuals), so its truncation does not add coherently to c.  Emulated near the true
// position (truncation modelled): rel-l 2.9e-6 (c2), 6.4e-7 (c3), 8.1e-7 (c4).
//
// Kernel (one persistent CTA per SM, 14 warps, warp-specialised):
//   warp 0       TMEM allocation; one lane streams the B chunks (1-D bulk TMA, prepared in the UMMA
//                canonical K-major no-swizzle layout by nb_prep_kernel) into the stage ring
//   warp 1       one lane issues tcgen05.mma (kind::f16, M = 128 hypotheses, N = 2 nbh <= 256 per pass,
//                four per K-step of 16) and tcgen05.commit's the stage / accumulator barriers
//   warps 2..9   generate A (two groups of 4 warps on alternate stages, one row per thread: fp64 set-up,
//                anchor x per-tile table of w^j, grid/fp16 split, f32x2 pairs) into the same ring
//   warps 10..13 epilogue: tcgen05.ld one TMEM lane (= one hypothesis) each, W = D1 + D2, contract with conj(a)
//                (fp32 rows of N_v, fp64 across rows), apply gain, carrier and the operand scales -> c_s
// Work item = (tile of 128 hypotheses of one PA, antenna pass); arrays with 2 ceil8(N_a) > 256 take several
// passes (A is regenerated per pass).  Accumulator pairs are double-buffered in TMEM when 4 nb <= 512.
#include <cuda_fp16.h>
#include <stdlib.h>

#include "cdms_internal.h"
#include "geometry.cuh"

namespace cdms {

namespace {

constexpr int NB_M = 128;          // hypotheses per tile = TMEM lanes = UMMA M
constexpr int NB_GEN_WARPS = 8;
constexpr int NB_EPI_WARPS = 4;
constexpr int NB_WARPS = 2 + NB_GEN_WARPS + NB_EPI_WARPS;
constexpr int NB_THREADS = 32 * NB_WARPS;
constexpr int NB_MAX_STAGES = 6;
constexpr int NB_MAX_PASS = 8;
constexpr size_t NB_SMEM_BUDGET = 220 * 1024;
constexpr int NB_SCALE_LOG2 = 8;   // operands scaled to magnitude <= 2^8 before the split

// ---------------------------------------------------------------------------- tcgen05 / TMEM helpers
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// UMMA shared-memory descriptor: canonical K-major, no swizzle, ((8,n),2):((16 B, SBO),LBO); version 1 (tcgen05)
__device__ __forceinline__ uint64_t umma_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}
// instruction descriptor kind::f16: D f32 (bit 4), A = B = f16 (formats 0), both K-major, N >> 3 at 17, M >> 4 at 24
__host__ __device__ constexpr uint32_t umma_idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// A from TMEM (lane = row, consecutive K elements packed two per 32-bit column), B from shared memory
__device__ __forceinline__ void umma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// four 8-column loads of this warp's 32 TMEM lanes, one wait
__device__ __forceinline__ void tmem_ld8x4(uint32_t t0, uint32_t t1, uint32_t t2, uint32_t t3, uint32_t (&a)[8],
                                           uint32_t (&b)[8], uint32_t (&c)[8], uint32_t (&d)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%32];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%8,%9,%10,%11,%12,%13,%14,%15}, [%33];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%16,%17,%18,%19,%20,%21,%22,%23}, [%34];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%24,%25,%26,%27,%28,%29,%30,%31}, [%35];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]), "=r"(a[7]),
        "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3]), "=r"(b[4]), "=r"(b[5]), "=r"(b[6]), "=r"(b[7]),
        "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3]), "=r"(c[4]), "=r"(c[5]), "=r"(c[6]), "=r"(c[7]),
        "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7])
      : "r"(t0), "r"(t1), "r"(t2), "r"(t3)
      : "memory");
}
// (x, y) -> fp16x2 with x in the low half (lower address)
__device__ __forceinline__ uint32_t pack_h2(float x, float y) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(y), "f"(x));
  return r;
}
// error-free split of a complex value (already scaled): hi = rint(x / grid) grid (exact in fp16: <= 11 bits),
// lo = fp16(x - hi) (x - hi is exact in fp32)
__device__ __forceinline__ void split_grid(float x, float y, float grid, float inv_grid, uint32_t& hi,
                                           uint32_t& lo) {
  const float hx = rintf(x * inv_grid) * grid, hy = rintf(y * inv_grid) * grid;
  hi = pack_h2(hx, hy);
  lo = pack_h2(x - hx, y - hy);
}

// packed fp32 pairs (FADD2 / FMUL2 / FFMA2 on sm_100): the A generator advances two subcarriers per instruction
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t f2(float lo, float hi) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_split(f2_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2_t f2_fma(f2_t a, f2_t b, f2_t c) {
  f2_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2_t f2_mul(f2_t a, f2_t b) {
  f2_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2_t f2_add(f2_t a, f2_t b) {
  f2_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2_t f2_sub(f2_t a, f2_t b) {
  f2_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// x -> (hi, lo) with hi = x rounded to a multiple of grid by the magic constant M = 1.5 2^23 grid
// ((x + M) - M, |x| < 2^22 grid; add.rn cannot be re-associated), lo = x - hi exactly
__device__ __forceinline__ void f2_grid_split(f2_t x, f2_t M, f2_t& hi, f2_t& lo) {
  hi = f2_sub(f2_add(x, M), M);
  lo = f2_sub(x, hi);
}

// Epilogue rows for N_v = NV (passes aligned to rows): c += sum_iy conj(a_y[iy]) sum_iv conj(a_v[iv]) W[iy, iv]
// with W = D1 + D2 read from TMEM, a_v[] precomputed in registers, a_y advanced by a hi + lo step per row.
template <int NV>
__device__ __forceinline__ void nb_epi_rows(uint32_t c1, uint32_t c2, int nbh, int nrows, const float (&avr)[NV],
                                            const float (&avi)[NV], float ayr, float ayi, float syr, float syi,
                                            float sylr, float syli, double& cr, double& ci) {
  for (int r = 0; r < nrows; ++r) {
    float sr0 = 0.f, si0 = 0.f, sr1 = 0.f, si1 = 0.f;
#pragma unroll
    for (int h8 = 0; h8 < NV / 8; ++h8) {
      const uint32_t o = (uint32_t)(r * NV + h8 * 8);
      uint32_t r1[8], i1[8], r2[8], i2[8];
      tmem_ld8x4(c1 + o, c1 + nbh + o, c2 + o, c2 + nbh + o, r1, i1, r2, i2);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int iv = h8 * 8 + e;
        const float wr = __uint_as_float(r1[e]) + __uint_as_float(r2[e]);
        const float wi = __uint_as_float(i1[e]) + __uint_as_float(i2[e]);
        if (e & 1) {
          sr1 = fmaf(avr[iv], wr, fmaf(avi[iv], wi, sr1));
          si1 = fmaf(avr[iv], wi, fmaf(-avi[iv], wr, si1));
        } else {
          sr0 = fmaf(avr[iv], wr, fmaf(avi[iv], wi, sr0));
          si0 = fmaf(avr[iv], wi, fmaf(-avi[iv], wr, si0));
        }
      }
    }
    const float sr = sr0 + sr1, si = si0 + si1;
    cr += (double)fmaf(ayr, sr, ayi * si);
    ci += (double)fmaf(ayr, si, -ayi * sr);
    cmul_df<float>(syr, syi, sylr, syli, ayr, ayi, ayr, ayi);
  }
}

// Position in a ring of n mbarrier-guarded slots: slot index, phase parity of the current use, and whether the
// slot has been used before (producers then wait for the consumer's release of the previous use, parity phase^1).
// 32-bit increments keep the counters warp-uniform (64-bit div/mod would go through a subroutine).
struct RingPos {
  int slot = 0, n = 1;
  uint32_t phase = 0;
  bool reused = false;
  __device__ __forceinline__ explicit RingPos(int n_) : n(n_) {}
  __device__ __forceinline__ void next() {
    if (++slot == n) {
      slot = 0;
      phase ^= 1u;
      reused = true;
    }
  }
};

// ---------------------------------------------------------------------------- per-hypothesis set-up (fp64)
struct NbHyp {
  double R, delta, uy, uz, gain;
  int flag;  // pflag bits: 1 degenerate (r' = 0 or non-finite), 2 invalid SFV
};
// hypothesis (p, s) of PA j (P:L57-61 layout, P:L2097 local ray, P:L2150-2157 path loss)
__device__ __forceinline__ NbHyp nb_setup(const SceneDev& sc, const NbArgs& a, int j, int64_t p, int s) {
  NbHyp o;
  const double* pos = a.particles + p * a.pstride;
  const double* sfv_s = nullptr;
  if (s > 0) sfv_s = a.sfv_pp ? a.sfv + (p * sc.K + (s - 1)) * 3 : a.sfv + (int64_t)(s - 1) * 3;
  double va[3], sh[3];
  const bool ok = anchor_va(sc, j, sfv_s, va, sh);
  o.flag = ok ? 0 : 2;
  if (!ok) {
    va[0] = pos[0] - 1.0; va[1] = pos[1]; va[2] = pos[2];
    sh[0] = sh[1] = sh[2] = 0.0;
  }
  const double r0 = pos[0] - va[0], r1 = pos[1] - va[1], r2 = pos[2] - va[2];
  const double rs2 = 2.0 * (r0 * sh[0] + r1 * sh[1] + r2 * sh[2]);
  const double h0 = r0 - rs2 * sh[0], h1 = r1 - rs2 * sh[1], h2 = r2 - rs2 * sh[2];  // H r
  const double* Rj = sc.pa_rot[j];
  const double ly = Rj[1] * h0 + Rj[4] * h1 + Rj[7] * h2;  // r' = R_j^T H r
  const double lz = Rj[2] * h0 + Rj[5] * h1 + Rj[8] * h2;
  double R = sqrt(r0 * r0 + r1 * r1 + r2 * r2);
  if (!(R > 0.0) || !isfinite(R)) {
    o.flag |= 1;
    R = 1.0;
    o.uy = 0.0; o.uz = 0.0;
  } else {
    o.uy = ly / R; o.uz = lz / R;
  }
  o.R = R;
  o.delta = R * sc.df_c;
  o.gain = sc.pathloss ? sc.lambda / (4.0 * PI * R) : 1.0;
  return o;
}

}  // namespace

// ---------------------------------------------------------------------------- plan
bool nb_tensor_plan(const SceneDev& sc, NbPlan* pl) {
  if (sc.wavefront != CDMS_PLANAR_NB) return false;
  NbPlan p{};
  const int na8 = (sc.Na + 7) / 8 * 8;
  p.n_pass = (2 * na8 + 255) / 256;  // UMMA N = 2 nbh <= 256 per pass (two accumulators <= 512 columns)
  if (p.n_pass > NB_MAX_PASS) return false;
  p.nbh = ((sc.Na + p.n_pass - 1) / p.n_pass + 7) / 8 * 8;
  p.nb = 2 * p.nbh;
  const int kmax = ((2 * sc.nf + 15) / 16) * 16;  // no more K per stage than the padded problem has
  int kc = 0, nst = 0;
  for (int cand : {64, 32, 16}) {
    if (cand > kmax && cand != 16) continue;
    const size_t stage = 4u * (size_t)cand * (NB_M + p.nb);
    const int n = (int)(NB_SMEM_BUDGET / stage);
    if (n >= 3 || cand == 16) {
      kc = cand;
      nst = n < NB_MAX_STAGES ? n : NB_MAX_STAGES;
      break;
    }
  }
  if (nst < 2) return false;
  p.kc = kc;
  p.nst = nst;
  p.nf_pad = (sc.nf + kc / 2 - 1) / (kc / 2) * (kc / 2);
  p.n_chunks = 2 * p.nf_pad / kc;
  p.a_bytes = (uint32_t)(NB_M * kc * 2);
  p.b_bytes = (uint32_t)(p.nb * kc * 2);
  p.nacc = (4 * p.nb <= 512) ? 2 : 1;
  int cols = 32;
  while (cols < p.nacc * 2 * p.nb) cols *= 2;
  p.tmem_cols = cols;
  // exactness of D1 = A_hi B_hi: |partial sum| <= K 2^(p+q) grid units <= 2^24  (K = 2 nf_pad)
  int lk = 0;
  while ((1 << lk) < 2 * p.nf_pad) ++lk;
  const int pq = 24 - lk;
  p.qexp = pq / 2 > 10 ? 10 : pq / 2;
  p.pexp = (pq - p.qexp) > 10 ? 10 : pq - p.qexp;
  if (p.pexp < 4 || p.qexp < 4) return false;  // K > 2^16: the exact grid gets too coarse
  p.smem = (size_t)nst * 2 * (p.a_bytes + p.b_bytes) + 1024;
  // A in TMEM when the accumulator pair leaves room for >= 3 stages of kc columns (hi and lo, kc/2 fp16x2 words each):
  // the MMA then reads only B from shared memory.  At N <= 128 every MMA re-reads its 4 KB A tile from shared
  // memory and the four MMAs of a K-step plus the generator and TMA writes exceed its bandwidth.
  // The accumulator pair is then single-buffered.  CDMS_NB_ATMEM=0 keeps A in shared memory.
  const char* ev = getenv("CDMS_NB_ATMEM");
  if ((ev == nullptr || atoi(ev) != 0) && 2 * p.nb <= 256 && kc == 64) {
    p.a_tmem = 1;
    p.nacc = 1;
    p.a_col0 = 256;
    int n = (512 - p.a_col0) / kc;
    p.nst = n < NB_MAX_STAGES ? n : NB_MAX_STAGES;
    p.tmem_cols = 512;
    p.smem = (size_t)p.nst * 2 * p.b_bytes + 1024;
  }
  *pl = p;
  return true;
}
size_t nb_operand_bytes(const SceneDev& sc, const NbPlan& pl) {
  return (size_t)sc.J * pl.n_pass * pl.n_chunks * 2 * pl.b_bytes;
}

// ---------------------------------------------------------------------------- B operand (per PA)
// bop[j][pass][q][piece][...]: pass pi covers antennas [pi nbh, (pi+1) nbh); chunk q holds kk in [q kc, (q+1) kc)
// (subcarriers q kc/2 ...); piece 0 = hi (grid 2^-q_exp of the scaled max), 1 = lo; element (n, kk) at byte
// (n/8) SBO + (kk/8) 128 + (n%8) 16 + (kk%8) 2 with SBO = 16 kc (UMMA canonical K-major, no swizzle).
// y is scaled by 2^(8-e_j) (max |Re|, |Im| in [2^7, 2^8)); yscale_inv[j] = 2^(e_j - 16) undoes both scales.
__global__ void nb_prep_kernel(const __grid_constant__ SceneDev sc, const NbPlan pl, const float2* __restrict__ y,
                               uint8_t* __restrict__ bop, float* __restrict__ yscale_inv) {
  const int j = blockIdx.y;
  const int64_t nz = (int64_t)sc.nf * sc.Na;
  const float2* yj = y + (int64_t)j * nz;
  __shared__ float red[32];
  float mx = 0.f;
  for (int64_t n = threadIdx.x; n < nz; n += blockDim.x) {
    const float2 v = yj[n];
    mx = fmaxf(mx, fmaxf(fabsf(v.x), fabsf(v.y)));
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    mx = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.f;
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (threadIdx.x == 0) red[0] = mx;
  }
  __syncthreads();
  mx = red[0];
  int e = 0;
  if (mx > 0.f && isfinite(mx)) frexpf(mx, &e);  // mx = f 2^e, f in [0.5, 1)
  const float scale = ldexpf(1.f, NB_SCALE_LOG2 - e);
  if (blockIdx.x == 0 && threadIdx.x == 0) yscale_inv[j] = ldexpf(1.f, e - 2 * NB_SCALE_LOG2);
  const float grid = ldexpf(1.f, NB_SCALE_LOG2 - pl.qexp), inv_grid = ldexpf(1.f, pl.qexp - NB_SCALE_LOG2);
  const int kc8 = pl.kc / 8;
  const uint32_t sbo = 16u * pl.kc;
  const int64_t units = (int64_t)pl.n_pass * pl.n_chunks * kc8 * pl.nb;  // 16-byte units (4 subcarriers)
  uint8_t* bj = bop + (size_t)j * pl.n_pass * pl.n_chunks * 2 * pl.b_bytes;
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < units; u += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(u % pl.nb);
    int64_t r = u / pl.nb;
    const int cc = (int)(r % kc8);
    r /= kc8;
    const int q = (int)(r % pl.n_chunks);
    const int pass = (int)(r / pl.n_chunks);
    const bool im = n >= pl.nbh;
    const int ml = im ? n - pl.nbh : n;
    const int m = pass * pl.nbh + ml;
    const bool mok = ml < pl.nbh && m < sc.Na;
    uint32_t hi[4], lo[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int k = q * (pl.kc / 2) + cc * 4 + t;
      float2 v = make_float2(0.f, 0.f);
      if (mok && k < sc.nf) v = yj[(int64_t)k * sc.Na + m];
      const float xr = (im ? v.y : v.x) * scale, xi = (im ? -v.x : v.y) * scale;
      split_grid(xr, xi, grid, inv_grid, hi[t], lo[t]);
    }
    const size_t off = (size_t)(n >> 3) * sbo + (size_t)cc * 128 + (size_t)(n & 7) * 16;
    uint8_t* base = bj + ((size_t)pass * pl.n_chunks + q) * 2 * pl.b_bytes;
    *reinterpret_cast<uint4*>(base + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<uint4*>(base + pl.b_bytes + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  }
}

// D_N(x) = sin(pi N x) / sin(pi x) (C-amb-13): x = n + xr, D_N(x) = (-1)^{n (N-1)} D_N(xr); both sines reduced in
// fp64 (sin(pi N xr) = sin(pi t), t = N xr mod 2 in [-1, 1]) and evaluated in fp32 (relative error ~1e-7, the
// precision of K1's per-antenna fp32 Gram terms); second-order series below |N xr| = 1e-4 (truncation < 1e-15).
__device__ __forceinline__ float dirichlet_rr(double x, int N) {
  const double n = rint(x);
  const double xr = x - n;
  double t = (double)N * xr;
  t -= 2.0 * rint(0.5 * t);
  const float fx = (float)xr;
  float d;
  if (fabsf(fx) * (float)N < 1e-4f) {
    d = (float)N * (1.f - (float)(PI * PI / 6.0) * ((float)N * (float)N - 1.f) * fx * fx);
  } else {
    d = sinpif((float)t) / sinpif(fx);
  }
  if (((N - 1) & 1) && (((long long)n) & 1)) d = -d;
  return d;
}

// ---------------------------------------------------------------------------- Gram (closed form)
// G_rc = psi_r^H psi_c = g_r g_c e^{j2pi f_c (R_r - R_c)/c} D_Nf(df (R_r - R_c)/c)
//        D_Ny(d_y (u'_y,c - u'_y,r)/lambda) D_Nv(d_v (u'_z,c - u'_z,r)/lambda),  G_ss = g_s^2 N_z
// (centred template and subcarrier grid: every factor is a real Dirichlet kernel, C-amb-13 for D_N).
// One thread per (particle, PA); also ORs the per-particle flags.
__global__ void nb_gram_kernel(const __grid_constant__ SceneDev sc, const NbArgs a, int* __restrict__ pflag) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int J = sc.J, S = sc.S, T = S + S * (S + 1) / 2;
  if (idx >= a.P * J) return;
  const int j = (int)(idx / a.P);  // consecutive threads: consecutive particles of one PA (term_idx)
  const int64_t p = idx - (int64_t)j * a.P;
  double R[MAXS], dl[MAXS], uy[MAXS], uz[MAXS], g[MAXS];
  int fl = 0;
  for (int s = 0; s < S; ++s) {
    const NbHyp h = nb_setup(sc, a, j, p, s);
    R[s] = h.R; dl[s] = h.delta; uy[s] = h.uy; uz[s] = h.uz; g[s] = h.gain;
    fl |= h.flag;
  }
  if (fl) atomicOr(&pflag[p], fl);
  const double nz = (double)sc.nf * (double)sc.Na;
  const double ky = sc.dy / sc.lambda, kv = sc.dv / sc.lambda;
  int t = 0;
  for (int r = 0; r < S; ++r) {
    for (int c = 0; c <= r; ++c, ++t) {
      if (r == c) {
        a.terms[term_idx(p, j, S + t, T, a.P)] = make_double2(nz * g[r] * g[r], 0.0);
        continue;
      }
      if (a.diag_only) {
        a.terms[term_idx(p, j, S + t, T, a.P)] = make_double2(0.0, 0.0);
        continue;
      }
      float sn, cs;
      sincospif(2.f * (float)frac_c((R[r] - R[c]) * sc.fc_c), &sn, &cs);
      const float D = dirichlet_rr(dl[r] - dl[c], sc.nf) * dirichlet_rr(ky * (uy[c] - uy[r]), sc.ny) *
                      dirichlet_rr(kv * (uz[c] - uz[r]), sc.nv);
      const double m = g[r] * g[c] * (double)D;
      a.terms[term_idx(p, j, S + t, T, a.P)] = make_double2(m * (double)cs, m * (double)sn);
    }
  }
}

// ---------------------------------------------------------------------------- K1 (tensor cores)
__global__ void __launch_bounds__(NB_THREADS, 1)
    nb_corr_kernel(const __grid_constant__ SceneDev sc, const NbPlan pl, const NbArgs a) {
  extern __shared__ __align__(1024) uint8_t nb_smem[];
  // warp index through a shuffle: provably warp-uniform, so role branches keep loop state and UMMA descriptors
  // in uniform registers (no per-MMA ELECT/R2UR waterfall)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int nst = pl.nst, kc = pl.kc, npass = pl.n_pass;
  const uint32_t stage_bytes = pl.a_tmem ? 2 * pl.b_bytes : 2 * (pl.a_bytes + pl.b_bytes);
  uint8_t* ring = nb_smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(nb_smem + (size_t)nst * stage_bytes);
  uint64_t* full_a = bars;
  uint64_t* full_b = bars + NB_MAX_STAGES;
  uint64_t* empty = bars + 2 * NB_MAX_STAGES;
  uint64_t* acc_full = bars + 3 * NB_MAX_STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  // stage s: [A_hi | A_lo | B_hi | B_lo] (A in TMEM: [B_hi | B_lo])
  auto A_hi = [&](int s) { return ring + (size_t)s * stage_bytes; };
  auto B_hi = [&](int s) { return ring + (size_t)s * stage_bytes + (pl.a_tmem ? 0 : 2 * pl.a_bytes); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full_a[s], NB_GEN_WARPS / 2);  // one group of generator warps per stage
      mbar_init(&full_b[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], NB_EPI_WARPS);
    }
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)pl.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int S = sc.S;
  const int64_t nhyp = a.P * S;
  const int n_chunks = pl.n_chunks;
  const uint32_t sbo = 16u * kc;

  if (warp == 0) {
    // ---------------- B producer
    if (lane == 0) {
      RingPos rp(nst);
      for (int64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
        const int j = (int)(tile / a.n_tiles_j);
        const uint8_t* src = a.bop + (size_t)j * npass * n_chunks * 2 * pl.b_bytes;
        for (int pass = 0; pass < npass; ++pass) {
          for (int q = 0; q < n_chunks; ++q, rp.next()) {
            const int slot = rp.slot;
            if (rp.reused) mbar_wait(&empty[slot], rp.phase ^ 1u);
            mbar_expect_tx(&full_b[slot], 2 * pl.b_bytes);
            tma_load_1d(B_hi(slot), src + ((size_t)pass * n_chunks + q) * 2 * pl.b_bytes, 2 * pl.b_bytes,
                        &full_b[slot]);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: D1 += A_hi B_hi (exact), D2 += A_hi B_lo + A_lo B_hi + A_lo B_lo
    // The whole warp runs the loop (barrier waits, descriptors: warp-uniform values in uniform registers); lane 0
    // issues.  Descriptors are the slot-0 ones plus address offsets in 16-byte units (the 14-bit start-address
    // field cannot carry: dynamic shared memory < 256 KB).  At N = 128 an MMA lasts ~64 clocks, so per-MMA issue
    // overhead decides whether the tensor pipe stays fed.
    {
      RingPos rp(nst), ap(pl.nacc);
      const uint32_t idesc = umma_idesc_f16(NB_M, pl.nb);
      const uint64_t dA0 = umma_sdesc(smem_u32(A_hi(0)), 128, sbo), dB0 = umma_sdesc(smem_u32(B_hi(0)), 128, sbo);
      const uint64_t slot_step = stage_bytes >> 4, a_lo_step = pl.a_bytes >> 4, b_lo_step = pl.b_bytes >> 4;
      const int nks = kc / 16;
      for (int64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
        for (int pass = 0; pass < npass; ++pass, ap.next()) {
          const int b = ap.slot;
          if (ap.reused) mbar_wait(&acc_empty[b], ap.phase ^ 1u);
          tc_fence_after();
          const uint32_t d1 = tmem + (uint32_t)(b * 2 * pl.nb), d2 = d1 + (uint32_t)pl.nb;
          for (int q = 0; q < n_chunks; ++q, rp.next()) {
            const int slot = rp.slot;
            const uint32_t par = rp.phase;
            mbar_wait(&full_b[slot], par);
            mbar_wait(&full_a[slot], par);
            tc_fence_after();
            const uint64_t sa = dA0 + (uint64_t)slot * slot_step, sb = dB0 + (uint64_t)slot * slot_step;
            if (lane == 0) {
              if (pl.a_tmem) {
                const uint32_t ta = tmem + (uint32_t)(pl.a_col0 + slot * kc);  // hi at +0, lo at +kc/2 columns
                for (int ks = 0; ks < nks; ++ks) {
                  const uint64_t dbh = sb + (uint64_t)(ks * 16), dbl = dbh + b_lo_step;
                  const uint32_t tah = ta + (uint32_t)(ks * 8), tal = tah + (uint32_t)(kc / 2);
                  const uint32_t acc0 = (q | ks) ? 1u : 0u;
                  umma_f16_ts(d1, tah, dbh, idesc, acc0);
                  umma_f16_ts(d2, tah, dbl, idesc, acc0);
                  umma_f16_ts(d2, tal, dbh, idesc, 1u);
                  umma_f16_ts(d2, tal, dbl, idesc, 1u);
                }
              } else {
                for (int ks = 0; ks < nks; ++ks) {
                  const uint64_t dah = sa + (uint64_t)(ks * 16), dbh = sb + (uint64_t)(ks * 16);
                  const uint64_t dal = dah + a_lo_step, dbl = dbh + b_lo_step;
                  const uint32_t acc0 = (q | ks) ? 1u : 0u;
                  umma_f16(d1, dah, dbh, idesc, acc0);
                  umma_f16(d2, dah, dbl, idesc, acc0);
                  umma_f16(d2, dal, dbh, idesc, 1u);
                  umma_f16(d2, dal, dbl, idesc, 1u);
                }
              }
              umma_commit(&empty[slot]);
            }
            __syncwarp();
          }
          if (lane == 0) umma_commit(&acc_full[b]);
          __syncwarp();
        }
      }
    }
  } else if (warp < 2 + NB_GEN_WARPS) {
    // ---------------- A generators: two groups of 4 warps take alternate stages; thread -> row h of its group
    // b_k = e^{-j2pi (k - kcen) delta} for the stage's kc/2 subcarriers as A_a t[j]: an anchor A_a per 16
    // subcarriers from the fp64-reduced phase and a per-tile table t[j] = w^j (j < 16, fp64, rounded once), so
    // each phasor carries one fp32 rounding (no coherent drift of a raised step) and no
    // dependency chain; pairs of subcarriers share f32x2 instructions.
    // row h = this thread's TMEM lane (warp w may only access lanes [32 (w % 4), +32)): rows of both groups cover
    // the 128 lanes, consecutive lanes -> consecutive rows (conflict-free 16-byte shared-memory stores as well)
    const int h = 32 * (warp & 3) + lane, grp = (warp - 2) >> 2;
    const uint32_t a_lane = (uint32_t)(32 * (warp & 3)) << 16;
    const int nsub = kc / 2;  // subcarriers per stage (8, 16 or 32)
    const double kcen = 0.5 * (sc.nf - 1);
    const float a_scale = (float)(1 << NB_SCALE_LOG2);
    const float gmag = 1.5f * 8388608.f * ldexpf(1.f, NB_SCALE_LOG2 - pl.pexp);  // 1.5 2^23 grid
    const f2_t M2 = f2(gmag, gmag);
    const uint32_t row_off = (uint32_t)(h >> 3) * sbo + (uint32_t)(h & 7) * 16u;
    RingPos rp(nst);
    int gs = 0;  // stage counter: this group generates the stages with gs % 2 == grp
    for (int64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
      const int j = (int)(tile / a.n_tiles_j);
      const int64_t hg = (tile - (int64_t)j * a.n_tiles_j) * NB_M + h;
      double delta = 0.0;
      if (hg < nhyp) {
        const int64_t p = hg / S;
        delta = nb_setup(sc, a, j, p, (int)(hg - p * S)).delta;
      }
      f2_t TR[8], TI[8];  // t[2i], t[2i+1] in the two lanes
      {
        double sw, cw;
        sincospi(2.0 * frac_c(delta), &sw, &cw);
        double tr = 1.0, ti = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double ur = tr * cw + ti * sw, ui = ti * cw - tr * sw;  // t w, w = e^{-j2pi delta}
          TR[i] = f2((float)tr, (float)ur);
          TI[i] = f2((float)ti, (float)ui);
          tr = ur * cw + ui * sw;
          ti = ui * cw - ur * sw;
        }
      }
      for (int pass = 0; pass < npass; ++pass) {
        for (int q = 0; q < n_chunks; ++q, rp.next(), ++gs) {
          if ((gs & 1) != grp) continue;
          const int slot = rp.slot;
          if (rp.reused) mbar_wait(&empty[slot], rp.phase ^ 1u);
          uint8_t* ahi = A_hi(slot);
          for (int a16 = 0; a16 < nsub; a16 += 16) {
            const int k0 = q * nsub + a16;
            const double ph = frac_c(-((double)k0 - kcen) * delta);  // anchor b_{k0}
            float ar, ai;
            sincospif(2.f * (float)ph, &ai, &ar);
            ar *= a_scale;
            ai *= a_scale;
            const f2_t AR = f2(ar, ar), AI = f2(ai, ai), nAI = f2(-ai, -ai);
            const int npair = (nsub - a16) < 16 ? (nsub - a16) / 2 : 8;
#pragma unroll
            for (int p4 = 0; p4 < 8; p4 += 2) {  // 4 subcarriers = one 16-byte chunk per piece
              if (p4 < npair) {
                uint32_t hi[4], lo[4];
#pragma unroll
                for (int t2 = 0; t2 < 2; ++t2) {
                  const f2_t BR = f2_fma(AR, TR[p4 + t2], f2_mul(nAI, TI[p4 + t2]));
                  const f2_t BI = f2_fma(AR, TI[p4 + t2], f2_mul(AI, TR[p4 + t2]));
                  f2_t hr, lr, hI, lI;
                  f2_grid_split(BR, M2, hr, lr);
                  f2_grid_split(BI, M2, hI, lI);
                  float x0, x1, y0, y1;
                  f2_split(hr, x0, x1);
                  f2_split(hI, y0, y1);
                  hi[2 * t2] = pack_h2(x0, y0);
                  hi[2 * t2 + 1] = pack_h2(x1, y1);
                  f2_split(lr, x0, x1);
                  f2_split(lI, y0, y1);
                  lo[2 * t2] = pack_h2(x0, y0);
                  lo[2 * t2 + 1] = pack_h2(x1, y1);
                }
                const int chunk = (a16 + 2 * p4) / 4;  // 4 subcarriers = 4 fp16x2 words per piece
                if (pl.a_tmem) {
                  const uint32_t ta = tmem + a_lane + (uint32_t)(pl.a_col0 + slot * kc + chunk * 4);
                  tmem_st4(ta, hi[0], hi[1], hi[2], hi[3]);
                  tmem_st4(ta + (uint32_t)(kc / 2), lo[0], lo[1], lo[2], lo[3]);
                } else {
                  const uint32_t off = row_off + (uint32_t)chunk * 128u;
                  *reinterpret_cast<uint4*>(ahi + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                  *reinterpret_cast<uint4*>(ahi + pl.a_bytes + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
                }
              }
            }
          }
          if (pl.a_tmem) {
            tmem_wait_st();     // this warp's TMEM stores complete, ordered before the arrive
            tc_fence_before();
          } else {
            fence_proxy_async();  // generic-proxy stores -> visible to the tensor core (async proxy)
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&full_a[slot]);
        }
      }
    }
  } else {
    // ---------------- epilogue: one TMEM lane (hypothesis) per thread
    const int quarter = warp & 3;  // TMEM lanes [32 quarter, 32 quarter + 32) of this warp
    const int h = quarter * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
    const int T = S + S * (S + 1) / 2;
    const double cy = 0.5 * (sc.ny - 1), cv = 0.5 * (sc.nv - 1);
    const double ky = sc.dy / sc.lambda, kv = sc.dv / sc.lambda;
    RingPos ap(pl.nacc);
    for (int64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
      const int j = (int)(tile / a.n_tiles_j);
      const int64_t hg = (tile - (int64_t)j * a.n_tiles_j) * NB_M + h;
      const bool valid = hg < nhyp;
      const int64_t p = valid ? hg / S : 0;
      const int s = valid ? (int)(hg - p * S) : 0;
      NbHyp hy;
      if (valid) hy = nb_setup(sc, a, j, p, s);
      else { hy.R = 1.0; hy.delta = 0.0; hy.uy = 0.0; hy.uz = 0.0; hy.gain = 1.0; hy.flag = 0; }
      const double ty = ky * hy.uy, tv = kv * hy.uz;  // cycles per antenna step along y / z
      double sv_, cv_;
      sincospi(2.0 * frac_c(tv), &sv_, &cv_);  // antenna step along z, hi + lo (raised to the iv-th power)
      const float svr = (float)cv_, svi = (float)sv_;
      const float svlr = (float)(cv_ - (double)svr), svli = (float)(sv_ - (double)svi);
      double sy_, cy_;
      sincospi(2.0 * frac_c(ty), &sy_, &cy_);  // antenna step along y (row to row), hi + lo
      const float syr = (float)cy_, syi = (float)sy_;
      const float sylr = (float)(cy_ - (double)syr), syli = (float)(sy_ - (double)syi);
      // rows of N_v = 8 / 16 with passes on row boundaries: a_v[] in registers (row-structured epilogue)
      const int rowmode = (sc.nv == 16 && pl.nbh % 16 == 0) ? 16 : (sc.nv == 8 ? 8 : 0);
      float avr[16], avi[16];
      if (rowmode) {
        sincospif(2.f * (float)frac_c(-cv * tv), &avi[0], &avr[0]);
#pragma unroll
        for (int t = 1; t < 16; ++t) cmul_df<float>(svr, svi, svlr, svli, avr[t - 1], avi[t - 1], avr[t], avi[t]);
      }
      double cr = 0.0, ci = 0.0;
      for (int pass = 0; pass < npass; ++pass, ap.next()) {
        const int b = ap.slot;
        const int mbeg = pass * pl.nbh;
        const int mend = (mbeg + pl.nbh < sc.Na) ? mbeg + pl.nbh : sc.Na;
        int iy = mbeg / sc.nv, iv = mbeg - iy * sc.nv;
        float pr = 0.f, pi = 0.f, ar = 1.f, ai = 0.f;
        bool anchor = true;
        float ayr = 1.f, ayi = 0.f;
        if (rowmode) sincospif(2.f * (float)frac_c(((double)iy - cy) * ty), &ayi, &ayr);
        mbar_wait(&acc_full[b], ap.phase);
        tc_fence_after();
        const uint32_t c1 = tmem + lane_addr + (uint32_t)(b * 2 * pl.nb), c2 = c1 + (uint32_t)pl.nb;
        if (rowmode == 16) {
          float r16[16], i16[16];
#pragma unroll
          for (int t = 0; t < 16; ++t) { r16[t] = avr[t]; i16[t] = avi[t]; }
          nb_epi_rows<16>(c1, c2, pl.nbh, (mend - mbeg) / 16, r16, i16, ayr, ayi, syr, syi, sylr, syli, cr, ci);
        } else if (rowmode == 8) {
          float r8[8], i8[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) { r8[t] = avr[t]; i8[t] = avi[t]; }
          nb_epi_rows<8>(c1, c2, pl.nbh, (mend - mbeg) / 8, r8, i8, ayr, ayi, syr, syi, sylr, syli, cr, ci);
        }
        for (int m0 = mbeg; m0 < (rowmode ? mbeg : mend); m0 += 8) {
          const uint32_t o = (uint32_t)(m0 - mbeg);
          uint32_t r1[8], i1[8], r2[8], i2[8];
          tmem_ld8x4(c1 + o, c1 + pl.nbh + o, c2 + o, c2 + pl.nbh + o, r1, i1, r2, i2);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            if (m0 + e < mend) {
              if (anchor || iv == 0) {  // row anchor a_{iy, iv} from an fp64-reduced phase
                const double ph = frac_c(((double)iy - cy) * ty + ((double)iv - cv) * tv);
                sincospif(2.f * (float)ph, &ai, &ar);
                anchor = false;
              }
              const float wr = __uint_as_float(r1[e]) + __uint_as_float(r2[e]);
              const float wi = __uint_as_float(i1[e]) + __uint_as_float(i2[e]);
              pr = fmaf(ar, wr, fmaf(ai, wi, pr));   // conj(a) W
              pi = fmaf(ar, wi, fmaf(-ai, wr, pi));
              cmul_df<float>(svr, svi, svlr, svli, ar, ai, ar, ai);
              if (++iv == sc.nv) {
                iv = 0;
                ++iy;
                cr += (double)pr;
                ci += (double)pi;
                pr = 0.f;
                pi = 0.f;
              }
            }
          }
        }
        cr += (double)pr;  // a pass may end inside a row
        ci += (double)pi;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[b]);
      }
      if (valid) {
        double sc_, cc_;
        sincospi(2.0 * frac_c(hy.R * sc.fc_c), &sc_, &cc_);  // conj(carrier) = e^{+j2pi f_c R/c}
        const double gs = hy.gain * (double)a.yscale_inv[j];
        const double xr = (cr * cc_ - ci * sc_) * gs, xi = (cr * sc_ + ci * cc_) * gs;
        a.terms[term_idx(p, j, s, T, a.P)] = make_double2(xr, xi);
      }
    }
  }
  __syncthreads();
  if (warp == 0) {
    __syncwarp();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)pl.tmem_cols)
                 : "memory");
  }
}

// ---------------------------------------------------------------------------- launchers
cudaError_t launch_nb_prep(const SceneDev& sc, const NbPlan& pl, const float2* y, uint8_t* bop, float* yscale_inv,
                           cudaStream_t st) {
  dim3 grid(8, sc.J);
  nb_prep_kernel<<<grid, 512, 0, st>>>(sc, pl, y, bop, yscale_inv);
  return cudaGetLastError();
}
cudaError_t launch_nb_gram(const SceneDev& sc, const NbArgs& a, int* pflag, cudaStream_t st) {
  const int64_t n = a.P * sc.J;
  nb_gram_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(sc, a, pflag);
  return cudaGetLastError();
}
cudaError_t launch_nb_corr(const SceneDev& sc, const NbPlan& pl, const NbArgs& a, int num_sms, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(nb_corr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem);
  if (e != cudaSuccess) return e;
  int64_t grid = a.n_tiles < num_sms ? a.n_tiles : num_sms;
  if (grid < 1) grid = 1;
  nb_corr_kernel<<<(unsigned)grid, NB_THREADS, pl.smem, st>>>(sc, pl, a);
  return cudaGetLastError();
}

}  // namespace cdms
