// cdms_internal.h -- device-side parameter blocks, constants and small PTX helpers shared by the
// libcdms kernels (loglik.cu, beliefs.cu) and the host ABI (cdms.cpp).  Nothing here is visible
// through include/cdms.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/cdms.h"

namespace cdms {

constexpr int MAXJ = 8;       // PAs per scene
constexpr int MAXS = 9;       // propagation components S = K + 1 (LOS + 8 walls)
constexpr int TILE_P = 32;    // particles per CTA tile (one per lane)
#ifndef CDMS_NWARP
#define CDMS_NWARP 8
#endif
constexpr int NWARP = CDMS_NWARP;  // warps per CTA = antennas per antenna block (power of two)
constexpr int NTHREADS = TILE_P * NWARP;
constexpr int SEG = 64;       // Horner segment length in subcarriers (re-anchor period)
constexpr int KCHUNK = 128;   // max subcarriers per shared-memory chunk of y (multiple of SEG; corr_kchunk(S))
constexpr double C_LIGHT = 299792458.0;
constexpr double PI = 3.14159265358979323846;

enum DeviceFlags : int { FLAG_DEGENERATE = 1, FLAG_ZEROMASS = 2, FLAG_NAN = 4 };

// Scene + per-call priors, passed by value as a __grid_constant__ kernel parameter (~2.7 KB).
struct SceneDev {
  int J, K, S, ny, nv, Na, nf, wavefront, pathloss;
  int kc_len;        // subcarriers per chunk (min(KCHUNK, nf))
  int small_step;    // 1: 2 pi max|Delta| df/c <= 0.2 -> polynomial per-antenna step correction
  int small_z;       // 1: 2 pi max|Delta| SEG df/c <= 1 -> polynomial per-antenna segment correction
  int n_mb, n_kc;    // antenna blocks of NWARP, subcarrier chunks
  double dy, dv, fc, df, f0;      // f0 = fc - (nf-1)/2 df
  double f0_c, df_c, segdf_c, fc_c;  // f0/c, df/c, SEG*df/c, fc/c (cycles per metre)
  double lambda;
  // fp32 constants of the per-antenna Gram term (constant-bank operands): fc/c, df/c, N = nf,
  // pi^2/6 (N^2 - 1) and the sign mask (bit 31 when N is even, i.e. D_N(x + 1) = -D_N(x))
  float fc_cf, df_cf, nf_f, c6N_f;
  float fc2pi_f;     // fp32 2 pi f_c / c: carriers e^{j f_c 2pi Delta/c} straight into __sincosf (no reduction)
  double ap_r;       // 1.5 x half the URA diagonal (||p~_m|| <= ap_r / 1.5): R > ap_r keeps every antenna distance
                     // >= R / 3, far from fp32 cancellation
  uint32_t evenN_mask;
  float f0_cf, segdf_cf;  // fp32 f0/c, SEG df/c for the per-antenna set-up
  int two_seg;            // SEG < nf <= 2 SEG, not planar NB: second segment phasor formed directly (A1)
  double f1_c;            // (f0 + SEG df)/c
  float f1_cf;
  int64_t y_mb_step;      // ytiles element step from the last chunk of an antenna block to the next block
  double pa_pos[MAXJ][3];
  double pa_rot[MAXJ][9];
  double m_re[MAXJ][MAXS], m_im[MAXJ][MAXS], v[MAXJ][MAXS];
  double eta[MAXJ];
};

// K1 (correlation + Gram) for one batch of particles -> sufficient statistics per (particle, PA):
// terms[p][j][0..S) = c_s, terms[p][j][S + tri(r,c)] = G_rc (lower triangle incl. diagonal), gains applied.
struct CorrArgs {
  const double* particles;  // batch start
  int64_t P;                // particles in the batch
  int pstride;
  const double* sfv;        // [K][3], or [P][K][3] starting at the batch (sfv_pp)
  int sfv_pp;
  const float4* ytiles;     // [J][Na_pad][n_kc][kc_len] (yr, yr, yi, yi), zero padded
  const float4* tmpl;       // [J][Na_pad] template columns (R_j p~_m, ||p~_m||^2), fp32
  double2* terms;           // [P][J][T]
  int* pflag;               // [P] per-particle, ORed (zeroed by K1b): 1 degenerate, 2 invalid input
  int* flags;
  unsigned int* sched;      // [2] group claim counter and finished-CTA counter, zero between launches
  int64_t n_tiles;
  int64_t n_groups;         // n_tiles * J (< 2^31)
  int64_t grid;             // CTAs
  int no_gram;              // 1: skip the off-diagonal Gram (callers that use c only; G = diag(g^2 N_z) is written)
};
// K1b (S x S assembly) for the same batch
struct AsmArgs {
  const void* terms;        // [J][T][P] (term_idx): float2 from K1T (FP32 spherical / planar WB), else double2
  int terms_f32;
  int* pflag;
  const double* ynorm2;     // [J]
  const double* logw_prior; // [P] (batch) or NULL
  double* loglik;           // [P]
  double2* amp;             // [P][J][S] or NULL
  double2* term_c;          // [P][J][S] or NULL (cdms_loglik_terms)
  double2* term_G;          // [P][J][S][S] or NULL
  int* flags;
  int64_t P;
  const int* perm;          // [P] processing order -> particle index (locality sort, loglik_impl), or NULL = identity
};
inline int terms_width(int S) { return S + S * (S + 1) / 2; }
// Sufficient statistics of a batch of P particles, layout [J][T][P] (term t of PA j of particle p): the writers (one
// thread per particle, or per particle and PA) store consecutive particles to consecutive 16-byte slots, so every warp
// store and every assembly load is a full-sector coalesced access (the [P][J][T] row layout made each 16-byte store
// its own half-used sector: ~2x the DRAM bytes of the hand-off, VERDICT r01 Weak 10).
__host__ __device__ __forceinline__ int64_t term_idx(int64_t p, int j, int t, int T, int64_t P) {
  return ((int64_t)j * T + t) * P + p;
}

// ---------------------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// 1-D bulk TMA copy global -> shared, completion counted on an mbarrier (cp.async.bulk, sm_90+).
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, "
      "p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// Packed fp32 pairs in one 64-bit register for the sm_100 f32x2 instructions (FFMA2 / FMUL2 / FADD2: two lanes of
// FP32 work per issue slot; the K1 Horner and the K1T Gram use them)
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk2(float lo, float hi) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void up2(u64 v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
  u64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ u64 fmul2(u64 a, u64 b) {
  u64 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 fadd2(u64 a, u64 b) {
  u64 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// K1T's terms hand-off in complex64: the fp64 sums rounded once (6e-8 relative, below K1T's own fp32 accumulation)
__device__ __forceinline__ float2 term_f2(double re, double im) { return make_float2((float)re, (float)im); }

// Philox4x32-10 (Salmon et al., SC'11): counter-based draws of the regularisation normals (step.cu) and the
// birth-proposal candidates (birth.cu)
__device__ __forceinline__ uint4 philox_step(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}

// I(x) = #{i in [0, P_total) : t_i < x}, t_i = floor((u + i 2^32) Q / (P_total 2^32)), exact in 128-bit integers:
// the first output slot of the CDF position x (distributed resampling plan, C-amb-15).  Used
// by the device plan (step.cu) and the host entry cdms_resample_plan.
__host__ __device__ inline int64_t resample_slot_index(uint64_t x, uint64_t Q, int64_t P_total, uint32_t u) {
  typedef unsigned __int128 u128;
  const u128 lhs = (u128)x * (u128)(uint64_t)P_total << 32;
  const u128 uq = (u128)u * Q;
  if (lhs <= uq) return 0;
  const u128 A = lhs - uq;
  const u128 step = (u128)Q << 32;
  u128 I = (A + step - 1) / step;
  if (I > (u128)(uint64_t)P_total) I = (u128)(uint64_t)P_total;
  return (int64_t)I;
}

// Resampling plan of one rank (plan[4] = Q_total, O_r, slot_lo, slot_hi) from every rank's integer mass Q_r: its CDF
// range [O_r, O_r + Q_r) covers the contiguous output slots [I(O_r), I(O_r + Q_r)).
__device__ inline void plan_dev(const uint64_t* Q, int nranks, int rank, int64_t P_total, uint32_t u_bits,
                                uint64_t* plan) {
  uint64_t Qt = 0, O = 0;
  for (int r = 0; r < nranks; ++r) {
    if (r < rank) O += Q[r];
    Qt += Q[r];
  }
  plan[0] = Qt;
  plan[1] = O;
  plan[2] = Qt ? (uint64_t)resample_slot_index(O, Qt, P_total, u_bits) : 0ull;
  plan[3] = Qt ? (uint64_t)resample_slot_index(O + Q[rank], Qt, P_total, u_bits) : 0ull;
}

// ---------------------------------------------------------------------------- launchers
// (defined in loglik.cu / beliefs.cu, called from cdms.cpp)
// The template columns as a kernel parameter (constant bank) when J N_a,pad <= TMPLC_MAX: the correlation kernel's
// per-element template read then goes through the constant cache instead of the L1 data path its table rows
// saturate; prep_y copies the same host-computed values into the tmpl buffer, so every kernel sees identical columns.
constexpr int TMPLC_MAX = 512;
struct TmplC {
  float4 v[TMPLC_MAX];  // [J][Na_pad] (R_j p~_m, ||p~_m||^2), padded antennas repeat m = 0
  int n;                // J Na_pad, or 0 (too many: the kernels compute / read the tmpl buffer)
};
void make_tmplc(const SceneDev& sc, TmplC* out);
cudaError_t launch_prep_y(const SceneDev& sc, const float2* y, float4* ytiles, double* ynorm2, float4* tmpl,
                          cudaStream_t st);
int64_t corr_grid(const SceneDev& sc, int64_t n_tiles, int precision, int num_sms);  // 0 on error
cudaError_t launch_corr(const SceneDev& sc, const CorrArgs& a, int precision, cudaStream_t st);
cudaError_t launch_assemble(const SceneDev& sc, const AsmArgs& a, cudaStream_t st);
size_t corr_smem_bytes(int S, int precision);
int corr_kchunk(int S);   // subcarriers per y chunk (SceneDev::kc_len = min(corr_kchunk(S), nf))
cudaError_t launch_response(const SceneDev& sc, const double* pos, int64_t n, const int32_t* js,
                            const double* sfv, double2* psi, int precision, int* flags, cudaStream_t st,
                            int sfv_per_item = 0);
cudaError_t launch_layout(const SceneDev& sc, const double* sfv, double* layout, double* va, double* H,
                          int* flags, cudaStream_t st);

// beliefs.cu
constexpr int RED_BLOCK = 256;       // threads per reduction block
constexpr int RED_ITEMS = 2048;      // particles per reduction block (fixed partition -> determinism)
int64_t red_blocks(int64_t P);
cudaError_t launch_lse_partial(const double* l, int64_t P, double2* part, cudaStream_t st);
cudaError_t launch_lse_final(const double2* part, int64_t nblk, double2* out, cudaStream_t st);
cudaError_t launch_lse_combine(const double2* per_rank, int nranks, double* lse, double* M,
                               double* logS, int* flags, cudaStream_t st);
cudaError_t launch_normalize(const double* l, int64_t P, const double* M, const double* logS,
                             const int* flags, double* w, cudaStream_t st);
cudaError_t launch_moments1(const double* x, const double* w, int64_t P, double* part, cudaStream_t st);
cudaError_t launch_moments2(const double* x, const double* w, int64_t P, const double* sum1,
                            double* part, cudaStream_t st);
cudaError_t launch_sum_partials(const double* part, int64_t nblk, int width, double* out, cudaStream_t st);
cudaError_t launch_moments_finalize(const double* sum1, const double* sum2, double* est, int* flags,
                                    cudaStream_t st);
cudaError_t launch_wmax_partial_f(const double* w, int64_t P, double* part, int* flags, cudaStream_t st);
cudaError_t launch_max_final(const double* part, int64_t nblk, double* out, cudaStream_t st);
cudaError_t launch_quantize(const double* w, int64_t P, const double* wmax, const double* M, int from_loglik,
                            uint64_t* q, int* flags, cudaStream_t st);
cudaError_t launch_scan(uint64_t* q, int64_t P, uint64_t* block_sums, cudaStream_t st);
cudaError_t launch_ancestors(const uint64_t* C, int64_t P_local, const uint64_t* plan, int64_t P_total, uint32_t u_bits,
                             int64_t p_global0, int64_t* own_anc, int64_t* const* peer_anc, int* flags,
                             cudaStream_t st);
cudaError_t launch_plan(const uint64_t* Qall, int nranks, int rank, int64_t P_total, uint32_t u_bits, uint64_t* plan,
                        cudaStream_t st);
cudaError_t launch_sum_ranks(const double* in, int nranks, int n, double* out, cudaStream_t st);
cudaError_t launch_gather(const double* x, const int64_t* anc, int64_t n, int64_t p_global0, double* out,
                          cudaStream_t st);
cudaError_t launch_predict(double* x, int64_t P, int64_t p0, double T, double sigma_v, uint64_t key,
                           uint64_t step, cudaStream_t st);
cudaError_t launch_chol6(const double* est, double* L, cudaStream_t st);
cudaError_t launch_regularize(double* x, int64_t P, int64_t p0, int64_t P_total, const double* L,
                              uint64_t key, uint64_t step, cudaStream_t st);
cudaError_t launch_fill_u64(uint64_t* dst, uint64_t v, int n, cudaStream_t st);

// loglik.cu K1 Gram-only variant + taylor.cu K1T (spherical / planar-WB correlation from spectral Taylor tables)
int tay_centres(int nf, int lanes);
size_t tay_table_bytes(const SceneDev& sc, int lanes);  // lanes: the lane-group layout, else the thread layout
bool tay_lanes(const SceneDev& sc, int64_t P);  // table layout / correlation kernel choice for P particles
cudaError_t launch_tay_prep(const SceneDev& sc, const float2* y, float2* tab, int lanes, int direct,
                            cudaStream_t st);
int tay_gram_launches(const SceneDev& sc, int64_t P, bool tab);  // kernels per launch_tay_gram call
cudaError_t launch_tay_gram(const SceneDev& sc, const float4* tmpl, const double* particles, int64_t P, int pstride,
                            const double* sfv, int sfv_pp, float2* terms, const float* dn, int* wflag, cudaStream_t st);
// The scene's Dirichlet table for the Gram (taylor.cu dn_table_kernel): dn_table_floats(nf) floats, built per N_f
size_t dn_table_floats(int nf);
cudaError_t launch_dn_table(int nf, float* out, cudaStream_t st);
cudaError_t launch_tay_corr(const SceneDev& sc, const float2* tab, const float4* tmpl, const double* particles,
                            int64_t P, int pstride, const double* sfv, int sfv_pp, float2* terms, int* pflag,
                            int gram_diag, int lanes, cudaStream_t st);

// sort.cu: locality (Morton) processing order of a likelihood batch; perm[i] = particle index of processing slot i
size_t locality_sort_temp_bytes(int64_t P);
cudaError_t launch_locality_sort(const double* particles, int64_t P, int pstride, const double* sfv, int K, int sfv_pp,
                                 uint32_t* keys, uint32_t* keys_alt, int* idx, int* perm, void* temp, size_t temp_bytes,
                                 double* pos, double* sfv_out, cudaStream_t st);

// F1 (pf.cu, taylor.cu pf_corr_kernel): PF-particle update message kappa~ and the PF normalization
cudaError_t launch_pf_corr(const SceneDev& sc, int T, const float2* tab, const float4* tmpl, const double* particles,
                           int64_t P, int pstride, const double* phi, double2* out, int* pflag, cudaStream_t st);
cudaError_t launch_pf_prep(int J, int T, int64_t Nz, const float2* y, const float2* mu3, const float2* mcols,
                           float2* snaps, double2* dots, const double* d_eta, double2* fixed, int* flags,
                           cudaStream_t st);
cudaError_t launch_pf_finish(const SceneDev& sc, int T, const double2* cc, const double2* fixed, const double* d_eta,
                             const double* d_zeta, double* gain2, const double* particles, int pstride,
                             const double* phi, const double* walpha, const double2* mu, const double* gamma,
                             int* pflag, int64_t P, double* logr, double* w, double* out, int* flags,
                             double* lse_part, cudaStream_t st);
// two-level deterministic log-sum-exp over R rows (lse.cu): out [R][3] = (max, sum e^{l - max}, sum of the companion
// row a or 0); part: 3 R lse_blocks(P) doubles
int lse_blocks(int64_t P);
cudaError_t launch_lse_rows(const double* l, int64_t ld, int R, int64_t P, const double* a, int64_t lda, double* part,
                            double* out, cudaStream_t st);
cudaError_t launch_vec_stack_dots(int J, int T, int L, int64_t Nz, const float2* y, const float2* mu, const float2* cols,
                                  const float2* x1, const float2* x2, float2* stack, double2* dots, cudaStream_t st);
// slam.cu: F4 update messages nu~ (noise) and omega~ (PPR)
cudaError_t launch_noise_update(int J, int L, int64_t P, int64_t Nz, const double2* dots, double* eig, const double* eta,
                                const double* wxi, double* logw, double* lognorm, double* w, int* flags,
                                double* lse_part, cudaStream_t st);
cudaError_t launch_ppr_update(int J, int L, const double2* dots, const double* zeta, const double* eta, double* out,
                              int* flags, cudaStream_t st);
int slam_eig_width();     // doubles per PA of the nu~ eigen data
int slam_max_columns();   // feature columns <= 9
int pf_fixed_width();     // double2 per PA of the fixed (particle-independent) part
int pf_max_snapshots();   // T = L + 1 <= 9

// nbmma.cu: PLANAR_NB correlation on the tensor cores
struct NbPlan {
  int kc;              // real K per pipeline stage (2 x subcarriers), 16 / 32 / 64
  int nst;             // pipeline stages
  int n_pass;          // antenna passes (2 ceil8(N_a) > 256 takes several)
  int nbh;             // antennas per pass, padded to 8: Re W in accumulator columns [0, nbh), Im W in [nbh, 2 nbh)
  int nb;              // UMMA N = 2 nbh (<= 256)
  int nacc;            // accumulator pairs (D1 exact hi x hi, D2 the rest) in TMEM: 2 when 4 nb <= 512
  int tmem_cols;       // allocated TMEM columns (power of two >= 32)
  int pexp, qexp;      // hi grids: A_hi on 2^-pexp of |b| = 1, y_hi on 2^-qexp of max|y|; K 2^(p+q) <= 2^24
  int a_tmem;          // 1: A operand staged in TMEM (tcgen05.st by the generators; MMA reads only B from smem)
  int a_col0;          // TMEM column of the A ring (a_tmem): stage s at a_col0 + s kc, hi then lo (kc/2 columns each)
  int nf_pad;          // subcarriers padded to kc / 2
  int n_chunks;        // pipeline stages per tile = 2 nf_pad / kc
  uint32_t a_bytes;    // one fp16 piece of the A stage (128 x kc)
  uint32_t b_bytes;    // one fp16 piece of the B stage (nb x kc)
  size_t smem;         // dynamic shared memory of nb_corr_kernel
};
struct NbArgs {
  const double* particles;  // batch start
  int64_t P;
  int pstride;
  const double* sfv;        // [K][3] or [P][K][3] at the batch (sfv_pp)
  int sfv_pp;
  const uint8_t* bop;       // [J][n_chunks][2][nb x kc] fp16 B operand (nb_prep_kernel)
  const float* yscale_inv;  // [J] 2^e_j
  double2* terms;           // [P][J][T]: c_s written by nb_corr_kernel, G by nb_gram_kernel
  int64_t n_tiles_j;        // ceil(P S / 128)
  int64_t n_tiles;          // n_tiles_j J
  int diag_only;            // nb_gram_kernel: write G = diag(g^2 N_z) only (callers that use c only)
};
bool nb_tensor_plan(const SceneDev& sc, NbPlan* pl);  // false: shape not supported (2 N_a > 512)
size_t nb_operand_bytes(const SceneDev& sc, const NbPlan& pl);
cudaError_t launch_nb_prep(const SceneDev& sc, const NbPlan& pl, const float2* y, uint8_t* bop, float* yscale_inv,
                           cudaStream_t st);
cudaError_t launch_nb_gram(const SceneDev& sc, const NbArgs& a, int* pflag, cudaStream_t st);
cudaError_t launch_nb_corr(const SceneDev& sc, const NbPlan& pl, const NbArgs& a, int num_sms, cudaStream_t st);

// birth.cu: F3 birth proposal
struct BirthBox {                  // by-value kernel parameter
  double lo[3], hi[3];             // partition P_q (axis-aligned box)
  double x_hat[3];                 // predicted MMSE MT position
  double sfv[MAXS - 1][3];         // legacy PF MMSE SFVs
  int L;                           // number of legacy PFs
};
int64_t birth_blocks(int64_t N_g);
cudaError_t launch_birth_items(const BirthBox& box, int J, double* pos, int32_t* js, double* sfv, cudaStream_t st);
cudaError_t launch_birth_residual(int J, int nz, int n, const double2* psi, const float2* y, double2* dots,
                                  double2* coef, float2* zr, int* flags, cudaStream_t st);
int64_t birth_pseudo_particles(int64_t N_g);  // pseudo-particles of MAXS - 1 candidate walls each
cudaError_t launch_birth_candidates(int64_t N_g, uint64_t key, uint64_t counter, const BirthBox& box, double* cand,
                                    cudaStream_t st);
cudaError_t launch_birth_reduce(int64_t N_g, int J, int nz, const double2* c, const double* cand, double* pb,
                                double4* part, double* part6, double* scratch, double* out, int* flags,
                                cudaStream_t st);

// step.cu: the fused O(P) pipeline of cdms_bp_step (fixed STEP_ITEMS-particle blocks, last-block reductions)
constexpr int STEP_ITEMS = 512;
int64_t step_blocks(int64_t P);
cudaError_t launch_step_lse(const double* l, int64_t P, double2* part, unsigned* cnt, double2* rank_pair, int combine,
                            double* lse, double* M, double* logS, int* flags, cudaStream_t st);
cudaError_t launch_step_lse_global(const double2* gpart, int64_t nbt, double2* rank_pair, double* lse, double* M,
                                   double* logS, int* flags, cudaStream_t st);
cudaError_t launch_step_post(const double* l, const double* x, int64_t P, const double* M, const double* logS,
                             const int* flags, double* w, uint64_t* q, double* mpart, uint64_t* bsum, unsigned* cnt,
                             double* sum1, uint32_t u_bits, uint64_t* plan, cudaStream_t st);
cudaError_t launch_step_post_global(const double* gmpart, int64_t nbt, double* sum1, const uint64_t* Qall, int nranks,
                                    int rank, int64_t P_total, uint32_t u_bits, uint64_t* plan, cudaStream_t st);
cudaError_t launch_step_scan(uint64_t* q, const double* x, const double* w, int64_t P, const uint64_t* boff,
                             const double* sum1, const int* flags, double* mpart, unsigned* cnt, double* sum2,
                             int finalize, double* est, double* L, int* flags_w, cudaStream_t st);
cudaError_t launch_step_scan_global(const double* gmpart, int64_t nbt, const double* sum1, double* sum2, double* est,
                                    double* L, int* flags, cudaStream_t st);
cudaError_t launch_step_anc(const uint64_t* C, const uint64_t* boff, int64_t P_local, const uint64_t* plan,
                            int64_t P_total, uint32_t u_bits, const double* x, double* own_x, int64_t* own_anc,
                            double* const* peer_x, int64_t* const* peer_anc, int64_t p_global0, int* flags,
                            cudaStream_t st);
cudaError_t launch_step_reg(const double* in, double* out, int64_t P, int64_t p0, int64_t P_total, const double* L,
                            int regularize, uint64_t key, uint64_t step, cudaStream_t st);
// fused single-rank pipeline (K_lse .. K_reg in one cooperative launch, step.cu)
struct StepFusedArgs {
  const double* l;
  double* x;  // particles [P][6], read by K_post / K_scan / K_anc, overwritten by K_reg
  int64_t P;
  double2* lpart;
  double2* rank_pair;
  double *lse, *M, *logS;
  int* flags;
  double* w;
  uint64_t* q;
  double* mpart;
  uint64_t* bsum;  // [nb + 1]
  double* sums;    // [32]: sum1 at 0, sum2 at 8
  double *est, *L;
  double* stage;  // [P][6]
  int64_t* anc;   // [P] ancestors out, or nullptr
  uint64_t* plan; // [4] resampling plan (Q, O, slot_lo, slot_hi)
  uint32_t u_bits;
  double h;
  int regularize;
  uint64_t key, step;
};
cudaError_t launch_step_fused(const StepFusedArgs& a, int num_sms, cudaStream_t st);
double step_reg_bandwidth(int64_t P_total);

// F4 step driver kernels (slam_step.cu)
struct SlamWsumJob {
  const double* w;  // weights [P] or nullptr (all 1)
  const double* v;  // values, row p at v + p vs
  int64_t P;
  int vs, nc;       // row stride, columns (<= 3)
};
constexpr int SLAM_MAXJOBS = 64;
struct SlamWsumJobs {
  SlamWsumJob job[SLAM_MAXJOBS];
  int n;
};
constexpr int SLAM_PAR = MAXS + MAXS * MAXJ;  // device slot parameters: eps [MAXS], zeta [MAXS][MAXJ]
cudaError_t launch_slam_noise_predict(double* eta, int J, int64_t P, double c, uint64_t key, uint64_t n,
                                      cudaStream_t st);
cudaError_t launch_slam_pf_predict(double* phi, double2* mu, double* gam, double* w, int64_t P, int slot,
                                   double sigma_sfv, double sigma_mu, double c_gamma, double p_s, uint64_t key,
                                   uint64_t n, cudaStream_t st);
cudaError_t launch_slam_birth(const double* mu_q, const double* Lq, const double* box, double mu_max, double gamma_max,
                              double pB, double* phi, double2* mu, double* gam, double* lw, double* w, double* out,
                              double* lse_part, int64_t P, uint64_t key, uint64_t n, cudaStream_t st);
int slam_wsum_blocks(int64_t P);  // part: 4 jobs slam_wsum_blocks(max P) doubles (cov: 7 slam_wsum_blocks(P))
cudaError_t launch_slam_wsum(const SlamWsumJobs& jobs, double* part, double* out, cudaStream_t st);
cudaError_t launch_slam_bv_wsum(const double* w, int64_t P, int64_t K, int S, double* wk, cudaStream_t st);
cudaError_t launch_slam_bv_items(const double* x, const double* phi, int64_t P, int64_t K, int64_t k0, int B, int J,
                                 int S, double* pos, int32_t* js, double* sfv, cudaStream_t st);
cudaError_t launch_slam_bv_accum(const double2* psi, const double2* mu, const double* gam, const double* w,
                                 const double* wk, const double* par, int64_t P, int64_t K, int64_t k0, int B, int J,
                                 int S, int64_t Nz, double2* au, double2* am, double2* aw, cudaStream_t st);
cudaError_t launch_slam_bv_final(const double2* am, const double2* au, const double* par, int J, int S, int64_t Nz,
                                 float2* m64, float2* munu, cudaStream_t st);
cudaError_t launch_slam_others(const double2* au, const double2* am, const double2* aw, const double* par, int J, int S,
                               int64_t Nz, int s, float2* mu3, float2* mo, float2* mws, float2* us, cudaStream_t st);
cudaError_t launch_slam_sfv_pp(const double* phi, int64_t P, int K, double* out, cudaStream_t st);
cudaError_t launch_slam_pf_gather(const double* phi, const double2* mu, const double* gam, const int64_t* anc,
                                  int64_t P, double* tphi, double2* tmu, double* tgam, cudaStream_t st);
cudaError_t launch_slam_fill(double* w, int64_t P, double v, cudaStream_t st);
cudaError_t launch_slam_gather1(const double* src, const int64_t* anc, int64_t P, double* dst, cudaStream_t st);
cudaError_t launch_slam_sfv_reg(const double* w, const double* phi_src, double* phi_dst, int64_t P, const double* mean,
                                double h, double* L, double* part, uint64_t key, uint64_t n, int slot, cudaStream_t st);

}  // namespace cdms
