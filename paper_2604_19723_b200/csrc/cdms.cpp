// cdms.cpp -- host side of libcdms: the extern "C" ABI of include/cdms.h.  Validation happens here,
// before any launch; every device step is one of the kernels in loglik.cu / response.cu / beliefs.cu,
// enqueued on the context's stream; cross-GPU steps are NCCL collectives on the context's
// communicator (one process per GPU).
#include <cuda_runtime.h>
#include <math.h>
#include <nccl.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>
#include <vector>

#include "cdms_internal.h"

using namespace cdms;

struct cdms_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  std::string err;
  int* d_flags = nullptr;
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  int64_t launches = 0;
  std::vector<void*> bufs;
  std::vector<size_t> sizes;
  uint64_t* h_pinned = nullptr;  // small pinned host staging (plan exchange)
  bool timing = false;           // bracket the likelihood kernel with events
  bool nb_tensor = true;         // PLANAR_NB fp32 on the tensor cores (nbmma.cu); CDMS_NB_TENSOR=0 selects K1
  bool taylor = true;            // spherical / planar-WB fp32 correlation by K1T (taylor.cu); CDMS_TAYLOR=0 selects K1
  int taylor_gram = 0;           // K1T's off-diagonal Gram: 0/2 tay_gram_kernel, 1 K1's Horner-free variant
                                 // (CDMS_TAYLOR_GRAM=k1 / tay, A/B only)
  int step_fused = 0;           // 1: single-rank bp_step O(P) phases in one cooperative kernel (CDMS_STEP_FUSED=1,
                                 // A/B; measured not faster: c2 0.409 vs 0.403 ms, the grid barriers and block 0's
                                 // epilogues cost what the launches did)
  int taylor_prep_direct = 0;   // K1T tables by the direct sum even when G is a power of two (CDMS_TAY_PREP=direct,
                                 // A/B only; default FFT)
  int taylor_lanes = -1;         // K1T correlation kernel: -1 by P J (tay_lanes), 1 lane groups, 0 thread per
                                 // particle (CDMS_TAY_LANES=1 / 0, A/B only)
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
};

namespace {

enum Slot {
  WS_YTILES, WS_YNORM, WS_LSE_PART, WS_LSE_RANK, WS_SCAL, WS_MOM_PART, WS_SUMS, WS_WMAX_PART, WS_Q, WS_BSUM,
  WS_QALL, WS_LOGLIK, WS_W, WS_ANC, WS_STAGE, WS_L6, WS_ANC2, WS_TERMS, WS_PFLAG, WS_TMPL, WS_SCHED, WS_STEP_CNT, WS_NBOP, WS_NBSCALE,
  WS_BPOS, WS_BJS, WS_BSFV, WS_BPSI, WS_BDOTS, WS_BCOEF, WS_BZR, WS_BCAND, WS_BC, WS_BLL, WS_BPB,
  WS_BPART, WS_BPART6, WS_BSCR, WS_TAY, WS_COUNT
};
constexpr size_t TERMS_BUDGET = (size_t)2 << 30;  // bytes of per-(particle, PA) sufficient statistics per batch

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

cdms_status fail(cdms_ctx ctx, cdms_status st, const char* fmt, ...) {
  if (ctx) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    ctx->err = buf;
  }
  return st;
}

#define CUDA_TRY(ctx, expr)                                                                  \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess) return fail(ctx, CDMS_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

#define NCCL_TRY(ctx, expr)                                                                  \
  do {                                                                                       \
    ncclResult_t r_ = (expr);                                                                \
    if (r_ != ncclSuccess) return fail(ctx, CDMS_ENCCL, "%s: %s", #expr, ncclGetErrorString(r_)); \
  } while (0)

template <typename T>
cdms_status ws(cdms_ctx ctx, int slot, size_t count, T** out) {
  const size_t bytes = count * sizeof(T) + 256;
  if (ctx->sizes[slot] < bytes) {
    if (ctx->bufs[slot]) cudaFree(ctx->bufs[slot]);
    ctx->bufs[slot] = nullptr;
    ctx->sizes[slot] = 0;
    size_t want = bytes + bytes / 4;
    cudaError_t e = cudaMalloc(&ctx->bufs[slot], want);
    if (e != cudaSuccess) return fail(ctx, CDMS_ENOMEM, "cudaMalloc(%zu): %s", want, cudaGetErrorString(e));
    ctx->sizes[slot] = want;
    // fresh workspaces start zeroed (K1's per-particle flags are OR-accumulated and cleared by K1b)
    e = cudaMemsetAsync(ctx->bufs[slot], 0, want, ctx->stream);
    if (e != cudaSuccess) return fail(ctx, CDMS_ECUDA, "cudaMemsetAsync: %s", cudaGetErrorString(e));
  }
  *out = static_cast<T*>(ctx->bufs[slot]);
  return CDMS_OK;
}

#define WS_TRY(ctx, slot, count, ptr)                  \
  do {                                                 \
    cdms_status s_ = ws(ctx, slot, (size_t)(count), ptr); \
    if (s_ != CDMS_OK) return s_;                      \
  } while (0)

bool is_fin(double x) { return x == x && x != INFINITY && x != -INFINITY; }

// Validate the scene and fill the device parameter block (priors / eta optional).
cdms_status build_scene(cdms_ctx ctx, const cdms_scene* sc, const double* f_pb, const cdms_prior* prior,
                        const double* eta, SceneDev* out) {
  if (!sc) return fail(ctx, CDMS_EINVAL, "scene is NULL");
  if (sc->J < 1 || sc->J > MAXJ) return fail(ctx, CDMS_EINVAL, "J=%d outside [1,%d]", sc->J, MAXJ);
  if (sc->K < 0 || sc->K + 1 > MAXS) return fail(ctx, CDMS_EINVAL, "K=%d outside [0,%d]", sc->K, MAXS - 1);
  if (sc->ny < 1 || sc->nv < 1 || (int64_t)sc->ny * sc->nv > 4096)
    return fail(ctx, CDMS_EINVAL, "URA %d x %d invalid", sc->ny, sc->nv);
  if (sc->nf < 1 || sc->nf > 65536) return fail(ctx, CDMS_EINVAL, "nf=%d invalid", sc->nf);
  if (sc->wavefront < 0 || sc->wavefront > 2) return fail(ctx, CDMS_EINVAL, "wavefront=%d invalid", sc->wavefront);
  if (sc->precision < 0 || sc->precision > 1) return fail(ctx, CDMS_EINVAL, "precision=%d invalid", sc->precision);
  if (!is_fin(sc->dy) || !is_fin(sc->dv) || !(sc->fc > 0.0) || !is_fin(sc->fc) || !is_fin(sc->df) || sc->df < 0.0)
    return fail(ctx, CDMS_EINVAL, "dy/dv/fc/df invalid");
  if (!sc->h_pa_pos || !sc->h_pa_rot) return fail(ctx, CDMS_EINVAL, "h_pa_pos / h_pa_rot NULL");
  memset(out, 0, sizeof(*out));
  out->J = sc->J;
  out->K = sc->K;
  out->S = sc->K + 1;
  out->ny = sc->ny;
  out->nv = sc->nv;
  out->Na = sc->ny * sc->nv;
  out->nf = sc->nf;
  out->wavefront = sc->wavefront;
  out->pathloss = sc->pathloss ? 1 : 0;
  {
    const int kc = corr_kchunk(out->S);
    out->kc_len = sc->nf < kc ? sc->nf : kc;
  }
  out->n_mb = (out->Na + NWARP - 1) / NWARP;
  out->n_kc = (sc->nf + out->kc_len - 1) / out->kc_len;
  out->dy = sc->dy;
  out->dv = sc->dv;
  out->fc = sc->fc;
  out->df = sc->df;
  out->f0 = sc->fc - 0.5 * (sc->nf - 1) * sc->df;
  out->f0_c = out->f0 / C_LIGHT;
  out->df_c = sc->df / C_LIGHT;
  out->segdf_c = (double)SEG * sc->df / C_LIGHT;
  out->fc_c = sc->fc / C_LIGHT;
  out->lambda = C_LIGHT / sc->fc;
  out->fc_cf = (float)out->fc_c;
  out->df_cf = (float)out->df_c;
  out->nf_f = (float)sc->nf;
  out->c6N_f = (float)(PI * PI / 6.0 * ((double)sc->nf * sc->nf - 1.0));
  out->evenN_mask = ((sc->nf - 1) & 1) ? 0x80000000u : 0u;
  out->f0_cf = (float)out->f0_c;
  out->segdf_cf = (float)out->segdf_c;
  out->two_seg = (sc->nf > SEG && sc->nf <= 2 * SEG && sc->wavefront != CDMS_PLANAR_NB) ? 1 : 0;
  out->f1_c = (out->f0 + (double)SEG * sc->df) / C_LIGHT;
  out->f1_cf = (float)out->f1_c;
  out->y_mb_step = (int64_t)(NWARP - 1) * out->n_kc * out->kc_len;
  {
    // |Delta_m| <= ||q_m|| = ||p~_m|| <= half the URA diagonal (H, R orthogonal)
    const double hy = 0.5 * (sc->ny - 1) * fabs(sc->dy), hv = 0.5 * (sc->nv - 1) * fabs(sc->dv);
    const double th = 2.0 * PI * sqrt(hy * hy + hv * hv) * out->df_c;
    out->small_step = (th <= 0.02) ? 2 : (th <= 0.2) ? 1 : 0;
    out->small_z = (2.0 * PI * sqrt(hy * hy + hv * hv) * out->segdf_c <= 1.0) ? 1 : 0;
  }
  for (int j = 0; j < sc->J; ++j) {
    const double* R = sc->h_pa_rot + 9 * j;
    for (int c = 0; c < 3; ++c) {
      if (!is_fin(sc->h_pa_pos[3 * j + c])) return fail(ctx, CDMS_EINVAL, "pa_pos[%d] not finite", j);
      out->pa_pos[j][c] = sc->h_pa_pos[3 * j + c];
    }
    double det = R[0] * (R[4] * R[8] - R[5] * R[7]) - R[1] * (R[3] * R[8] - R[5] * R[6]) +
                 R[2] * (R[3] * R[7] - R[4] * R[6]);
    double orth = 0.0;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double s = 0.0;
        for (int c = 0; c < 3; ++c) s += R[a * 3 + c] * R[b * 3 + c];
        orth = fmax(orth, fabs(s - (a == b ? 1.0 : 0.0)));
      }
    if (!(orth <= 1e-9) || !(fabs(det - 1.0) <= 1e-9))
      return fail(ctx, CDMS_EINVAL, "pa_rot[%d] not in SO(3) (|RR^T-I|=%.3g, det=%.12g)", j, orth, det);
    for (int c = 0; c < 9; ++c) out->pa_rot[j][c] = R[c];
  }
  if (f_pb) {
    for (int k = 0; k < sc->nf; ++k) {
      const double want = out->f0 + k * sc->df;
      if (!(fabs(f_pb[k] - want) <= 1e-9 * sc->fc))
        return fail(ctx, CDMS_EINVAL, "f_pb[%d]=%.17g does not match the uniform grid (%.17g)", k, f_pb[k], want);
    }
  }
  if (prior) {
    for (int j = 0; j < sc->J; ++j)
      for (int s = 0; s < out->S; ++s) {
        const cdms_prior& q = prior[j * out->S + s];
        if (!is_fin(q.m_re) || !is_fin(q.m_im) || !is_fin(q.v) || q.v < 0.0)
          return fail(ctx, CDMS_EINVAL, "prior[%d][%d] invalid", j, s);
        out->m_re[j][s] = q.m_re;
        out->m_im[j][s] = q.m_im;
        out->v[j][s] = q.v;
      }
  }
  if (eta) {
    for (int j = 0; j < sc->J; ++j) {
      if (!(eta[j] > 0.0) || !is_fin(eta[j])) return fail(ctx, CDMS_EINVAL, "eta[%d] must be > 0", j);
      out->eta[j] = eta[j];
    }
  }
  return CDMS_OK;
}

// Philox4x32-10 on the host (for the per-step resampling offset u = first word of (0, 0, step, 3)).
uint32_t host_step_u_bits(uint64_t key, uint64_t step) {
  uint32_t c0 = 0, c1 = 0, c2 = (uint32_t)step, c3 = 3u, k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n1 = (uint32_t)p1, n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1,
                   n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  return c0;
}

// I(x) = #{i in [0, P_total) : t_i < x}, t_i = floor((u + i 2^32) Q / (P_total 2^32)) (exact, 128-bit)
int64_t slot_index(uint64_t x, uint64_t Q, int64_t P_total, uint32_t u) {
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

// ---------------------------------------------------------------------------- internal pipelines
cdms_status run_lse(cdms_ctx ctx, const double* d_l, int64_t P, double* d_lse) {
  const int64_t nb = red_blocks(P);
  double2 *part, *per_rank;
  double* scal;
  WS_TRY(ctx, WS_LSE_PART, nb + 1, &part);
  WS_TRY(ctx, WS_LSE_RANK, ctx->nranks + 1, &per_rank);
  WS_TRY(ctx, WS_SCAL, 8, &scal);
  CUDA_TRY(ctx, launch_lse_partial(d_l, P, part, ctx->stream));
  if (ctx->comm) {
    CUDA_TRY(ctx, launch_lse_final(part, nb, part + nb, ctx->stream));
    NCCL_TRY(ctx, ncclAllGather(part + nb, per_rank, 2, ncclDouble, ctx->comm, ctx->stream));
  } else {
    CUDA_TRY(ctx, launch_lse_final(part, nb, per_rank, ctx->stream));
  }
  CUDA_TRY(ctx, launch_lse_combine(per_rank, ctx->nranks, d_lse, scal + 0, scal + 1, ctx->d_flags, ctx->stream));
  ctx->launches += 3;
  return CDMS_OK;
}

cdms_status run_moments(cdms_ctx ctx, const double* d_x, const double* d_w, int64_t P, double* d_est) {
  const int64_t nb = red_blocks(P);
  double *part, *sums;
  WS_TRY(ctx, WS_MOM_PART, (nb + 1) * 21, &part);
  WS_TRY(ctx, WS_SUMS, 32, &sums);
  CUDA_TRY(ctx, launch_moments1(d_x, d_w, P, part, ctx->stream));
  CUDA_TRY(ctx, launch_sum_partials(part, nb, 7, sums, ctx->stream));
  if (ctx->comm) NCCL_TRY(ctx, ncclAllReduce(sums, sums, 7, ncclDouble, ncclSum, ctx->comm, ctx->stream));
  CUDA_TRY(ctx, launch_moments2(d_x, d_w, P, sums, part, ctx->stream));
  CUDA_TRY(ctx, launch_sum_partials(part, nb, 21, sums + 8, ctx->stream));
  if (ctx->comm)
    NCCL_TRY(ctx, ncclAllReduce(sums + 8, sums + 8, 21, ncclDouble, ncclSum, ctx->comm, ctx->stream));
  CUDA_TRY(ctx, launch_moments_finalize(sums, sums + 8, d_est, ctx->d_flags, ctx->stream));
  ctx->launches += 5;
  return CDMS_OK;
}

// Quantize + scan + ancestors for this rank's CDF range.  from_loglik: r_p = e^{l_p - M} (M = global max,
// in WS_SCAL[0]); else r_p = w_p / w_max (global).  Results: the global ancestor ids of the slots
// [slot_lo, slot_hi) that this rank's CDF range covers, in *d_anc_out (WS_ANC), plus the plan.
struct Plan {
  int64_t lo = 0, hi = 0;
  std::vector<int64_t> lo_all, hi_all;
};

cdms_status run_resample_core(cdms_ctx ctx, const double* d_in, int64_t P_local, uint32_t u_bits, int from_loglik,
                              Plan* plan, int64_t** d_anc_out) {
  const int64_t nb = red_blocks(P_local);
  const int64_t P_total = P_local * ctx->nranks;
  if (P_total > ((int64_t)1 << 26)) return fail(ctx, CDMS_EINVAL, "P_total=%lld exceeds 2^26", (long long)P_total);
  uint64_t *q, *bsum, *qall;
  double *scal, *wpart;
  int64_t* anc;
  WS_TRY(ctx, WS_Q, P_local, &q);
  WS_TRY(ctx, WS_BSUM, nb + 2, &bsum);
  WS_TRY(ctx, WS_QALL, 2 * ctx->nranks + 4, &qall);
  WS_TRY(ctx, WS_SCAL, 8, &scal);
  if (!from_loglik) {
    WS_TRY(ctx, WS_WMAX_PART, nb + 1, &wpart);
    CUDA_TRY(ctx, launch_wmax_partial_f(d_in, P_local, wpart, ctx->d_flags, ctx->stream));
    CUDA_TRY(ctx, launch_max_final(wpart, nb, scal + 2, ctx->stream));
    if (ctx->comm)
      NCCL_TRY(ctx, ncclAllReduce(scal + 2, scal + 2, 1, ncclDouble, ncclMax, ctx->comm, ctx->stream));
    ctx->launches += 2;
  }
  CUDA_TRY(ctx, launch_quantize(d_in, P_local, scal + 2, scal + 0, from_loglik, q, ctx->d_flags, ctx->stream));
  CUDA_TRY(ctx, launch_scan(q, P_local, bsum, ctx->stream));
  ctx->launches += 4;
  if (!(ctx->comm)) {
    WS_TRY(ctx, WS_ANC, P_local, &anc);
    CUDA_TRY(ctx, launch_ancestors(q, P_local, bsum + nb, nullptr, 0, P_local, P_local, u_bits, 0, anc, ctx->d_flags,
                                   ctx->stream));
    ctx->launches += 1;
    plan->lo = 0;
    plan->hi = P_local;
    plan->lo_all.assign(1, 0);
    plan->hi_all.assign(1, P_local);
    *d_anc_out = anc;
    return CDMS_OK;
  }
  // multi-rank: all-gather Q_r, host plan (one small D2H + stream sync per step)
  NCCL_TRY(ctx, ncclAllGather(bsum + nb, qall, 1, ncclUint64, ctx->comm, ctx->stream));
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_pinned, qall, sizeof(uint64_t) * ctx->nranks, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  std::vector<uint64_t> Q(ctx->h_pinned, ctx->h_pinned + ctx->nranks);
  uint64_t Qtot = 0;
  for (uint64_t v : Q) Qtot += v;
  if (Qtot == 0) return fail(ctx, CDMS_EZEROMASS, "all resampling weights are zero");
  plan->lo_all.resize(ctx->nranks);
  plan->hi_all.resize(ctx->nranks);
  uint64_t O = 0, Omine = 0;
  for (int r = 0; r < ctx->nranks; ++r) {
    plan->lo_all[r] = slot_index(O, Qtot, P_total, u_bits);
    plan->hi_all[r] = slot_index(O + Q[r], Qtot, P_total, u_bits);
    if (r == ctx->rank) Omine = O;
    O += Q[r];
  }
  plan->lo = plan->lo_all[ctx->rank];
  plan->hi = plan->hi_all[ctx->rank];
  ctx->h_pinned[ctx->nranks] = Qtot;
  ctx->h_pinned[ctx->nranks + 1] = Omine;
  CUDA_TRY(ctx, cudaMemcpyAsync(qall + ctx->nranks, ctx->h_pinned + ctx->nranks, 2 * sizeof(uint64_t),
                                cudaMemcpyHostToDevice, ctx->stream));
  const int64_t n = plan->hi - plan->lo;
  WS_TRY(ctx, WS_ANC, n > 0 ? n : 1, &anc);
  CUDA_TRY(ctx, launch_ancestors(q, P_local, qall + ctx->nranks, qall + ctx->nranks + 1, plan->lo, plan->hi, P_total,
                                 u_bits, (int64_t)ctx->rank * P_local, anc, ctx->d_flags, ctx->stream));
  ctx->launches += 1;
  *d_anc_out = anc;
  return CDMS_OK;
}

// Redistribute `width` 8-byte words per slot from the staging rows of this rank's CDF slots
// [plan.lo, plan.hi) to the owners of those slots (slot i lives on rank i / P_local, row i % P_local).
cdms_status exchange(cdms_ctx ctx, const Plan& plan, int64_t P_local, const void* src, void* dst, int width) {
  const int R = ctx->nranks;
  const size_t row = (size_t)width * 8;
  NCCL_TRY(ctx, ncclGroupStart());
  for (int d = 0; d < R; ++d) {  // sends
    const int64_t a = plan.lo > d * P_local ? plan.lo : d * P_local;
    const int64_t b = plan.hi < (d + 1) * P_local ? plan.hi : (d + 1) * P_local;
    if (b <= a || d == ctx->rank) continue;
    NCCL_TRY(ctx, ncclSend((const char*)src + (size_t)(a - plan.lo) * row, (size_t)(b - a) * width, ncclUint64, d,
                           ctx->comm, ctx->stream));
  }
  for (int s = 0; s < R; ++s) {  // receives
    const int64_t a = plan.lo_all[s] > ctx->rank * P_local ? plan.lo_all[s] : ctx->rank * P_local;
    const int64_t b = plan.hi_all[s] < (ctx->rank + 1) * P_local ? plan.hi_all[s] : (ctx->rank + 1) * P_local;
    if (b <= a || s == ctx->rank) continue;
    NCCL_TRY(ctx, ncclRecv((char*)dst + (size_t)(a - ctx->rank * P_local) * row, (size_t)(b - a) * width, ncclUint64, s,
                           ctx->comm, ctx->stream));
  }
  NCCL_TRY(ctx, ncclGroupEnd());
  const int64_t a = plan.lo > ctx->rank * P_local ? plan.lo : ctx->rank * P_local;
  const int64_t b = plan.hi < (ctx->rank + 1) * P_local ? plan.hi : (ctx->rank + 1) * P_local;
  if (b > a)
    CUDA_TRY(ctx, cudaMemcpyAsync((char*)dst + (size_t)(a - ctx->rank * P_local) * row,
                                  (const char*)src + (size_t)(a - plan.lo) * row, (size_t)(b - a) * row,
                                  cudaMemcpyDeviceToDevice, ctx->stream));
  return CDMS_OK;
}

cdms_status loglik_impl(cdms_ctx ctx, const SceneDev& sd, int precision, const double* d_particles, int64_t P,
                        int32_t pstride, const double* d_sfv, int32_t sfv_pp, const void* d_y, const double* d_logw,
                        double* d_loglik, void* d_amp, void* d_c = nullptr, void* d_G = nullptr,
                        bool no_gram = false) {
  float4* yt;
  double* yn;
  double2* terms;
  float4* tmpl;
  unsigned int* sched;
  int* pflag;
  const int64_t tiles = (int64_t)sd.J * sd.n_mb * sd.n_kc * sd.kc_len * NWARP;
  WS_TRY(ctx, WS_YTILES, tiles, &yt);
  WS_TRY(ctx, WS_YNORM, MAXJ, &yn);
  WS_TRY(ctx, WS_TMPL, (int64_t)sd.J * sd.n_mb * NWARP, &tmpl);
  CUDA_TRY(ctx, launch_prep_y(sd, static_cast<const float2*>(d_y), yt, yn, tmpl, ctx->stream));
  ctx->launches += 1;
  // PLANAR_NB in fp32: the correlation runs as a tensor-core GEMM (nbmma.cu) with the closed-form Gram
  NbPlan nbp{};
  const bool nbt = ctx->nb_tensor && precision == CDMS_FP32 && nb_tensor_plan(sd, &nbp);
  uint8_t* nbop = nullptr;
  float* nbscale = nullptr;
  // spherical / planar WB in FP32: c from spectral Taylor tables (K1T), G from K1's Horner-free variant
  const bool tay = !nbt && ctx->taylor && precision == CDMS_FP32 && sd.wavefront != CDMS_PLANAR_NB &&
                   tay_table_bytes(sd) <= ((size_t)96 << 20);
  float2* taytab = nullptr;
  const int tlanes = tay && (ctx->taylor_lanes >= 0 ? ctx->taylor_lanes == 1 : tay_lanes(sd, P)) ? 1 : 0;  // taylor.cu
  if (tay) {
    WS_TRY(ctx, WS_TAY, tay_table_bytes(sd) / sizeof(float2), &taytab);
    CUDA_TRY(ctx, launch_tay_prep(sd, static_cast<const float2*>(d_y), taytab, tlanes, ctx->taylor_prep_direct,
                                  ctx->stream));
    ctx->launches += 1;
  }
  if (nbt) {
    WS_TRY(ctx, WS_NBOP, nb_operand_bytes(sd, nbp), &nbop);
    WS_TRY(ctx, WS_NBSCALE, MAXJ, &nbscale);
    CUDA_TRY(ctx, launch_nb_prep(sd, nbp, static_cast<const float2*>(d_y), nbop, nbscale, ctx->stream));
    ctx->launches += 1;
  }
  // particles go through K1 (correlation + Gram -> HBM terms) and K1b (assembly) in batches whose terms
  // buffer stays under TERMS_BUDGET bytes
  const int T = terms_width(sd.S);
  const size_t per_particle = (size_t)sd.J * T * sizeof(double2);
  int64_t PB = (int64_t)(TERMS_BUDGET / per_particle);
  PB = PB < TILE_P ? TILE_P : (PB / TILE_P) * TILE_P;
  if (PB > P) PB = P;
  WS_TRY(ctx, WS_TERMS, (size_t)PB * sd.J * T, &terms);
  WS_TRY(ctx, WS_PFLAG, PB, &pflag);
  WS_TRY(ctx, WS_SCHED, 2, &sched);  // zeroed at allocation, reset by the last K1 CTA of every launch
  if ((PB + TILE_P - 1) / TILE_P * sd.J >= (int64_t)1 << 31) return fail(ctx, CDMS_EINVAL, "loglik: batch too large");
  for (int64_t b0 = 0; b0 < P; b0 += PB) {
    const int64_t nb = (P - b0 < PB) ? P - b0 : PB;
    CorrArgs a;
    a.particles = d_particles + b0 * pstride;
    a.P = nb;
    a.pstride = pstride;
    a.sfv = (d_sfv && sfv_pp) ? d_sfv + b0 * 3 * sd.K : d_sfv;
    a.sfv_pp = sfv_pp;
    a.ytiles = yt;
    a.tmpl = tmpl;
    a.terms = terms;
    a.pflag = pflag;
    a.flags = ctx->d_flags;
    a.n_tiles = (nb + TILE_P - 1) / TILE_P;
    a.n_groups = a.n_tiles * sd.J;
    a.grid = tay ? corr_grid_gram_only(sd, a.n_tiles, ctx->num_sms) : corr_grid(sd, a.n_tiles, precision, ctx->num_sms);
    if (a.grid < 1) return fail(ctx, CDMS_ECUDA, "corr_kernel occupancy query failed");
    a.sched = sched;
    a.no_gram = no_gram ? 1 : 0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ctx->timing) {
      while (ctx->ev_pool.size() < ctx->ev_used + 2) {
        cudaEvent_t e;
        CUDA_TRY(ctx, cudaEventCreate(&e));
        ctx->ev_pool.push_back(e);
      }
      e0 = ctx->ev_pool[ctx->ev_used];
      e1 = ctx->ev_pool[ctx->ev_used + 1];
      ctx->ev_used += 2;
      CUDA_TRY(ctx, cudaEventRecord(e0, ctx->stream));
    }
    if (nbt) {
      NbArgs na;
      na.particles = a.particles;
      na.P = nb;
      na.pstride = pstride;
      na.sfv = a.sfv;
      na.sfv_pp = sfv_pp;
      na.bop = nbop;
      na.yscale_inv = nbscale;
      na.terms = terms;
      na.n_tiles_j = (nb * sd.S + 127) / 128;
      na.n_tiles = na.n_tiles_j * sd.J;
      na.diag_only = no_gram ? 1 : 0;
      CUDA_TRY(ctx, launch_nb_gram(sd, na, pflag, ctx->stream));
      CUDA_TRY(ctx, launch_nb_corr(sd, nbp, na, ctx->num_sms, ctx->stream));
      ctx->launches += 1;
    } else if (tay) {
      // c and G_ss from K1T; the off-diagonal Gram from tay_gram_kernel (thread per particle, all pairs), or with
      // CDMS_TAYLOR_GRAM=k1 from K1's Horner-free variant, which writes every term (c as zeros) and so runs first.
      // Measured (profiles/r01_k1t_gram_select.txt): since its pair loops unroll fully tay_gram wins at every S
      // (c3, S = 7: 8.97 vs 12.45 ms per step; c5 shard, S = 9: 60.0 vs 73.6; c2: 0.40 vs 0.48)
      const bool k1g = !no_gram && ctx->taylor_gram == 1;
      if (k1g) CUDA_TRY(ctx, launch_corr_gram_only(sd, a, ctx->stream));
      CUDA_TRY(ctx, launch_tay_corr(sd, taytab, tmpl, a.particles, nb, pstride, a.sfv, sfv_pp, terms, pflag,
                                    no_gram ? 1 : 0, tlanes, ctx->stream));
      if (!no_gram && !k1g)
        CUDA_TRY(ctx, launch_tay_gram(sd, tmpl, a.particles, nb, pstride, a.sfv, sfv_pp, terms, ctx->stream));
      ctx->launches += no_gram ? 0 : 1;
    } else {
      CUDA_TRY(ctx, launch_corr(sd, a, precision, ctx->stream));
    }
    if (ctx->timing) CUDA_TRY(ctx, cudaEventRecord(e1, ctx->stream));
    AsmArgs s;
    s.terms = terms;
    s.pflag = pflag;
    s.ynorm2 = yn;
    s.logw_prior = d_logw ? d_logw + b0 : nullptr;
    s.loglik = d_loglik + b0;
    s.amp = d_amp ? static_cast<double2*>(d_amp) + b0 * sd.J * sd.S : nullptr;
    s.term_c = d_c ? static_cast<double2*>(d_c) + b0 * sd.J * sd.S : nullptr;
    s.term_G = d_G ? static_cast<double2*>(d_G) + b0 * sd.J * sd.S * sd.S : nullptr;
    s.flags = ctx->d_flags;
    s.P = nb;
    CUDA_TRY(ctx, launch_assemble(sd, s, ctx->stream));
    ctx->launches += 2;
  }
  return CDMS_OK;
}

}  // namespace

// ============================================================================ ABI
extern "C" {

cdms_status cdms_create(cdms_ctx* out, int device, void* cuda_stream) {
  if (!out) return CDMS_EINVAL;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return CDMS_ECUDA;
  cdms_ctx ctx = new cdms_ctx_s();
  ctx->device = device;
  ctx->stream = static_cast<cudaStream_t>(cuda_stream);
  ctx->bufs.assign(WS_COUNT, nullptr);
  ctx->sizes.assign(WS_COUNT, 0);
  DeviceGuard g(device);
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (const char* e = getenv("CDMS_NB_TENSOR")) ctx->nb_tensor = atoi(e) != 0;
  if (const char* e = getenv("CDMS_TAYLOR")) ctx->taylor = atoi(e) != 0;
  if (const char* e = getenv("CDMS_STEP_FUSED")) ctx->step_fused = atoi(e) ? 1 : 0;
  if (const char* e = getenv("CDMS_TAY_PREP")) ctx->taylor_prep_direct = strcmp(e, "direct") == 0 ? 1 : 0;
  if (const char* e = getenv("CDMS_TAY_LANES")) ctx->taylor_lanes = atoi(e) ? 1 : 0;
  if (const char* e = getenv("CDMS_TAYLOR_GRAM")) ctx->taylor_gram = strcmp(e, "k1") == 0 ? 1 : (strcmp(e, "tay") == 0 ? 2 : 0);
  if (cudaMalloc(&ctx->d_flags, sizeof(int)) != cudaSuccess || cudaMemset(ctx->d_flags, 0, sizeof(int)) != cudaSuccess ||
      cudaMallocHost(&ctx->h_pinned, 4096) != cudaSuccess) {
    delete ctx;
    return CDMS_ECUDA;
  }
  *out = ctx;
  return CDMS_OK;
}

cdms_status cdms_destroy(cdms_ctx ctx) {
  if (!ctx) return CDMS_EINVAL;
  DeviceGuard g(ctx->device);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  for (void* b : ctx->bufs)
    if (b) cudaFree(b);
  for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->d_flags) cudaFree(ctx->d_flags);
  if (ctx->h_pinned) cudaFreeHost(ctx->h_pinned);
  delete ctx;
  return CDMS_OK;
}

cdms_status cdms_set_stream(cdms_ctx ctx, void* cuda_stream) {
  if (!ctx) return CDMS_EINVAL;
  ctx->stream = static_cast<cudaStream_t>(cuda_stream);
  return CDMS_OK;
}

const char* cdms_last_error(cdms_ctx ctx) { return ctx ? ctx->err.c_str() : "NULL context"; }

int64_t cdms_launch_count(cdms_ctx ctx) { return ctx ? ctx->launches : -1; }

cdms_status cdms_timing_enable(cdms_ctx ctx, int on) {
  if (!ctx) return CDMS_EINVAL;
  ctx->timing = on != 0;
  ctx->ev_used = 0;
  return CDMS_OK;
}

cdms_status cdms_timing_read(cdms_ctx ctx, double* loglik_ms, int64_t* n_launches) {
  if (!ctx || !loglik_ms || !n_launches) return CDMS_EINVAL;
  DeviceGuard g(ctx->device);
  double tot = 0.0;
  for (size_t i = 0; i + 1 < ctx->ev_used; i += 2) {
    CUDA_TRY(ctx, cudaEventSynchronize(ctx->ev_pool[i + 1]));
    float ms = 0.f;
    CUDA_TRY(ctx, cudaEventElapsedTime(&ms, ctx->ev_pool[i], ctx->ev_pool[i + 1]));
    tot += ms;
  }
  *loglik_ms = tot;
  *n_launches = (int64_t)(ctx->ev_used / 2);
  return CDMS_OK;
}

cdms_status cdms_sync(cdms_ctx ctx) {
  if (!ctx) return CDMS_EINVAL;
  DeviceGuard g(ctx->device);
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  int flags = 0;
  CUDA_TRY(ctx, cudaMemcpy(&flags, ctx->d_flags, sizeof(int), cudaMemcpyDeviceToHost));
  CUDA_TRY(ctx, cudaMemset(ctx->d_flags, 0, sizeof(int)));
  if (flags & FLAG_NAN) return fail(ctx, CDMS_EINVAL, "device detected NaN / invalid input (flags=%d)", flags);
  if (flags & FLAG_ZEROMASS) return fail(ctx, CDMS_EZEROMASS, "all weights zero (flags=%d)", flags);
  if (flags & FLAG_DEGENERATE) return fail(ctx, CDMS_EDEGENERATE, "degenerate ray: MT on a phase centre or antenna");
  return CDMS_OK;
}

cdms_status cdms_reserve(cdms_ctx ctx, const cdms_scene* scene, int64_t P_local) {
  if (!ctx || P_local <= 0) return fail(ctx, CDMS_EINVAL, "reserve: bad arguments");
  DeviceGuard g(ctx->device);
  SceneDev sd;
  cdms_status st = build_scene(ctx, scene, nullptr, nullptr, nullptr, &sd);
  if (st) return st;
  // partial buffers sized for the finer of the two partitions (beliefs.cu RED_ITEMS, step.cu STEP_ITEMS)
  const int64_t nb = red_blocks(P_local) > step_blocks(P_local) ? red_blocks(P_local) : step_blocks(P_local);
  float4* f4;
  double* d;
  double2* d2;
  uint64_t* u;
  int64_t* i64;
  int* i32;
  WS_TRY(ctx, WS_YTILES, (int64_t)sd.J * sd.n_mb * sd.n_kc * sd.kc_len * NWARP, &f4);
  {
    const int T = terms_width(sd.S);
    const size_t per_particle = (size_t)sd.J * T * sizeof(double2);
    int64_t PB = (int64_t)(TERMS_BUDGET / per_particle);
    PB = PB < TILE_P ? TILE_P : (PB / TILE_P) * TILE_P;
    if (PB > P_local) PB = P_local;
    WS_TRY(ctx, WS_TERMS, (size_t)PB * sd.J * T, &d2);
    WS_TRY(ctx, WS_PFLAG, PB, &i32);
    unsigned int* sch;
    WS_TRY(ctx, WS_SCHED, 2, &sch);
    WS_TRY(ctx, WS_STEP_CNT, 4, &sch);
    WS_TRY(ctx, WS_TMPL, (int64_t)sd.J * sd.n_mb * NWARP, &f4);
    NbPlan nbp{};  // the tensor-core path's per-PA B operand and scales (PLANAR_NB, FP32)
    if (ctx->nb_tensor && scene->precision == CDMS_FP32 && nb_tensor_plan(sd, &nbp)) {
      uint8_t* nbop;
      float* nbs;
      WS_TRY(ctx, WS_NBOP, nb_operand_bytes(sd, nbp), &nbop);
      WS_TRY(ctx, WS_NBSCALE, MAXJ, &nbs);
    }
  }
  WS_TRY(ctx, WS_YNORM, MAXJ, &d);
  WS_TRY(ctx, WS_LSE_PART, nb + 1, &d2);
  WS_TRY(ctx, WS_LSE_RANK, ctx->nranks + 1, &d2);
  WS_TRY(ctx, WS_SCAL, 8, &d);
  WS_TRY(ctx, WS_MOM_PART, (nb + 1) * 21, &d);
  WS_TRY(ctx, WS_SUMS, 32, &d);
  WS_TRY(ctx, WS_WMAX_PART, nb + 1, &d);
  WS_TRY(ctx, WS_Q, P_local, &u);
  WS_TRY(ctx, WS_BSUM, nb + 2, &u);
  WS_TRY(ctx, WS_QALL, 2 * ctx->nranks + 4, &u);
  WS_TRY(ctx, WS_LOGLIK, P_local, &d);
  WS_TRY(ctx, WS_W, P_local, &d);
  WS_TRY(ctx, WS_ANC, P_local, &i64);
  WS_TRY(ctx, WS_STAGE, P_local * 6, &d);
  WS_TRY(ctx, WS_L6, 36, &d);
  return CDMS_OK;
}

cdms_status cdms_get_unique_id(unsigned char id_out[128]) {
  if (!id_out) return CDMS_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return CDMS_ENCCL;
  memcpy(id_out, id.internal, 128);
  return CDMS_OK;
}

cdms_status cdms_comm_init(cdms_ctx ctx, const unsigned char id_in[128], int rank, int nranks) {
  if (!ctx || !id_in || nranks < 1 || rank < 0 || rank >= nranks) return fail(ctx, CDMS_EINVAL, "comm_init: bad args");
  DeviceGuard g(ctx->device);
  ncclUniqueId id;
  memcpy(id.internal, id_in, 128);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  ctx->comm = nullptr;
  NCCL_TRY(ctx, ncclCommInitRank(&ctx->comm, nranks, id, rank));
  ctx->rank = rank;
  ctx->nranks = nranks;
  return CDMS_OK;
}

cdms_status cdms_layout(cdms_ctx ctx, const cdms_scene* scene, const double* d_sfv, double* d_layout, double* d_va,
                        double* d_H) {
  if (!ctx) return CDMS_EINVAL;
  DeviceGuard g(ctx->device);
  SceneDev sd;
  cdms_status st = build_scene(ctx, scene, nullptr, nullptr, nullptr, &sd);
  if (st) return st;
  if ((sd.K > 0 && !d_sfv) || !d_layout || !d_va || !d_H) return fail(ctx, CDMS_EINVAL, "layout: NULL pointer");
  CUDA_TRY(ctx, launch_layout(sd, d_sfv, d_layout, d_va, d_H, ctx->d_flags, ctx->stream));
  ctx->launches += 1;
  return CDMS_OK;
}

cdms_status cdms_loglik(cdms_ctx ctx, const cdms_scene* scene, const double* d_particles, int64_t P, int32_t pstride,
                        const double* d_sfv, int32_t sfv_per_particle, const void* d_y, const double* h_f_pb,
                        const cdms_prior* h_prior, const double* h_eta, const double* d_logw_prior, double* d_loglik,
                        void* d_amp) {
  if (!ctx) return CDMS_EINVAL;
  DeviceGuard g(ctx->device);
  if (!d_particles || !d_y || !h_f_pb || !h_prior || !h_eta || !d_loglik) return fail(ctx, CDMS_EINVAL, "loglik: NULL pointer");
  if (P <= 0 || pstride < 3) return fail(ctx, CDMS_EINVAL, "loglik: P=%lld pstride=%d", (long long)P, pstride);
  SceneDev sd;
  cdms_status st = build_scene(ctx, scene, h_f_pb, h_prior, h_eta, &sd);
  if (st) return st;
  if (sd.K > 0 && !d_sfv) return fail(ctx, CDMS_EINVAL, "loglik: d_sfv NULL with K > 0");
  return loglik_impl(ctx, sd, scene->precision, d_particles, P, pstride, d_sfv, sfv_per_particle ? 1 : 0, d_y,
                     d_logw_prior, d_loglik, d_amp);
}

cdms_status cdms_loglik_terms(cdms_ctx ctx, const cdms_scene* scene, const double* d_particles, int64_t P,
                              int32_t pstride, const double* d_sfv, int32_t sfv_per_particle, const void* d_y,
                              const double* h_f_pb, const cdms_prior* h_prior, const double* h_eta, double* d_loglik,
                              void* d_c, void* d_G) {
  if (!ctx) return CDMS_EINVAL;
  DeviceGuard g(ctx->device);
  if (!d_particles || !d_y || !h_f_pb || !h_prior || !h_eta || !d_loglik || !d_c || !d_G)
    return fail(ctx, CDMS_EINVAL, "loglik_terms: NULL pointer");
  if (P <= 0 || pstride < 3) return fail(ctx, CDMS_EINVAL, "loglik_terms: P=%lld pstride=%d", (long long)P, pstride);
  SceneDev sd;
  cdms_status st = build_scene(ctx, scene, h_f_pb, h_prior, h_eta, &sd);
  if (st) return st;
  if (sd.K > 0 && !d_sfv) return fail(ctx, CDMS_EINVAL, "loglik_terms: d_sfv NULL with K > 0");
  return loglik_impl(ctx, sd, scene->precision, d_particles, P, pstride, d_sfv, sfv_per_particle ? 1 : 0, d_y,
                     nullptr, d_loglik, nullptr, d_c, d_G);
}

cdms_status cdms_birth_proposal(cdms_ctx ctx, const cdms_scene* scene, const double* h_f_pb, const double* h_x_hat,
                                const double* h_sfv_legacy, int32_t L, const void* d_y, const double* h_box,
                                int64_t N_g, uint64_t key, uint64_t counter, double* d_out, double* d_pb,
                                double* d_cand) {
  if (!ctx) return CDMS_EINVAL;
  DeviceGuard g(ctx->device);
  if (!scene || !h_f_pb || !h_x_hat || !d_y || !h_box || !d_out || N_g <= 0 || L < 0 || L > MAXS - 1 ||
      (L > 0 && !h_sfv_legacy))
    return fail(ctx, CDMS_EINVAL, "birth_proposal: bad arguments (L=%d, N_g=%lld)", L, (long long)N_g);
  BirthBox box{};
  for (int a = 0; a < 3; ++a) {
    box.lo[a] = h_box[a];
    box.hi[a] = h_box[3 + a];
    box.x_hat[a] = h_x_hat[a];
    if (!is_fin(box.lo[a]) || !is_fin(box.hi[a]) || box.hi[a] < box.lo[a] || !is_fin(box.x_hat[a]))
      return fail(ctx, CDMS_EINVAL, "birth_proposal: box / x_hat invalid");
  }
  for (int l = 0; l < L; ++l)
    for (int a = 0; a < 3; ++a) {
      box.sfv[l][a] = h_sfv_legacy[3 * l + a];
      if (!is_fin(box.sfv[l][a])) return fail(ctx, CDMS_EINVAL, "birth_proposal: legacy SFV not finite");
    }
  box.L = L;
  static const bool dbg_sync = getenv("CDMS_BIRTH_DEBUG") != nullptr;  // debug aid: sync + check per stage
  auto stage = [&](const char* what) -> cdms_status {
    if (!dbg_sync) return CDMS_OK;
    const cudaError_t e = cudaStreamSynchronize(ctx->stream);
    return e == cudaSuccess ? CDMS_OK : fail(ctx, CDMS_ECUDA, "birth_proposal stage %s: %s", what, cudaGetErrorString(e));
  };
  // (1) residual z~ = Pi_perp z against LOS + legacy components at x_hat (fp64 responses, scene with K = L)
  cdms_scene s1 = *scene;
  s1.K = L;
  SceneDev sd1;
  cdms_status st = build_scene(ctx, &s1, h_f_pb, nullptr, nullptr, &sd1);
  if (st) return st;
  const int J = sd1.J, n = L + 1;
  const int nz = sd1.nf * sd1.Na;
  double *pos, *sfvb, *cand, *ll, *pb, *part6, *scr;
  int32_t* js;
  double2 *psi, *dots, *coef, *cbuf;
  float2* zr;
  double4* part;
  WS_TRY(ctx, WS_BPOS, (size_t)3 * J * n, &pos);
  WS_TRY(ctx, WS_BJS, (size_t)2 * J * n, &js);
  WS_TRY(ctx, WS_BSFV, (size_t)3 * (L > 0 ? L : 1), &sfvb);
  WS_TRY(ctx, WS_BPSI, (size_t)J * n * nz, &psi);
  WS_TRY(ctx, WS_BDOTS, (size_t)J * (n * (n + 1) / 2 + n), &dots);
  WS_TRY(ctx, WS_BCOEF, (size_t)J * n, &coef);
  WS_TRY(ctx, WS_BZR, (size_t)J * nz, &zr);
  CUDA_TRY(ctx, launch_birth_items(box, J, pos, js, sfvb, ctx->stream));
  if ((st = stage("items"))) return st;
  CUDA_TRY(ctx, launch_response(sd1, pos, (int64_t)J * n, js, sfvb, psi, CDMS_FP64, ctx->d_flags, ctx->stream));
  if ((st = stage("response"))) return st;
  CUDA_TRY(ctx, launch_birth_residual(J, nz, n, psi, static_cast<const float2*>(d_y), dots, coef, zr, ctx->d_flags,
                                      ctx->stream));
  ctx->launches += 5;
  if ((st = stage("residual"))) return st;
  // (2) candidates p_i, padded to whole pseudo-particles (copies of the last candidate)
  const int64_t npp = birth_pseudo_particles(N_g);
  const int pack = MAXS - 1;
  WS_TRY(ctx, WS_BCAND, (size_t)3 * npp * pack, &cand);
  CUDA_TRY(ctx, launch_birth_candidates(N_g, key, counter, box, cand, ctx->stream));
  ctx->launches += 1;
  if (d_cand)
    CUDA_TRY(ctx, cudaMemcpyAsync(d_cand, cand, sizeof(double) * 3 * N_g, cudaMemcpyDeviceToDevice, ctx->stream));
  if ((st = stage("candidates"))) return st;
  // (3) c = psi(x_hat, p_i)^H z~_j on the likelihood engine: pseudo-particles at x_hat (pstride 0: pos[0..2] is
  //     x_hat) with the candidates as their K = 8 per-particle walls, neutral prior (the assembled likelihood is not
  //     used), snapshot z~
  cdms_scene s0 = *scene;
  s0.K = pack;
  cdms_prior pr[MAXJ * MAXS];
  double eta1[MAXJ];
  for (int q = 0; q < J * MAXS; ++q) {
    pr[q].m_re = 0.0;
    pr[q].m_im = 0.0;
    pr[q].v = 1.0;
  }
  for (int j = 0; j < J; ++j) eta1[j] = 1.0;
  SceneDev sd0;
  st = build_scene(ctx, &s0, h_f_pb, pr, eta1, &sd0);
  if (st) return st;
  WS_TRY(ctx, WS_BC, (size_t)npp * J * MAXS, &cbuf);
  WS_TRY(ctx, WS_BLL, (size_t)npp, &ll);
  st = loglik_impl(ctx, sd0, scene->precision, pos, npp, 0, cand, 1, zr, nullptr, ll, nullptr, cbuf, nullptr,
                   /*no_gram=*/true);
  if (st) return st;
  if ((st = stage("correlation"))) return st;
  // (4) Bartlett spectrum, mode and weighted second moment
  if (d_pb) pb = d_pb;
  else WS_TRY(ctx, WS_BPB, (size_t)N_g, &pb);
  const int64_t nblk = birth_blocks(N_g);
  WS_TRY(ctx, WS_BPART, (size_t)nblk, &part);
  WS_TRY(ctx, WS_BPART6, (size_t)6 * nblk, &part6);
  WS_TRY(ctx, WS_BSCR, 8, &scr);
  CUDA_TRY(ctx, launch_birth_reduce(N_g, J, nz, cbuf, cand, pb, part, part6, scr, d_out, ctx->d_flags, ctx->stream));
  ctx->launches += 4;
  return stage("reduce");
}

cdms_status cdms_weights_normalize(cdms_ctx ctx, const double* d_logw, int64_t P_local, double* d_w, double* d_lse) {
  if (!ctx) return CDMS_EINVAL;
  DeviceGuard g(ctx->device);
  if (!d_logw || !d_w || !d_lse || P_local <= 0) return fail(ctx, CDMS_EINVAL, "normalize: bad arguments");
  cdms_status st = run_lse(ctx, d_logw, P_local, d_lse);
  if (st) return st;
  double* scal;
  WS_TRY(ctx, WS_SCAL, 8, &scal);
  CUDA_TRY(ctx, launch_normalize(d_logw, P_local, scal + 0, scal + 1, ctx->d_flags, d_w, ctx->stream));
  ctx->launches += 1;
  return CDMS_OK;
}

cdms_status cdms_moments(cdms_ctx ctx, const double* d_particles, const double* d_w, int64_t P_local, double* d_est) {
  if (!ctx) return CDMS_EINVAL;
  DeviceGuard g(ctx->device);
  if (!d_particles || !d_w || !d_est || P_local <= 0) return fail(ctx, CDMS_EINVAL, "moments: bad arguments");
  return run_moments(ctx, d_particles, d_w, P_local, d_est);
}

cdms_status cdms_resample(cdms_ctx ctx, const double* d_w, int64_t P_local, uint32_t u_bits, int64_t* d_ancestors) {
  if (!ctx) return CDMS_EINVAL;
  DeviceGuard g(ctx->device);
  if (!d_w || !d_ancestors || P_local <= 0) return fail(ctx, CDMS_EINVAL, "resample: bad arguments");
  Plan plan;
  int64_t* anc;
  cdms_status st = run_resample_core(ctx, d_w, P_local, u_bits, 0, &plan, &anc);
  if (st) return st;
  if (!(ctx->comm)) {
    CUDA_TRY(ctx, cudaMemcpyAsync(d_ancestors, anc, sizeof(int64_t) * P_local, cudaMemcpyDeviceToDevice, ctx->stream));
    return CDMS_OK;
  }
  return exchange(ctx, plan, P_local, anc, d_ancestors, 1);
}

cdms_status cdms_bp_step(cdms_ctx ctx, const cdms_scene* scene, double* d_particles, int64_t P_local, const double* d_sfv,
                         const void* d_y, const double* h_f_pb, const cdms_prior* h_prior, const double* h_eta,
                         const cdms_step_params* prm, double* d_est, double* d_lse) {
  if (!ctx) return CDMS_EINVAL;
  DeviceGuard g(ctx->device);
  if (!d_particles || !d_y || !h_f_pb || !h_prior || !h_eta || !prm || !d_est || !d_lse || P_local <= 0)
    return fail(ctx, CDMS_EINVAL, "bp_step: bad arguments");
  if (!is_fin(prm->T) || !is_fin(prm->sigma_v) || prm->sigma_v < 0.0) return fail(ctx, CDMS_EINVAL, "bp_step: T/sigma_v");
  SceneDev sd;
  cdms_status st = build_scene(ctx, scene, h_f_pb, h_prior, h_eta, &sd);
  if (st) return st;
  if (sd.K > 0 && !d_sfv) return fail(ctx, CDMS_EINVAL, "bp_step: d_sfv NULL with K > 0");
  const int64_t p0 = (int64_t)ctx->rank * P_local;
  const int64_t P_total = P_local * ctx->nranks;
  double *l, *w, *stage, *L6, *scal;
  WS_TRY(ctx, WS_LOGLIK, P_local, &l);
  WS_TRY(ctx, WS_W, P_local, &w);
  WS_TRY(ctx, WS_L6, 36, &L6);
  WS_TRY(ctx, WS_SCAL, 8, &scal);
  // (1) prediction (row A9)
  CUDA_TRY(ctx, launch_predict(d_particles, P_local, p0, prm->T, prm->sigma_v, prm->philox_key, prm->step, ctx->stream));
  ctx->launches += 1;
  // (2) coherent log-likelihood, uniform w_beta (rows A1-A5)
  st = loglik_impl(ctx, sd, scene->precision, d_particles, P_local, 6, d_sfv, 0, d_y, nullptr, l, nullptr);
  if (st) return st;
  // (3)-(6) the fused O(P) pipeline (step.cu): LSE (A6), weights + quantized masses + moments (A7),
  // scan + ancestors + gather (A8), regularization (A9).  With a communicator the collectives sit between the
  // kernels; the combine / finalize arithmetic is the same device code either way.
  const bool comm = ctx->comm != nullptr;
  const int R = ctx->nranks;
  if (P_total > ((int64_t)1 << 26)) return fail(ctx, CDMS_EINVAL, "P_total=%lld exceeds 2^26", (long long)P_total);
  const int64_t nb = step_blocks(P_local);
  double2 *lpart, *pairs;
  double *mpart, *sums;
  uint64_t *q, *bsum, *qall;
  unsigned* cnt;
  WS_TRY(ctx, WS_LSE_PART, nb + 1, &lpart);
  WS_TRY(ctx, WS_LSE_RANK, R + 1, &pairs);
  WS_TRY(ctx, WS_MOM_PART, (nb + 1) * 21, &mpart);
  WS_TRY(ctx, WS_SUMS, 32, &sums);
  WS_TRY(ctx, WS_Q, P_local, &q);
  WS_TRY(ctx, WS_BSUM, nb + 2, &bsum);
  WS_TRY(ctx, WS_QALL, 2 * R + 4, &qall);
  WS_TRY(ctx, WS_STEP_CNT, 4, &cnt);  // zeroed at allocation, reset by each kernel's last block
  if (!comm && ctx->step_fused) {
    // one rank: the five kernels' bodies in one cooperative launch (grid barriers instead of launches and
    // last-block tails), identical arithmetic and block partition, so identical results
    WS_TRY(ctx, WS_STAGE, P_local * 6, &stage);
    StepFusedArgs fa;
    fa.l = l;
    fa.x = d_particles;
    fa.P = P_local;
    fa.lpart = lpart;
    fa.rank_pair = pairs;
    fa.lse = d_lse;
    fa.M = scal + 0;
    fa.logS = scal + 1;
    fa.flags = ctx->d_flags;
    fa.w = w;
    fa.q = q;
    fa.mpart = mpart;
    fa.bsum = bsum;
    fa.sums = sums;
    fa.est = d_est;
    fa.L = L6;
    fa.stage = stage;
    fa.u_bits = host_step_u_bits(prm->philox_key, prm->step);
    fa.h = step_reg_bandwidth(P_total);
    fa.regularize = prm->regularize ? 1 : 0;
    fa.key = prm->philox_key;
    fa.step = prm->step;
    CUDA_TRY(ctx, launch_step_fused(fa, ctx->num_sms, ctx->stream));
    ctx->launches += 1;
    return CDMS_OK;
  }
  CUDA_TRY(ctx, launch_step_lse(l, P_local, lpart, cnt + 0, comm ? pairs + R : pairs, comm ? 0 : 1, d_lse, scal + 0,
                                scal + 1, ctx->d_flags, ctx->stream));
  ctx->launches += 1;
  if (comm) {
    NCCL_TRY(ctx, ncclAllGather(pairs + R, pairs, 2, ncclDouble, ctx->comm, ctx->stream));
    CUDA_TRY(ctx, launch_step_lse_combine(pairs, R, d_lse, scal + 0, scal + 1, ctx->d_flags, ctx->stream));
    ctx->launches += 1;
  }
  CUDA_TRY(ctx, launch_step_post(l, d_particles, P_local, scal + 0, scal + 1, ctx->d_flags, w, q, mpart, bsum, cnt + 1,
                                 sums, ctx->stream));
  ctx->launches += 1;
  if (comm) NCCL_TRY(ctx, ncclAllReduce(sums, sums, 7, ncclDouble, ncclSum, ctx->comm, ctx->stream));
  CUDA_TRY(ctx, launch_step_scan(q, d_particles, w, P_local, bsum, sums, ctx->d_flags, mpart, cnt + 2, sums + 8,
                                 comm ? 0 : 1, d_est, L6, ctx->d_flags, ctx->stream));
  ctx->launches += 1;
  if (comm) {
    NCCL_TRY(ctx, ncclAllReduce(sums + 8, sums + 8, 21, ncclDouble, ncclSum, ctx->comm, ctx->stream));
    CUDA_TRY(ctx, launch_step_finalize(sums, sums + 8, d_est, L6, ctx->d_flags, ctx->stream));
    ctx->launches += 1;
  }
  // systematic resampling on r_p = e^{l_p - M} (C-amb-23): slots of this rank's CDF range, states gathered
  const uint32_t u_bits = host_step_u_bits(prm->philox_key, prm->step);
  Plan plan;
  const uint64_t* Qtot = bsum + nb;
  const uint64_t* Ooff = nullptr;
  if (!comm) {
    plan.lo = 0;
    plan.hi = P_local;
  } else {
    // all-gather Q_r, host plan (one small D2H + stream sync per step)
    NCCL_TRY(ctx, ncclAllGather(bsum + nb, qall, 1, ncclUint64, ctx->comm, ctx->stream));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_pinned, qall, sizeof(uint64_t) * R, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    std::vector<uint64_t> Q(ctx->h_pinned, ctx->h_pinned + R);
    uint64_t Qt = 0;
    for (uint64_t v : Q) Qt += v;
    if (Qt == 0) return fail(ctx, CDMS_EZEROMASS, "all resampling weights are zero");
    plan.lo_all.resize(R);
    plan.hi_all.resize(R);
    uint64_t O = 0, Omine = 0;
    for (int r = 0; r < R; ++r) {
      plan.lo_all[r] = slot_index(O, Qt, P_total, u_bits);
      plan.hi_all[r] = slot_index(O + Q[r], Qt, P_total, u_bits);
      if (r == ctx->rank) Omine = O;
      O += Q[r];
    }
    plan.lo = plan.lo_all[ctx->rank];
    plan.hi = plan.hi_all[ctx->rank];
    ctx->h_pinned[R] = Qt;
    ctx->h_pinned[R + 1] = Omine;
    CUDA_TRY(ctx, cudaMemcpyAsync(qall + R, ctx->h_pinned + R, 2 * sizeof(uint64_t), cudaMemcpyHostToDevice,
                                  ctx->stream));
    Qtot = qall + R;
    Ooff = qall + R + 1;
  }
  const int64_t n = plan.hi - plan.lo;
  WS_TRY(ctx, WS_STAGE, (n > 0 ? n : 1) * 6, &stage);
  CUDA_TRY(ctx, launch_step_anc(q, bsum, P_local, Qtot, Ooff, plan.lo, plan.hi, P_total, u_bits, d_particles, stage,
                                ctx->d_flags, ctx->stream));
  ctx->launches += 1;
  if (comm) {
    st = exchange(ctx, plan, P_local, stage, d_particles, 6);
    if (st) return st;
    if (prm->regularize) {
      CUDA_TRY(ctx, launch_step_reg(d_particles, d_particles, P_local, p0, P_total, L6, 1, prm->philox_key, prm->step,
                                    ctx->stream));
      ctx->launches += 1;
    }
  } else {
    // regularization with the pre-resampling covariance (A9), reading the staged states (no extra copy)
    CUDA_TRY(ctx, launch_step_reg(stage, d_particles, P_local, p0, P_total, L6, prm->regularize ? 1 : 0,
                                  prm->philox_key, prm->step, ctx->stream));
    ctx->launches += 1;
  }
  return CDMS_OK;
}

cdms_status cdms_response(cdms_ctx ctx, const cdms_scene* scene, const double* d_pos, int64_t n, const int32_t* d_js,
                          const double* d_sfv, void* d_psi) {
  if (!ctx) return CDMS_EINVAL;
  DeviceGuard g(ctx->device);
  if (!d_pos || !d_js || !d_psi || n <= 0) return fail(ctx, CDMS_EINVAL, "response: bad arguments");
  SceneDev sd;
  cdms_status st = build_scene(ctx, scene, nullptr, nullptr, nullptr, &sd);
  if (st) return st;
  if (sd.K > 0 && !d_sfv) return fail(ctx, CDMS_EINVAL, "response: d_sfv NULL with K > 0");
  CUDA_TRY(ctx, launch_response(sd, d_pos, n, d_js, d_sfv, static_cast<double2*>(d_psi), scene->precision, ctx->d_flags,
                                ctx->stream));
  ctx->launches += 1;
  return CDMS_OK;
}

cdms_status cdms_moment_match(double mu_re, double mu_im, double gamma, double exist, cdms_prior* out) {
  if (!out || !is_fin(mu_re) || !is_fin(mu_im) || !is_fin(gamma) || gamma < 0.0 || !(exist >= 0.0 && exist <= 1.0))
    return CDMS_EINVAL;
  out->m_re = exist * mu_re;
  out->m_im = exist * mu_im;
  out->v = exist * (gamma + (mu_re * mu_re + mu_im * mu_im) * (1.0 - exist));
  return CDMS_OK;
}

cdms_status cdms_resample_plan(const uint64_t* h_Q, int nranks, int rank, int64_t P_local, uint32_t u_bits,
                               int64_t* slot_lo, int64_t* slot_hi, int64_t* h_send_counts) {
  if (!h_Q || nranks < 1 || rank < 0 || rank >= nranks || P_local <= 0 || !slot_lo || !slot_hi) return CDMS_EINVAL;
  const int64_t P_total = P_local * nranks;
  if (P_total > ((int64_t)1 << 26)) return CDMS_EINVAL;
  uint64_t Qtot = 0, O = 0;
  for (int r = 0; r < nranks; ++r) {
    if (r < rank) O += h_Q[r];
    Qtot += h_Q[r];
  }
  if (Qtot == 0) return CDMS_EZEROMASS;
  const int64_t lo = slot_index(O, Qtot, P_total, u_bits);
  const int64_t hi = slot_index(O + h_Q[rank], Qtot, P_total, u_bits);
  *slot_lo = lo;
  *slot_hi = hi;
  if (h_send_counts)
    for (int d = 0; d < nranks; ++d) {
      const int64_t a = lo > d * P_local ? lo : d * P_local;
      const int64_t b = hi < (d + 1) * P_local ? hi : (d + 1) * P_local;
      h_send_counts[d] = b > a ? b - a : 0;
    }
  return CDMS_OK;
}

}  // extern "C"
