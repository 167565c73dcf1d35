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

#include <algorithm>
#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "cdms_internal.h"

using namespace cdms;

namespace {
// NVTX range around each ABI call and each phase of the step (nsys / ncu --nvtx timelines)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace

namespace {
struct Coll;
}

struct cdms_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  std::string err;
  int* d_flags = nullptr;
  ncclComm_t comm = nullptr;     // NCCL backend (owned by the NcclColl in coll)
  Coll* coll = nullptr;           // collective backend once a communicator is attached (NCCL or test loopback)
  int rank = 0, nranks = 1;
  // peer-writable redistribution buffers (multi-rank): this rank's stage [pcap][6] f64 and ancestor ids [pcap] i64,
  // and device arrays of every rank's buffers as addressable from this device (d_peer_x[r], d_peer_anc[r])
  double* pstage = nullptr;
  int64_t* panc = nullptr;
  int64_t pcap = 0;
  double** d_peer_x = nullptr;
  int64_t** d_peer_anc = nullptr;
  int* d_barrier = nullptr;
  int64_t launches = 0;
  std::vector<void*> bufs;
  std::vector<size_t> sizes;
  uint64_t* h_pinned = nullptr;  // small pinned host staging (plan exchange)
  bool timing = false;           // bracket the likelihood kernel with events
  bool nb_tensor = true;         // PLANAR_NB fp32 on the tensor cores (nbmma.cu); CDMS_NB_TENSOR=0 selects K1
  bool taylor = true;            // spherical / planar-WB fp32 correlation by K1T (taylor.cu); CDMS_TAYLOR=0 selects K1
  int step_fused = 0;           // 1: single-rank bp_step O(P) phases in one cooperative kernel (CDMS_STEP_FUSED=1,
                                 // A/B; measured not faster: c2 0.409 vs 0.403 ms, the grid barriers and block 0's
                                 // epilogues cost what the launches did)
  int taylor_prep_direct = 0;   // K1T tables by the direct sum even when G is a power of two (CDMS_TAY_PREP=direct,
                                 // A/B only; default FFT)
  int gram_tab = 1;              // K1T Gram's D_N from the Taylor table (taylor.cu GramTab) at every S; CDMS_GRAM_TAB=0/2
  int dn_nf = -1;                // N_f the table in WS_DN was built for
  void* dn_ptr = nullptr;
  int locality = 0;              // 1: K1T batches in Morton processing order (sort.cu; CDMS_LOCALITY=1, A/B only).
                                 // Measured (4M c5 particles, final kernels): Gram 44.9 vs 45.0 ms, correlation 25.9
                                 // vs 25.6 sorted / unsorted, c2 step 0.477 vs 0.409 ms: at warm-cache rates the
                                 // correlation is issue-bound (81%) and the Gram latency-bound at its occupancy, so
                                 // the halved L1 wavefronts (cold-cache ncu) buy nothing
                                 // (profiles/r02_warm_k1t_c5_summary.txt)
  int taylor_lanes = -1;         // K1T correlation kernel: -1 by P J (tay_lanes), 1 lane groups, 0 thread per
                                 // particle (CDMS_TAY_LANES=1 / 0, A/B only)
  std::vector<cudaEvent_t> ev_pool;  // timing: 4 events per likelihood batch (before / between the correlation and
  size_t ev_used = 0;                // Gram kernels / before / after the assembly)
  std::vector<uint8_t> ev_gram_first;  // per batch: 1 when the Gram kernel runs first (tensor-core path)
};

namespace {

enum Slot {
  WS_YTILES, WS_YNORM, WS_LSE_PART, WS_LSE_RANK, WS_SCAL, WS_MOM_PART, WS_SUMS, WS_WMAX_PART, WS_Q, WS_BSUM,
  WS_QALL, WS_LOGLIK, WS_W, WS_ANC, WS_STAGE, WS_L6, WS_ANC2, WS_TERMS, WS_PFLAG, WS_TMPL, WS_SCHED, WS_STEP_CNT, WS_NBOP, WS_NBSCALE,
  WS_BPOS, WS_BJS, WS_BSFV, WS_BPSI, WS_BDOTS, WS_BCOEF, WS_BZR, WS_BCAND, WS_BC, WS_BLL, WS_BPB,
  WS_BPART, WS_BPART6, WS_BSCR, WS_TAY, WS_GPART, WS_PLAN, WS_RANKS, WS_PF_SNAP, WS_PF_TAB, WS_PF_DOTS, WS_PF_FIXED,
  WS_PF_CC, WS_PF_FLAG, WS_PF_GAIN, WS_PF_PAR, WS_LSE2, WS_SL_STACK, WS_SL_DOTS, WS_SL_EIG, WS_SL_PAR, WS_LOC_KEYS, WS_LOC_IDX,
  WS_LOC_TEMP, WS_LOC_POS, WS_LOC_SFV, WS_DN, WS_COUNT
};
// bytes of per-(particle, PA) sufficient statistics per likelihood batch: 32 GiB of the 180 GB holds the whole c5
// step (16M particles, 27.6 GB of complex64 terms) in one batch -- fewer kernel tails than round 2's 2 GiB batches of
// 1.24M particles (measured c5 step 209.2 ms at 2 GiB, 205.8 at 8, 205.0 at 32; profiles/r02_gram_onechunk.txt)
#ifndef CDMS_TERMS_BUDGET_GB
#define CDMS_TERMS_BUDGET_GB 32
#endif
constexpr size_t TERMS_BUDGET = (size_t)CDMS_TERMS_BUDGET_GB << 30;
constexpr int64_t LOCALITY_MIN_P = 32768;         // K1T batches from this size run in Morton order (sort.cu)

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
  out->fc2pi_f = (float)(2.0 * PI * out->fc_c);
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
    out->ap_r = 1.5 * sqrt(hy * hy + hv * hv) + 1e-9;
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

// ---------------------------------------------------------------------------- collective backends
// Everything that crosses ranks goes through one of these (multi-GPU semantics):
//  allgather  every rank contributes `bytes` of device data, recv gets all ranks' contributions rank-major;
//  barrier    stream-ordered: work enqueued before it on every rank (including writes into peers' buffers) is
//             complete and visible to work enqueued after it on any rank;
//  register   make this rank's peer-writable buffers addressable from every rank (collective; fills the ctx's
//             d_peer_x / d_peer_anc arrays).
// NcclColl is the product backend (one process per GPU; NCCL all-gathers over NVLink / NVSwitch, CUDA IPC for the
// peer buffers).  LoopbackColl is the TEST backend behind cdms_loopback_*: several contexts of one process (one
// thread each, any number on one GPU) exchange through host barriers and device copies, so the multi-rank device
// path runs on a single GPU without ranks whose kernels wait on each other.
struct Coll {
  virtual ~Coll() {}
  virtual cdms_status allgather(cdms_ctx ctx, const void* send, void* recv, size_t bytes) = 0;
  virtual cdms_status barrier(cdms_ctx ctx) = 0;
  virtual cdms_status register_peers(cdms_ctx ctx) = 0;
};

cdms_status fail(cdms_ctx ctx, cdms_status st, const char* fmt, ...);

struct NcclColl : Coll {
  std::vector<void*> opened;  // IPC-mapped peer buffers to close
  cdms_status allgather(cdms_ctx ctx, const void* send, void* recv, size_t bytes) override {
    ncclResult_t r = ncclAllGather(send, recv, bytes, ncclChar, ctx->comm, ctx->stream);
    return r == ncclSuccess ? CDMS_OK : fail(ctx, CDMS_ENCCL, "ncclAllGather: %s", ncclGetErrorString(r));
  }
  cdms_status barrier(cdms_ctx ctx) override {
    // a 4-byte all-reduce: it completes on a rank only after every rank's stream reached it, i.e. after their
    // preceding kernels (whose peer stores end with __threadfence_system) completed
    ncclResult_t r = ncclAllReduce(ctx->d_barrier, ctx->d_barrier, 1, ncclInt32, ncclSum, ctx->comm, ctx->stream);
    return r == ncclSuccess ? CDMS_OK : fail(ctx, CDMS_ENCCL, "barrier ncclAllReduce: %s", ncclGetErrorString(r));
  }
  cdms_status register_peers(cdms_ctx ctx) override {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    opened.clear();
    const int R = ctx->nranks;
    cudaIpcMemHandle_t h[2];
    cudaError_t e = cudaIpcGetMemHandle(&h[0], ctx->pstage);
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h[1], ctx->panc);
    if (e != cudaSuccess) return fail(ctx, CDMS_ECUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    char *dsend = nullptr, *drecv = nullptr;
    std::vector<char> hall((size_t)R * sizeof(h));
    e = cudaMalloc(&dsend, sizeof(h) * (R + 1));
    if (e != cudaSuccess) return fail(ctx, CDMS_ENOMEM, "register_peers: %s", cudaGetErrorString(e));
    drecv = dsend + sizeof(h);
    cdms_status st = CDMS_OK;
    if (cudaMemcpyAsync(dsend, h, sizeof(h), cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess ||
        ncclAllGather(dsend, drecv, sizeof(h), ncclChar, ctx->comm, ctx->stream) != ncclSuccess ||
        cudaMemcpyAsync(hall.data(), drecv, hall.size(), cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)
      st = fail(ctx, CDMS_ENCCL, "register_peers: handle exchange failed");
    cudaFree(dsend);
    if (st) return st;
    std::vector<double*> px(R);
    std::vector<int64_t*> pa(R);
    for (int r = 0; r < R; ++r) {
      if (r == ctx->rank) {
        px[r] = ctx->pstage;
        pa[r] = ctx->panc;
        continue;
      }
      cudaIpcMemHandle_t hr[2];
      memcpy(hr, hall.data() + (size_t)r * sizeof(h), sizeof(h));
      void *a = nullptr, *b = nullptr;
      e = cudaIpcOpenMemHandle(&a, hr[0], cudaIpcMemLazyEnablePeerAccess);
      if (e == cudaSuccess) e = cudaIpcOpenMemHandle(&b, hr[1], cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) return fail(ctx, CDMS_ECUDA, "cudaIpcOpenMemHandle(rank %d): %s", r, cudaGetErrorString(e));
      opened.push_back(a);
      opened.push_back(b);
      px[r] = static_cast<double*>(a);
      pa[r] = static_cast<int64_t*>(b);
    }
    if (cudaMemcpy(ctx->d_peer_x, px.data(), sizeof(double*) * R, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(ctx->d_peer_anc, pa.data(), sizeof(int64_t*) * R, cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(ctx, CDMS_ECUDA, "register_peers: pointer upload failed");
    return barrier(ctx);
  }
  ~NcclColl() override {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
  }
};

}  // namespace
struct cdms_loopback_s {
  int nranks;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<const void*> send;
  std::vector<double*> stage;
  std::vector<int64_t*> anc;
  explicit cdms_loopback_s(int n) : nranks(n), send(n), stage(n), anc(n) {}
  void host_barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == nranks) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};
namespace {

struct LoopbackColl : Coll {
  cdms_loopback_s* g;
  explicit LoopbackColl(cdms_loopback_s* grp) : g(grp) {}
  cdms_status allgather(cdms_ctx ctx, const void* send, void* recv, size_t bytes) override {
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return fail(ctx, CDMS_ECUDA, "loopback: sync");
    g->send[ctx->rank] = send;
    g->host_barrier();
    for (int r = 0; r < g->nranks; ++r)
      if (cudaMemcpyAsync(static_cast<char*>(recv) + (size_t)r * bytes, g->send[r], bytes, cudaMemcpyDeviceToDevice,
                          ctx->stream) != cudaSuccess)
        return fail(ctx, CDMS_ECUDA, "loopback: copy");
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return fail(ctx, CDMS_ECUDA, "loopback: sync");
    g->host_barrier();  // nobody reuses its send buffer before every rank has copied it
    return CDMS_OK;
  }
  cdms_status barrier(cdms_ctx ctx) override {
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return fail(ctx, CDMS_ECUDA, "loopback: sync");
    g->host_barrier();
    return CDMS_OK;
  }
  cdms_status register_peers(cdms_ctx ctx) override {
    g->stage[ctx->rank] = ctx->pstage;
    g->anc[ctx->rank] = ctx->panc;
    g->host_barrier();
    if (cudaMemcpy(ctx->d_peer_x, g->stage.data(), sizeof(double*) * g->nranks, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(ctx->d_peer_anc, g->anc.data(), sizeof(int64_t*) * g->nranks, cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(ctx, CDMS_ECUDA, "loopback: pointer upload");
    g->host_barrier();
    return CDMS_OK;
  }
};

// This rank's peer-writable buffers for P_local particles (collective when they grow: every rank calls with the same
// P_local, so all ranks re-register together).  Not capturable when it (re)allocates: cdms_reserve first.
cdms_status ensure_peer(cdms_ctx ctx, int64_t P_local) {
  if (ctx->pcap >= P_local && ctx->d_peer_x) return CDMS_OK;
  if (ctx->pstage) cudaFree(ctx->pstage);
  if (ctx->panc) cudaFree(ctx->panc);
  ctx->pstage = nullptr;
  ctx->panc = nullptr;
  ctx->pcap = 0;
  if (!ctx->d_peer_x) {
    if (cudaMalloc(&ctx->d_peer_x, sizeof(double*) * ctx->nranks) != cudaSuccess ||
        cudaMalloc(&ctx->d_peer_anc, sizeof(int64_t*) * ctx->nranks) != cudaSuccess ||
        cudaMalloc(&ctx->d_barrier, 16) != cudaSuccess || cudaMemset(ctx->d_barrier, 0, 16) != cudaSuccess)
      return fail(ctx, CDMS_ENOMEM, "peer pointer arrays");
  }
  if (cudaMalloc(&ctx->pstage, sizeof(double) * 6 * P_local) != cudaSuccess ||
      cudaMalloc(&ctx->panc, sizeof(int64_t) * P_local) != cudaSuccess)
    return fail(ctx, CDMS_ENOMEM, "peer buffers for %lld particles", (long long)P_local);
  ctx->pcap = P_local;
  return ctx->coll->register_peers(ctx);
}

#define COLL_TRY(expr)              \
  do {                              \
    cdms_status s_ = (expr);        \
    if (s_ != CDMS_OK) return s_;   \
  } while (0)

// K1T (taylor.cu) serves FP32 spherical / planar-WB likelihoods whose tables fit the budget
bool tay_engine(cdms_ctx ctx, const SceneDev& sd, int precision, bool nb_tensor) {
  return !nb_tensor && ctx->taylor && precision == CDMS_FP32 && sd.wavefront != CDMS_PLANAR_NB &&
         std::max(tay_table_bytes(sd, 0), tay_table_bytes(sd, 1)) <= ((size_t)160 << 20);
}

cdms_status loglik_impl(cdms_ctx ctx, const SceneDev& sd, int precision, const double* d_particles, int64_t P,
                        int32_t pstride, const double* d_sfv, int32_t sfv_pp, const void* d_y, const double* d_logw,
                        double* d_loglik, void* d_amp, void* d_c = nullptr, void* d_G = nullptr,
                        bool no_gram = false) {
  NvtxRange nv_("loglik (A1-A5)");
  float4* yt;
  double* yn;
  double2* terms;
  float4* tmpl;
  unsigned int* sched;
  int* pflag;
  const int64_t tiles = (int64_t)sd.J * sd.n_mb * sd.n_kc * sd.kc_len * NWARP;
  WS_TRY(ctx, WS_YTILES, tiles, &yt);
  WS_TRY(ctx, WS_YNORM, MAXJ, &yn);
  WS_TRY(ctx, WS_TMPL, (int64_t)(sd.J + 1) * sd.n_mb * NWARP, &tmpl);
  CUDA_TRY(ctx, launch_prep_y(sd, static_cast<const float2*>(d_y), yt, yn, tmpl, ctx->stream));
  ctx->launches += 1;
  // PLANAR_NB in fp32: the correlation runs as a tensor-core GEMM (nbmma.cu) with the closed-form Gram
  NbPlan nbp{};
  const bool nbt = ctx->nb_tensor && precision == CDMS_FP32 && nb_tensor_plan(sd, &nbp);
  uint8_t* nbop = nullptr;
  float* nbscale = nullptr;
  // spherical / planar WB in FP32: c from spectral Taylor tables (K1T), G from K1's Horner-free variant
  const bool tay = tay_engine(ctx, sd, precision, nbt);
  float2* taytab = nullptr;
  const int tlanes = tay && (ctx->taylor_lanes >= 0 ? ctx->taylor_lanes == 1 : tay_lanes(sd, P)) ? 1 : 0;  // taylor.cu
  if (tay) {
    WS_TRY(ctx, WS_TAY, tay_table_bytes(sd, tlanes) / sizeof(float2), &taytab);
    CUDA_TRY(ctx, launch_tay_prep(sd, static_cast<const float2*>(d_y), taytab, tlanes, ctx->taylor_prep_direct,
                                  ctx->stream));
    ctx->launches += 1;
  }
  // the Gram's Dirichlet table (depends on N_f only: built once per context and N_f, taylor.cu dn_table_kernel).
  // Measured (Gram ms per step, profiles/r02_dn_table.txt): 16-byte rows (degree 3, even-symmetric) vs the sine
  // quotient c5 (S = 9, 4M) 49.3 vs 64.1, c3 (S = 7) 3.37 vs 4.27, c4 (S = 5) 3.43 vs 3.98, c2 0.132 vs 0.132; round 2's
  // first 32-byte rows (degree 7) had lost at S <= 6 (in-flight rows raised the registers) and were kept for S >= 7 only
  float* dn = nullptr;
  if (tay && ctx->gram_tab && sd.small_step >= 1 && (sd.S >= 7 || ctx->gram_tab == 1)) {
    WS_TRY(ctx, WS_DN, dn_table_floats(sd.nf) + 4, &dn);  // + the Gram's W != 0 flag
    if (ctx->dn_nf != sd.nf || ctx->dn_ptr != dn) {
      CUDA_TRY(ctx, launch_dn_table(sd.nf, dn, ctx->stream));
      ctx->launches += 1;
      ctx->dn_nf = sd.nf;
      ctx->dn_ptr = dn;
    }
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
  const bool f32t = tay;  // K1T hands its terms over in complex64 (term_f2), K1 and the tensor-core path in complex128
  const size_t per_particle = (size_t)sd.J * T * (f32t ? sizeof(float2) : sizeof(double2));
  int64_t PB = (int64_t)(TERMS_BUDGET / per_particle);
  PB = PB < TILE_P ? TILE_P : (PB / TILE_P) * TILE_P;
  if (PB > P) PB = P;
  WS_TRY(ctx, WS_TERMS, f32t ? ((size_t)PB * sd.J * T + 1) / 2 : (size_t)PB * sd.J * T, &terms);
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
    a.grid = tay ? 1 : corr_grid(sd, a.n_tiles, precision, ctx->num_sms);  // K1T does not launch K1
    if (a.grid < 1) return fail(ctx, CDMS_ECUDA, "corr_kernel occupancy query failed");
    a.sched = sched;
    a.no_gram = no_gram ? 1 : 0;
    const int* perm = nullptr;  // locality processing order of this batch (K1T path), or identity
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    if (ctx->timing) {
      while (ctx->ev_pool.size() < ctx->ev_used + 4) {
        cudaEvent_t e;
        CUDA_TRY(ctx, cudaEventCreate(&e));
        ctx->ev_pool.push_back(e);
      }
      for (int k = 0; k < 4; ++k) ev[k] = ctx->ev_pool[ctx->ev_used + k];
      ctx->ev_used += 4;
      ctx->ev_gram_first.push_back(nbt ? 1 : 0);
      CUDA_TRY(ctx, cudaEventRecord(ev[0], ctx->stream));
    }
    auto mark = [&](int k) -> cdms_status {
      if (ctx->timing) CUDA_TRY(ctx, cudaEventRecord(ev[k], ctx->stream));
      return CDMS_OK;
    };
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
      COLL_TRY(mark(1));
      CUDA_TRY(ctx, launch_nb_corr(sd, nbp, na, ctx->num_sms, ctx->stream));
      ctx->launches += 1;
    } else if (tay) {
      // c and G_ss from K1T; the off-diagonal Gram from tay_gram_kernel (thread per particle, all pairs).  Measured
      // against K1's Horner-free Gram (profiles/r01_k1t_gram_select.txt; that A/B option was removed in round 2 when
      // the K1T terms went to complex64): tay_gram wins at every S (c3: 8.97 vs 12.45 ms per step; c5 shard: 60.0 vs
      // 73.6; c2: 0.40 vs 0.48)
      float2* terms32 = reinterpret_cast<float2*>(terms);
      // locality order (sort.cu): the batch's positions (and per-particle SFVs) gathered in Morton order; the kernels
      // run on the sorted copy, the assembly writes each result back to its particle (bit-identical results)
      const double* bpart = a.particles;
      const double* bsfv = a.sfv;
      int bstride = pstride;
      if (ctx->locality && nb >= LOCALITY_MIN_P) {
        uint32_t* keys;
        int *idx, *permb;
        unsigned char* temp;
        double *spos, *ssfv = nullptr;
        const size_t tb = locality_sort_temp_bytes(nb);
        WS_TRY(ctx, WS_LOC_KEYS, 2 * (size_t)nb, &keys);
        WS_TRY(ctx, WS_LOC_IDX, 2 * (size_t)nb, &idx);
        WS_TRY(ctx, WS_LOC_TEMP, tb, &temp);
        WS_TRY(ctx, WS_LOC_POS, 3 * (size_t)nb, &spos);
        if (sfv_pp) WS_TRY(ctx, WS_LOC_SFV, 3 * (size_t)sd.K * nb, &ssfv);
        permb = idx + nb;
        CUDA_TRY(ctx, launch_locality_sort(a.particles, nb, pstride, a.sfv, sd.K, sfv_pp, keys, keys + nb, idx, permb,
                                           temp, tb, spos, ssfv, ctx->stream));
        ctx->launches += 3;
        bpart = spos;
        bstride = 3;
        bsfv = sfv_pp ? ssfv : a.sfv;
        perm = permb;
      }
      CUDA_TRY(ctx, launch_tay_corr(sd, taytab, tmpl, bpart, nb, bstride, bsfv, sfv_pp, terms32, pflag,
                                    no_gram ? 1 : 0, tlanes, ctx->stream));
      COLL_TRY(mark(1));
      if (!no_gram)
        CUDA_TRY(ctx, launch_tay_gram(sd, tmpl, bpart, nb, bstride, bsfv, sfv_pp, terms32, dn,
                                      dn ? reinterpret_cast<int*>(dn + dn_table_floats(sd.nf)) : nullptr, ctx->stream));
      ctx->launches += no_gram ? 0 : tay_gram_launches(sd, nb, dn != nullptr);
    } else {
      CUDA_TRY(ctx, launch_corr(sd, a, precision, ctx->stream));
      COLL_TRY(mark(1));
    }
    COLL_TRY(mark(2));
    AsmArgs s;
    s.terms = terms;
    s.terms_f32 = f32t ? 1 : 0;
    s.pflag = pflag;
    s.ynorm2 = yn;
    s.logw_prior = d_logw ? d_logw + b0 : nullptr;
    s.loglik = d_loglik + b0;
    s.amp = d_amp ? static_cast<double2*>(d_amp) + b0 * sd.J * sd.S : nullptr;
    s.term_c = d_c ? static_cast<double2*>(d_c) + b0 * sd.J * sd.S : nullptr;
    s.term_G = d_G ? static_cast<double2*>(d_G) + b0 * sd.J * sd.S * sd.S : nullptr;
    s.flags = ctx->d_flags;
    s.P = nb;
    s.perm = perm;
    CUDA_TRY(ctx, launch_assemble(sd, s, ctx->stream));
    COLL_TRY(mark(3));
    ctx->launches += 2;
  }
  return CDMS_OK;
}

// ---------------------------------------------------------------------------- standalone A6-A8 entries
// (beliefs.cu kernels, RED_ITEMS partition).  Cross-rank combines are all-gathers followed by a fixed rank-order
// combine on the device (deterministic for a given rank count).
cdms_status run_lse(cdms_ctx ctx, const double* d_l, int64_t P, double* d_lse) {
  const int64_t nb = red_blocks(P);
  double2 *part, *per_rank;
  double* scal;
  WS_TRY(ctx, WS_LSE_PART, nb + 1, &part);
  WS_TRY(ctx, WS_LSE_RANK, ctx->nranks + 1, &per_rank);
  WS_TRY(ctx, WS_SCAL, 8, &scal);
  CUDA_TRY(ctx, launch_lse_partial(d_l, P, part, ctx->stream));
  if (ctx->coll) {
    CUDA_TRY(ctx, launch_lse_final(part, nb, part + nb, ctx->stream));
    COLL_TRY(ctx->coll->allgather(ctx, part + nb, per_rank, sizeof(double2)));
  } else {
    CUDA_TRY(ctx, launch_lse_final(part, nb, per_rank, ctx->stream));
  }
  CUDA_TRY(ctx, launch_lse_combine(per_rank, ctx->nranks, d_lse, scal + 0, scal + 1, ctx->d_flags, ctx->stream));
  ctx->launches += 3;
  return CDMS_OK;
}

cdms_status run_moments(cdms_ctx ctx, const double* d_x, const double* d_w, int64_t P, double* d_est) {
  const int64_t nb = red_blocks(P);
  double *part, *sums, *ranks;
  WS_TRY(ctx, WS_MOM_PART, (nb + 1) * 21, &part);
  WS_TRY(ctx, WS_SUMS, 32, &sums);
  WS_TRY(ctx, WS_RANKS, (size_t)ctx->nranks * 21, &ranks);
  CUDA_TRY(ctx, launch_moments1(d_x, d_w, P, part, ctx->stream));
  CUDA_TRY(ctx, launch_sum_partials(part, nb, 7, sums, ctx->stream));
  if (ctx->coll) {
    COLL_TRY(ctx->coll->allgather(ctx, sums, ranks, 7 * sizeof(double)));
    CUDA_TRY(ctx, launch_sum_ranks(ranks, ctx->nranks, 7, sums, ctx->stream));
  }
  CUDA_TRY(ctx, launch_moments2(d_x, d_w, P, sums, part, ctx->stream));
  CUDA_TRY(ctx, launch_sum_partials(part, nb, 21, sums + 8, ctx->stream));
  if (ctx->coll) {
    COLL_TRY(ctx->coll->allgather(ctx, sums + 8, ranks, 21 * sizeof(double)));
    CUDA_TRY(ctx, launch_sum_ranks(ranks, ctx->nranks, 21, sums + 8, ctx->stream));
  }
  CUDA_TRY(ctx, launch_moments_finalize(sums, sums + 8, d_est, ctx->d_flags, ctx->stream));
  ctx->launches += ctx->coll ? 7 : 5;
  return CDMS_OK;
}

// ---------------------------------------------------------------------------- rows A6-A9 after the likelihood
// The belief update of cdms_bp_step / cdms_bp_update (step.cu): normalize, moments, systematic resampling of the masses
// e^{l - M} (C-amb-23) with the gather of the ancestors' states, regularization.  One rank: the five step.cu kernels
// with last-block epilogues.  Several ranks: the same per-block bodies; the block partials of every rank are
// all-gathered and reduced in the single-rank order (bit-identical results for block-aligned shards); the resampling
// plan is formed on the device from the all-gathered masses and K_anc writes each output slot's state straight into
// the owner rank's stage buffer, then a barrier and the regularization from the own stage buffer.  No host
// synchronization in either case.
cdms_status bp_update_impl(cdms_ctx ctx, const double* l, double* x, int64_t P_local, const cdms_step_params* prm,
                           double* d_est, double* d_lse, int64_t* d_anc) {
  NvtxRange nv_("update (A6-A9)");
  const bool comm = ctx->coll != nullptr;
  const int R = ctx->nranks;
  const int64_t P_total = P_local * R, p0 = (int64_t)ctx->rank * P_local;
  const int64_t nb = step_blocks(P_local);
  double2 *lpart, *pairs;
  double *mpart, *sums, *w, *L6, *scal, *stage;
  uint64_t *q, *bsum, *qall, *plan;
  unsigned* cnt;
  WS_TRY(ctx, WS_LSE_PART, nb + 1, &lpart);
  WS_TRY(ctx, WS_LSE_RANK, R + 1, &pairs);
  WS_TRY(ctx, WS_MOM_PART, (nb + 1) * 21, &mpart);
  WS_TRY(ctx, WS_SUMS, 32, &sums);
  WS_TRY(ctx, WS_Q, P_local, &q);
  WS_TRY(ctx, WS_BSUM, nb + 2, &bsum);
  WS_TRY(ctx, WS_QALL, 2 * R + 4, &qall);
  WS_TRY(ctx, WS_PLAN, 8, &plan);
  WS_TRY(ctx, WS_STEP_CNT, 4, &cnt);  // zeroed at allocation, reset by each kernel's last block
  WS_TRY(ctx, WS_W, P_local, &w);
  WS_TRY(ctx, WS_L6, 36, &L6);
  WS_TRY(ctx, WS_SCAL, 8, &scal);
  const uint32_t u_bits = host_step_u_bits(prm->philox_key, prm->step);
  const int reg = prm->regularize ? 1 : 0;
  if (!comm) {
    WS_TRY(ctx, WS_STAGE, P_local * 6, &stage);
    if (ctx->step_fused) {
      // the five kernels' bodies in one cooperative launch (grid barriers instead of launches and last-block tails),
      // identical arithmetic and block partition, so identical results
      StepFusedArgs fa;
      fa.l = l;
      fa.x = x;
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
      fa.anc = d_anc;
      fa.plan = plan;
      fa.u_bits = u_bits;
      fa.h = step_reg_bandwidth(P_total);
      fa.regularize = reg;
      fa.key = prm->philox_key;
      fa.step = prm->step;
      CUDA_TRY(ctx, launch_step_fused(fa, ctx->num_sms, ctx->stream));
      ctx->launches += 1;
      return CDMS_OK;
    }
    CUDA_TRY(ctx, launch_step_lse(l, P_local, lpart, cnt + 0, pairs, 1, d_lse, scal + 0, scal + 1, ctx->d_flags,
                                  ctx->stream));
    CUDA_TRY(ctx, launch_step_post(l, x, P_local, scal + 0, scal + 1, ctx->d_flags, w, q, mpart, bsum, cnt + 1, sums,
                                   u_bits, plan, ctx->stream));
    CUDA_TRY(ctx, launch_step_scan(q, x, w, P_local, bsum, sums, ctx->d_flags, mpart, cnt + 2, sums + 8, 1, d_est, L6,
                                   ctx->d_flags, ctx->stream));
    CUDA_TRY(ctx, launch_step_anc(q, bsum, P_local, plan, P_local, u_bits, x, stage, d_anc, nullptr, nullptr, 0,
                                  ctx->d_flags, ctx->stream));
    // regularization with the pre-resampling covariance (A9), reading the staged states (no extra copy)
    CUDA_TRY(ctx, launch_step_reg(stage, x, P_local, 0, P_total, L6, reg, prm->philox_key, prm->step, ctx->stream));
    ctx->launches += 5;
    return CDMS_OK;
  }
  cdms_status st = ensure_peer(ctx, P_local);
  if (st) return st;
  double* gpart;
  WS_TRY(ctx, WS_GPART, (size_t)R * nb * 21, &gpart);
  const int64_t nbt = (int64_t)R * nb;
  // (A6) block partials of every rank -> M, ln S, lse in the single-rank combine order
  CUDA_TRY(ctx, launch_step_lse(l, P_local, lpart, cnt + 0, nullptr, 0, nullptr, nullptr, nullptr, ctx->d_flags,
                                ctx->stream));
  COLL_TRY(ctx->coll->allgather(ctx, lpart, gpart, (size_t)nb * sizeof(double2)));
  CUDA_TRY(ctx, launch_step_lse_global(reinterpret_cast<double2*>(gpart), nbt, pairs, d_lse, scal + 0, scal + 1,
                                       ctx->d_flags, ctx->stream));
  // (A7, A8) weights, masses e^{l - M}, first-moment partials, local scan of the block masses; then all ranks' first
  // moments and this rank's resampling plan from the all-gathered Q_r
  CUDA_TRY(ctx, launch_step_post(l, x, P_local, scal + 0, scal + 1, ctx->d_flags, w, q, mpart, bsum, cnt + 1, nullptr,
                                 u_bits, nullptr, ctx->stream));
  COLL_TRY(ctx->coll->allgather(ctx, mpart, gpart, (size_t)nb * 7 * sizeof(double)));
  COLL_TRY(ctx->coll->allgather(ctx, bsum + nb, qall, sizeof(uint64_t)));
  CUDA_TRY(ctx, launch_step_post_global(gpart, nbt, sums, qall, R, ctx->rank, P_total, u_bits, plan, ctx->stream));
  // (A7) inclusive scan + second-moment partials; all ranks' covariance, est and its Cholesky factor
  CUDA_TRY(ctx, launch_step_scan(q, x, w, P_local, bsum, sums, ctx->d_flags, mpart, cnt + 2, nullptr, 0, nullptr,
                                 nullptr, ctx->d_flags, ctx->stream));
  COLL_TRY(ctx->coll->allgather(ctx, mpart, gpart, (size_t)nb * 21 * sizeof(double)));
  CUDA_TRY(ctx, launch_step_scan_global(gpart, nbt, sums, sums + 8, d_est, L6, ctx->d_flags, ctx->stream));
  // (A8) ancestors of this rank's slots, states written into the owners' stage buffers; barrier; (A9) regularize
  CUDA_TRY(ctx, launch_step_anc(q, bsum, P_local, plan, P_total, u_bits, x, nullptr, nullptr, ctx->d_peer_x,
                                d_anc ? ctx->d_peer_anc : nullptr, p0, ctx->d_flags, ctx->stream));
  COLL_TRY(ctx->coll->barrier(ctx));
  CUDA_TRY(ctx, launch_step_reg(ctx->pstage, x, P_local, p0, P_total, L6, reg, prm->philox_key, prm->step,
                                ctx->stream));
  if (d_anc)
    CUDA_TRY(ctx, cudaMemcpyAsync(d_anc, ctx->panc, sizeof(int64_t) * P_local, cudaMemcpyDeviceToDevice, ctx->stream));
  ctx->launches += 8;
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
  if (const char* e = getenv("CDMS_LOCALITY")) ctx->locality = atoi(e) ? 1 : 0;
  if (const char* e = getenv("CDMS_GRAM_TAB")) ctx->gram_tab = atoi(e);  // A/B: 0 off, 2 S >= 7 only
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
  delete ctx->coll;  // closes IPC mappings of peers' buffers before the communicator goes
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  if (ctx->pstage) cudaFree(ctx->pstage);
  if (ctx->panc) cudaFree(ctx->panc);
  if (ctx->d_peer_x) cudaFree(ctx->d_peer_x);
  if (ctx->d_peer_anc) cudaFree(ctx->d_peer_anc);
  if (ctx->d_barrier) cudaFree(ctx->d_barrier);
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
  ctx->ev_gram_first.clear();
  return CDMS_OK;
}

cdms_status cdms_timing_read_stages(cdms_ctx ctx, double* ms, int64_t* n_launches) {
  if (!ctx || !ms || !n_launches) return CDMS_EINVAL;
  DeviceGuard g(ctx->device);
  ms[0] = ms[1] = ms[2] = 0.0;
  for (size_t i = 0, b = 0; i + 3 < ctx->ev_used; i += 4, ++b) {
    CUDA_TRY(ctx, cudaEventSynchronize(ctx->ev_pool[i + 3]));
    float t[3] = {0.f, 0.f, 0.f};
    for (int k = 0; k < 3; ++k) CUDA_TRY(ctx, cudaEventElapsedTime(&t[k], ctx->ev_pool[i + k], ctx->ev_pool[i + k + 1]));
    const bool gf = ctx->ev_gram_first[b] != 0;
    ms[0] += gf ? t[1] : t[0];  // correlation kernel
    ms[1] += gf ? t[0] : t[1];  // Gram kernel
    ms[2] += t[2];              // assembly
  }
  *n_launches = (int64_t)(ctx->ev_used / 4);
  return CDMS_OK;
}

cdms_status cdms_timing_read(cdms_ctx ctx, double* loglik_ms, int64_t* n_launches) {
  if (!ctx || !loglik_ms || !n_launches) return CDMS_EINVAL;
  double ms[3];
  cdms_status st = cdms_timing_read_stages(ctx, ms, n_launches);
  if (st) return st;
  *loglik_ms = ms[0] + ms[1];
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
  NvtxRange nv_("cdms_reserve");
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
    NbPlan nbp{};  // the tensor-core path's per-PA B operand and scales (PLANAR_NB, FP32)
    const bool nbt = ctx->nb_tensor && scene->precision == CDMS_FP32 && nb_tensor_plan(sd, &nbp);
    const bool f32t = tay_engine(ctx, sd, scene->precision, nbt);  // the batch and terms sizes loglik_impl uses
    const int T = terms_width(sd.S);
    const size_t per_particle = (size_t)sd.J * T * (f32t ? sizeof(float2) : sizeof(double2));
    int64_t PB = (int64_t)(TERMS_BUDGET / per_particle);
    PB = PB < TILE_P ? TILE_P : (PB / TILE_P) * TILE_P;
    if (PB > P_local) PB = P_local;
    WS_TRY(ctx, WS_TERMS, f32t ? ((size_t)PB * sd.J * T + 1) / 2 : (size_t)PB * sd.J * T, &d2);
    WS_TRY(ctx, WS_PFLAG, PB, &i32);
    unsigned int* sch;
    WS_TRY(ctx, WS_SCHED, 2, &sch);
    WS_TRY(ctx, WS_STEP_CNT, 4, &sch);
    WS_TRY(ctx, WS_TMPL, (int64_t)(sd.J + 1) * sd.n_mb * NWARP, &f4);
    if (nbt) {
      uint8_t* nbop;
      float* nbs;
      WS_TRY(ctx, WS_NBOP, nb_operand_bytes(sd, nbp), &nbop);
      WS_TRY(ctx, WS_NBSCALE, MAXJ, &nbs);
    }
    if (tay_engine(ctx, sd, scene->precision, nbt)) {  // K1T's tables (the same choice loglik_impl makes)
      float2* tab;
      WS_TRY(ctx, WS_TAY, std::max(tay_table_bytes(sd, 0), tay_table_bytes(sd, 1)) / sizeof(float2), &tab);
      if (ctx->locality && PB >= LOCALITY_MIN_P) {  // the locality sort's buffers (shared-SFV batches)
        uint32_t* keys;
        unsigned char* temp;
        double* spos;
        WS_TRY(ctx, WS_LOC_KEYS, 2 * (size_t)PB, &keys);
        WS_TRY(ctx, WS_LOC_IDX, 2 * (size_t)PB, &i32);
        WS_TRY(ctx, WS_LOC_TEMP, locality_sort_temp_bytes(PB), &temp);
        WS_TRY(ctx, WS_LOC_POS, 3 * (size_t)PB, &spos);
      }
      if (ctx->gram_tab && sd.small_step >= 1 && (sd.S >= 7 || ctx->gram_tab == 1)) {  // the Gram's D_N table,
        float* dn;                                                                     // built here, outside captures
        WS_TRY(ctx, WS_DN, dn_table_floats(sd.nf) + 4, &dn);  // + the Gram's W != 0 flag
        if (ctx->dn_nf != sd.nf || ctx->dn_ptr != dn) {
          CUDA_TRY(ctx, launch_dn_table(sd.nf, dn, ctx->stream));
          ctx->launches += 1;
          ctx->dn_nf = sd.nf;
          ctx->dn_ptr = dn;
        }
      }
    }
  }
  WS_TRY(ctx, WS_PLAN, 8, &u);
  WS_TRY(ctx, WS_RANKS, (size_t)ctx->nranks * 21, &d);
  if (ctx->coll) {
    WS_TRY(ctx, WS_GPART, (size_t)ctx->nranks * step_blocks(P_local) * 21, &d);
    cdms_status st2 = ensure_peer(ctx, P_local);  // collective with a communicator (all ranks reserve alike)
    if (st2) return st2;
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
  delete ctx->coll;
  ctx->coll = nullptr;
  NCCL_TRY(ctx, ncclCommInitRank(&ctx->comm, nranks, id, rank));
  ctx->rank = rank;
  ctx->nranks = nranks;
  ctx->coll = new NcclColl();
  ctx->pcap = 0;  // peer buffers are (re)registered collectively on first use
  return CDMS_OK;
}

cdms_status cdms_loopback_create(int nranks, cdms_loopback* out) {
  if (!out || nranks < 1) return CDMS_EINVAL;
  *out = new cdms_loopback_s(nranks);
  return CDMS_OK;
}
cdms_status cdms_loopback_destroy(cdms_loopback g) {
  if (!g) return CDMS_EINVAL;
  delete g;
  return CDMS_OK;
}
cdms_status cdms_comm_init_loopback(cdms_ctx ctx, cdms_loopback g, int rank) {
  if (!ctx || !g || rank < 0 || rank >= g->nranks) return fail(ctx, CDMS_EINVAL, "comm_init_loopback: bad args");
  if (ctx->comm || ctx->coll) return fail(ctx, CDMS_EINVAL, "comm_init_loopback: a communicator is attached");
  ctx->rank = rank;
  ctx->nranks = g->nranks;
  ctx->coll = new LoopbackColl(g);
  ctx->pcap = 0;
  return CDMS_OK;
}

cdms_status cdms_layout(cdms_ctx ctx, const cdms_scene* scene, const double* d_sfv, double* d_layout, double* d_va,
                        double* d_H) {
  if (!ctx) return CDMS_EINVAL;
  DeviceGuard g(ctx->device);
  NvtxRange nv_("cdms_layout");
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
  NvtxRange nv_("cdms_loglik");
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
  NvtxRange nv_("cdms_loglik_terms");
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
  NvtxRange nv_("cdms_birth_proposal");
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

cdms_status cdms_pf_update(cdms_ctx ctx, const cdms_scene* scene, const double* h_f_pb, const double* d_particles,
                           int64_t P, int32_t pstride, const double* d_phi, const double* d_walpha, const void* d_mu,
                           const double* d_gamma, const double* h_zeta, const double* h_eta, const void* d_y,
                           const void* d_mu3, const void* d_mcols, int32_t L, double* d_logr, double* d_w,
                           double* d_out) {
  if (!ctx) return CDMS_EINVAL;
  DeviceGuard g(ctx->device);
  NvtxRange nv_("cdms_pf_update");
  if (!scene || !h_f_pb || !d_particles || !d_walpha || !d_mu || !d_gamma || !h_zeta || !h_eta || !d_y ||
      !d_mu3 || (L > 0 && !d_mcols) || !d_logr || !d_out || P <= 0 || pstride < 3 || L < 0 ||
      L + 1 > pf_max_snapshots())
    return fail(ctx, CDMS_EINVAL, "pf_update: bad arguments (P=%lld, L=%d)", (long long)P, L);
  // the PF's component: one wall whose SFV is per particle (K = 1, component 1), on the K1T tables; d_phi == NULL: the
  // LOS PF s = 0 (F4)
  cdms_scene s1 = *scene;
  s1.K = 1;
  SceneDev sd;
  cdms_status st = build_scene(ctx, &s1, h_f_pb, nullptr, nullptr, &sd);
  if (st) return st;
  if (scene->precision != CDMS_FP32 || sd.wavefront == CDMS_PLANAR_NB)
    return fail(ctx, CDMS_EUNSUPPORTED, "pf_update: FP32 spherical / planar-WB only (K1T tables)");
  double par[2 * MAXJ];
  for (int j = 0; j < sd.J; ++j) {
    if (!(h_eta[j] > 0.0) || !is_fin(h_eta[j])) return fail(ctx, CDMS_EINVAL, "pf_update: eta[%d] must be > 0", j);
    if (!(h_zeta[j] >= 0.0 && h_zeta[j] <= 1.0)) return fail(ctx, CDMS_EINVAL, "pf_update: zeta[%d] not in [0, 1]", j);
    par[j] = h_eta[j];
    par[MAXJ + j] = h_zeta[j];
  }
  const int J = sd.J, T = L + 1;
  const int64_t Nz = (int64_t)sd.nf * sd.Na;
  SceneDev sdt = sd;  // the T snapshots of every PA as J T "PAs" for the table builder
  sdt.J = J * T;
  const size_t tab_bytes = tay_table_bytes(sdt, 0);
  if (tab_bytes > ((size_t)1 << 30)) return fail(ctx, CDMS_EUNSUPPORTED, "pf_update: tables of %zu bytes", tab_bytes);
  float2 *snaps, *tab;
  double2 *dots, *fixed, *cc;
  double *gain2, *dpar;
  int* pflag;
  float4 *yt, *tmpl;
  double* yn;
  WS_TRY(ctx, WS_PF_SNAP, (size_t)J * T * Nz, &snaps);
  WS_TRY(ctx, WS_PF_TAB, tab_bytes / sizeof(float2), &tab);
  WS_TRY(ctx, WS_PF_DOTS, (size_t)J * T * T, &dots);
  WS_TRY(ctx, WS_PF_FIXED, (size_t)J * pf_fixed_width(), &fixed);
  WS_TRY(ctx, WS_PF_CC, (size_t)P * J * T, &cc);
  WS_TRY(ctx, WS_PF_FLAG, P, &pflag);
  WS_TRY(ctx, WS_PF_GAIN, (size_t)P * J, &gain2);
  WS_TRY(ctx, WS_PF_PAR, 2 * MAXJ, &dpar);
  double* lse2;
  WS_TRY(ctx, WS_LSE2, (size_t)3 * MAXJ * (lse_blocks(P) + 1), &lse2);
  WS_TRY(ctx, WS_YTILES, (int64_t)sd.J * sd.n_mb * sd.n_kc * sd.kc_len * NWARP, &yt);
  WS_TRY(ctx, WS_YNORM, MAXJ, &yn);
  WS_TRY(ctx, WS_TMPL, (int64_t)(sd.J + 1) * sd.n_mb * NWARP, &tmpl);
  CUDA_TRY(ctx, cudaMemcpyAsync(dpar, par, sizeof(par), cudaMemcpyHostToDevice, ctx->stream));
  // (1) template columns of the PAs; snapshots e0 = z - mu3, m_l; their fp64 dot products and the particle-independent
  //     factor of A^-1; K1T tables of every snapshot
  CUDA_TRY(ctx, launch_prep_y(sd, static_cast<const float2*>(d_y), yt, yn, tmpl, ctx->stream));
  CUDA_TRY(ctx, launch_pf_prep(J, T, Nz, static_cast<const float2*>(d_y), static_cast<const float2*>(d_mu3),
                               static_cast<const float2*>(d_mcols), snaps, dots, dpar, fixed, ctx->d_flags,
                               ctx->stream));
  CUDA_TRY(ctx, launch_tay_prep(sdt, snaps, tab, 0, ctx->taylor_prep_direct, ctx->stream));
  // (2) per (particle, PA): psi_p^H v_t for the T snapshots
  CUDA_TRY(ctx, launch_pf_corr(sd, T, tab, tmpl, d_particles, P, pstride, d_phi, cc, pflag, ctx->stream));
  // (3) per particle: log kappa~(phi_p, 1) - log kappa~(., 0) summed over PAs + log w_alpha; M_y, existence, weights
  CUDA_TRY(ctx, launch_pf_finish(sd, T, cc, fixed, dpar, dpar + MAXJ, gain2, d_particles, pstride, d_phi, d_walpha,
                                 static_cast<const double2*>(d_mu), d_gamma, pflag, P, d_logr, d_w, d_out,
                                 ctx->d_flags, lse2, ctx->stream));
  ctx->launches += 12 + (d_w ? 1 : 0);
  return CDMS_OK;
}

cdms_status cdms_noise_update(cdms_ctx ctx, const cdms_scene* scene, const double* d_eta, const double* d_wxi,
                              int64_t P, const void* d_y, const void* d_mu, const void* d_mcols, int32_t S,
                              double* d_logw, double* d_w, double* d_lognorm) {
  if (!ctx) return CDMS_EINVAL;
  DeviceGuard g(ctx->device);
  NvtxRange nv_("cdms_noise_update");
  if (!scene || !d_eta || !d_wxi || !d_y || !d_mu || (S > 0 && !d_mcols) || !d_logw || !d_lognorm || P <= 0 || S < 0 ||
      S > slam_max_columns())
    return fail(ctx, CDMS_EINVAL, "noise_update: bad arguments (P=%lld, S=%d)", (long long)P, S);
  SceneDev sd;
  cdms_status st = build_scene(ctx, scene, nullptr, nullptr, nullptr, &sd);
  if (st) return st;
  const int J = sd.J, T = S + 1;
  const int64_t Nz = (int64_t)sd.nf * sd.Na;
  float2* stack;
  double2* dots;
  double* eig;
  WS_TRY(ctx, WS_SL_STACK, (size_t)J * T * Nz, &stack);
  WS_TRY(ctx, WS_SL_DOTS, (size_t)J * T * T, &dots);
  WS_TRY(ctx, WS_SL_EIG, (size_t)J * slam_eig_width(), &eig);
  double* lse2;
  WS_TRY(ctx, WS_LSE2, (size_t)3 * MAXJ * (lse_blocks(P) + 1), &lse2);
  // e = z - mu_nu and the columns: their dot products (fp64), then per PA the eigen data of M^H M, per particle nu~
  CUDA_TRY(ctx, launch_vec_stack_dots(J, T, S, Nz, static_cast<const float2*>(d_y), static_cast<const float2*>(d_mu),
                                      static_cast<const float2*>(d_mcols), nullptr, nullptr, stack, dots, ctx->stream));
  CUDA_TRY(ctx, launch_noise_update(J, S, P, Nz, dots, eig, d_eta, d_wxi, d_logw, d_lognorm, d_w, ctx->d_flags,
                                    lse2, ctx->stream));
  ctx->launches += 6;
  return CDMS_OK;
}

cdms_status cdms_ppr_update(cdms_ctx ctx, const cdms_scene* scene, const double* h_zeta, const double* h_eta,
                            const void* d_y, const void* d_mu3, const void* d_mcols, int32_t L, const void* d_momega,
                            const void* d_mu4, double* d_out) {
  if (!ctx) return CDMS_EINVAL;
  DeviceGuard g(ctx->device);
  NvtxRange nv_("cdms_ppr_update");
  if (!scene || !h_zeta || !h_eta || !d_y || !d_mu3 || (L > 0 && !d_mcols) || !d_momega || !d_mu4 || !d_out || L < 0 ||
      L > slam_max_columns())
    return fail(ctx, CDMS_EINVAL, "ppr_update: bad arguments (L=%d)", L);
  SceneDev sd;
  cdms_status st = build_scene(ctx, scene, nullptr, nullptr, nullptr, &sd);
  if (st) return st;
  double par[2 * MAXJ];
  for (int j = 0; j < sd.J; ++j) {
    if (!(h_eta[j] > 0.0) || !is_fin(h_eta[j])) return fail(ctx, CDMS_EINVAL, "ppr_update: eta[%d] must be > 0", j);
    if (!(h_zeta[j] > 0.0 && h_zeta[j] < 1.0)) return fail(ctx, CDMS_EINVAL, "ppr_update: zeta[%d] not in (0, 1)", j);
    par[j] = h_zeta[j];
    par[MAXJ + j] = h_eta[j];
  }
  const int J = sd.J, T = L + 3;
  const int64_t Nz = (int64_t)sd.nf * sd.Na;
  float2* stack;
  double2* dots;
  double* dpar;
  WS_TRY(ctx, WS_SL_STACK, (size_t)J * T * Nz, &stack);
  WS_TRY(ctx, WS_SL_DOTS, (size_t)J * T * T, &dots);
  WS_TRY(ctx, WS_SL_PAR, 2 * MAXJ, &dpar);
  CUDA_TRY(ctx, cudaMemcpyAsync(dpar, par, sizeof(par), cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(ctx, launch_vec_stack_dots(J, T, L, Nz, static_cast<const float2*>(d_y), static_cast<const float2*>(d_mu3),
                                      static_cast<const float2*>(d_mcols), static_cast<const float2*>(d_momega),
                                      static_cast<const float2*>(d_mu4), stack, dots, ctx->stream));
  CUDA_TRY(ctx, launch_ppr_update(J, L, dots, dpar, dpar + MAXJ, d_out, ctx->d_flags, ctx->stream));
  ctx->launches += 3;
  return CDMS_OK;
}

cdms_status cdms_weights_normalize(cdms_ctx ctx, const double* d_logw, int64_t P_local, double* d_w, double* d_lse) {
  if (!ctx) return CDMS_EINVAL;
  DeviceGuard g(ctx->device);
  NvtxRange nv_("cdms_weights_normalize");
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
  NvtxRange nv_("cdms_moments");
  if (!d_particles || !d_w || !d_est || P_local <= 0) return fail(ctx, CDMS_EINVAL, "moments: bad arguments");
  return run_moments(ctx, d_particles, d_w, P_local, d_est);
}

cdms_status cdms_resample(cdms_ctx ctx, const double* d_w, int64_t P_local, uint32_t u_bits, int64_t* d_ancestors) {
  if (!ctx) return CDMS_EINVAL;
  DeviceGuard g(ctx->device);
  NvtxRange nv_("cdms_resample");
  if (!d_w || !d_ancestors || P_local <= 0) return fail(ctx, CDMS_EINVAL, "resample: bad arguments");
  const int R = ctx->nranks;
  const int64_t P_total = P_local * R;
  if (P_total > ((int64_t)1 << 26)) return fail(ctx, CDMS_EINVAL, "P_total=%lld exceeds 2^26", (long long)P_total);
  if (ctx->coll) {
    cdms_status st = ensure_peer(ctx, P_local);
    if (st) return st;
  }
  const int64_t nb = red_blocks(P_local);
  uint64_t *q, *bsum, *qall, *plan;
  double *scal, *wpart, *ranks;
  WS_TRY(ctx, WS_Q, P_local, &q);
  WS_TRY(ctx, WS_BSUM, nb + 2, &bsum);
  WS_TRY(ctx, WS_QALL, 2 * R + 4, &qall);
  WS_TRY(ctx, WS_PLAN, 8, &plan);
  WS_TRY(ctx, WS_SCAL, 8, &scal);
  WS_TRY(ctx, WS_WMAX_PART, nb + 1, &wpart);
  WS_TRY(ctx, WS_RANKS, (size_t)R * 21, &ranks);
  // q_p = rint(ldexp(w_p / w_max, 36)) with the global w_max (max is order-independent, hence exact)
  CUDA_TRY(ctx, launch_wmax_partial_f(d_w, P_local, wpart, ctx->d_flags, ctx->stream));
  CUDA_TRY(ctx, launch_max_final(wpart, nb, scal + 2, ctx->stream));
  if (ctx->coll) {
    COLL_TRY(ctx->coll->allgather(ctx, scal + 2, ranks, sizeof(double)));
    CUDA_TRY(ctx, launch_max_final(ranks, R, scal + 2, ctx->stream));
  }
  CUDA_TRY(ctx, launch_quantize(d_w, P_local, scal + 2, scal + 0, 0, q, ctx->d_flags, ctx->stream));
  CUDA_TRY(ctx, launch_scan(q, P_local, bsum, ctx->stream));  // bsum[nb] = Q_r
  if (!ctx->coll) {
    CUDA_TRY(ctx, launch_plan(bsum + nb, 1, 0, P_local, u_bits, plan, ctx->stream));
    CUDA_TRY(ctx, launch_ancestors(q, P_local, plan, P_local, u_bits, 0, d_ancestors, nullptr, ctx->d_flags,
                                   ctx->stream));
    ctx->launches += 7;
    return CDMS_OK;
  }
  // all ranks' masses -> this rank's plan on the device; ancestor ids written into the slot owners' buffers
  COLL_TRY(ctx->coll->allgather(ctx, bsum + nb, qall, sizeof(uint64_t)));
  CUDA_TRY(ctx, launch_plan(qall, R, ctx->rank, P_total, u_bits, plan, ctx->stream));
  CUDA_TRY(ctx, launch_ancestors(q, P_local, plan, P_total, u_bits, (int64_t)ctx->rank * P_local, nullptr,
                                 ctx->d_peer_anc, ctx->d_flags, ctx->stream));
  COLL_TRY(ctx->coll->barrier(ctx));
  CUDA_TRY(ctx, cudaMemcpyAsync(d_ancestors, ctx->panc, sizeof(int64_t) * P_local, cudaMemcpyDeviceToDevice,
                                ctx->stream));
  ctx->launches += 8;
  return CDMS_OK;
}

static cdms_status check_step_params(cdms_ctx ctx, const cdms_step_params* prm, int64_t P_local) {
  if (!prm) return fail(ctx, CDMS_EINVAL, "step params NULL");
  if (!is_fin(prm->T) || !is_fin(prm->sigma_v) || prm->sigma_v < 0.0) return fail(ctx, CDMS_EINVAL, "T/sigma_v");
  if (P_local <= 0 || P_local * ctx->nranks > ((int64_t)1 << 26))
    return fail(ctx, CDMS_EINVAL, "P_total=%lld outside [1, 2^26]", (long long)(P_local * ctx->nranks));
  return CDMS_OK;
}

cdms_status cdms_bp_step(cdms_ctx ctx, const cdms_scene* scene, double* d_particles, int64_t P_local, const double* d_sfv,
                         const void* d_y, const double* h_f_pb, const cdms_prior* h_prior, const double* h_eta,
                         const cdms_step_params* prm, double* d_est, double* d_lse) {
  if (!ctx) return CDMS_EINVAL;
  DeviceGuard g(ctx->device);
  NvtxRange nv_("cdms_bp_step");
  if (!d_particles || !d_y || !h_f_pb || !h_prior || !h_eta || !prm || !d_est || !d_lse || P_local <= 0)
    return fail(ctx, CDMS_EINVAL, "bp_step: bad arguments");
  cdms_status st = check_step_params(ctx, prm, P_local);  // every host check before the first launch
  if (st) return st;
  SceneDev sd;
  st = build_scene(ctx, scene, h_f_pb, h_prior, h_eta, &sd);
  if (st) return st;
  if (sd.K > 0 && !d_sfv) return fail(ctx, CDMS_EINVAL, "bp_step: d_sfv NULL with K > 0");
  const int64_t p0 = (int64_t)ctx->rank * P_local;
  double* l;
  WS_TRY(ctx, WS_LOGLIK, P_local, &l);
  // (1) prediction (row A9)
  {
    NvtxRange r("predict");
    CUDA_TRY(ctx, launch_predict(d_particles, P_local, p0, prm->T, prm->sigma_v, prm->philox_key, prm->step,
                                 ctx->stream));
  }
  ctx->launches += 1;
  // (2) coherent log-likelihood, uniform w_beta (rows A1-A5)
  st = loglik_impl(ctx, sd, scene->precision, d_particles, P_local, 6, d_sfv, 0, d_y, nullptr, l, nullptr);
  if (st) return st;
  // (3)-(6) normalize, moments, resample + redistribute, regularize (rows A6-A9)
  return bp_update_impl(ctx, l, d_particles, P_local, prm, d_est, d_lse, nullptr);
}

cdms_status cdms_bp_update(cdms_ctx ctx, const double* d_loglik, double* d_particles, int64_t P_local,
                           const cdms_step_params* prm, double* d_est, double* d_lse, int64_t* d_ancestors) {
  if (!ctx) return CDMS_EINVAL;
  DeviceGuard g(ctx->device);
  NvtxRange nv_("cdms_bp_update");
  if (!d_loglik || !d_particles || !prm || !d_est || !d_lse || P_local <= 0)
    return fail(ctx, CDMS_EINVAL, "bp_update: bad arguments");
  cdms_status st = check_step_params(ctx, prm, P_local);
  if (st) return st;
  return bp_update_impl(ctx, d_loglik, d_particles, P_local, prm, d_est, d_lse, d_ancestors);
}

cdms_status cdms_response(cdms_ctx ctx, const cdms_scene* scene, const double* d_pos, int64_t n, const int32_t* d_js,
                          const double* d_sfv, void* d_psi) {
  if (!ctx) return CDMS_EINVAL;
  DeviceGuard g(ctx->device);
  NvtxRange nv_("cdms_response");
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
  const int64_t lo = resample_slot_index(O, Qtot, P_total, u_bits);
  const int64_t hi = resample_slot_index(O + h_Q[rank], Qtot, P_total, u_bits);
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

// =========================================================================================================== F4 driver
// cdms_slam_step: one time step of the synthetic SLAM method in the paper's schedule -- prediction and
// birth messages, every update message from the same prediction messages (flooding), beliefs, resampling, estimates,
// declaration and pruning -- composed from the library's own entries (cdms_loglik, cdms_noise_update, cdms_pf_update,
// cdms_ppr_update, cdms_birth_proposal, cdms_bp_update, cdms_resample) and the kernels of slam_step.cu.  Readings F4a-k
// (DESIGN.md section 3).  Single-rank contexts only; four host synchronizations per step (predicted means for the
// birth proposal and the host-side priors, the birth's proposal, its normalization, the posterior statistics).
namespace {

constexpr int SLS = MAXS;  // slots: LOS + 8 PFs

uint32_t host_philox_word0(uint64_t key, uint64_t index, uint64_t step, uint32_t stream) {
  uint32_t c0 = (uint32_t)index, c1 = (uint32_t)(index >> 32), c2 = (uint32_t)step, c3 = stream;
  uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
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

// 3 x 3 Cholesky (row-major lower L of A), false on a non-positive pivot
bool chol3(const double* A, double* L) {
  for (int i = 0; i < 9; ++i) L[i] = 0.0;
  for (int j = 0; j < 3; ++j) {
    double d = A[4 * j];
    for (int k = 0; k < j; ++k) d -= L[3 * j + k] * L[3 * j + k];
    if (!(d > 0.0)) return false;
    L[4 * j] = sqrt(d);
    for (int i = j + 1; i < 3; ++i) {
      double a = A[3 * i + j];
      for (int k = 0; k < j; ++k) a -= L[3 * i + k] * L[3 * j + k];
      L[3 * i + j] = a / L[4 * j];
    }
  }
  return true;
}

}  // namespace

struct cdms_slam_s {
  cdms_ctx ctx = nullptr;
  cdms_scene scene{};
  std::vector<double> pa_pos, pa_rot, f_pb;
  cdms_slam_params prm{};
  int64_t P = 0;
  int J = 0;
  int64_t Nz = 0;
  // state
  double *x = nullptr, *eta = nullptr, *phi = nullptr, *gam = nullptr, *w = nullptr;
  double2* mu = nullptr;
  int n_slots = 0;
  int ident[SLS] = {};
  double zeta[SLS][MAXJ] = {};
  double phi_hat[SLS][3] = {};
  int64_t n = 1;
  int next_id = 1;
  // scratch
  double *l = nullptr, *wnew = nullptr, *logr = nullptr, *weta = nullptr, *logweta = nullptr, *wxi = nullptr;
  double *tphi = nullptr, *tgam = nullptr, *teta = nullptr, *lw = nullptr, *sfvpp = nullptr, *par = nullptr;
  double2* tmu = nullptr;
  int64_t* anc = nullptr;
  double *wpart = nullptr, *lpart = nullptr;
  double *stats = nullptr, *bout = nullptr, *bnorm = nullptr, *est = nullptr, *lse = nullptr, *pfout = nullptr,
         *pprout = nullptr, *lnorm = nullptr, *wk = nullptr;
  double2 *au = nullptr, *am = nullptr, *aw = nullptr, *psi = nullptr;
  float2 *m64 = nullptr, *munu = nullptr, *mu3o = nullptr, *mo = nullptr, *mws = nullptr, *us = nullptr;
  double *bpos = nullptr, *bsfv = nullptr;
  int32_t* bjs = nullptr;
  int64_t bv_chunk = 1;
  // debug copies
  double *x_pred = nullptr, *eta_pred = nullptr, *phi_pr = nullptr, *gam_pr = nullptr, *w_pr = nullptr;
  double2* mu_pr = nullptr;
  std::vector<void*> allocs;
  int n_feat_last = 0;
};

namespace {

template <typename T>
cudaError_t slam_alloc(cdms_slam sl, T** p, size_t count) {
  void* q = nullptr;
  const cudaError_t e = cudaMalloc(&q, (count ? count : 1) * sizeof(T));
  if (e != cudaSuccess) return e;
  sl->allocs.push_back(q);
  *p = static_cast<T*>(q);
  return cudaSuccess;
}

void slam_free(cdms_slam sl) {
  for (void* p : sl->allocs) cudaFree(p);
  sl->allocs.clear();
}

double* slot_phi(cdms_slam s, int i) { return s->phi + (size_t)i * s->P * 3; }
double2* slot_mu(cdms_slam s, int i) { return s->mu + (size_t)i * s->P; }
double* slot_gam(cdms_slam s, int i) { return s->gam + (size_t)i * s->P; }
double* slot_w(cdms_slam s, int i) { return s->w + (size_t)i * s->P; }

// weighted sums of the slots' (phi, mu, gamma) under weights w (or the posterior weights wnew) + x-hat and eta-bar
// (uniform weights) or eta-hat (weights weta); out layout: job order
void slot_jobs(cdms_slam s, SlamWsumJobs& jb, int first, int last, const double* wts, bool posterior) {
  for (int i = first; i < last; ++i) {
    const double* wi = wts + (size_t)i * s->P;
    jb.job[jb.n++] = SlamWsumJob{wi, reinterpret_cast<const double*>(slot_mu(s, i)), s->P, 2, 2};
    jb.job[jb.n++] = SlamWsumJob{wi, slot_gam(s, i), s->P, 1, 1};
    jb.job[jb.n++] = SlamWsumJob{wi, slot_phi(s, i), s->P, 3, i ? 3 : 0};
  }
  (void)posterior;
}

}  // namespace

extern "C" {

cdms_status cdms_slam_create(cdms_ctx ctx, const cdms_scene* scene, const double* h_f_pb, int64_t P,
                             const cdms_slam_params* prm, cdms_slam* out) {
  if (!ctx || !out) return CDMS_EINVAL;
  DeviceGuard g(ctx->device);
  *out = nullptr;
  if (!scene || !h_f_pb || !prm || P <= 0 || P > ((int64_t)1 << 26))
    return fail(ctx, CDMS_EINVAL, "slam_create: bad arguments (P=%lld)", (long long)P);
  if (ctx->coll) return fail(ctx, CDMS_EUNSUPPORTED, "slam_create: single-rank contexts only");
  if (prm->P_m <= 0 || prm->N_g <= 0 || !(prm->c_eta >= 1.0) || !(prm->c_gamma >= 1.0) || !(prm->p_s >= 0.0) ||
      !(prm->p_s <= 1.0) || !(prm->mu_b >= 0.0))
    return fail(ctx, CDMS_EINVAL, "slam_create: bad parameters");
  cdms_scene s0 = *scene;
  s0.K = 0;
  SceneDev sd;
  cdms_status st = build_scene(ctx, &s0, h_f_pb, nullptr, nullptr, &sd);
  if (st) return st;
  cdms_slam sl = new cdms_slam_s();
  sl->ctx = ctx;
  sl->prm = *prm;
  sl->P = P;
  sl->J = sd.J;
  sl->Nz = (int64_t)sd.nf * sd.Na;
  sl->pa_pos.assign(scene->h_pa_pos, scene->h_pa_pos + 3 * sd.J);
  sl->pa_rot.assign(scene->h_pa_rot, scene->h_pa_rot + 9 * sd.J);
  sl->f_pb.assign(h_f_pb, h_f_pb + sd.nf);
  sl->scene = *scene;
  sl->scene.h_pa_pos = sl->pa_pos.data();
  sl->scene.h_pa_rot = sl->pa_rot.data();
  const int J = sl->J;
  const int64_t Nz = sl->Nz;
  // belief-average chunk: at most 256 MiB of fp64 responses per chunk
  const int64_t K = P < prm->P_m ? P : prm->P_m;
  const int64_t per = (int64_t)J * SLS * Nz * 16;
  sl->bv_chunk = std::max<int64_t>(1, std::min<int64_t>(K, ((int64_t)256 << 20) / per));
  const int64_t nit = sl->bv_chunk * J * SLS;
  cudaError_t e = cudaSuccess;
  auto A = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
  A(slam_alloc(sl, &sl->x, (size_t)P * 6));
  A(slam_alloc(sl, &sl->eta, (size_t)J * P));
  A(slam_alloc(sl, &sl->phi, (size_t)SLS * P * 3));
  A(slam_alloc(sl, &sl->mu, (size_t)SLS * P));
  A(slam_alloc(sl, &sl->gam, (size_t)SLS * P));
  A(slam_alloc(sl, &sl->w, (size_t)SLS * P));
  A(slam_alloc(sl, &sl->l, (size_t)P));
  A(slam_alloc(sl, &sl->wnew, (size_t)SLS * P));
  A(slam_alloc(sl, &sl->logr, (size_t)SLS * P));
  A(slam_alloc(sl, &sl->weta, (size_t)J * P));
  A(slam_alloc(sl, &sl->logweta, (size_t)J * P));
  A(slam_alloc(sl, &sl->wxi, (size_t)J * P));
  A(slam_alloc(sl, &sl->tphi, (size_t)P * 3));
  A(slam_alloc(sl, &sl->tmu, (size_t)P));
  A(slam_alloc(sl, &sl->tgam, (size_t)P));
  A(slam_alloc(sl, &sl->teta, (size_t)P));
  A(slam_alloc(sl, &sl->lw, (size_t)P));
  A(slam_alloc(sl, &sl->sfvpp, (size_t)P * (SLS - 1) * 3));
  A(slam_alloc(sl, &sl->par, (size_t)SLAM_PAR));
  A(slam_alloc(sl, &sl->anc, (size_t)P));
  A(slam_alloc(sl, &sl->stats, (size_t)4 * SLAM_MAXJOBS));
  A(slam_alloc(sl, &sl->wpart, (size_t)4 * SLAM_MAXJOBS * slam_wsum_blocks(P)));
  A(slam_alloc(sl, &sl->lpart, (size_t)3 * (lse_blocks(P) + 1)));
  A(slam_alloc(sl, &sl->bout, (size_t)16));
  A(slam_alloc(sl, &sl->bnorm, (size_t)4));
  A(slam_alloc(sl, &sl->est, (size_t)28));
  A(slam_alloc(sl, &sl->lse, (size_t)4));
  A(slam_alloc(sl, &sl->pfout, (size_t)SLS * 2));
  A(slam_alloc(sl, &sl->pprout, (size_t)SLS * MAXJ * 3));
  A(slam_alloc(sl, &sl->lnorm, (size_t)MAXJ));
  A(slam_alloc(sl, &sl->wk, (size_t)SLS));
  A(slam_alloc(sl, &sl->au, (size_t)J * SLS * Nz));
  A(slam_alloc(sl, &sl->am, (size_t)J * SLS * Nz));
  A(slam_alloc(sl, &sl->aw, (size_t)J * SLS * Nz));
  A(slam_alloc(sl, &sl->psi, (size_t)nit * Nz));
  A(slam_alloc(sl, &sl->m64, (size_t)J * SLS * Nz));
  A(slam_alloc(sl, &sl->munu, (size_t)J * Nz));
  A(slam_alloc(sl, &sl->mu3o, (size_t)J * Nz));
  A(slam_alloc(sl, &sl->mo, (size_t)J * (SLS - 1) * Nz));
  A(slam_alloc(sl, &sl->mws, (size_t)J * Nz));
  A(slam_alloc(sl, &sl->us, (size_t)J * Nz));
  A(slam_alloc(sl, &sl->bpos, (size_t)nit * 3));
  A(slam_alloc(sl, &sl->bsfv, (size_t)nit * 3));
  A(slam_alloc(sl, &sl->bjs, (size_t)nit * 2));
  if (prm->keep_debug) {
    A(slam_alloc(sl, &sl->x_pred, (size_t)P * 6));
    A(slam_alloc(sl, &sl->eta_pred, (size_t)J * P));
    A(slam_alloc(sl, &sl->phi_pr, (size_t)SLS * P * 3));
    A(slam_alloc(sl, &sl->mu_pr, (size_t)SLS * P));
    A(slam_alloc(sl, &sl->gam_pr, (size_t)SLS * P));
    A(slam_alloc(sl, &sl->w_pr, (size_t)SLS * P));
  }
  if (e == cudaSuccess) e = cudaMemsetAsync(sl->phi, 0, sizeof(double) * SLS * P * 3, ctx->stream);
  if (e == cudaSuccess) e = launch_slam_fill(sl->wxi, (int64_t)J * P, 1.0 / (double)P, ctx->stream);
  if (e != cudaSuccess) {
    slam_free(sl);
    delete sl;
    return fail(ctx, e == cudaErrorMemoryAllocation ? CDMS_ENOMEM : CDMS_ECUDA, "slam_create: %s",
                cudaGetErrorString(e));
  }
  *out = sl;
  return CDMS_OK;
}

cdms_status cdms_slam_destroy(cdms_slam sl) {
  if (!sl) return CDMS_EINVAL;
  DeviceGuard g(sl->ctx->device);
  cudaStreamSynchronize(sl->ctx->stream);
  slam_free(sl);
  delete sl;
  return CDMS_OK;
}

cdms_status cdms_slam_get_view(cdms_slam sl, cdms_slam_view* v) {
  if (!sl || !v) return CDMS_EINVAL;
  *v = cdms_slam_view{};
  v->P = sl->P;
  v->J = sl->J;
  v->n_slots = sl->n_slots;
  v->n_feat = sl->n_feat_last;
  v->x = sl->x;
  v->eta = sl->eta;
  v->phi = sl->phi;
  v->mu = sl->mu;
  v->gamma = sl->gam;
  v->w = sl->w;
  v->x_pred = sl->x_pred;
  v->eta_pred = sl->eta_pred;
  v->phi_prior = sl->phi_pr;
  v->mu_prior = sl->mu_pr;
  v->gamma_prior = sl->gam_pr;
  v->w_prior = sl->w_pr;
  v->loglik = sl->l;
  v->w_eta = sl->weta;
  v->logr = sl->logr;
  v->w_post = sl->wnew;
  v->m_cols = sl->m64;
  v->mu_nu = sl->munu;
  v->u_sums = sl->au;
  v->m_sums = sl->am;
  v->mw_sums = sl->aw;
  v->pf_out = sl->pfout;
  v->ppr_out = sl->pprout;
  v->n = sl->n;
  v->next_id = sl->next_id;
  for (int i = 0; i < SLS; ++i) {
    v->ident[i] = sl->ident[i];
    for (int j = 0; j < MAXJ; ++j) v->zeta[i][j] = sl->zeta[i][j];
    for (int c = 0; c < 3; ++c) v->phi_hat[i][c] = sl->phi_hat[i][c];
  }
  return CDMS_OK;
}

cdms_status cdms_slam_set_slots(cdms_slam sl, int32_t n_slots, const int32_t* h_ident, const double* h_zeta,
                                const double* h_phi_hat, int64_t n, int32_t next_id) {
  if (!sl) return CDMS_EINVAL;
  if (n_slots < 1 || n_slots > SLS || !h_ident || !h_zeta || n < 1 || next_id < 1)
    return fail(sl->ctx, CDMS_EINVAL, "slam_set_slots: bad arguments");
  sl->n_slots = n_slots;
  for (int i = 0; i < n_slots; ++i) {
    sl->ident[i] = h_ident[i];
    for (int j = 0; j < sl->J; ++j) sl->zeta[i][j] = h_zeta[(size_t)i * sl->J + j];
    for (int c = 0; c < 3; ++c) sl->phi_hat[i][c] = h_phi_hat ? h_phi_hat[3 * i + c] : 0.0;
  }
  sl->n = n;
  sl->next_id = next_id;
  return CDMS_OK;
}

cdms_status cdms_slam_init(cdms_slam sl, const double* d_x0, const double* d_eta0) {
  if (!sl) return CDMS_EINVAL;
  cdms_ctx ctx = sl->ctx;
  DeviceGuard g(ctx->device);
  if (!d_x0 || !d_eta0) return fail(ctx, CDMS_EINVAL, "slam_init: NULL pointer");
  const cdms_slam_params& q = sl->prm;
  CUDA_TRY(ctx, cudaMemcpyAsync(sl->x, d_x0, sizeof(double) * sl->P * 6, cudaMemcpyDeviceToDevice, ctx->stream));
  CUDA_TRY(ctx, cudaMemcpyAsync(sl->eta, d_eta0, sizeof(double) * sl->P * sl->J, cudaMemcpyDeviceToDevice,
                                ctx->stream));
  // the LOS at n = 0 "the same way as new PFs": hyperprior amplitudes, weights p_B / P (reading F4j)
  const double pB = q.mu_b / (1.0 + q.mu_b);
  CUDA_TRY(ctx, launch_slam_birth(nullptr, nullptr, nullptr, q.mu_max, q.gamma_max, pB, nullptr, slot_mu(sl, 0),
                                  slot_gam(sl, 0), sl->lw, nullptr, nullptr, sl->lpart, sl->P, q.key, 0, ctx->stream));
  CUDA_TRY(ctx, launch_slam_fill(slot_w(sl, 0), sl->P, pB / (double)sl->P, ctx->stream));
  sl->n_slots = 1;
  sl->ident[0] = 0;
  for (int j = 0; j < sl->J; ++j) sl->zeta[0][j] = q.p_b_pr;
  sl->n = 1;
  sl->next_id = 1;
  ctx->launches += 2;
  return CDMS_OK;
}

cdms_status cdms_slam_step(cdms_slam sl, const void* d_y, cdms_slam_report* rep) {
  if (!sl) return CDMS_EINVAL;
  cdms_ctx ctx = sl->ctx;
  DeviceGuard g(ctx->device);
  NvtxRange nv_("cdms_slam_step");
  if (!d_y) return fail(ctx, CDMS_EINVAL, "slam_step: d_y NULL");
  if (sl->n_slots < 1) return fail(ctx, CDMS_EINVAL, "slam_step: no state (cdms_slam_init first)");
  const cdms_slam_params& q = sl->prm;
  cudaStream_t stm = ctx->stream;
  const int J = sl->J;
  const int64_t P = sl->P, Nz = sl->Nz;
  const uint64_t n = (uint64_t)sl->n;
  const bool dbg = q.keep_debug != 0;
  cdms_status st;
  // ---- (i) prediction messages: beta (NCV), xi (Gamma), alpha (legacy PFs), zeta (PPRs)
  CUDA_TRY(ctx, launch_predict(sl->x, P, 0, q.T, q.sigma_v, q.key, n, stm));
  CUDA_TRY(ctx, launch_slam_noise_predict(sl->eta, J, P, q.c_eta, q.key, n, stm));
  int S = sl->n_slots;
  double zeta_pr[SLS][MAXJ];
  for (int i = 0; i < S; ++i) {
    CUDA_TRY(ctx, launch_slam_pf_predict(i ? slot_phi(sl, i) : nullptr, slot_mu(sl, i), slot_gam(sl, i), slot_w(sl, i),
                                         P, i, q.sigma_sfv, q.sigma_mu, q.c_gamma, q.p_s, q.key, n, stm));
    for (int j = 0; j < J; ++j) zeta_pr[i][j] = q.p_s_pr * sl->zeta[i][j] + q.p_rev_pr * (1.0 - sl->zeta[i][j]);
  }
  ctx->launches += 2 + S;
  if (dbg) {
    CUDA_TRY(ctx, cudaMemcpyAsync(sl->x_pred, sl->x, sizeof(double) * P * 6, cudaMemcpyDeviceToDevice, stm));
    CUDA_TRY(ctx, cudaMemcpyAsync(sl->eta_pred, sl->eta, sizeof(double) * P * J, cudaMemcpyDeviceToDevice, stm));
  }
  // predicted means: x^_{n|n-1}, eta-bar, per slot (eps, mu-bar, gamma-bar, phi-bar)
  SlamWsumJobs jb{};
  jb.job[jb.n++] = SlamWsumJob{nullptr, sl->x, P, 6, 3};
  for (int j = 0; j < J; ++j) jb.job[jb.n++] = SlamWsumJob{nullptr, sl->eta + (size_t)j * P, P, 1, 1};
  const int j0 = jb.n;
  slot_jobs(sl, jb, 0, S, sl->w, false);
  double h[4 * SLAM_MAXJOBS];
  CUDA_TRY(ctx, launch_slam_wsum(jb, sl->wpart, sl->stats, stm));
  CUDA_TRY(ctx, cudaMemcpyAsync(h, sl->stats, sizeof(double) * 4 * jb.n, cudaMemcpyDeviceToHost, stm));
  ctx->launches += 2;
  if ((st = cdms_sync(ctx))) return st;
  double x_hat[3], eta_bar[MAXJ], eps[SLS], mub[SLS][2], gab[SLS];
  for (int c = 0; c < 3; ++c) x_hat[c] = h[1 + c] / (double)P;
  for (int j = 0; j < J; ++j) eta_bar[j] = h[4 * (1 + j) + 1] / (double)P;
  auto read_slot = [&](int i, int base) {
    eps[i] = h[4 * base];
    const double e = eps[i] > 0.0 ? eps[i] : 1.0;
    mub[i][0] = h[4 * base + 1] / e;
    mub[i][1] = h[4 * base + 2] / e;
    gab[i] = h[4 * (base + 1) + 1] / e;
  };
  for (int i = 0; i < S; ++i) read_slot(i, j0 + 3 * i);
  // ---- birth message of one new PF (Q = 1) on the F3 proposal (reading F4h)
  if (S < SLS) {
    double legacy[SLS * 3];
    for (int i = 1; i < S; ++i)
      for (int c = 0; c < 3; ++c) legacy[3 * (i - 1) + c] = sl->phi_hat[i][c];
    st = cdms_birth_proposal(ctx, &sl->scene, sl->f_pb.data(), x_hat, S > 1 ? legacy : nullptr, S - 1, d_y, q.box,
                             q.N_g, q.key, n, sl->bout, nullptr, nullptr);
    if (st) return st;
    double bo[13];
    CUDA_TRY(ctx, cudaMemcpyAsync(bo, sl->bout, sizeof(bo), cudaMemcpyDeviceToHost, stm));
    st = cdms_sync(ctx);
    bool born = false;
    if (st == CDMS_OK) {
      double C[9], Lq[9];
      const double tr = bo[3] + bo[7] + bo[11];
      for (int c = 0; c < 9; ++c) C[c] = bo[3 + c];
      for (int c = 0; c < 3; ++c) C[4 * c] += 1e-12 * tr;
      if (chol3(C, Lq)) {
        const double pB = q.mu_b / (1.0 + q.mu_b);
        CUDA_TRY(ctx, launch_slam_birth(bo, Lq, q.box, q.mu_max, q.gamma_max, pB, slot_phi(sl, S), slot_mu(sl, S),
                                        slot_gam(sl, S), sl->lw, slot_w(sl, S), sl->bnorm, sl->lpart, P, q.key, n,
                                        stm));
        SlamWsumJobs jn{};
        slot_jobs(sl, jn, S, S + 1, sl->w, false);
        CUDA_TRY(ctx, launch_slam_wsum(jn, sl->wpart, sl->stats, stm));
        double hb[4 * 3 + 1];
        CUDA_TRY(ctx, cudaMemcpyAsync(hb, sl->stats, sizeof(double) * 12, cudaMemcpyDeviceToHost, stm));
        CUDA_TRY(ctx, cudaMemcpyAsync(hb + 12, sl->bnorm, sizeof(double), cudaMemcpyDeviceToHost, stm));
        ctx->launches += 6;  // sample, 2 LSE levels, weights, 2 weighted-sum levels
        if ((st = cdms_sync(ctx))) return st;
        if (hb[12] > 0.0) {  // some particle inside the birth box
          for (int c = 0; c < 12; ++c) h[4 * j0 + 4 * 3 * S + c] = hb[c];
          read_slot(S, j0 + 3 * S);
          sl->ident[S] = sl->next_id++;
          for (int j = 0; j < J; ++j) zeta_pr[S][j] = q.p_b_pr;
          ++S;
          born = true;
        }
      }
    } else if (st != CDMS_EZEROMASS) {
      return st;  // a residual without power is no birth, anything else an error
    }
    (void)born;
  }
  sl->n_feat_last = S;
  if (dbg) {
    CUDA_TRY(ctx, cudaMemcpyAsync(sl->phi_pr, sl->phi, sizeof(double) * SLS * P * 3, cudaMemcpyDeviceToDevice, stm));
    CUDA_TRY(ctx, cudaMemcpyAsync(sl->mu_pr, sl->mu, sizeof(double2) * SLS * P, cudaMemcpyDeviceToDevice, stm));
    CUDA_TRY(ctx, cudaMemcpyAsync(sl->gam_pr, sl->gam, sizeof(double) * SLS * P, cudaMemcpyDeviceToDevice, stm));
    CUDA_TRY(ctx, cudaMemcpyAsync(sl->w_pr, sl->w, sizeof(double) * SLS * P, cudaMemcpyDeviceToDevice, stm));
  }
  // device slot parameters: eps, zeta of the prediction messages
  double hp[SLAM_PAR] = {};
  for (int i = 0; i < S; ++i) {
    hp[i] = eps[i];
    for (int j = 0; j < J; ++j) hp[MAXS + i * MAXJ + j] = zeta_pr[i][j];
  }
  CUDA_TRY(ctx, cudaMemcpyAsync(sl->par, hp, sizeof(hp), cudaMemcpyHostToDevice, stm));
  // ---- belief-averaged columns over the paired particles (reading F4c)
  {
    const int64_t K = P < q.P_m ? P : q.P_m;
    cdms_scene s1 = sl->scene;
    s1.K = 1;
    s1.precision = CDMS_FP64;
    SceneDev sd1;
    if ((st = build_scene(ctx, &s1, sl->f_pb.data(), nullptr, nullptr, &sd1))) return st;
    CUDA_TRY(ctx, cudaMemsetAsync(sl->au, 0, sizeof(double2) * J * S * Nz, stm));
    CUDA_TRY(ctx, cudaMemsetAsync(sl->am, 0, sizeof(double2) * J * S * Nz, stm));
    CUDA_TRY(ctx, cudaMemsetAsync(sl->aw, 0, sizeof(double2) * J * S * Nz, stm));
    CUDA_TRY(ctx, launch_slam_bv_wsum(sl->w, P, K, S, sl->wk, stm));
    for (int64_t k0 = 0; k0 < K; k0 += sl->bv_chunk) {
      const int B = (int)std::min<int64_t>(sl->bv_chunk, K - k0);
      CUDA_TRY(ctx, launch_slam_bv_items(sl->x, sl->phi, P, K, k0, B, J, S, sl->bpos, sl->bjs, sl->bsfv, stm));
      CUDA_TRY(ctx, launch_response(sd1, sl->bpos, (int64_t)B * J * S, sl->bjs, sl->bsfv, sl->psi, CDMS_FP64,
                                    ctx->d_flags, stm, 1));
      CUDA_TRY(ctx, launch_slam_bv_accum(sl->psi, sl->mu, sl->gam, sl->w, sl->wk, sl->par, P, K, k0, B, J, S, Nz,
                                         sl->au, sl->am, sl->aw, stm));
      ctx->launches += 3;
    }
    CUDA_TRY(ctx, launch_slam_bv_final(sl->am, sl->au, sl->par, J, S, Nz, sl->m64, sl->munu, stm));
    ctx->launches += 2;
  }
  // ---- (iii) update messages from the same prediction messages (flooding)
  // iota~: the MT likelihood with the moment-matched amplitude priors (C-amb-7) and the paired SFVs (C-amb-8)
  {
    cdms_scene sK = sl->scene;
    sK.K = S - 1;
    cdms_prior pr[MAXJ * MAXS];
    for (int j = 0; j < J; ++j)
      for (int i = 0; i < S; ++i) {
        const double ex = std::min(1.0, std::max(0.0, eps[i] * zeta_pr[i][j]));
        if (cdms_moment_match(mub[i][0], mub[i][1], gab[i], ex, &pr[j * S + i]))
          return fail(ctx, CDMS_EINVAL, "slam_step: moment matching of slot %d", i);
      }
    CUDA_TRY(ctx, launch_slam_sfv_pp(sl->phi, P, S - 1, sl->sfvpp, stm));
    if ((st = cdms_loglik(ctx, &sK, sl->x, P, 6, sl->sfvpp, 1, d_y, sl->f_pb.data(), pr, eta_bar, nullptr, sl->l,
                          nullptr)))
      return st;
  }
  // nu~ with every slot's column
  if ((st = cdms_noise_update(ctx, &sl->scene, sl->eta, sl->wxi, P, d_y, sl->munu, sl->m64, S, sl->logweta, sl->weta,
                              sl->lnorm)))
    return st;
  // kappa~ and omega~ of every slot with the other slots' terms
  cdms_scene s32 = sl->scene;
  s32.precision = CDMS_FP32;
  for (int i = 0; i < S; ++i) {
    CUDA_TRY(ctx, launch_slam_others(sl->au, sl->am, sl->aw, sl->par, J, S, Nz, i, sl->mu3o, sl->mo, sl->mws, sl->us,
                                     stm));
    ctx->launches += 1;
    if ((st = cdms_pf_update(ctx, &s32, sl->f_pb.data(), sl->x, P, 6, i ? slot_phi(sl, i) : nullptr, slot_w(sl, i),
                             slot_mu(sl, i), slot_gam(sl, i), zeta_pr[i], eta_bar, d_y, sl->mu3o, sl->mo, S - 1,
                             sl->logr + (size_t)i * P, sl->wnew + (size_t)i * P, sl->pfout + 2 * i)))
      return st;
    if ((st = cdms_ppr_update(ctx, &sl->scene, zeta_pr[i], eta_bar, d_y, sl->mu3o, sl->mo, S - 1, sl->mws, sl->us,
                              sl->pprout + (size_t)3 * MAXJ * i)))
      return st;
  }
  // ---- beliefs: MT (normalize, estimate, resample, regularize; rows A6-A9)
  cdms_step_params sp{};
  sp.T = q.T;
  sp.sigma_v = q.sigma_v;
  sp.philox_key = q.key;
  sp.step = n;
  sp.regularize = q.regularize;
  if ((st = cdms_bp_update(ctx, sl->l, sl->x, P, &sp, sl->est, sl->lse, nullptr))) return st;
  // posterior statistics of the PFs (weights wnew) and eta-hat (weights w_eta)
  SlamWsumJobs jp{};
  slot_jobs(sl, jp, 0, S, sl->wnew, true);
  for (int j = 0; j < J; ++j)
    jp.job[jp.n++] = SlamWsumJob{sl->weta + (size_t)j * P, sl->eta + (size_t)j * P, P, 1, 1};
  CUDA_TRY(ctx, launch_slam_wsum(jp, sl->wpart, sl->stats, stm));
  double hs[4 * SLAM_MAXJOBS], pfo[SLS * 2], ppo[SLS * MAXJ * 3], est[28], lse;
  CUDA_TRY(ctx, cudaMemcpyAsync(hs, sl->stats, sizeof(double) * 4 * jp.n, cudaMemcpyDeviceToHost, stm));
  CUDA_TRY(ctx, cudaMemcpyAsync(pfo, sl->pfout, sizeof(double) * 2 * S, cudaMemcpyDeviceToHost, stm));
  CUDA_TRY(ctx, cudaMemcpyAsync(ppo, sl->pprout, sizeof(double) * 3 * MAXJ * S, cudaMemcpyDeviceToHost, stm));
  CUDA_TRY(ctx, cudaMemcpyAsync(est, sl->est, sizeof(est), cudaMemcpyDeviceToHost, stm));
  CUDA_TRY(ctx, cudaMemcpyAsync(&lse, sl->lse, sizeof(double), cudaMemcpyDeviceToHost, stm));
  ctx->launches += 2;
  if ((st = cdms_sync(ctx))) return st;
  // ---- estimates, declaration, pruning; resampling of the kept PFs and of the noise
  cdms_slam_report r{};
  r.n = (int64_t)n;
  r.n_feat = S;
  int kept = 0;
  int new_ident[SLS];
  double new_zeta[SLS][MAXJ], new_phi_hat[SLS][3];
  for (int i = 0; i < S; ++i) {
    const double ex = pfo[2 * i + 1];
    const int b = 3 * i;
    const double e = hs[4 * b] > 0.0 ? hs[4 * b] : 1.0;
    r.ident[i] = sl->ident[i];
    r.exist[i] = ex;
    r.mu_hat[i][0] = hs[4 * b + 1] / e;
    r.mu_hat[i][1] = hs[4 * b + 2] / e;
    r.gamma_hat[i] = hs[4 * (b + 1) + 1] / e;
    for (int c = 0; c < 3; ++c) r.phi_hat[i][c] = i ? hs[4 * (b + 2) + 1 + c] / e : 0.0;
    for (int j = 0; j < J; ++j) r.zeta[i][j] = ppo[(size_t)3 * MAXJ * i + 3 * j + 2];
    r.declared[i] = ex > q.T_dec;
    r.pruned[i] = (i > 0 && ex < q.T_pru) ? 1 : 0;
    if (r.pruned[i]) continue;
    const int d = kept++;
    if (ex > 0.0) {
      const uint32_t u = host_philox_word0(q.key, 0, n, 0x400u + (uint32_t)i);
      if ((st = cdms_resample(ctx, sl->wnew + (size_t)i * P, P, u, sl->anc))) return st;
      CUDA_TRY(ctx, launch_slam_pf_gather(i ? slot_phi(sl, i) : nullptr, slot_mu(sl, i), slot_gam(sl, i), sl->anc, P,
                                          sl->tphi, sl->tmu, sl->tgam, stm));
      if (i && q.regularize) {  // SFV regularization (reading F4k): h for d = 3, the posterior's Sigma
        const double h = pow(4.0 / (5.0 * (double)P), 1.0 / 7.0);
        CUDA_TRY(ctx, launch_slam_sfv_reg(sl->wnew + (size_t)i * P, slot_phi(sl, i), sl->tphi, P, r.phi_hat[i], h,
                                          sl->bout, sl->wpart, q.key, n, i, stm));
        ctx->launches += 3;
      }
      if (i)
        CUDA_TRY(ctx, cudaMemcpyAsync(slot_phi(sl, d), sl->tphi, sizeof(double) * P * 3, cudaMemcpyDeviceToDevice,
                                      stm));
      CUDA_TRY(ctx, cudaMemcpyAsync(slot_mu(sl, d), sl->tmu, sizeof(double2) * P, cudaMemcpyDeviceToDevice, stm));
      CUDA_TRY(ctx, cudaMemcpyAsync(slot_gam(sl, d), sl->tgam, sizeof(double) * P, cudaMemcpyDeviceToDevice, stm));
      CUDA_TRY(ctx, launch_slam_fill(slot_w(sl, d), P, ex / (double)P, stm));
      ctx->launches += 2;
    } else if (d != i) {
      return fail(ctx, CDMS_EZEROMASS, "slam_step: the LOS PF lost all mass");
    }
    new_ident[d] = sl->ident[i];
    for (int j = 0; j < J; ++j) new_zeta[d][j] = r.zeta[i][j];
    for (int c = 0; c < 3; ++c) new_phi_hat[d][c] = r.phi_hat[i][c];
  }
  for (int j = 0; j < J; ++j) {
    const int b = 3 * S + j;
    r.eta_hat[j] = hs[4 * b + 1] / (hs[4 * b] > 0.0 ? hs[4 * b] : 1.0);
    r.eta_bar[j] = eta_bar[j];
    const uint32_t u = host_philox_word0(q.key, 0, n, 0x500u + (uint32_t)j);
    if ((st = cdms_resample(ctx, sl->weta + (size_t)j * P, P, u, sl->anc))) return st;
    CUDA_TRY(ctx, launch_slam_gather1(sl->eta + (size_t)j * P, sl->anc, P, sl->teta, stm));
    CUDA_TRY(ctx, cudaMemcpyAsync(sl->eta + (size_t)j * P, sl->teta, sizeof(double) * P, cudaMemcpyDeviceToDevice,
                                  stm));
    ctx->launches += 1;
  }
  sl->n_slots = kept;
  for (int i = 0; i < kept; ++i) {
    sl->ident[i] = new_ident[i];
    for (int j = 0; j < J; ++j) sl->zeta[i][j] = new_zeta[i][j];
    for (int c = 0; c < 3; ++c) sl->phi_hat[i][c] = new_phi_hat[i][c];
  }
  sl->n = (int64_t)n + 1;
  r.n_slots = kept;
  for (int c = 0; c < 28; ++c) r.est[c] = est[c];
  r.lse = lse;
  for (int c = 0; c < 3; ++c) r.x_pred_hat[c] = x_hat[c];
  if (rep) *rep = r;
  return CDMS_OK;
}

}  // extern "C"
