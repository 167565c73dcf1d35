// step.cu -- the O(P) part of cdms_bp_step (rows A6-A9) as a fused pipeline of five kernels:
//   K_lse   per-block (max l, sum e^{l - max}); the last block to finish reduces the partials in a fixed
//           order and, without a communicator, combines them into (M, ln S, lse)
//   K_post  one pass over the particles: w = e^{(l - M) - ln S}, q = rint(ldexp(e^{l - M}, 36)) (C-amb-15, 23),
//           first-moment partials [sum w, sum w x]; block sums of q.  Last block: the fixed-order moment sum
//           and the exclusive scan of the block sums of q
//   K_scan  inclusive scan C of q (block offset + local scan); second-moment partials sum w (x - mu)(x - mu)^T.
//           Last block (no communicator): est and the Cholesky factor of its covariance (C-amb-16)
//   K_anc   per output slot: ancestor = min{p : C_p > t_i} with the exact 128-bit t_i, gather of the state
//
//   K_reg   x = staged state + h chol(Sigma) n (Philox streams 1, 2), or a plain copy
// Block partitions are fixed (STEP_ITEMS particles per block) and every cross-block reduction runs in a fixed
// order in the last block, so results depend only on P, never on scheduling.  With a communicator the host
// inserts the NCCL collectives between the kernels and runs the same combine / finalize device code.
#include <math.h>

#include <cooperative_groups.h>

#include "cdms_internal.h"

namespace cg = cooperative_groups;

namespace cdms {

constexpr int STEP_BLOCK = 256;
constexpr int STEP_PER = STEP_ITEMS / STEP_BLOCK;  // contiguous particles per thread
static_assert(STEP_ITEMS % STEP_BLOCK == 0, "STEP_ITEMS");

int64_t step_blocks(int64_t P) { return P <= 0 ? 0 : (P + STEP_ITEMS - 1) / STEP_ITEMS; }

// ---------------------------------------------------------------------------- helpers
// Fixed-order block sum of N doubles per thread: warp tree by shuffles, then the 8 warp results in order.
template <int N>
__device__ __forceinline__ void block_sum(double (&v)[N], double* sh /* [8][N] */, double* out /* [N] */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < N; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < N; ++k) sh[warp * N + k] = v[k];
  }
  __syncthreads();
  if ((int)threadIdx.x < N) {
    double s = 0.0;
    for (int w = 0; w < STEP_BLOCK / 32; ++w) s += sh[w * N + threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

// Arrive on the grid-wide counter; true in the last block to arrive (which then owns the fixed-order
// cross-block reduction and resets the counter for the next launch).
__device__ __forceinline__ bool last_block(unsigned* cnt) {
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) am_last = atomicAdd(cnt, 1u) == gridDim.x - 1;
  __syncthreads();
  if (am_last) {
    __threadfence();
    if (threadIdx.x == 0) *cnt = 0u;
  }
  return am_last;
}

// Column sums of part[nb][N]: G = STEP_BLOCK / N threads per column, thread g sums rows g, g + G, ... ascending
// (four independent loads in flight), then one thread per column adds the G partials in order -- deterministic.
// out is visible to the block after the trailing __syncthreads.  (One warp per column with one dependent L2 load
// per step made the single-block epilogues the longest serial part of the step.)
template <int N>
__device__ void sum_columns(const double* part, int64_t nb, double* out) {
  constexpr int G = STEP_BLOCK / N;
  __shared__ double red[STEP_BLOCK];
  const int c = threadIdx.x / G, g = threadIdx.x - c * G;
  double s = 0.0;
  if (c < N) {
    int64_t b = g;
    for (; b + 3 * G < nb; b += 4 * G) {
      const double v0 = __ldcg(&part[b * N + c]), v1 = __ldcg(&part[(b + G) * N + c]);
      const double v2 = __ldcg(&part[(b + 2 * G) * N + c]), v3 = __ldcg(&part[(b + 3 * G) * N + c]);
      s += v0;
      s += v1;
      s += v2;
      s += v3;
    }
    for (; b < nb; b += G) s += __ldcg(&part[b * N + c]);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  if ((int)threadIdx.x < N) {
    double tot = 0.0;
    for (int k = 0; k < G; ++k) tot += red[threadIdx.x * G + k];
    out[threadIdx.x] = tot;
  }
  __syncthreads();
}

// Ranks' (M_r, S_r) in rank order -> lse, M, ln S, flags (the same code with and without a communicator)
__device__ void lse_combine_dev(const double2* per_rank, int nranks, double* lse, double* Mout, double* logS,
                                int* flags) {
  double M = -INFINITY;
  bool nan = false;
  for (int r = 0; r < nranks; ++r) {
    nan |= !(per_rank[r].x == per_rank[r].x) || !(per_rank[r].y == per_rank[r].y);
    M = fmax(M, per_rank[r].x);
  }
  double S = 0.0;
  if (M > -INFINITY)
    for (int r = 0; r < nranks; ++r)
      if (per_rank[r].x > -INFINITY) S += per_rank[r].y * exp(per_rank[r].x - M);
  if (nan) {
    atomicOr(flags, FLAG_NAN);
    *lse = NAN;
  } else if (!(M > -INFINITY) || !(S > 0.0)) {
    atomicOr(flags, FLAG_ZEROMASS);
    *lse = -INFINITY;
  } else {
    *lse = M + log(S);
  }
  *Mout = M;
  *logS = (S > 0.0) ? log(S) : -INFINITY;
}

// est = [sum w, mean (6), covariance upper triangle (21)] and L = chol(Sigma + 1e-12 tr(Sigma) I), run by one
// full warp: lanes 0..27 form est in parallel, lane 0 then factors the 6 x 6 covariance (one reciprocal per
// pivot).  The same code serves the single-rank kernel epilogue and the multi-rank finalize kernel.
__device__ void finalize_dev(const double* sum1, const double* sum2, double* est, double* L, int* flags) {
  const int lane = threadIdx.x & 31;
  const double sw = sum1[0];
  if (lane == 0 && !(sw > 0.0)) atomicOr(flags, FLAG_ZEROMASS);
  if (lane < 28) est[lane] = lane == 0 ? sw : (lane < 7 ? sum1[lane] : sum2[lane - 7]) / sw;
  __syncwarp();
  if (L == nullptr || lane != 0) return;
  // fully unrolled with compile-time indices: the 6 x 6 factors stay in registers (a rolled version lived in
  // local memory on the single thread that runs it)
  double Sg[36];
#pragma unroll
  for (int a = 0; a < 6; ++a)
#pragma unroll
    for (int b = 0; b < 6; ++b) {
      if (b < a) continue;
      const int t = a * 6 - a * (a - 1) / 2 + (b - a);  // upper-triangle index, row-major
      Sg[a * 6 + b] = est[7 + t];
      Sg[b * 6 + a] = est[7 + t];
    }
  double tr = 0.0;
#pragma unroll
  for (int a = 0; a < 6; ++a) tr += Sg[a * 6 + a];
#pragma unroll
  for (int a = 0; a < 6; ++a) Sg[a * 6 + a] += 1e-12 * tr;
  double Lr[36];
#pragma unroll
  for (int i = 0; i < 36; ++i) Lr[i] = 0.0;
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    double d = Sg[j * 6 + j];
#pragma unroll
    for (int k = 0; k < 6; ++k)
      if (k < j) d -= Lr[j * 6 + k] * Lr[j * 6 + k];
    const bool ok = d > 0.0;
    const double lj = ok ? sqrt(d) : 0.0;
    const double inv = ok ? 1.0 / lj : 0.0;
    Lr[j * 6 + j] = lj;
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      if (i <= j) continue;
      double acc = Sg[i * 6 + j];
#pragma unroll
      for (int k = 0; k < 6; ++k)
        if (k < j) acc -= Lr[i * 6 + k] * Lr[j * 6 + k];
      Lr[i * 6 + j] = ok ? acc * inv : 0.0;
    }
  }
#pragma unroll
  for (int i = 0; i < 36; ++i) L[i] = Lr[i];
}

// ---------------------------------------------------------------------------- K_lse
// Each phase is a per-block body of virtual block vb (STEP_ITEMS particles) and a cross-block epilogue; the
// separate kernels run the epilogue in the last block to arrive, the fused single-rank kernel (below) in block 0
// after a grid barrier -- the same code either way, so results are identical.  Data written by other blocks in
// the same launch is read with __ldcg (L2), never through the non-coherent path.
__device__ void lse_block(int64_t vb, const double* l, int64_t P, double2* part) {
  __shared__ double sh[STEP_BLOCK];
  const int64_t base = vb * STEP_ITEMS + threadIdx.x * STEP_PER;
  double v[STEP_PER];
  double m = -INFINITY;
#pragma unroll
  for (int i = 0; i < STEP_PER; ++i) {
    v[i] = (base + i < P) ? l[base + i] : -INFINITY;
    m = fmax(m, v[i]);
  }
  sh[threadIdx.x] = m;
  __syncthreads();
  for (int o = STEP_BLOCK / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  const double Mb = sh[0];
  __syncthreads();
  double s = 0.0;
  if (Mb > -INFINITY) {
#pragma unroll
    for (int i = 0; i < STEP_PER; ++i)
      if (base + i < P) s += exp(v[i] - Mb);
  }
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = STEP_BLOCK / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[vb] = make_double2(Mb, sh[0]);
  __syncthreads();
}
__device__ void lse_final(int64_t nb, const double2* part, double2* rank_pair, int combine, double* lse, double* M,
                          double* logS, int* flags) {
  __shared__ double sh[STEP_BLOCK];
  // fixed-order combine of the block partials -> this rank's (M_r, S_r)
  double mm = -INFINITY;
  for (int64_t b = threadIdx.x; b < nb; b += STEP_BLOCK) mm = fmax(mm, __ldcg(&part[b].x));
  sh[threadIdx.x] = mm;
  __syncthreads();
  for (int o = STEP_BLOCK / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  const double Mr = sh[0];
  __syncthreads();
  double ss = 0.0;
  if (Mr > -INFINITY)
    for (int64_t b = threadIdx.x; b < nb; b += STEP_BLOCK) {
      const double2 q = __ldcg(&part[b]);
      if (q.x > -INFINITY) ss += q.y * exp(q.x - Mr);
    }
  sh[threadIdx.x] = ss;
  __syncthreads();
  for (int o = STEP_BLOCK / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *rank_pair = make_double2(Mr, sh[0]);
    if (combine) lse_combine_dev(rank_pair, 1, lse, M, logS, flags);
  }
  __syncthreads();
}
__global__ void __launch_bounds__(STEP_BLOCK) step_lse_kernel(const double* __restrict__ l, int64_t P,
                                                             double2* __restrict__ part, unsigned* cnt,
                                                             double2* rank_pair, int combine, double* lse,
                                                             double* M, double* logS, int* flags) {
  lse_block(blockIdx.x, l, P, part);
  if (rank_pair == nullptr || !last_block(cnt)) return;  // multi-rank: the block partials are all-gathered instead
  lse_final(gridDim.x, part, rank_pair, combine, lse, M, logS, flags);
}
// Multi-rank: the same fixed-order combine over the all-gathered block partials of every rank (rank-major), so with
// block-aligned shards (P_local a multiple of STEP_ITEMS) it reduces exactly the partials a single rank holding all
// particles would, in the same order -- M, ln S and lse are bit-identical for any rank count.
__global__ void __launch_bounds__(STEP_BLOCK) step_lse_global_kernel(const double2* gpart, int64_t nbt,
                                                                    double2* rank_pair, double* lse, double* M,
                                                                    double* logS, int* flags) {
  lse_final(nbt, gpart, rank_pair, 1, lse, M, logS, flags);
}


// ---------------------------------------------------------------------------- K_post
__device__ void post_block(int64_t vb, const double* l, const double* x, int64_t P, const double* Mp,
                           const double* logSp, const int* flags, double* w, uint64_t* q, double* mpart,
                           uint64_t* bsum) {
  __shared__ double sh[STEP_BLOCK * 4];
  __shared__ double red[8];
  __shared__ uint64_t shq[STEP_BLOCK];
  const bool bad = (__ldcg(flags) & (FLAG_ZEROMASS | FLAG_NAN)) != 0;
  const double M = __ldcg(Mp), ls = __ldcg(logSp);
  const int64_t base = vb * STEP_ITEMS + threadIdx.x * STEP_PER;
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  uint64_t qs = 0;
#pragma unroll
  for (int i = 0; i < STEP_PER; ++i) {
    const int64_t p = base + i;
    if (p >= P) continue;
    const double d = l[p] - M;
    const double wp = exp(d - ls);
    if (!bad) w[p] = wp;
    double r = exp(d);
    if (!(r >= 0.0)) r = 0.0;
    const uint64_t qp = (uint64_t)rint(scalbn(r, 36));
    q[p] = qp;
    qs += qp;
    const double wa = bad ? 0.0 : wp;
    acc[0] += wa;
#pragma unroll
    for (int a = 0; a < 6; ++a) acc[1 + a] += wa * x[p * 6 + a];
  }
  block_sum<7>(acc, sh, red);
  if (threadIdx.x < 7) mpart[vb * 7 + threadIdx.x] = red[threadIdx.x];
  // block total of q (exact)
  shq[threadIdx.x] = qs;
  __syncthreads();
  for (int o = STEP_BLOCK / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) shq[threadIdx.x] += shq[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) bsum[vb] = shq[0];
  __syncthreads();
}
__device__ void post_final(int64_t nb, const double* mpart, uint64_t* bsum, double* sum1, int64_t P, uint32_t u_bits,
                           uint64_t* plan) {
  __shared__ uint64_t shq[STEP_BLOCK];
  if (sum1) sum_columns<7>(mpart, nb, sum1);
  // exclusive scan of the block totals in place; bsum[nb] = Q (this rank)
  const int64_t chunk = (nb + STEP_BLOCK - 1) / STEP_BLOCK;
  const int64_t b0 = threadIdx.x * chunk, b1 = min(nb, b0 + chunk);
  uint64_t run = 0;
  for (int64_t b = b0; b < b1; ++b) run += __ldcg(&bsum[b]);
  shq[threadIdx.x] = run;
  __syncthreads();
  for (int off = 1; off < STEP_BLOCK; off <<= 1) {  // Hillis-Steele inclusive scan of the thread totals
    const uint64_t add = ((int)threadIdx.x >= off) ? shq[threadIdx.x - off] : 0ull;
    __syncthreads();
    shq[threadIdx.x] += add;
    __syncthreads();
  }
  uint64_t ex = (threadIdx.x > 0) ? shq[threadIdx.x - 1] : 0ull;
  for (int64_t b = b0; b < b1; ++b) {
    const uint64_t v = __ldcg(&bsum[b]);
    bsum[b] = ex;
    ex += v;
  }
  if (threadIdx.x == STEP_BLOCK - 1) {
    bsum[nb] = shq[STEP_BLOCK - 1];
    if (plan) plan_dev(&shq[STEP_BLOCK - 1], 1, 0, P, u_bits, plan);  // single rank: slots [0, P)
  }
  __syncthreads();
}
// sum1 == nullptr (multi-rank): the last block only scans the local block totals; the moment sums follow from the
// all-gathered block partials (step_post_global_kernel)
__global__ void __launch_bounds__(STEP_BLOCK) step_post_kernel(const double* l, const double* x, int64_t P,
                                                              const double* Mp, const double* logSp, const int* flags,
                                                              double* w, uint64_t* q, double* mpart, uint64_t* bsum,
                                                              unsigned* cnt, double* sum1, uint32_t u_bits,
                                                              uint64_t* plan) {
  post_block(blockIdx.x, l, x, P, Mp, logSp, flags, w, q, mpart, bsum);
  if (!last_block(cnt)) return;
  post_final(gridDim.x, mpart, bsum, sum1, P, u_bits, plan);
}
// Multi-rank: first moments over every rank's block partials (fixed order, as a single rank would) and the plan of
// this rank from the all-gathered masses Q_r.
__global__ void __launch_bounds__(STEP_BLOCK) step_post_global_kernel(const double* gmpart, int64_t nbt, double* sum1,
                                                                     const uint64_t* Qall, int nranks, int rank,
                                                                     int64_t P_total, uint32_t u_bits, uint64_t* plan) {
  sum_columns<7>(gmpart, nbt, sum1);
  if (threadIdx.x == 0) plan_dev(Qall, nranks, rank, P_total, u_bits, plan);
}

// ---------------------------------------------------------------------------- K_scan
__device__ void scan_block(int64_t vb, uint64_t* q, const double* x, const double* w, int64_t P, const uint64_t* boff,
                           const double* sum1, const int* flags, double* mpart) {
  __shared__ double sh[STEP_BLOCK * 21 / 8 + 32];
  __shared__ double red[24];
  __shared__ uint64_t shq[STEP_BLOCK];
  const bool bad = (__ldcg(flags) & (FLAG_ZEROMASS | FLAG_NAN)) != 0;
  const int64_t base = vb * STEP_ITEMS + threadIdx.x * STEP_PER;
  // inclusive scan: thread-contiguous runs, Hillis-Steele over the thread totals, + block offset
  uint64_t v[STEP_PER];
  uint64_t run = 0;
#pragma unroll
  for (int i = 0; i < STEP_PER; ++i) {
    run += (base + i < P) ? q[base + i] : 0ull;
    v[i] = run;
  }
  shq[threadIdx.x] = run;
  __syncthreads();
  for (int off = 1; off < STEP_BLOCK; off <<= 1) {
    const uint64_t add = ((int)threadIdx.x >= off) ? shq[threadIdx.x - off] : 0ull;
    __syncthreads();
    shq[threadIdx.x] += add;
    __syncthreads();
  }
  const uint64_t ex = ((threadIdx.x > 0) ? shq[threadIdx.x - 1] : 0ull) + __ldcg(&boff[vb]);
#pragma unroll
  for (int i = 0; i < STEP_PER; ++i)
    if (base + i < P) q[base + i] = v[i] + ex;
  // second moments about the global mean
  double mu[6];
#pragma unroll
  for (int a = 0; a < 6; ++a) mu[a] = __ldcg(&sum1[1 + a]) / __ldcg(&sum1[0]);
  double acc[21];
#pragma unroll
  for (int t = 0; t < 21; ++t) acc[t] = 0.0;
#pragma unroll
  for (int i = 0; i < STEP_PER; ++i) {
    const int64_t p = base + i;
    if (p >= P || bad) continue;
    const double wp = w[p];
    double d[6];
#pragma unroll
    for (int a = 0; a < 6; ++a) d[a] = x[p * 6 + a] - mu[a];
    int t = 0;
#pragma unroll
    for (int a = 0; a < 6; ++a)
#pragma unroll
      for (int b = a; b < 6; ++b) acc[t++] += wp * d[a] * d[b];
  }
  block_sum<21>(acc, sh, red);
  if (threadIdx.x < 21) mpart[vb * 21 + threadIdx.x] = red[threadIdx.x];
  __syncthreads();
}
__device__ void scan_final(int64_t nb, const double* mpart, double* sum2, int finalize, const double* sum1,
                           double* est, double* L, int* flags_w) {
  sum_columns<21>(mpart, nb, sum2);
  if (finalize && threadIdx.x < 32) finalize_dev(sum1, sum2, est, L, flags_w);  // warp 0
  __syncthreads();
}
__global__ void __launch_bounds__(STEP_BLOCK) step_scan_kernel(uint64_t* q, const double* x, const double* w,
                                                              int64_t P, const uint64_t* boff, const double* sum1,
                                                              const int* flags, double* mpart, unsigned* cnt,
                                                              double* sum2, int finalize, double* est, double* L,
                                                              int* flags_w) {
  scan_block(blockIdx.x, q, x, w, P, boff, sum1, flags, mpart);
  if (sum2 == nullptr || !last_block(cnt)) return;  // multi-rank: partials all-gathered, step_scan_global_kernel
  scan_final(gridDim.x, mpart, sum2, finalize, sum1, est, L, flags_w);
}
__global__ void __launch_bounds__(STEP_BLOCK) step_scan_global_kernel(const double* gmpart, int64_t nbt,
                                                                     const double* sum1, double* sum2, double* est,
                                                                     double* L, int* flags) {
  scan_final(nbt, gmpart, sum2, 1, sum1, est, L, flags);
}


// ---------------------------------------------------------------------------- K_anc (+ gather)
// Output slot g in this rank's range [slot_lo, slot_hi) (plan, written on the device: no host round trip):
// t_g = floor((u + g 2^32) Q / (P_total 2^32)); ancestor = min{p : C_p > t_g - O_r} (local index lo, global
// p_global0 + lo); the state x[lo] goes to row g mod P_local of the stage buffer of the slot's owner rank
// g / P_local -- written directly into that rank's memory (peer_x[owner]: its own buffer on one rank, NVLink peer
// memory (CUDA IPC) under NCCL, another context's buffer for the loopback test backend), so the redistribution of
// DESIGN.md section 9 is fused into the gather instead of a separate send/recv round.  Grid-stride over the slots.
// Two-level search when the rank has at most ANC_SMEM blocks: the block ends E_b = boff[b + 1] (boff[nb] = this
// rank's total) in shared memory give the block holding the ancestor (C is non-decreasing, so it is the first block
// whose last C exceeds t), then 9 steps inside its STEP_ITEMS entries; above ANC_SMEM blocks every ANC_SUP-th block
// end is staged (three-level search).
constexpr int ANC_SMEM = 2048;
__device__ void anc_range(int64_t i0, int64_t stride, const uint64_t* C, const uint64_t* boff, int64_t nb,
                          int64_t P_local, const uint64_t* plan, int64_t P_total, uint32_t u_bits, const double* x,
                          double* own_x, int64_t* own_anc, double* const* peer_x, int64_t* const* peer_anc,
                          int64_t p_global0, int* flags) {
  __shared__ uint64_t sE[ANC_SMEM];
  const int64_t sup = (nb + ANC_SMEM - 1) / ANC_SMEM;  // blocks per staged end (1: every block end)
  const int64_t ns = (nb + sup - 1) / sup;
  for (int64_t b = threadIdx.x; b < ns; b += blockDim.x) sE[b] = __ldcg(&boff[min(nb, (b + 1) * sup)]);
  __syncthreads();
  const uint64_t Q = __ldcg(&plan[0]), O = __ldcg(&plan[1]);
  const int64_t slot_lo = (int64_t)__ldcg(&plan[2]), n = (int64_t)__ldcg(&plan[3]) - slot_lo;
  if (Q == 0) {
    if (i0 == 0) atomicOr(flags, FLAG_ZEROMASS);
    return;
  }
  const unsigned __int128 den = (unsigned __int128)(uint64_t)P_total << 32;
  for (int64_t i = i0; i < n; i += stride) {
    const uint64_t g = (uint64_t)(slot_lo + i);
    const unsigned __int128 num = ((unsigned __int128)u_bits + ((unsigned __int128)g << 32)) * Q;
    const uint64_t t = (uint64_t)(num / den) - O;
    int64_t bl = 0, bh = ns - 1;  // smallest staged group with end > t
    while (bl < bh) {
      const int64_t mid = (bl + bh) >> 1;
      if (sE[mid] > t) bh = mid; else bl = mid + 1;
    }
    int64_t b0 = bl * sup, b1 = min(nb, b0 + sup) - 1;  // then the block inside the group (sup > 1 only)
    while (b0 < b1) {
      const int64_t mid = (b0 + b1) >> 1;
      if (__ldcg(&boff[mid + 1]) > t) b1 = mid; else b0 = mid + 1;
    }
    int64_t lo = b0 * STEP_ITEMS, hi = min(P_local, lo + STEP_ITEMS) - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldcg(&C[mid]) > t) hi = mid; else lo = mid + 1;
    }
    const int64_t own = (int64_t)(g / (uint64_t)P_local), row = (int64_t)g - own * P_local;
    int64_t* da = peer_x ? (peer_anc ? peer_anc[own] : nullptr) : own_anc;  // peer_x == nullptr: one rank
    if (da) da[row] = p_global0 + lo;
    const double2* src = reinterpret_cast<const double2*>(x + lo * 6);
    double2* dst = reinterpret_cast<double2*>((peer_x ? peer_x[own] : own_x) + row * 6);
    dst[0] = src[0];
    dst[1] = src[1];
    dst[2] = src[2];
  }
  __threadfence_system();  // peer writes ordered before the barrier collective that follows the kernel
}
__global__ void step_anc_kernel(const uint64_t* C, const uint64_t* boff, int64_t nb, int64_t P_local,
                                const uint64_t* plan, int64_t P_total, uint32_t u_bits, const double* x, double* own_x,
                                int64_t* own_anc, double* const* peer_x, int64_t* const* peer_anc, int64_t p_global0,
                                int* flags) {
  anc_range((int64_t)blockIdx.x * blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x, C, boff, nb, P_local,
            plan, P_total, u_bits, x, own_x, own_anc, peer_x, peer_anc, p_global0, flags);
}

// ---------------------------------------------------------------------------- K_reg
// Philox4x32-10 and Box-Muller exactly as beliefs.cu (streams 1, 2 of the global slot index).
__device__ __forceinline__ void normals4_step(uint64_t key, uint64_t step, uint64_t index, uint32_t stream,
                                              double n[4]) {
  const uint4 x = philox_step(make_uint4((uint32_t)index, (uint32_t)(index >> 32), (uint32_t)step, stream),
                              make_uint2((uint32_t)key, (uint32_t)(key >> 32)));
  const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const double ua = ((double)xs[2 * h] + 0.5) * 0x1p-32;
    const double ub = ((double)xs[2 * h + 1] + 0.5) * 0x1p-32;
    const double r = sqrt(-2.0 * log(ua));
    n[2 * h] = r * cos(2.0 * PI * ub);
    n[2 * h + 1] = r * sin(2.0 * PI * ub);
  }
}

// out[p] = in[p] + h L n_p (regularize) or in[p]; in may equal out
__device__ void reg_range(int64_t i0, int64_t stride, const double* in, double* out, int64_t P, int64_t p0, double h,
                          const double* Lg, int regularize, uint64_t key, uint64_t step) {
  __shared__ double L[36];
  if (threadIdx.x < 36) L[threadIdx.x] = regularize ? __ldcg(&Lg[threadIdx.x]) : 0.0;
  __syncthreads();
  for (int64_t p = i0; p < P; p += stride) {
    double s[6];
#pragma unroll
    for (int a = 0; a < 6; ++a) s[a] = __ldcg(&in[p * 6 + a]);
    if (regularize) {
      double n[8];
      normals4_step(key, step, (uint64_t)(p0 + p), 1u, n);
      normals4_step(key, step, (uint64_t)(p0 + p), 2u, n + 4);
#pragma unroll
      for (int a = 0; a < 6; ++a) {
        double acc = 0.0;
#pragma unroll
        for (int b = 0; b <= a; ++b) acc += L[a * 6 + b] * n[b];
        s[a] += h * acc;
      }
    }
#pragma unroll
    for (int a = 0; a < 6; ++a) out[p * 6 + a] = s[a];
  }
}
__global__ void step_reg_kernel(const double* in, double* out, int64_t P, int64_t p0, double h, const double* Lg,
                                int regularize, uint64_t key, uint64_t step) {
  reg_range((int64_t)blockIdx.x * blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x, in, out, P, p0, h, Lg,
            regularize, key, step);
}

// ---------------------------------------------------------------------------- fused single-rank pipeline
// All five phases in one cooperative launch (no communicator): the per-block bodies over virtual blocks, block 0
// runs each cross-block epilogue between grid barriers.  Tried because the kernels above are latency-bound
// (196-391 blocks, 17-30% warps active, 8-17 us each at P = 1e5); measured not faster (c2 step 0.409 vs 0.403 ms:
// 7 grid barriers and the serial epilogues cost what the launches did), so it is an A/B option (CDMS_STEP_FUSED=1),
// tested bit-identical to the separate kernels.
__global__ void __launch_bounds__(STEP_BLOCK) step_fused_kernel(StepFusedArgs a) {
  cg::grid_group grid = cg::this_grid();
  const int64_t nb = (a.P + STEP_ITEMS - 1) / STEP_ITEMS;  // step_blocks(P)
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t vb = blockIdx.x; vb < nb; vb += gridDim.x) lse_block(vb, a.l, a.P, a.lpart);
  grid.sync();
  if (blockIdx.x == 0) lse_final(nb, a.lpart, a.rank_pair, 1, a.lse, a.M, a.logS, a.flags);
  grid.sync();
  for (int64_t vb = blockIdx.x; vb < nb; vb += gridDim.x)
    post_block(vb, a.l, a.x, a.P, a.M, a.logS, a.flags, a.w, a.q, a.mpart, a.bsum);
  grid.sync();
  if (blockIdx.x == 0) post_final(nb, a.mpart, a.bsum, a.sums, a.P, a.u_bits, a.plan);
  grid.sync();
  for (int64_t vb = blockIdx.x; vb < nb; vb += gridDim.x)
    scan_block(vb, a.q, a.x, a.w, a.P, a.bsum, a.sums, a.flags, a.mpart);
  grid.sync();
  if (blockIdx.x == 0) scan_final(nb, a.mpart, a.sums + 8, 1, a.sums, a.est, a.L, a.flags);
  grid.sync();
  anc_range(i0, stride, a.q, a.bsum, nb, a.P, a.plan, a.P, a.u_bits, a.x, a.stage, a.anc, nullptr, nullptr, 0,
            a.flags);
  grid.sync();
  reg_range(i0, stride, a.stage, a.x, a.P, 0, a.h, a.L, a.regularize, a.key, a.step);
}

// ---------------------------------------------------------------------------- launchers
static unsigned grid_cap(int64_t n, int threads, int cap = 8192) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

cudaError_t launch_step_lse(const double* l, int64_t P, double2* part, unsigned* cnt, double2* rank_pair, int combine,
                            double* lse, double* M, double* logS, int* flags, cudaStream_t st) {
  const int64_t nb = step_blocks(P);
  step_lse_kernel<<<(unsigned)nb, STEP_BLOCK, 0, st>>>(l, P, part, cnt, rank_pair, combine, lse, M, logS, flags);
  return cudaGetLastError();
}
cudaError_t launch_step_lse_global(const double2* gpart, int64_t nbt, double2* rank_pair, double* lse, double* M,
                                   double* logS, int* flags, cudaStream_t st) {
  step_lse_global_kernel<<<1, STEP_BLOCK, 0, st>>>(gpart, nbt, rank_pair, lse, M, logS, flags);
  return cudaGetLastError();
}
cudaError_t launch_step_post(const double* l, const double* x, int64_t P, const double* M, const double* logS,
                             const int* flags, double* w, uint64_t* q, double* mpart, uint64_t* bsum, unsigned* cnt,
                             double* sum1, uint32_t u_bits, uint64_t* plan, cudaStream_t st) {
  const int64_t nb = step_blocks(P);
  step_post_kernel<<<(unsigned)nb, STEP_BLOCK, 0, st>>>(l, x, P, M, logS, flags, w, q, mpart, bsum, cnt, sum1, u_bits,
                                                       plan);
  return cudaGetLastError();
}
cudaError_t launch_step_post_global(const double* gmpart, int64_t nbt, double* sum1, const uint64_t* Qall, int nranks,
                                    int rank, int64_t P_total, uint32_t u_bits, uint64_t* plan, cudaStream_t st) {
  step_post_global_kernel<<<1, STEP_BLOCK, 0, st>>>(gmpart, nbt, sum1, Qall, nranks, rank, P_total, u_bits, plan);
  return cudaGetLastError();
}
cudaError_t launch_step_scan(uint64_t* q, const double* x, const double* w, int64_t P, const uint64_t* boff,
                             const double* sum1, const int* flags, double* mpart, unsigned* cnt, double* sum2,
                             int finalize, double* est, double* L, int* flags_w, cudaStream_t st) {
  const int64_t nb = step_blocks(P);
  step_scan_kernel<<<(unsigned)nb, STEP_BLOCK, 0, st>>>(q, x, w, P, boff, sum1, flags, mpart, cnt, sum2, finalize, est,
                                                       L, flags_w);
  return cudaGetLastError();
}
cudaError_t launch_step_scan_global(const double* gmpart, int64_t nbt, const double* sum1, double* sum2, double* est,
                                    double* L, int* flags, cudaStream_t st) {
  step_scan_global_kernel<<<1, STEP_BLOCK, 0, st>>>(gmpart, nbt, sum1, sum2, est, L, flags);
  return cudaGetLastError();
}
// The plan's slot count is only known on the device: a fixed grid (enough for one slot per thread when the rank keeps
// its own P_local slots, grid-stride beyond) of threads reads it.
cudaError_t launch_step_anc(const uint64_t* C, const uint64_t* boff, int64_t P_local, const uint64_t* plan,
                            int64_t P_total, uint32_t u_bits, const double* x, double* own_x, int64_t* own_anc,
                            double* const* peer_x, int64_t* const* peer_anc, int64_t p_global0, int* flags,
                            cudaStream_t st) {
  step_anc_kernel<<<grid_cap(P_local, 256), 256, 0, st>>>(C, boff, step_blocks(P_local), P_local, plan, P_total,
                                                         u_bits, x, own_x, own_anc, peer_x, peer_anc, p_global0, flags);
  return cudaGetLastError();
}
__global__ void plan_kernel(const uint64_t* Qall, int nranks, int rank, int64_t P_total, uint32_t u_bits,
                            uint64_t* plan) {
  if (threadIdx.x == 0 && blockIdx.x == 0) plan_dev(Qall, nranks, rank, P_total, u_bits, plan);
}
cudaError_t launch_plan(const uint64_t* Qall, int nranks, int rank, int64_t P_total, uint32_t u_bits, uint64_t* plan,
                        cudaStream_t st) {
  plan_kernel<<<1, 32, 0, st>>>(Qall, nranks, rank, P_total, u_bits, plan);
  return cudaGetLastError();
}
cudaError_t launch_step_reg(const double* in, double* out, int64_t P, int64_t p0, int64_t P_total, const double* L,
                            int regularize, uint64_t key, uint64_t step, cudaStream_t st) {
  if (P <= 0) return cudaSuccess;
  const double h = step_reg_bandwidth(P_total);  // h_opt, d = 6 (C-amb-16)
  step_reg_kernel<<<grid_cap(P, 256), 256, 0, st>>>(in, out, P, p0, h, L, regularize, key, step);
  return cudaGetLastError();
}

cudaError_t launch_step_fused(const StepFusedArgs& a, int num_sms, cudaStream_t st) {
  if (a.P <= 0) return cudaSuccess;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, step_fused_kernel, STEP_BLOCK, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  // enough blocks for one pass of the per-particle phases, never more than can be co-resident
  int64_t g = (a.P + STEP_BLOCK - 1) / STEP_BLOCK;
  const int64_t cap = (int64_t)per_sm * num_sms;
  if (g > cap) g = cap;
  StepFusedArgs args = a;
  void* params[] = {&args};
  e = cudaLaunchCooperativeKernel((const void*)step_fused_kernel, dim3((unsigned)g), dim3(STEP_BLOCK), params, 0, st);
  return e != cudaSuccess ? e : cudaGetLastError();
}
double step_reg_bandwidth(int64_t P_total) { return pow(4.0 / (8.0 * (double)P_total), 1.0 / 10.0); }

}  // namespace cdms
