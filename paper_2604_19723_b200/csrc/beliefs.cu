// beliefs.cu -- rows A6-A9 on sm_100a: log-sum-exp weight normalization, belief moments, integer
// systematic resampling (quantize, scan, ancestors, gather), NCV prediction and the Gaussian
// regularization kernel with a counter-based Philox4x32-10 generator.  All reductions use a fixed
// partition of the particles into blocks of RED_ITEMS and a fixed tree order, so results depend only
// on the particle order, not on the launch configuration.
#include <math.h>

#include "cdms_internal.h"

namespace cdms {

int64_t red_blocks(int64_t P) { return P <= 0 ? 0 : (P + RED_ITEMS - 1) / RED_ITEMS; }

// ---------------------------------------------------------------------------- block helpers
template <typename T, typename Op>
__device__ __forceinline__ T block_reduce(T v, T* sh, Op op) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int s = RED_BLOCK / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) sh[threadIdx.x] = op(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  T r = sh[0];
  __syncthreads();
  return r;
}
struct OpMax {
  __device__ double operator()(double a, double b) const { return a > b ? a : b; }
};
struct OpAdd {
  __device__ double operator()(double a, double b) const { return a + b; }
};

// ---------------------------------------------------------------------------- row A6: LSE
// Block b covers particles [b*RED_ITEMS, (b+1)*RED_ITEMS); out part[b] = (max l, sum e^{l - max}).
__global__ void lse_partial_kernel(const double* __restrict__ l, int64_t P, double2* __restrict__ part) {
  __shared__ double sh[RED_BLOCK];
  const int64_t base = (int64_t)blockIdx.x * RED_ITEMS;
  double m = -INFINITY;
  for (int i = threadIdx.x; i < RED_ITEMS; i += RED_BLOCK) {
    const int64_t p = base + i;
    if (p < P) m = fmax(m, l[p]);
  }
  const double M = block_reduce(m, sh, OpMax());
  double s = 0.0;
  if (M > -INFINITY) {
    for (int i = threadIdx.x; i < RED_ITEMS; i += RED_BLOCK) {
      const int64_t p = base + i;
      if (p < P) s += exp(l[p] - M);
    }
  }
  const double S = block_reduce(s, sh, OpAdd());
  if (threadIdx.x == 0) part[blockIdx.x] = make_double2(M, S);
}

// Single block: combine the block partials in a fixed tree -> (M_r, S_r) of this rank.
__global__ void lse_final_kernel(const double2* __restrict__ part, int64_t nblk, double2* __restrict__ out) {
  __shared__ double sh[RED_BLOCK];
  double m = -INFINITY;
  for (int64_t b = threadIdx.x; b < nblk; b += RED_BLOCK) m = fmax(m, part[b].x);
  const double M = block_reduce(m, sh, OpMax());
  double s = 0.0;
  if (M > -INFINITY)
    for (int64_t b = threadIdx.x; b < nblk; b += RED_BLOCK) {
      const double2 q = part[b];
      if (q.x > -INFINITY) s += q.y * exp(q.x - M);
    }
  const double S = block_reduce(s, sh, OpAdd());
  if (threadIdx.x == 0) out[0] = make_double2(M, S);
}

// Combine the ranks' (M_r, S_r) in rank order: M = max M_r, S = sum_r S_r e^{M_r - M};
// lse = M + ln S.  All -inf -> FLAG_ZEROMASS, lse = -inf; NaN -> FLAG_NAN.
__global__ void lse_combine_kernel(const double2* __restrict__ per_rank, int nranks, double* lse, double* Mout,
                                   double* logS, int* flags) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
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

// w_p = e^{(l_p - M) - ln S} (l_p - M is exact, so w keeps full relative precision)
__global__ void normalize_kernel(const double* __restrict__ l, int64_t P, const double* __restrict__ M,
                                 const double* __restrict__ logS, const int* __restrict__ flags,
                                 double* __restrict__ w) {
  if (*flags & (FLAG_ZEROMASS | FLAG_NAN)) return;
  const double m = *M, ls = *logS;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x)
    w[p] = exp((l[p] - m) - ls);
}

static unsigned grid_for(int64_t n, int threads, int cap = 4096) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

cudaError_t launch_lse_partial(const double* l, int64_t P, double2* part, cudaStream_t st) {
  const int64_t nb = red_blocks(P);
  if (nb > 0) lse_partial_kernel<<<(unsigned)nb, RED_BLOCK, 0, st>>>(l, P, part);
  return cudaGetLastError();
}
cudaError_t launch_lse_final(const double2* part, int64_t nblk, double2* out, cudaStream_t st) {
  lse_final_kernel<<<1, RED_BLOCK, 0, st>>>(part, nblk, out);
  return cudaGetLastError();
}
cudaError_t launch_lse_combine(const double2* per_rank, int nranks, double* lse, double* M, double* logS, int* flags,
                               cudaStream_t st) {
  lse_combine_kernel<<<1, 32, 0, st>>>(per_rank, nranks, lse, M, logS, flags);
  return cudaGetLastError();
}
cudaError_t launch_normalize(const double* l, int64_t P, const double* M, const double* logS, const int* flags,
                             double* w, cudaStream_t st) {
  normalize_kernel<<<grid_for(P, 256), 256, 0, st>>>(l, P, M, logS, flags, w);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------- row A7: moments
// pass 1: per block [sum w, sum w x_0..x_5]; pass 2: per block sum w (x - mu)(x - mu)^T (upper tri, 21)
__global__ void moments1_kernel(const double* __restrict__ x, const double* __restrict__ w, int64_t P,
                                double* __restrict__ part) {
  __shared__ double sh[RED_BLOCK];
  const int64_t base = (int64_t)blockIdx.x * RED_ITEMS;
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int i = threadIdx.x; i < RED_ITEMS; i += RED_BLOCK) {
    const int64_t p = base + i;
    if (p < P) {
      const double wp = w[p];
      acc[0] += wp;
      for (int a = 0; a < 6; ++a) acc[1 + a] += wp * x[p * 6 + a];
    }
  }
  for (int a = 0; a < 7; ++a) {
    const double r = block_reduce(acc[a], sh, OpAdd());
    if (threadIdx.x == 0) part[blockIdx.x * 7 + a] = r;
  }
}

__global__ void moments2_kernel(const double* __restrict__ x, const double* __restrict__ w, int64_t P,
                                const double* __restrict__ sum1, double* __restrict__ part) {
  __shared__ double sh[RED_BLOCK];
  const int64_t base = (int64_t)blockIdx.x * RED_ITEMS;
  double mu[6];
  for (int a = 0; a < 6; ++a) mu[a] = sum1[1 + a] / sum1[0];
  double acc[21];
  for (int t = 0; t < 21; ++t) acc[t] = 0.0;
  for (int i = threadIdx.x; i < RED_ITEMS; i += RED_BLOCK) {
    const int64_t p = base + i;
    if (p < P) {
      const double wp = w[p];
      double d[6];
      for (int a = 0; a < 6; ++a) d[a] = x[p * 6 + a] - mu[a];
      int t = 0;
      for (int a = 0; a < 6; ++a)
        for (int b = a; b < 6; ++b) acc[t++] += wp * d[a] * d[b];
    }
  }
  for (int t = 0; t < 21; ++t) {
    const double r = block_reduce(acc[t], sh, OpAdd());
    if (threadIdx.x == 0) part[blockIdx.x * 21 + t] = r;
  }
}

// out[c] = sum_b part[b * width + c], b ascending (one thread per column, fixed order)
__global__ void sum_partials_kernel(const double* __restrict__ part, int64_t nblk, int width, double* __restrict__ out) {
  const int c = threadIdx.x;
  if (c >= width) return;
  double s = 0.0;
  for (int64_t b = 0; b < nblk; ++b) s += part[b * width + c];
  out[c] = s;
}

__global__ void moments_finalize_kernel(const double* __restrict__ sum1, const double* __restrict__ sum2,
                                        double* __restrict__ est, int* flags) {
  if (threadIdx.x != 0) return;
  const double sw = sum1[0];
  if (!(sw > 0.0)) atomicOr(flags, FLAG_ZEROMASS);
  est[0] = sw;
  for (int a = 0; a < 6; ++a) est[1 + a] = sum1[1 + a] / sw;
  for (int t = 0; t < 21; ++t) est[7 + t] = sum2[t] / sw;
}

cudaError_t launch_moments1(const double* x, const double* w, int64_t P, double* part, cudaStream_t st) {
  const int64_t nb = red_blocks(P);
  if (nb > 0) moments1_kernel<<<(unsigned)nb, RED_BLOCK, 0, st>>>(x, w, P, part);
  return cudaGetLastError();
}
cudaError_t launch_moments2(const double* x, const double* w, int64_t P, const double* sum1, double* part,
                            cudaStream_t st) {
  const int64_t nb = red_blocks(P);
  if (nb > 0) moments2_kernel<<<(unsigned)nb, RED_BLOCK, 0, st>>>(x, w, P, sum1, part);
  return cudaGetLastError();
}
cudaError_t launch_sum_partials(const double* part, int64_t nblk, int width, double* out, cudaStream_t st) {
  sum_partials_kernel<<<1, 32, 0, st>>>(part, nblk, width, out);
  return cudaGetLastError();
}
cudaError_t launch_moments_finalize(const double* sum1, const double* sum2, double* est, int* flags, cudaStream_t st) {
  moments_finalize_kernel<<<1, 32, 0, st>>>(sum1, sum2, est, flags);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------- row A8: resampling
__global__ void wmax_partial_kernel(const double* __restrict__ w, int64_t P, double* __restrict__ part, int* flags) {
  __shared__ double sh[RED_BLOCK];
  const int64_t base = (int64_t)blockIdx.x * RED_ITEMS;
  double m = 0.0;
  bool bad = false;
  for (int i = threadIdx.x; i < RED_ITEMS; i += RED_BLOCK) {
    const int64_t p = base + i;
    if (p < P) {
      const double v = w[p];
      bad |= !(v >= 0.0);
      m = fmax(m, v);
    }
  }
  if (bad) atomicOr(flags, FLAG_NAN);
  const double M = block_reduce(m, sh, OpMax());
  if (threadIdx.x == 0) part[blockIdx.x] = M;
}
__global__ void max_final_kernel(const double* __restrict__ part, int64_t nblk, double* __restrict__ out) {
  __shared__ double sh[RED_BLOCK];
  double m = 0.0;
  for (int64_t b = threadIdx.x; b < nblk; b += RED_BLOCK) m = fmax(m, part[b]);
  const double M = block_reduce(m, sh, OpMax());
  if (threadIdx.x == 0) out[0] = M;
}

// q_p = rint(ldexp(r_p, 36)), r_p = w_p / w_max (from_loglik = 0) or e^{l_p - M} (= 1) (C-amb-15)
__global__ void quantize_kernel(const double* __restrict__ w, int64_t P, const double* __restrict__ wmax,
                                const double* __restrict__ M, int from_loglik, uint64_t* __restrict__ q, int* flags) {
  const double wm = from_loglik ? 0.0 : *wmax;
  const double m = from_loglik ? *M : 0.0;
  if (!from_loglik && !(wm > 0.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(flags, FLAG_ZEROMASS);
  }
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
    double r = from_loglik ? exp(w[p] - m) : (wm > 0.0 ? w[p] / wm : 0.0);
    if (!(r >= 0.0)) r = 0.0;
    q[p] = (uint64_t)rint(scalbn(r, 36));
  }
}

// inclusive scan of uint64 (exact): per-block scan + block sums, then block offsets
__global__ void scan_block_kernel(uint64_t* __restrict__ q, int64_t P, uint64_t* __restrict__ bsum) {
  __shared__ uint64_t sh[RED_BLOCK];
  const int64_t base = (int64_t)blockIdx.x * RED_ITEMS;
  constexpr int PER = RED_ITEMS / RED_BLOCK;
  uint64_t v[PER];
  uint64_t run = 0;
  for (int i = 0; i < PER; ++i) {  // thread t owns the contiguous run [t*PER, (t+1)*PER)
    const int64_t p = base + threadIdx.x * PER + i;
    run += (p < P) ? q[p] : 0ull;
    v[i] = run;
  }
  sh[threadIdx.x] = run;
  __syncthreads();
  for (int off = 1; off < RED_BLOCK; off <<= 1) {  // Hillis-Steele inclusive scan of thread totals
    uint64_t add = (threadIdx.x >= (unsigned)off) ? sh[threadIdx.x - off] : 0ull;
    __syncthreads();
    sh[threadIdx.x] += add;
    __syncthreads();
  }
  const uint64_t excl = (threadIdx.x > 0) ? sh[threadIdx.x - 1] : 0ull;
  for (int i = 0; i < PER; ++i) {
    const int64_t p = base + threadIdx.x * PER + i;
    if (p < P) q[p] = v[i] + excl;
  }
  if (threadIdx.x == RED_BLOCK - 1) bsum[blockIdx.x] = sh[RED_BLOCK - 1];
}
__global__ void scan_sums_kernel(uint64_t* __restrict__ bsum, int64_t nblk) {
  if (threadIdx.x != 0) return;
  uint64_t run = 0;
  for (int64_t b = 0; b < nblk; ++b) {  // exclusive prefix in place
    const uint64_t v = bsum[b];
    bsum[b] = run;
    run += v;
  }
  bsum[nblk] = run;  // total Q
}
__global__ void scan_add_kernel(uint64_t* __restrict__ q, int64_t P, const uint64_t* __restrict__ bsum) {
  const int64_t base = (int64_t)blockIdx.x * RED_ITEMS;
  const uint64_t off = bsum[blockIdx.x];
  for (int i = threadIdx.x; i < RED_ITEMS; i += RED_BLOCK) {
    const int64_t p = base + i;
    if (p < P) q[p] += off;
  }
}

// Output slot g of this rank's range [slot_lo, slot_hi) (plan on the device): t_g = floor((u + g 2^32) Q /
// (P_total 2^32)), ancestor = min{p : C_p > t_g - O_r} (binary search in this rank's inclusive scan C), written to
// row g mod P_local of the slot owner's ancestor buffer peer_anc[g / P_local].
__global__ void ancestors_kernel(const uint64_t* __restrict__ C, int64_t P_local, const uint64_t* __restrict__ plan,
                                 int64_t P_total, uint32_t u_bits, int64_t p_global0, int64_t* own_anc,
                                 int64_t* const* peer_anc, int* flags) {
  const uint64_t Q = plan[0], O = plan[1];
  const int64_t slot_lo = (int64_t)plan[2], n = (int64_t)plan[3] - slot_lo;
  if (Q == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(flags, FLAG_ZEROMASS);
    return;
  }
  const unsigned __int128 den = (unsigned __int128)(uint64_t)P_total << 32;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t g = (uint64_t)(slot_lo + i);
    const unsigned __int128 num = ((unsigned __int128)u_bits + ((unsigned __int128)g << 32)) * Q;
    const uint64_t t = (uint64_t)(num / den) - O;
    int64_t lo = 0, hi = P_local - 1;  // smallest p with C[p] > t
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (C[mid] > t) hi = mid; else lo = mid + 1;
    }
    const int64_t own = (int64_t)(g / (uint64_t)P_local);
    (peer_anc ? peer_anc[own] : own_anc)[(int64_t)g - own * P_local] = p_global0 + lo;
  }
  __threadfence_system();
}

// out[n] = sum over ranks r (in rank order) of in[r][n]: deterministic combine of all-gathered per-rank sums
__global__ void sum_ranks_kernel(const double* __restrict__ in, int nranks, int n, double* __restrict__ out) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < nranks; ++r) s += in[(int64_t)r * n + i];
    out[i] = s;
  }
}
cudaError_t launch_sum_ranks(const double* in, int nranks, int n, double* out, cudaStream_t st) {
  sum_ranks_kernel<<<1, 64, 0, st>>>(in, nranks, n, out);
  return cudaGetLastError();
}

// out[i] = x[anc[i] - p_global0] (6 doubles per particle)
__global__ void gather_kernel(const double* __restrict__ x, const int64_t* __restrict__ anc, int64_t n,
                              int64_t p_global0, double* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n * 6; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / 6;
    const int c = (int)(t - i * 6);
    out[t] = x[(anc[i] - p_global0) * 6 + c];
  }
}

cudaError_t launch_max_final(const double* part, int64_t nblk, double* out, cudaStream_t st) {
  max_final_kernel<<<1, RED_BLOCK, 0, st>>>(part, nblk, out);
  return cudaGetLastError();
}
cudaError_t launch_quantize(const double* w, int64_t P, const double* wmax, const double* M, int from_loglik,
                            uint64_t* q, int* flags, cudaStream_t st) {
  quantize_kernel<<<grid_for(P, 256), 256, 0, st>>>(w, P, wmax, M, from_loglik, q, flags);
  return cudaGetLastError();
}
// block_sums must hold red_blocks(P) + 1 entries; the total Q lands in block_sums[red_blocks(P)]
cudaError_t launch_scan(uint64_t* q, int64_t P, uint64_t* block_sums, cudaStream_t st) {
  const int64_t nb = red_blocks(P);
  if (nb == 0) return cudaSuccess;
  scan_block_kernel<<<(unsigned)nb, RED_BLOCK, 0, st>>>(q, P, block_sums);
  scan_sums_kernel<<<1, 32, 0, st>>>(block_sums, nb);
  scan_add_kernel<<<(unsigned)nb, RED_BLOCK, 0, st>>>(q, P, block_sums);
  return cudaGetLastError();
}
cudaError_t launch_ancestors(const uint64_t* C, int64_t P_local, const uint64_t* plan, int64_t P_total, uint32_t u_bits,
                             int64_t p_global0, int64_t* own_anc, int64_t* const* peer_anc, int* flags,
                             cudaStream_t st) {
  ancestors_kernel<<<grid_for(P_local, 256), 256, 0, st>>>(C, P_local, plan, P_total, u_bits, p_global0, own_anc,
                                                          peer_anc, flags);
  return cudaGetLastError();
}
cudaError_t launch_gather(const double* x, const int64_t* anc, int64_t n, int64_t p_global0, double* out,
                          cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  gather_kernel<<<grid_for(n * 6, 256), 256, 0, st>>>(x, anc, n, p_global0, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------- row A9: RNG, predict, regularize
// Philox4x32-10 (Salmon et al., SC'11): 10 rounds of the (M0, M1) multiply-xor round with a Weyl key
// schedule (W0, W1).
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
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

// four N(0,1) draws for (key, step, index, stream): u = (x + 1/2) 2^-32, Box-Muller on (u0,u1), (u2,u3)
__device__ __forceinline__ void normals4(uint64_t key, uint64_t step, uint64_t index, uint32_t stream, double n[4]) {
  const uint4 x = philox4x32_10(make_uint4((uint32_t)index, (uint32_t)(index >> 32), (uint32_t)step, stream),
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

// NCV: x_n = F x_{n-1} + Gamma a, a ~ N(0, sigma_v^2 I3), Gamma = [T^2/2 I; T I]
__global__ void predict_kernel(double* __restrict__ x, int64_t P, int64_t p0, double T, double sigma_v, uint64_t key,
                               uint64_t step) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
    double n[4];
    normals4(key, step, (uint64_t)(p0 + p), 0u, n);
    double* s = x + p * 6;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double acc = sigma_v * n[a];
      s[a] = s[a] + T * s[3 + a] + 0.5 * T * T * acc;
      s[3 + a] = s[3 + a] + T * acc;
    }
  }
}

// Cholesky of Sigma + 1e-12 tr(Sigma) I (C-amb-16), non-positive pivots zero their column; one thread.
__global__ void chol6_kernel(const double* __restrict__ est, double* __restrict__ L) {
  if (threadIdx.x != 0) return;
  double Sg[36];
  int t = 0;
  for (int a = 0; a < 6; ++a)
    for (int b = a; b < 6; ++b) {
      Sg[a * 6 + b] = est[7 + t];
      Sg[b * 6 + a] = est[7 + t];
      ++t;
    }
  double tr = 0.0;
  for (int a = 0; a < 6; ++a) tr += Sg[a * 6 + a];
  for (int a = 0; a < 6; ++a) Sg[a * 6 + a] += 1e-12 * tr;
  for (int i = 0; i < 36; ++i) L[i] = 0.0;
  for (int j = 0; j < 6; ++j) {
    double d = Sg[j * 6 + j];
    for (int k = 0; k < j; ++k) d -= L[j * 6 + k] * L[j * 6 + k];
    if (!(d > 0.0)) continue;
    const double l = sqrt(d);
    L[j * 6 + j] = l;
    for (int i = j + 1; i < 6; ++i) {
      double acc = Sg[i * 6 + j];
      for (int k = 0; k < j; ++k) acc -= L[i * 6 + k] * L[j * 6 + k];
      L[i * 6 + j] = acc / l;
    }
  }
}

// x <- x + h chol(Sigma) n, n ~ N(0, I6) from streams 1 and 2 of the global slot index
__global__ void regularize_kernel(double* __restrict__ x, int64_t P, int64_t p0, double h, const double* __restrict__ Lg,
                                  uint64_t key, uint64_t step) {
  __shared__ double L[36];
  if (threadIdx.x < 36) L[threadIdx.x] = Lg[threadIdx.x];
  __syncthreads();
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
    double n[8];
    normals4(key, step, (uint64_t)(p0 + p), 1u, n);
    normals4(key, step, (uint64_t)(p0 + p), 2u, n + 4);
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      double acc = 0.0;
      for (int b = 0; b <= a; ++b) acc += L[a * 6 + b] * n[b];
      x[p * 6 + a] += h * acc;
    }
  }
}

__global__ void fill_u64_kernel(uint64_t* dst, uint64_t v, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = v;
}

cudaError_t launch_predict(double* x, int64_t P, int64_t p0, double T, double sigma_v, uint64_t key, uint64_t step,
                           cudaStream_t st) {
  if (P <= 0) return cudaSuccess;
  predict_kernel<<<grid_for(P, 256), 256, 0, st>>>(x, P, p0, T, sigma_v, key, step);
  return cudaGetLastError();
}
cudaError_t launch_chol6(const double* est, double* L, cudaStream_t st) {
  chol6_kernel<<<1, 32, 0, st>>>(est, L);
  return cudaGetLastError();
}
cudaError_t launch_regularize(double* x, int64_t P, int64_t p0, int64_t P_total, const double* L, uint64_t key,
                              uint64_t step, cudaStream_t st) {
  if (P <= 0) return cudaSuccess;
  const double h = pow(4.0 / (8.0 * (double)P_total), 1.0 / 10.0);  // h_opt, d = 6 (C-amb-16)
  regularize_kernel<<<grid_for(P, 256), 256, 0, st>>>(x, P, p0, h, L, key, step);
  return cudaGetLastError();
}
cudaError_t launch_fill_u64(uint64_t* dst, uint64_t v, int n, cudaStream_t st) {
  fill_u64_kernel<<<(n + 127) / 128, 128, 0, st>>>(dst, v, n);
  return cudaGetLastError();
}

cudaError_t launch_wmax_partial_f(const double* w, int64_t P, double* part, int* flags, cudaStream_t st) {
  const int64_t nb = red_blocks(P);
  if (nb > 0) wmax_partial_kernel<<<(unsigned)nb, RED_BLOCK, 0, st>>>(w, P, part, flags);
  return cudaGetLastError();
}

}  // namespace cdms
