// response.cu -- test entry cdms_response (materialized steering vectors) and cdms_layout (row A1),
// built from exactly the device functions and recurrences of the likelihood kernel (geometry.cuh).
#include <math.h>

#include "cdms_internal.h"
#include "geometry.cuh"

namespace cdms {

// ---------------------------------------------------------------------------- response (test entry)
// psi[k*Na + m] = conj(A_seg w^i), k = k0 + i, with exactly the per-(p,s) and per-(s,m) set-up and the
// segment recurrence (A_seg <- A_seg Z every SEG subcarriers) of the likelihood kernel.  sfv_per_item: item i's wall
// (s >= 1) is sfv[i] instead of sfv[s - 1] (the F4 belief averages over paired particles, slam_step.cu).
template <typename RT>
__global__ void response_kernel(const __grid_constant__ SceneDev sc, const double* __restrict__ pos,
                                int64_t n, const int32_t* __restrict__ js, const double* __restrict__ sfv,
                                double2* __restrict__ psi, int* flags, int sfv_per_item) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * sc.Na) return;
  const int64_t item = t / sc.Na;
  const int m = (int)(t - item * sc.Na);
  const int j = js[2 * item], s = js[2 * item + 1];
  const double p[3] = {pos[3 * item], pos[3 * item + 1], pos[3 * item + 2]};
  PSField<RT> f;
  double R64;
  const int st = (j >= 0 && j < sc.J && s >= 0 && s < sc.S)
                     ? setup_ps<RT>(sc, j, p, s ? sfv + 3 * (sfv_per_item ? item : s - 1) : nullptr, f, R64)
                     : PS_BADSFV;
  if (st != PS_OK) {
    atomicOr(flags, st == PS_DEGENERATE ? FLAG_DEGENERATE : FLAG_NAN);
    for (int k = 0; k < sc.nf; ++k) psi[item * (int64_t)sc.nf * sc.Na + (int64_t)k * sc.Na + m] = make_double2(NAN, NAN);
    return;
  }
  double v64[3], q264;
  template_col(sc, j, m, v64, q264);
  const RT v[3] = {(RT)v64[0], (RT)v64[1], (RT)v64[2]};
  SMPhasors<RT> o;
  bool dg;
  setup_sm<RT>(sc, f, v, (RT)q264, m, s, o, dg);
  if (dg) atomicOr(flags, FLAG_DEGENERATE);
  RT Ar = o.Ar, Ai = o.Ai;
  const RT g = f.gain;
  for (int k0 = 0; k0 < sc.nf; k0 += SEG) {
    RT er = Ar, ei = Ai;
    const int k1 = min(k0 + SEG, sc.nf);
    for (int k = k0; k < k1; ++k) {
      psi[item * (int64_t)sc.nf * sc.Na + (int64_t)k * sc.Na + m] = make_double2((double)(g * er), -(double)(g * ei));
      const RT nr = er * o.wr - ei * o.wi;
      const RT ni = er * o.wi + ei * o.wr;
      er = nr;
      ei = ni;
    }
    if (sc.two_seg) {  // the kernel's second segment starts at A1 (carried in Z)
      Ar = o.Zr;
      Ai = o.Zi;
    } else {
      const RT nAr = Ar * o.Zr - Ai * o.Zi;
      const RT nAi = Ar * o.Zi + Ai * o.Zr;
      Ar = nAr;
      Ai = nAi;
    }
  }
}

cudaError_t launch_response(const SceneDev& sc, const double* pos, int64_t n, const int32_t* js, const double* sfv,
                            double2* psi, int precision, int* flags, cudaStream_t st, int sfv_per_item) {
  const int64_t threads = n * sc.Na;
  if (threads == 0) return cudaSuccess;
  const unsigned grid = (unsigned)((threads + 127) / 128);
  if (precision == CDMS_FP64)
    response_kernel<double><<<grid, 128, 0, st>>>(sc, pos, n, js, sfv, psi, flags, sfv_per_item);
  else
    response_kernel<float><<<grid, 128, 0, st>>>(sc, pos, n, js, sfv, psi, flags, sfv_per_item);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------- layout (row A1)
// One thread per (j, s, m): H_s, p_VA,js, P_{j,s}[:, m] = p_VA + H_s R_j p~_m
// (P:L57-61), with the kernel's anchor_va / template_col.
__global__ void layout_kernel(const __grid_constant__ SceneDev sc, const double* __restrict__ sfv,
                              double* __restrict__ layout, double* __restrict__ va_out, double* __restrict__ H_out,
                              int* flags) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int total = sc.J * sc.S * sc.Na;
  if (t >= total) return;
  const int m = t % sc.Na, js = t / sc.Na, s = js % sc.S, j = js / sc.S;
  double va[3], sh[3];
  if (!anchor_va(sc, j, s ? sfv + 3 * (s - 1) : nullptr, va, sh)) {
    atomicOr(flags, FLAG_NAN);
    return;
  }
  double v[3], q2;
  template_col(sc, j, m, v, q2);
  const double sv = sh[0] * v[0] + sh[1] * v[1] + sh[2] * v[2];
  for (int c = 0; c < 3; ++c)
    layout[(((int64_t)j * sc.S + s) * 3 + c) * sc.Na + m] = va[c] + v[c] - 2.0 * sh[c] * sv;
  if (m == 0) {
    for (int c = 0; c < 3; ++c) va_out[((int64_t)j * sc.S + s) * 3 + c] = va[c];
    if (j == 0)
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) H_out[s * 9 + r * 3 + c] = (r == c ? 1.0 : 0.0) - 2.0 * sh[r] * sh[c];
  }
}

cudaError_t launch_layout(const SceneDev& sc, const double* sfv, double* layout, double* va, double* H, int* flags,
                          cudaStream_t st) {
  const int total = sc.J * sc.S * sc.Na;
  layout_kernel<<<(total + 127) / 128, 128, 0, st>>>(sc, sfv, layout, va, H, flags);
  return cudaGetLastError();
}

}  // namespace cdms

