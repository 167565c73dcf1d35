// Carrier e^{j2pi f_c Delta/c} in fp32: (A) centred reduction x - rint(x) then __sincosf(2 pi x) (cis2pi_fast) vs
// (B) __sincosf(Delta * (2 pi f_c/c)) with no reduction (MUFU.SIN/COS reduce the revolutions themselves).  Max
// |error| against fp64 sincospi(2 Delta f_c/c) over |Delta f_c/c| <= XMAX cycles.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sincos_range sincos_range.cu && ./sincos_range
#include <cstdio>
#include <cmath>
__global__ void k(float fc_cf, float fc2pi, double fc_c, float dmax, int n, float* err) {
  float ea = 0.f, eb = 0.f;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float d = dmax * (2.f * (i + 0.5f) / n - 1.f);  // Delta, metres
    double s, c;
    sincospi(2.0 * (double)d * fc_c, &s, &c);
    float x = d * fc_cf;
    x = x - ((x + 12582912.f) - 12582912.f);
    float sa, ca, sb, cb;
    __sincosf(6.28318530717958647692f * x, &sa, &ca);
    __sincosf(d * fc2pi, &sb, &cb);
    ea = fmaxf(ea, fmaxf(fabsf(sa - (float)s), fabsf(ca - (float)c)));
    eb = fmaxf(eb, fmaxf(fabsf(sb - (float)s), fabsf(cb - (float)c)));
  }
  atomicMax(reinterpret_cast<int*>(err), __float_as_int(ea));
  atomicMax(reinterpret_cast<int*>(err + 1), __float_as_int(eb));
}
int main() {
  const double fc = 3.5e9, c0 = 299792458.0, fc_c = fc / c0;
  float* e;
  cudaMallocManaged(&e, 8);
  for (double xmax : {0.5, 2.0, 4.0, 8.0, 16.0}) {
    e[0] = e[1] = 0.f;
    const float dmax = (float)(xmax / fc_c);
    k<<<1184, 256>>>((float)fc_c, (float)(2.0 * M_PI * fc_c), fc_c, dmax, 1 << 26, e);
    cudaDeviceSynchronize();
    printf("|x| <= %5.1f cycles: reduced %.3e  direct %.3e (abs, vs fp64)\n", xmax, e[0], e[1]);
  }
  return 0;
}
