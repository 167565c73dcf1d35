/*
 * cdms_oracle.c -- plain, slow, fp64 CPU ORACLE for the coherent-likelihood hot path of
 * "Coherent Direct Multipath SLAM" (arxiv 2604.19723).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code, header,
 * table or constant generator with the CUDA path (paper_2604_19723_b200/csrc) and neither
 * includes the other.
 *
 * Citations: "P:Lnnn" is a line of /root/reference/PAPER.md, "S:Lnnn" one of SPEC.md,
 * "C-amb-n" a reading listed in SURVEY.md section 8(c) / DESIGN.md.
 *
 * Conventions: IEEE fp64, round-to-nearest, built with -O2 -fno-fast-math -ffp-contract=off;
 * every sum runs in index order (p; j; s; k; m) (C-amb-22).  OpenMP only splits the
 * outermost particle loop, so each particle's result is independent of the thread count.
 *
 * Parity pins (tests/test_oracle_*.py): geometry invariants, an independent reflection
 * construction of the VA layout, unit modulus, Kronecker == per-element, far-field 1/d law,
 * the dense N_z x N_z log-density (numpy), Sherman-Morrison at S=1, the v->0 and v->inf
 * limits, phase-rotation invariance, matched-filter Cauchy-Schwarz, moment matching by
 * enumeration, resampling hand trace + float Alg.2 agreement, Philox KAT vectors.
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_C 299792458.0 /* speed of light, m/s (C-amb-3) */
#define ORC_PI 3.14159265358979323846

enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_EDEGENERATE = 2, ORC_EZEROMASS = 3 };
enum { ORC_SPHERICAL = 0, ORC_PLANAR_WB = 1, ORC_PLANAR_NB = 2 };

typedef struct {
  int32_t J, K;          /* PAs; walls (S~ = K+1 components, s = 0 is LOS) */
  int32_t ny, nv;        /* URA N_y x N_v, column m = iy*nv + iv */
  int32_t nf;            /* subcarriers */
  int32_t wavefront;     /* ORC_SPHERICAL / ORC_PLANAR_WB / ORC_PLANAR_NB */
  int32_t pathloss;      /* 1: psi = lambda/(4 pi ||r'||) psi~ (C-amb-6) */
  int32_t pad_;
  double dy, dv;         /* element spacing */
  double fc;             /* carrier */
  const double* pa_pos;  /* [J][3] */
  const double* pa_rot;  /* [J][3][3] row-major */
  const double* f_pb;    /* [nf] passband frequencies f_pb = f_c 1 + f */
} orc_scene;

/* ------------------------------------------------------------------ L0 geometry (A1) */

/* Template URA P~ in the local yz-plane, symmetric about the origin:
 * row x = 0, row y = p_y^T (x) 1_{1 x N_v}, row z = 1_{1 x N_y} (x) p_z^T. */
void orc_template(int ny, int nv, double dy, double dv, double* pt /*[3][Na]*/) {
  int na = ny * nv;
  for (int iy = 0; iy < ny; ++iy)
    for (int iv = 0; iv < nv; ++iv) {
      int m = iy * nv + iv;
      pt[0 * na + m] = 0.0;
      pt[1 * na + m] = (iy - 0.5 * (ny - 1)) * dy;
      pt[2 * na + m] = (iv - 0.5 * (nv - 1)) * dv;
    }
}

/* Householder H_k = I - 2 s s^T / ||s||^2; H_0 = I for LOS. */
int orc_householder(const double* s /*[3] or NULL for LOS*/, double* H /*[3][3]*/) {
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) H[a * 3 + b] = (a == b) ? 1.0 : 0.0;
  if (!s) return ORC_OK;
  double n2 = s[0] * s[0] + s[1] * s[1] + s[2] * s[2];
  if (!(n2 > 0.0)) return ORC_EINVAL; /* p_sfv in R^3 \ {0} */
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) H[a * 3 + b] -= 2.0 * s[a] * s[b] / n2;
  return ORC_OK;
}

/* SFV -> VA: p_VA = p_j - (2 p_j^T s / ||s||^2 - 1) s; LOS: p_VA = p_j. */
int orc_va(const double* pj, const double* s /*or NULL*/, double* va) {
  if (!s) { va[0] = pj[0]; va[1] = pj[1]; va[2] = pj[2]; return ORC_OK; }
  double n2 = s[0] * s[0] + s[1] * s[1] + s[2] * s[2];
  if (!(n2 > 0.0)) return ORC_EINVAL;
  double c = 2.0 * (pj[0] * s[0] + pj[1] * s[1] + pj[2] * s[2]) / n2 - 1.0;
  for (int a = 0; a < 3; ++a) va[a] = pj[a] - c * s[a];
  return ORC_OK;
}

/* VA layout P_{j,k} = p_VA 1^T + H_k R_j P~; k = 0 gives the PA layout. */
int orc_anchor_layout(const orc_scene* sc, int j, const double* s /*or NULL*/,
                      double* layout /*[3][Na]*/, double* va /*[3]*/, double* H /*[3][3]*/) {
  int na = sc->ny * sc->nv;
  double* pt = (double*)malloc(sizeof(double) * 3 * na);
  orc_template(sc->ny, sc->nv, sc->dy, sc->dv, pt);
  int st = orc_householder(s, H);
  if (st == ORC_OK) st = orc_va(sc->pa_pos + 3 * j, s, va);
  if (st == ORC_OK) {
    const double* R = sc->pa_rot + 9 * j;
    double HR[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double acc = 0.0;
        for (int c = 0; c < 3; ++c) acc += H[a * 3 + c] * R[c * 3 + b];
        HR[a * 3 + b] = acc;
      }
    for (int m = 0; m < na; ++m)
      for (int a = 0; a < 3; ++a) {
        double acc = 0.0;
        for (int c = 0; c < 3; ++c) acc += HR[a * 3 + c] * pt[c * na + m];
        layout[a * na + m] = va[a] + acc;
      }
  }
  free(pt);
  return st;
}

/* cdms_layout counterpart: all (j, s) anchors at once.  layout[J][S][3][Na], va[J][S][3], H[S][3][3]. */
int orc_layout(const orc_scene* sc, const double* sfv /*[K][3]*/, double* layout, double* va,
               double* H) {
  int S = sc->K + 1, na = sc->ny * sc->nv;
  for (int j = 0; j < sc->J; ++j)
    for (int s = 0; s < S; ++s) {
      const double* sv = (s == 0) ? NULL : sfv + 3 * (s - 1);
      int st = orc_anchor_layout(sc, j, sv, layout + ((size_t)(j * S + s)) * 3 * na,
                                 va + (j * S + s) * 3, H + s * 9);
      if (st) return st;
    }
  return ORC_OK;
}

/* Local ray r' = R_j^T H_k (p - p_VA); LOS: R_j^T (p - p_j). */
void orc_local_ray(const orc_scene* sc, int j, const double* H, const double* va, const double* p,
                   double* rl) {
  const double* R = sc->pa_rot + 9 * j;
  double g[3], h[3];
  for (int a = 0; a < 3; ++a) g[a] = p[a] - va[a];
  for (int a = 0; a < 3; ++a) h[a] = H[a * 3 + 0] * g[0] + H[a * 3 + 1] * g[1] + H[a * 3 + 2] * g[2];
  for (int a = 0; a < 3; ++a) rl[a] = R[0 * 3 + a] * h[0] + R[1 * 3 + a] * h[1] + R[2 * 3 + a] * h[2];
}

/* ------------------------------------------------------------------ L1 array responses */

/* Steering vector psi in C^{N_z} of MT position p for anchor (j, s), element n = k*N_a + m
 * (vec of the N_a x N_f matrix, antenna fastest; C-amb-1).  Modes:
 *  SPHERICAL: psi = vec(exp(-j 2 pi / c vecnorm(p 1^T - P_{j,s})^T f_pb^T)).
 *  PLANAR_WB: vecnorm replaced by (p 1^T - P)^T u, u = r/||r||, r = p - p_VA.
 *  PLANAR_NB: (b(tau) (x) a_y (x) a_z) exp(-j 2 pi f_c ||r'|| / c), tau = ||r'||/c,
 *     theta = arccos(r'_z/||r'||), phi = atan2(r'_y, r'_x), b = exp(-j 2 pi f tau),
 *     a_y = exp(j 2 pi / lambda p_y sin(theta) sin(phi)), a_z = exp(j 2 pi / lambda p_z cos(theta)).
 * pathloss: times lambda / (4 pi ||r'||).  Returns ORC_EDEGENERATE if the MT sits
 * on the phase centre (r' = 0 excluded) or on an antenna (spherical). */
int orc_response(const orc_scene* sc, const double* p /*[3]*/, int j, int s,
                 const double* sfv_s /*[3] for s>0, ignored for s=0*/, int wavefront,
                 double complex* psi /*[Nz]*/) {
  int na = sc->ny * sc->nv, nf = sc->nf;
  double* lay = (double*)malloc(sizeof(double) * 3 * na);
  double va[3], H[9], rl[3];
  int st = orc_anchor_layout(sc, j, s == 0 ? NULL : sfv_s, lay, va, H);
  if (st) { free(lay); return st; }
  orc_local_ray(sc, j, H, va, p, rl);
  double rn = sqrt(rl[0] * rl[0] + rl[1] * rl[1] + rl[2] * rl[2]);
  if (!(rn > 0.0)) { free(lay); return ORC_EDEGENERATE; }
  double lam = ORC_C / sc->fc;
  double gain = sc->pathloss ? lam / (4.0 * ORC_PI * rn) : 1.0;
  if (wavefront == ORC_SPHERICAL) {
    for (int m = 0; m < na; ++m) {
      double dx = p[0] - lay[0 * na + m], dyy = p[1] - lay[1 * na + m], dz = p[2] - lay[2 * na + m];
      double d = sqrt(dx * dx + dyy * dyy + dz * dz);
      if (!(d > 0.0)) { free(lay); return ORC_EDEGENERATE; }
      for (int k = 0; k < nf; ++k) {
        double ph = -2.0 * ORC_PI / ORC_C * d * sc->f_pb[k];
        psi[(size_t)k * na + m] = gain * (cos(ph) + I * sin(ph));
      }
    }
  } else if (wavefront == ORC_PLANAR_WB) {
    double r[3] = {p[0] - va[0], p[1] - va[1], p[2] - va[2]};
    double rr = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
    double u[3] = {r[0] / rr, r[1] / rr, r[2] / rr};
    for (int m = 0; m < na; ++m) {
      double proj = (p[0] - lay[0 * na + m]) * u[0] + (p[1] - lay[1 * na + m]) * u[1] +
                    (p[2] - lay[2 * na + m]) * u[2];
      for (int k = 0; k < nf; ++k) {
        double ph = -2.0 * ORC_PI / ORC_C * proj * sc->f_pb[k];
        psi[(size_t)k * na + m] = gain * (cos(ph) + I * sin(ph));
      }
    }
  } else if (wavefront == ORC_PLANAR_NB) {
    double tau = rn / ORC_C;
    double theta = acos(rl[2] / rn);
    double phi = atan2(rl[1], rl[0]);
    double* pt = (double*)malloc(sizeof(double) * 3 * na);
    orc_template(sc->ny, sc->nv, sc->dy, sc->dv, pt);
    double complex carrier = cexp(-I * 2.0 * ORC_PI / ORC_C * sc->fc * rn);
    for (int k = 0; k < nf; ++k) {
      double fbb = sc->f_pb[k] - sc->fc; /* baseband f */
      double complex b = cexp(-I * 2.0 * ORC_PI * fbb * tau);
      for (int iy = 0; iy < sc->ny; ++iy) {
        double py = pt[1 * na + iy * sc->nv];
        double complex ay = cexp(I * 2.0 * ORC_PI / lam * py * sin(theta) * sin(phi));
        for (int iv = 0; iv < sc->nv; ++iv) {
          double pz = pt[2 * na + iv];
          double complex az = cexp(I * 2.0 * ORC_PI / lam * pz * cos(theta));
          psi[(size_t)k * na + iy * sc->nv + iv] = gain * (b * ay * az) * carrier;
        }
      }
    }
    free(pt);
  } else {
    free(lay);
    return ORC_EINVAL;
  }
  free(lay);
  return ORC_OK;
}

/* ------------------------------------------------------------------ small dense helpers */

/* In-place lower Cholesky A = L L^H of an n x n Hermitian PD matrix (row-major, lower part used). */
static int orc_cholesky(double complex* A, int n) {
  for (int j = 0; j < n; ++j) {
    double d = creal(A[j * n + j]);
    for (int k = 0; k < j; ++k) d -= creal(A[j * n + k] * conj(A[j * n + k]));
    if (!(d > 0.0)) return ORC_EINVAL;
    double l = sqrt(d);
    A[j * n + j] = l;
    for (int i = j + 1; i < n; ++i) {
      double complex acc = A[i * n + j];
      for (int k = 0; k < j; ++k) acc -= A[i * n + k] * conj(A[j * n + k]);
      A[i * n + j] = acc / l;
    }
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------ L2 likelihood (A3-A5) */

/* Approximate MT update message iota~ at one particle for PA j (Supplement S-V-C):
 *   iota~ = exp(-e^H A^-1 e) / ((pi eta)^Nz det(I + M^H M / eta)),  A = eta I + M M^H,
 *   e^H A^-1 e = ||e||^2/eta - ||(I + M^H M/eta)^{-1/2} M^H e||^2 / eta^2,
 * with the moment-matched reading (C-amb-7/8): columns m_s = sqrt(v_s) psi_s (so M = Psi V^1/2)
 * and mean mu^iota = sum_s m_s-prior psi_s, i.e. e = z - Psi m.  This reaches exactly the dense
 * log CN(z; Psi m, eta I + Psi V Psi^H) of P:L2217-2224 (pinned against numpy in the tests).
 * Steps follow the paper: responses, m-vectors, error vector e, Gram M^H M, M^H e, then the
 * S x S Cholesky for the inverse square root and the determinant.  Also returns the LMMSE
 * amplitude a = m + V^1/2 K^-1 M^H e / eta (K = I + M^H M / eta). */
static int orc_iota(const orc_scene* sc, const double* p, int j, const double* sfv /*[K][3]*/,
                    const double complex* z, const double complex* mprior /*[S]*/,
                    const double* vprior /*[S]*/, double eta, double complex* psi_work /*[S][Nz]*/,
                    double* out_l, double complex* out_amp /*[S] or NULL*/) {
  int S = sc->K + 1;
  size_t nz = (size_t)sc->nf * sc->ny * sc->nv;
  for (int s = 0; s < S; ++s) {
    int st = orc_response(sc, p, j, s, s ? sfv + 3 * (s - 1) : NULL, sc->wavefront,
                          psi_work + (size_t)s * nz);
    if (st) return st;
  }
  /* error vector e = z - mu^iota, mu^iota = sum_s m_s psi_s */
  double complex* e = (double complex*)malloc(sizeof(double complex) * nz);
  double e2 = 0.0;
  for (size_t n = 0; n < nz; ++n) {
    double complex mu = 0.0;
    for (int s = 0; s < S; ++s) mu += mprior[s] * psi_work[(size_t)s * nz + n];
    e[n] = z[n] - mu;
    e2 += creal(e[n] * conj(e[n]));
  }
  /* M^H e and M^H M by direct sums (m-vectors m_s = sqrt(v_s) psi_s) */
  double complex Mhe[16], K[256];
  for (int s = 0; s < S; ++s) {
    double sv = sqrt(vprior[s]);
    double complex acc = 0.0;
    for (size_t n = 0; n < nz; ++n) acc += conj(sv * psi_work[(size_t)s * nz + n]) * e[n];
    Mhe[s] = acc;
  }
  for (int a = 0; a < S; ++a)
    for (int b = 0; b < S; ++b) {
      double sa = sqrt(vprior[a]), sb = sqrt(vprior[b]);
      double complex acc = 0.0;
      for (size_t n = 0; n < nz; ++n)
        acc += conj(sa * psi_work[(size_t)a * nz + n]) * (sb * psi_work[(size_t)b * nz + n]);
      K[a * S + b] = (a == b ? 1.0 : 0.0) + acc / eta; /* I + M^H M / eta */
    }
  free(e);
  int st = orc_cholesky(K, S);
  if (st) return ORC_EINVAL;
  /* ||L^-1 M^H e||^2 = ||(I + M^H M/eta)^{-1/2} M^H e||^2 ; log det = 2 sum log L_ii */
  double complex x[16];
  double logdet = 0.0, q2 = 0.0;
  for (int a = 0; a < S; ++a) {
    double complex acc = Mhe[a];
    for (int b = 0; b < a; ++b) acc -= K[a * S + b] * x[b];
    x[a] = acc / creal(K[a * S + a]);
    q2 += creal(x[a] * conj(x[a]));
    logdet += 2.0 * log(creal(K[a * S + a]));
  }
  double quad = e2 / eta - q2 / (eta * eta);
  *out_l = -(double)nz * log(ORC_PI * eta) - logdet - quad;
  if (out_amp) {
    /* K^-1 b: back substitution L^H y = x */
    double complex y[16];
    for (int a = S - 1; a >= 0; --a) {
      double complex acc = x[a];
      for (int b = a + 1; b < S; ++b) acc -= conj(K[b * S + a]) * y[b];
      y[a] = acc / creal(K[a * S + a]);
    }
    for (int s = 0; s < S; ++s) out_amp[s] = mprior[s] + sqrt(vprior[s]) * y[s] / eta;
  }
  return ORC_OK;
}

/* Per-particle MT log-weight: l_p = log w_beta(p) + sum_j log iota~(x_p; z^(j)).
 * particles: [P][pstride] doubles, position = first 3.  sfv: [K][3] shared, or [P][K][3] when
 * sfv_per_particle (C-amb-8).  y: [J][nf][Na] complex (paper vec order).  m: [J][S] complex,
 * v: [J][S], eta: [J].  logw_prior: [P] or NULL (= 0).  loglik out [P]; amp out [P][J][S] or NULL.
 * Degenerate particles get l = -inf and the call returns ORC_EDEGENERATE. */
int orc_loglik(const orc_scene* sc, const double* particles, int64_t P, int pstride,
               const double* sfv, int sfv_per_particle, const double complex* y,
               const double complex* m, const double* v, const double* eta,
               const double* logw_prior, double* loglik, double complex* amp) {
  if (sc->K < 0 || sc->K > 15 || sc->J <= 0 || P < 0) return ORC_EINVAL;
  int S = sc->K + 1;
  size_t nz = (size_t)sc->nf * sc->ny * sc->nv;
  int status = ORC_OK;
#pragma omp parallel
  {
    double complex* work = (double complex*)malloc(sizeof(double complex) * nz * S);
#pragma omp for schedule(dynamic, 1)
    for (int64_t p = 0; p < P; ++p) {
      const double* x = particles + p * pstride;
      const double* sf = sfv_per_particle ? sfv + (size_t)p * 3 * sc->K : sfv;
      double l = logw_prior ? logw_prior[p] : 0.0;
      for (int j = 0; j < sc->J; ++j) {
        double lj;
        int st = orc_iota(sc, x, j, sf, y + (size_t)j * nz, m + j * S, v + j * S, eta[j], work, &lj,
                          amp ? amp + ((size_t)p * sc->J + j) * S : NULL);
        if (st) {
          l = -INFINITY;
#pragma omp critical
          status = (status == ORC_OK) ? st : status;
          break;
        }
        l += lj;
      }
      loglik[p] = l;
    }
    free(work);
  }
  return status;
}

/* Sufficient statistics of the low-rank evaluation at each particle: the correlation
 * c_s = psi_s^H z^(j) (the M^H e products of P:L755-769 with e = z, V = I) and the Gram
 * G_ab = psi_a^H psi_b (P:L769 fn), by direct summation over n in index order.
 * c out [P][J][S] complex, G out [P][J][S][S] complex. */
int orc_terms(const orc_scene* sc, const double* particles, int64_t P, int pstride, const double* sfv,
              int sfv_per_particle, const double complex* y, double complex* c_out, double complex* G_out) {
  int S = sc->K + 1;
  size_t nz = (size_t)sc->nf * sc->ny * sc->nv;
  int status = ORC_OK;
#pragma omp parallel
  {
    double complex* psi = (double complex*)malloc(sizeof(double complex) * nz * S);
#pragma omp for schedule(dynamic, 1)
    for (int64_t p = 0; p < P; ++p) {
      const double* x = particles + p * pstride;
      const double* sf = sfv_per_particle ? sfv + (size_t)p * 3 * sc->K : sfv;
      for (int j = 0; j < sc->J; ++j) {
        int st = ORC_OK;
        for (int s = 0; s < S && st == ORC_OK; ++s)
          st = orc_response(sc, x, j, s, s ? sf + 3 * (s - 1) : NULL, sc->wavefront, psi + (size_t)s * nz);
        if (st) {
#pragma omp critical
          status = (status == ORC_OK) ? st : status;
          continue;
        }
        const double complex* z = y + (size_t)j * nz;
        for (int a = 0; a < S; ++a) {
          double complex acc = 0.0;
          for (size_t n = 0; n < nz; ++n) acc += conj(psi[(size_t)a * nz + n]) * z[n];
          c_out[((size_t)p * sc->J + j) * S + a] = acc;
          for (int b = 0; b < S; ++b) {
            double complex g = 0.0;
            for (size_t n = 0; n < nz; ++n) g += conj(psi[(size_t)a * nz + n]) * psi[(size_t)b * nz + n];
            G_out[(((size_t)p * sc->J + j) * S + a) * S + b] = g;
          }
        }
      }
    }
    free(psi);
  }
  return status;
}

/* ------------------------------------------------------------------ L3 beliefs (A6-A8) */

/* Weight normalization in the log domain with max subtraction:
 * M = max l, S = sum e^{l - M} (index order), lse = M + ln S, w = e^{(l - M) - ln S}
 * (l - M is exact for |l| up to 1e7 nats, so w keeps full relative precision). */
int orc_normalize(const double* l, int64_t P, double* w, double* lse) {
  double M = -INFINITY;
  for (int64_t p = 0; p < P; ++p) {
    if (l[p] != l[p]) return ORC_EINVAL;
    if (l[p] > M) M = l[p];
  }
  if (P == 0 || M == -INFINITY) { *lse = -INFINITY; return ORC_EZEROMASS; }
  double s = 0.0;
  for (int64_t p = 0; p < P; ++p) s += exp(l[p] - M);
  double ls = log(s);
  for (int64_t p = 0; p < P; ++p) w[p] = exp((l[p] - M) - ls);
  *lse = M + ls;
  return ORC_OK;
}

/* MMSE moments of the weighted set and the belief's second central moment used by
 * the regularization kernel, two-pass: est = [sum w, mean(6), cov upper-tri(21)]. */
int orc_moments(const double* x /*[P][6]*/, const double* w, int64_t P, double* est /*[28]*/) {
  double sw = 0.0, mean[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t p = 0; p < P; ++p) {
    sw += w[p];
    for (int a = 0; a < 6; ++a) mean[a] += w[p] * x[p * 6 + a];
  }
  if (!(sw > 0.0)) return ORC_EZEROMASS;
  for (int a = 0; a < 6; ++a) mean[a] /= sw;
  double cov[21] = {0};
  for (int64_t p = 0; p < P; ++p) {
    double d[6];
    for (int a = 0; a < 6; ++a) d[a] = x[p * 6 + a] - mean[a];
    int t = 0;
    for (int a = 0; a < 6; ++a)
      for (int b = a; b < 6; ++b) cov[t++] += w[p] * d[a] * d[b];
  }
  est[0] = sw;
  for (int a = 0; a < 6; ++a) est[1 + a] = mean[a];
  for (int t = 0; t < 21; ++t) est[7 + t] = cov[t] / sw;
  return ORC_OK;
}

/* Systematic resampling [Arulampalam et al., Alg. 2] on integer quantities (C-amb-15):
 * given the masses q_p, C_p = sum_{p' <= p} q_p', Q = C_{P-1}, t_i = floor((u + i 2^32) Q / (P 2^32)),
 * ancestor a_i = min{p : C_p > t_i}.  Textbook serial sweep: the pointer p advances while C_p <= t_i. */
static int orc_systematic_sweep(const uint64_t* q, int64_t P, uint32_t u_bits, int64_t* anc) {
  uint64_t* C = (uint64_t*)malloc(sizeof(uint64_t) * P);
  uint64_t run = 0;
  for (int64_t p = 0; p < P; ++p) {
    run += q[p];
    C[p] = run;
  }
  uint64_t Q = run;
  if (Q == 0) { free(C); return ORC_EZEROMASS; }
  unsigned __int128 den = (unsigned __int128)P << 32;
  int64_t ptr = 0;
  for (int64_t i = 0; i < P; ++i) {
    unsigned __int128 num = ((unsigned __int128)u_bits + ((unsigned __int128)i << 32)) * Q;
    uint64_t t = (uint64_t)(num / den);
    while (C[ptr] <= t) ++ptr;
    anc[i] = ptr;
  }
  free(C);
  return ORC_OK;
}

/* Resampling of normalized weights w (cdms_resample): q_p = rint(ldexp(w_p / w_max, 36)). */
int orc_resample(const double* w, int64_t P, uint32_t u_bits, int64_t* anc) {
  if (P <= 0 || P > ((int64_t)1 << 26)) return ORC_EINVAL;
  double wmax = 0.0;
  for (int64_t p = 0; p < P; ++p) {
    if (!(w[p] >= 0.0)) return ORC_EINVAL;
    if (w[p] > wmax) wmax = w[p];
  }
  if (!(wmax > 0.0)) return ORC_EZEROMASS;
  uint64_t* q = (uint64_t*)malloc(sizeof(uint64_t) * P);
  for (int64_t p = 0; p < P; ++p) q[p] = (uint64_t)rint(ldexp(w[p] / wmax, 36));
  int st = orc_systematic_sweep(q, P, u_bits, anc);
  free(q);
  return st;
}

/* Resampling of the BP step from the log-weights l (reading C-amb-23): the same sweep on
 * q_p = rint(ldexp(r_p, 36)), r_p = e^{l_p - M}, M = max_p l_p.  r_p equals w_p / w_max of the
 * normalized weights w_p = e^{l_p - lse} in exact arithmetic (w_max = e^{M - lse}), and r_p depends only
 * on l_p and M, so it is the quantity a sharded implementation can form per particle. */
int orc_resample_loglik(const double* l, int64_t P, uint32_t u_bits, int64_t* anc) {
  if (P <= 0 || P > ((int64_t)1 << 26)) return ORC_EINVAL;
  double M = -INFINITY;
  for (int64_t p = 0; p < P; ++p) {
    if (l[p] != l[p]) return ORC_EINVAL;
    if (l[p] > M) M = l[p];
  }
  if (M == -INFINITY) return ORC_EZEROMASS;
  uint64_t* q = (uint64_t*)malloc(sizeof(uint64_t) * P);
  for (int64_t p = 0; p < P; ++p) q[p] = (uint64_t)rint(ldexp(exp(l[p] - M), 36));
  int st = orc_systematic_sweep(q, P, u_bits, anc);
  free(q);
  return st;
}

/* ------------------------------------------------------------------ RNG + BP step (A9) */

/* Philox4x32-10 (Salmon et al., SC'11), written out; pinned by the Random123 KAT vectors. */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Four N(0,1) draws for (key, step, index, stream): Philox block -> u = (x + 1/2) 2^-32 ->
 * Box-Muller pairs (u0,u1), (u2,u3): r = sqrt(-2 ln u_a), (r cos 2 pi u_b, r sin 2 pi u_b). */
void orc_normals4(uint64_t key, uint64_t step, uint64_t index, uint32_t stream, double n[4]) {
  uint32_t ctr[4] = {(uint32_t)index, (uint32_t)(index >> 32), (uint32_t)step, stream};
  uint32_t k[2] = {(uint32_t)key, (uint32_t)(key >> 32)};
  uint32_t x[4];
  orc_philox4x32_10(ctr, k, x);
  for (int h = 0; h < 2; ++h) {
    double ua = ((double)x[2 * h] + 0.5) * 0x1p-32;
    double ub = ((double)x[2 * h + 1] + 0.5) * 0x1p-32;
    double r = sqrt(-2.0 * log(ua));
    n[2 * h] = r * cos(2.0 * ORC_PI * ub);
    n[2 * h + 1] = r * sin(2.0 * ORC_PI * ub);
  }
}

/* The resampling offset of step n: the first word of Philox(key, (0, 0, step, 3)). */
uint32_t orc_step_u_bits(uint64_t key, uint64_t step) {
  uint32_t ctr[4] = {0u, 0u, (uint32_t)step, 3u};
  uint32_t k[2] = {(uint32_t)key, (uint32_t)(key >> 32)};
  uint32_t x[4];
  orc_philox4x32_10(ctr, k, x);
  return x[0];
}

/* NCV prediction: x_n = F x_{n-1} + Gamma a, a ~ N(0, sigma_v^2 I3),
 * F = [I T I; 0 I], Gamma = [T^2/2 I; T I].  Normals: stream 0 of particle index p0 + p. */
void orc_predict(double* x /*[P][6]*/, int64_t P, int64_t p0, double T, double sigma_v,
                 uint64_t key, uint64_t step) {
  for (int64_t p = 0; p < P; ++p) {
    double n[4];
    orc_normals4(key, step, (uint64_t)(p0 + p), 0u, n);
    double* s = x + p * 6;
    for (int a = 0; a < 3; ++a) {
      double acc = sigma_v * n[a];
      s[a] = s[a] + T * s[3 + a] + 0.5 * T * T * acc;
      s[3 + a] = s[3 + a] + T * acc;
    }
  }
}

/* Regularization: x <- x + h_opt chol(Sigma) n, n ~ N(0, I6) (streams 1, 2 of the
 * slot index), h_opt = (4 / ((d + 2) P_total))^{1/(d+4)}, d = 6 (C-amb-16), Cholesky of
 * Sigma + 1e-12 tr(Sigma) I with non-positive pivots zeroing their column. */
void orc_regularize(double* x, int64_t P, int64_t p0, int64_t P_total, const double* cov21,
                    uint64_t key, uint64_t step) {
  double Sg[36], L[36];
  int t = 0;
  for (int a = 0; a < 6; ++a)
    for (int b = a; b < 6; ++b) { Sg[a * 6 + b] = cov21[t]; Sg[b * 6 + a] = cov21[t]; ++t; }
  double tr = 0.0;
  for (int a = 0; a < 6; ++a) tr += Sg[a * 6 + a];
  for (int a = 0; a < 6; ++a) Sg[a * 6 + a] += 1e-12 * tr;
  memset(L, 0, sizeof(L));
  for (int j = 0; j < 6; ++j) {
    double d = Sg[j * 6 + j];
    for (int k = 0; k < j; ++k) d -= L[j * 6 + k] * L[j * 6 + k];
    if (!(d > 0.0)) continue;
    double l = sqrt(d);
    L[j * 6 + j] = l;
    for (int i = j + 1; i < 6; ++i) {
      double acc = Sg[i * 6 + j];
      for (int k = 0; k < j; ++k) acc -= L[i * 6 + k] * L[j * 6 + k];
      L[i * 6 + j] = acc / l;
    }
  }
  double h = pow(4.0 / (8.0 * (double)P_total), 1.0 / 10.0);
  for (int64_t p = 0; p < P; ++p) {
    double n[8];
    orc_normals4(key, step, (uint64_t)(p0 + p), 1u, n);
    orc_normals4(key, step, (uint64_t)(p0 + p), 2u, n + 4);
    for (int a = 0; a < 6; ++a) {
      double acc = 0.0;
      for (int b = 0; b <= a; ++b) acc += L[a * 6 + b] * n[b];
      x[p * 6 + a] += h * acc;
    }
  }
}

/* The MT belief update that follows the likelihood (the BP step from w~_x on): normalize the log-weights l
 * (P:L3409-3410), MMSE moments of the weighted set, systematic resampling of the masses
 * e^{l - M} (orc_resample_loglik, u = orc_step_u_bits), gather of the ancestors' states, and regularization
 * with the covariance of the weighted (pre-resampling) set.
 * particles [P][6] in/out; est [28]; lse; ancestors [P] out (may be NULL). */
int orc_step_update(const double* l, double* particles, int64_t P, uint64_t key, uint64_t step, int regularize,
                    double* est, double* lse, int64_t* ancestors) {
  double* w = (double*)malloc(sizeof(double) * P);
  int64_t* a = (int64_t*)malloc(sizeof(int64_t) * P);
  double* tmp = (double*)malloc(sizeof(double) * P * 6);
  int st = orc_normalize(l, P, w, lse);
  if (st == ORC_OK) st = orc_moments(particles, w, P, est);
  if (st == ORC_OK) st = orc_resample_loglik(l, P, orc_step_u_bits(key, step), a);
  if (st == ORC_OK) {
    for (int64_t i = 0; i < P; ++i) memcpy(tmp + i * 6, particles + a[i] * 6, sizeof(double) * 6);
    memcpy(particles, tmp, sizeof(double) * P * 6);
    if (ancestors) memcpy(ancestors, a, sizeof(int64_t) * P);
    if (regularize) orc_regularize(particles, P, 0, P, est + 7, key, step);
  }
  free(w); free(a); free(tmp);
  return st;
}

/* One MT BP time step (message schedule P:L2494-2508 restricted to the MT belief):
 * predict -> loglik with uniform w_beta (dropped) -> orc_step_update.
 * particles [P][6] in/out; est [28]; lse; ancestors [P] out (may be NULL). */
int orc_bp_step(const orc_scene* sc, double* particles, int64_t P, const double* sfv,
                const double complex* y, const double complex* m, const double* v,
                const double* eta, double T, double sigma_v, uint64_t key, uint64_t step,
                int regularize, double* est, double* lse, int64_t* ancestors) {
  orc_predict(particles, P, 0, T, sigma_v, key, step);
  double* l = (double*)malloc(sizeof(double) * P);
  int st = orc_loglik(sc, particles, P, 6, sfv, 0, y, m, v, eta, NULL, l, NULL);
  if (st == ORC_OK || st == ORC_EDEGENERATE) st = orc_step_update(l, particles, P, key, step, regularize, est, lse,
                                                                   ancestors);
  free(l);
  return st;
}

/* Moment matching of the amplitude prior seen by the MT update (Prop. 1; reading
 * C-amb-7): the effective amplitude r r' rho with existence probability exist = eps * zeta and
 * rho ~ CN(mu, gamma) has mean exist mu and variance exist (gamma + |mu|^2 (1 - exist)). */
void orc_moment_match(double mu_re, double mu_im, double gamma, double exist, double* out /*m_re,m_im,v*/) {
  out[0] = exist * mu_re;
  out[1] = exist * mu_im;
  out[2] = exist * (gamma + (mu_re * mu_re + mu_im * mu_im) * (1.0 - exist));
}

/* ------------------------------------------------------------------ F3 birth proposal */

/* Observation residual z~_j = Pi_perp_j z_j, Pi_perp_j = I - Psi_j Psi_j^dagger with
 * Psi_j = [psi(x_hat, LOS) psi(x_hat, sfv_1) ... psi(x_hat, sfv_L)] in C^{Nz x (L+1)}, the
 * steering vectors at the predicted MMSE state for the LOS and the legacy PFs' MMSE SFVs.  Psi^dagger is the
 * pseudo-inverse of a full-column-rank Psi: Psi^dagger z = (Psi^H Psi)^{-1} Psi^H z, solved by Cholesky.
 * y, z~: [J][Nz] (n = k Na + m).  ORC_EINVAL if Psi^H Psi is singular. */
int orc_birth_residual(const orc_scene* sc, const double* x_hat /*[3]*/, const double* sfv_legacy /*[L][3]*/,
                       int L, const double complex* y, double complex* zr) {
  int n = L + 1, J = sc->J;
  size_t nz = (size_t)sc->nf * sc->ny * sc->nv;
  double complex* Psi = (double complex*)malloc(sizeof(double complex) * nz * n);
  double complex* G = (double complex*)malloc(sizeof(double complex) * n * n);
  double complex* b = (double complex*)malloc(sizeof(double complex) * n);
  int st = ORC_OK;
  for (int j = 0; j < J && !st; ++j) {
    for (int s = 0; s < n && !st; ++s)
      st = orc_response(sc, x_hat, j, s, s ? sfv_legacy + 3 * (s - 1) : NULL, sc->wavefront, Psi + (size_t)s * nz);
    if (st) break;
    const double complex* z = y + (size_t)j * nz;
    for (int r = 0; r < n; ++r) {  /* Psi^H Psi (lower part) and Psi^H z */
      for (int c = 0; c <= r; ++c) {
        double complex acc = 0.0;
        for (size_t k = 0; k < nz; ++k) acc += conj(Psi[(size_t)r * nz + k]) * Psi[(size_t)c * nz + k];
        G[r * n + c] = acc;
      }
      double complex acc = 0.0;
      for (size_t k = 0; k < nz; ++k) acc += conj(Psi[(size_t)r * nz + k]) * z[k];
      b[r] = acc;
    }
    st = orc_cholesky(G, n);  /* G = L L^H */
    if (st) break;
    for (int r = 0; r < n; ++r) {  /* L w = b */
      double complex acc = b[r];
      for (int c = 0; c < r; ++c) acc -= G[r * n + c] * b[c];
      b[r] = acc / G[r * n + r];
    }
    for (int r = n - 1; r >= 0; --r) {  /* L^H a = w */
      double complex acc = b[r];
      for (int c = r + 1; c < n; ++c) acc -= conj(G[c * n + r]) * b[c];
      b[r] = acc / G[r * n + r];
    }
    double complex* out = zr + (size_t)j * nz;
    for (size_t k = 0; k < nz; ++k) {  /* z~ = z - Psi a */
      double complex acc = z[k];
      for (int s = 0; s < n; ++s) acc -= Psi[(size_t)s * nz + k] * b[s];
      out[k] = acc;
    }
  }
  free(Psi);
  free(G);
  free(b);
  return st;
}

/* Candidate i of the draw (key, counter): p_i = lo + u (hi - lo), u_a = (x_a + 1/2) 2^-32 from the Philox block
 * (key; i, i >> 32, counter, 7) (reading C-amb-F3b: the partition P_q is the axis-aligned box [lo, hi]). */
void orc_birth_candidate(uint64_t key, uint64_t counter, int64_t i, const double* box /*[6] lo, hi*/,
                         double* p /*[3]*/) {
  uint32_t ctr[4] = {(uint32_t)i, (uint32_t)((uint64_t)i >> 32), (uint32_t)counter, 7u};
  uint32_t k[2] = {(uint32_t)key, (uint32_t)(key >> 32)};
  uint32_t x[4];
  orc_philox4x32_10(ctr, k, x);
  for (int a = 0; a < 3; ++a) {
    double u = ((double)x[a] + 0.5) * 0x1p-32;
    p[a] = box[a] + u * (box[3 + a] - box[a]);
  }
}

/* Bartlett birth proposal for one new PF:
 *   candidates p_i ~ U(P_q), i < N_g (orc_birth_candidate);
 *   P_B(p_i, z~) = | sum_j (1/N_z) z~_j^H psi(x_hat, p_i) |^2  (coherent over the PAs; psi of the wall p_i,
 *   component s = 1 of PA j);
 *   w_i = P_B_i / sum P_B;  mu = p_{i*}, i* = argmax_i P_B_i (first index on ties);
 *   C = sum_i w_i (p_i - mu)(p_i - mu)^T.
 * Outputs pb[N_g], cand[N_g][3] (either may be NULL), mu[3], C[9] (row-major), *istar.  ORC_EZEROMASS when
 * sum P_B = 0 (the residual has no power), errors of the responses / residual are passed on. */
int orc_birth_proposal(const orc_scene* sc, const double* x_hat, const double* sfv_legacy, int L,
                       const double complex* y, const double* box, int64_t N_g, uint64_t key, uint64_t counter,
                       double* pb, double* cand, double* mu, double* Cov, int64_t* istar) {
  int J = sc->J;
  size_t nz = (size_t)sc->nf * sc->ny * sc->nv;
  if (N_g <= 0) return ORC_EINVAL;
  double complex* zr = (double complex*)malloc(sizeof(double complex) * nz * J);
  int st = orc_birth_residual(sc, x_hat, sfv_legacy, L, y, zr);
  double* P = (double*)malloc(sizeof(double) * N_g);
  double* X = (double*)malloc(sizeof(double) * 3 * N_g);
  double complex* psi = (double complex*)malloc(sizeof(double complex) * nz);
  for (int64_t i = 0; i < N_g && !st; ++i) {
    orc_birth_candidate(key, counter, i, box, X + 3 * i);
    double complex acc = 0.0;
    for (int j = 0; j < J && !st; ++j) {
      st = orc_response(sc, x_hat, j, 1, X + 3 * i, sc->wavefront, psi);
      double complex cj = 0.0;
      for (size_t k = 0; k < nz; ++k) cj += conj(zr[(size_t)j * nz + k]) * psi[k];
      acc += cj / (double)nz;
    }
    P[i] = creal(acc) * creal(acc) + cimag(acc) * cimag(acc);
  }
  double sum = 0.0;
  int64_t best = 0;
  if (!st) {
    for (int64_t i = 0; i < N_g; ++i) {
      sum += P[i];
      if (P[i] > P[best]) best = i;
    }
    if (!(sum > 0.0)) st = ORC_EZEROMASS;
  }
  if (!st) {
    for (int a = 0; a < 3; ++a) mu[a] = X[3 * best + a];
    for (int q = 0; q < 9; ++q) Cov[q] = 0.0;
    for (int64_t i = 0; i < N_g; ++i) {
      double w = P[i] / sum, d[3];
      for (int a = 0; a < 3; ++a) d[a] = X[3 * i + a] - mu[a];
      for (int a = 0; a < 3; ++a)
        for (int b2 = 0; b2 < 3; ++b2) Cov[3 * a + b2] += w * d[a] * d[b2];
    }
    *istar = best;
    if (pb) memcpy(pb, P, sizeof(double) * N_g);
    if (cand) memcpy(cand, X, sizeof(double) * 3 * N_g);
  }
  free(zr);
  free(P);
  free(X);
  free(psi);
  return st;
}

/* ------------------------------------------------------------------ F1 PF-particle update (S-V) */

/* a^H A^{-1} b with A = eta I + M M^H through the inversion lemma (eq. S-Maha-expression):
 *   a^H b / eta - (a^H M) (I + M^H M / eta)^{-1} (M^H b) / eta^2.
 * M = [m_1 .. m_L] (columns of length nz); Kc = the Cholesky factor (lower, row-major L x L) of I + M^H M / eta. */
static double complex orc_maha(const double complex* a, const double complex* b, const double complex* M, int L,
                               const double complex* Kc, double eta, size_t nz) {
  double complex ab = 0.0, u[16], v[16];
  for (size_t n = 0; n < nz; ++n) ab += conj(a[n]) * b[n];
  for (int l = 0; l < L; ++l) {
    double complex am = 0.0, mb = 0.0;
    for (size_t n = 0; n < nz; ++n) {
      am += conj(a[n]) * M[(size_t)l * nz + n];
      mb += conj(M[(size_t)l * nz + n]) * b[n];
    }
    u[l] = conj(am);  /* M^H a */
    v[l] = mb;        /* M^H b */
  }
  /* (M^H a)^H K^{-1} (M^H b) = (L^{-1} M^H a)^H (L^{-1} M^H b) */
  for (int r = 0; r < L; ++r) {
    for (int c = 0; c < r; ++c) {
      u[r] -= Kc[r * L + c] * u[c];
      v[r] -= Kc[r * L + c] * v[c];
    }
    u[r] /= creal(Kc[r * L + r]);
    v[r] /= creal(Kc[r * L + r]);
  }
  double complex q = 0.0;
  for (int l = 0; l < L; ++l) q += conj(u[l]) * v[l];
  return ab / eta - q / (eta * eta);
}

/* F1: the approximate PF update message kappa~(phi_p, r; z^(j)) (Supplement S-V "PF State Update
 * Message") evaluated at the particles of one PF s, and the PF weights with the normalization constant
 * M_{y,s,n} (Supplement S-IV).  Readings (C-amb-F1a..d):
 *   - the PF particles are paired with the MT particles by index (C-amb-8): psi_p = psi^(j)(x_p, phi_p), the response
 *     of PA j at MT particle x_p through the wall of SFV phi_p (component 1 of orc_response);
 *   - covariance C^kappa = r q_p psi_p psi_p^H + A, A = eta_j I + M M^H, q_p = (gamma_p +
 *     |mu_p|^2 (1 - zeta_j)) zeta_j; mean mu^kappa = r zeta_j mu_p psi_p + mu3_j;
 *   - the particle-independent terms mu3_j = sum_{s' != s} mu~_3 and the columns m_l of M (l < L) are inputs
 *     ("precomputed once");
 *   - det A and pi^Nz cancel between r = 1 and the H0 branch r = 0, so the per-particle result
 *     is logr_p = log w_alpha_p + sum_j [log kappa~(phi_p, 1; z_j) - log kappa~(., 0; z_j)], with
 *       log kappa~(phi_p, 1) - log kappa~(., 0) = q |psi^H A^-1 e|^2 / (1 + q psi^H A^-1 psi) - e^H A^-1 e
 *                                                - ln(1 + q psi^H A^-1 psi) + e0^H A^-1 e0,
 *     e = z_j - mu^kappa(phi_p, 1), e0 = z_j - mu3_j (the determinant lemma and the inversion lemma of);
 *   - normalization in units of prod_j kappa~(., 0): M_y = sum_p e^{logr_p} + (1 - sum_p w_alpha_p) (S-IV),
 *     PF weights w_p = e^{logr_p} / M_y, posterior existence sum_p w_p (eq. existenceProb).
 * y, mu3: [J][Nz]; mcols: [J][L][Nz]; x: [P][pstride]; phi: [P][3], or NULL for the LOS PF s = 0.
 * out[0] = log M_y, out[1] = existence. */
int orc_pf_update(const orc_scene* sc, const double* x, int64_t P, int pstride, const double* phi,
                  const double* walpha, const double complex* mu, const double* gamma, const double* zeta,
                  const double* eta, const double complex* y, const double complex* mu3,
                  const double complex* mcols, int L, double* logr, double* w, double* out) {
  int J = sc->J;
  size_t nz = (size_t)sc->nf * sc->ny * sc->nv;
  if (P <= 0 || L < 0 || L > 15) return ORC_EINVAL;
  int status = ORC_OK;
  for (int64_t p = 0; p < P; ++p) logr[p] = log(walpha[p]);
  double complex* e0 = (double complex*)malloc(sizeof(double complex) * nz);
  double complex* psi = (double complex*)malloc(sizeof(double complex) * nz);
  double complex* e = (double complex*)malloc(sizeof(double complex) * nz);
  double complex Kc[256];
  for (int j = 0; j < J && status == ORC_OK; ++j) {
    const double complex* M = mcols + (size_t)j * L * nz;
    /* the H0 error vector and the Cholesky factor of I + M^H M / eta (particle independent) */
    for (size_t n = 0; n < nz; ++n) e0[n] = y[(size_t)j * nz + n] - mu3[(size_t)j * nz + n];
    for (int a = 0; a < L; ++a)
      for (int b = 0; b < L; ++b) {
        double complex g = 0.0;
        for (size_t n = 0; n < nz; ++n) g += conj(M[(size_t)a * nz + n]) * M[(size_t)b * nz + n];
        Kc[a * L + b] = (a == b ? 1.0 : 0.0) + g / eta[j];
      }
    if (L > 0 && orc_cholesky(Kc, L)) { status = ORC_EINVAL; break; }
    double t0 = creal(orc_maha(e0, e0, M, L, Kc, eta[j], nz));
    for (int64_t p = 0; p < P && status == ORC_OK; ++p) {
      /* phi == NULL: the PF is the LOS s = 0 (no SFV, component 0 of orc_response) */
      int st = phi ? orc_response(sc, x + p * pstride, j, 1, phi + 3 * p, sc->wavefront, psi)
                   : orc_response(sc, x + p * pstride, j, 0, NULL, sc->wavefront, psi);
      if (st) { status = st; logr[p] = -INFINITY; continue; }
      double complex c = zeta[j] * mu[p];
      for (size_t n = 0; n < nz; ++n) e[n] = e0[n] - c * psi[n];   /* e = z - mu^kappa(phi_p, 1) */
      double beta = creal(orc_maha(psi, psi, M, L, Kc, eta[j], nz));
      double complex b = orc_maha(psi, e, M, L, Kc, eta[j], nz);
      double t1 = creal(orc_maha(e, e, M, L, Kc, eta[j], nz));
      double q = (gamma[p] + creal(mu[p] * conj(mu[p])) * (1.0 - zeta[j])) * zeta[j];
      double den = 1.0 + q * beta;
      logr[p] += q * creal(b * conj(b)) / den - t1 - log(den) + t0;
    }
  }
  free(e0); free(psi); free(e);
  if (status) return status;
  /* M_y = sum_p e^{logr_p} + (1 - sum_p w_alpha_p), in index order with the max taken out */
  double mx = -INFINITY, sa = 0.0;
  for (int64_t p = 0; p < P; ++p) {
    if (logr[p] > mx) mx = logr[p];
    sa += walpha[p];
  }
  double h0 = 1.0 - sa;
  if (h0 < 0.0) h0 = 0.0;
  double s = 0.0;
  if (mx > -INFINITY)
    for (int64_t p = 0; p < P; ++p) s += exp(logr[p] - mx);
  double logM;
  if (mx == -INFINITY) logM = log(h0);
  else logM = mx + log(s + h0 * exp(-mx));
  double ex = 0.0;
  for (int64_t p = 0; p < P; ++p) {
    double wp = exp(logr[p] - logM);
    if (w) w[p] = wp;
    ex += wp;
  }
  out[0] = logM;
  out[1] = ex;
  return ORC_OK;
}

/* ------------------------------------------------------------------ F4 parts: noise (nu~) and PPR (omega~) updates */

/* Noise variance update message nu~ (Supplement S-V "Noise Variance Update Message") at the noise
 * particles eta_p^(j) of every PA, and the normalized noise weights:
 *   A_p = eta_p I + M M^H, M = [m_0 .. m_{S-1}] (all features' columns), e = z - mu_nu (mu_nu = sum_s mu~_3),
 *   log nu~ = -Nz ln(pi eta_p) - ln det(I + M^H M / eta_p) - ||e||^2/eta_p
 *             + ||(I + M^H M/eta_p)^{-1/2} M^H e||^2 / eta_p^2,
 *   w~_p = w_xi,p nu~_p,  w_p = w~_p / sum_p w~_p (per PA).
 * Per particle: the S x S Cholesky of I + M^H M / eta_p (the paper's order: Gram once, factor per particle).
 * eta, wxi, logw, w: [J][P]; y, mu: [J][Nz]; mcols [J][S][Nz].  lognorm [J] = log sum_p w~_p. */
int orc_noise_update(const orc_scene* sc, const double* eta, const double* wxi, int64_t P, const double complex* y,
                     const double complex* mu, const double complex* mcols, int S, double* logw, double* w,
                     double* lognorm) {
  int J = sc->J;
  size_t nz = (size_t)sc->nf * sc->ny * sc->nv;
  if (P <= 0 || S < 0 || S > 15) return ORC_EINVAL;
  double complex* e = (double complex*)malloc(sizeof(double complex) * nz);
  double complex G[256], Me[16], K[256];
  int status = ORC_OK;
  for (int j = 0; j < J && status == ORC_OK; ++j) {
    const double complex* M = mcols + (size_t)j * S * nz;
    double e2 = 0.0;
    for (size_t n = 0; n < nz; ++n) {
      e[n] = y[(size_t)j * nz + n] - mu[(size_t)j * nz + n];
      e2 += creal(e[n] * conj(e[n]));
    }
    for (int a = 0; a < S; ++a) {
      double complex acc = 0.0;
      for (size_t n = 0; n < nz; ++n) acc += conj(M[(size_t)a * nz + n]) * e[n];
      Me[a] = acc;
      for (int b = 0; b < S; ++b) {
        double complex g = 0.0;
        for (size_t n = 0; n < nz; ++n) g += conj(M[(size_t)a * nz + n]) * M[(size_t)b * nz + n];
        G[a * S + b] = g;
      }
    }
    double mx = -INFINITY;
    for (int64_t p = 0; p < P; ++p) {
      double et = eta[(size_t)j * P + p];
      if (!(et > 0.0)) { status = ORC_EINVAL; break; }
      for (int a = 0; a < S; ++a)
        for (int b = 0; b < S; ++b) K[a * S + b] = (a == b ? 1.0 : 0.0) + G[a * S + b] / et;
      if (S > 0 && orc_cholesky(K, S)) { status = ORC_EINVAL; break; }
      double logdet = 0.0, q2 = 0.0;
      double complex x[16];
      for (int a = 0; a < S; ++a) {  /* L x = M^H e */
        double complex acc = Me[a];
        for (int b = 0; b < a; ++b) acc -= K[a * S + b] * x[b];
        x[a] = acc / creal(K[a * S + a]);
        q2 += creal(x[a] * conj(x[a]));
        logdet += 2.0 * log(creal(K[a * S + a]));
      }
      double lnu = -(double)nz * log(ORC_PI * et) - logdet - e2 / et + q2 / (et * et);
      logw[(size_t)j * P + p] = log(wxi[(size_t)j * P + p]) + lnu;
      if (logw[(size_t)j * P + p] > mx) mx = logw[(size_t)j * P + p];
    }
    if (status) break;
    double s = 0.0;
    for (int64_t p = 0; p < P; ++p) s += exp(logw[(size_t)j * P + p] - mx);
    lognorm[j] = mx + log(s);
    if (w)
      for (int64_t p = 0; p < P; ++p) w[(size_t)j * P + p] = exp(logw[(size_t)j * P + p] - lognorm[j]);
  }
  free(e);
  return status;
}

/* PPR update message omega~ (Supplement S-V "PR State Update Message") and the PPR existence revival
 * (Supplement S-VI) of one PF s at every PA j:
 *   C^omega(r) = r m_omega m_omega^H + A, A = eta_j I + M M^H (M^omega = M^kappa: the other features' columns),
 *   mu^omega(r) = r mu~_4 + mu3,
 *   log omega~(1) - log omega~(0) = |m_omega^H A^-1 e1|^2 / (1 + m_omega^H A^-1 m_omega) - e1^H A^-1 e1
 *                                   + e0^H A^-1 e0 - ln(1 + m_omega^H A^-1 m_omega),  e_r = z - mu^omega(r)
 *   (rank-1 inversion and determinant lemmas; det A and pi^Nz cancel between r = 1 and r = 0),
 *   u = log(zeta / (1 - zeta)) + that log ratio, posterior existence sigma(u) = 1 / (1 + e^-u).
 * y, mu3, momega, mu4: [J][Nz]; mcols [J][L][Nz]; zeta, eta [J].  out [J][3] = (log ratio, u, sigma(u)). */
int orc_ppr_update(const orc_scene* sc, const double* zeta, const double* eta, const double complex* y,
                   const double complex* mu3, const double complex* mcols, int L, const double complex* momega,
                   const double complex* mu4, double* out) {
  int J = sc->J;
  size_t nz = (size_t)sc->nf * sc->ny * sc->nv;
  if (L < 0 || L > 15) return ORC_EINVAL;
  double complex* e0 = (double complex*)malloc(sizeof(double complex) * nz);
  double complex* e1 = (double complex*)malloc(sizeof(double complex) * nz);
  double complex Kc[256];
  int status = ORC_OK;
  for (int j = 0; j < J && status == ORC_OK; ++j) {
    const double complex* M = mcols + (size_t)j * L * nz;
    const double complex* mw = momega + (size_t)j * nz;
    for (size_t n = 0; n < nz; ++n) {
      e0[n] = y[(size_t)j * nz + n] - mu3[(size_t)j * nz + n];
      e1[n] = e0[n] - mu4[(size_t)j * nz + n];
    }
    for (int a = 0; a < L; ++a)
      for (int b = 0; b < L; ++b) {
        double complex g = 0.0;
        for (size_t n = 0; n < nz; ++n) g += conj(M[(size_t)a * nz + n]) * M[(size_t)b * nz + n];
        Kc[a * L + b] = (a == b ? 1.0 : 0.0) + g / eta[j];
      }
    if (L > 0 && orc_cholesky(Kc, L)) { status = ORC_EINVAL; break; }
    double alpha = creal(orc_maha(mw, mw, M, L, Kc, eta[j], nz));
    double complex b1 = orc_maha(mw, e1, M, L, Kc, eta[j], nz);
    double t1 = creal(orc_maha(e1, e1, M, L, Kc, eta[j], nz));
    double t0 = creal(orc_maha(e0, e0, M, L, Kc, eta[j], nz));
    double lr = creal(b1 * conj(b1)) / (1.0 + alpha) - t1 + t0 - log(1.0 + alpha);
    double u = log(zeta[j] / (1.0 - zeta[j])) + lr;
    out[3 * j + 0] = lr;
    out[3 * j + 1] = u;
    out[3 * j + 2] = 1.0 / (1.0 + exp(-u));
  }
  free(e0); free(e1);
  return status;
}

/* ------------------------------------------------------------------ F4: Gamma transitions */

/* One Gamma(c, 1) draw, c >= 1, by Marsaglia and Tsang's squeeze-free acceptance test (ACM TOMS 26(3), 2000):
 * d = c - 1/3, k = 1/sqrt(9 d); attempt a = 0, 1, ...: z ~ N(0, 1), u ~ U(0, 1), v = (1 + k z)^3; accept d v if v > 0
 * and ln u < z^2/2 + d - d v + d ln v.  Attempt a draws the Philox block (key; index, index >> 32, step,
 * stream + a): z = sqrt(-2 ln u0) cos(2 pi u1) from words 0, 1 and u from word 2 (u_i = (x_i + 1/2) 2^-32), a < 16;
 * after 16 rejections the draw is d (probability below 1e-25 for c >= 10; reading F4-g).
 * The transitions of P:L3783-3795 use it as eta_n = eta_{n-1} g / c_eta and gamma_n = gamma_{n-1} g / c_gamma,
 * g ~ Gamma(c, 1): the Gamma pdf G(.; c, theta / c) with mean theta. */
double orc_gamma_draw(uint64_t key, uint64_t step, uint64_t index, uint32_t stream, double c) {
  double d = c - 1.0 / 3.0, k = 1.0 / sqrt(9.0 * d);
  uint32_t kk[2] = {(uint32_t)key, (uint32_t)(key >> 32)};
  for (uint32_t a = 0; a < 16; ++a) {
    uint32_t ctr[4] = {(uint32_t)index, (uint32_t)(index >> 32), (uint32_t)step, stream + a};
    uint32_t x[4];
    orc_philox4x32_10(ctr, kk, x);
    double u0 = ((double)x[0] + 0.5) * 0x1p-32, u1 = ((double)x[1] + 0.5) * 0x1p-32;
    double u = ((double)x[2] + 0.5) * 0x1p-32;
    double z = sqrt(-2.0 * log(u0)) * cos(2.0 * ORC_PI * u1);
    double t = 1.0 + k * z;
    if (t <= 0.0) continue;
    double v = t * t * t;
    if (log(u) < 0.5 * z * z + d - d * v + d * log(v)) return d * v;
  }
  return d;
}
