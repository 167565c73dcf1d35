/*
 * cdms.h -- C ABI of libcdms, the B200-native (sm_100a) coherent-likelihood engine for the MT
 * belief update of "Coherent Direct Multipath SLAM" (arxiv 2604.19723).
 *
 * Citations: P:Lnnn = line of PAPER.md (the paper), S:Lnnn = line of SPEC.md, C-amb-n = reading of
 * an ambiguous passage (section "Readings").
 *
 * Conventions (all entry points):
 *  - d_* arguments are CUDA DEVICE pointers owned by the CALLER (e.g. torch tensors) on the device
 *    of the context; h_* arguments are HOST pointers owned by the caller and read only during the
 *    call (the library copies what it keeps).  Arrays are dense, row-major, no padding.
 *  - complex64 = interleaved (re, im) float32 pairs; complex128 = interleaved float64 pairs.
 *  - Every device operation is enqueued on the context's stream; nothing synchronizes the host
 *    except cdms_sync() (and the test-only loopback backend's host barriers).  With several ranks the
 *    distributed resampling plan is formed on the device from the all-gathered masses and the
 *    redistribution is fused into the ancestor gather (each slot's state is written into its owner
 *    rank's buffer over NVLink peer memory), so calls are capturable into a CUDA graph once their
 *    workspaces exist (first call outside capture, or cdms_reserve(), collective with a communicator).
 *  - Concurrency: a context is one in-order worker -- its workspaces (including the device-side
 *    work-claim counters of the likelihood kernel and the step pipeline, which the last CTA of each
 *    launch resets) are shared by its calls, so calls on one context must not overlap on different
 *    streams.  Separate contexts are independent.
 *  - Errors: host-checkable problems (NULL pointers, sizes <= 0, ||sfv|| = 0, R not in SO(3),
 *    non-uniform f_pb, non-finite or negative priors) return CDMS_EINVAL BEFORE any launch and
 *    leave outputs untouched.  Device-detected conditions set a sticky flag that cdms_sync()
 *    returns: CDMS_EDEGENERATE (MT on a phase centre or antenna, P:L2137 -- that particle gets
 *    l = -inf), CDMS_EZEROMASS (all weights zero / all l = -inf: outputs untouched, lse = -inf),
 *    CDMS_EINVAL (NaN in device inputs).  cdms_last_error() gives a message.
 *  - Determinism: per-particle results do not depend on launch geometry, tile placement or rank
 *    count (fixed per-particle reduction order); cross-particle reductions are fp64 in a fixed
 *    order; resampling is integer arithmetic and therefore exact.
 *  - Multi-GPU: after cdms_comm_init(), cdms_weights_normalize, cdms_moments, cdms_resample and
 *    cdms_bp_step are COLLECTIVE over the ranks (every rank calls them, each with its P_local
 *    particles; global particle index = rank * P_local + local index, P_local equal on all ranks).
 *    cdms_loglik, cdms_response and cdms_layout are purely local.
 *  - Engines: FP32 spherical and planar-WB likelihoods evaluate the correlation from per-call spectral Taylor
 *    tables of the snapshot (K1T; tables in the context workspace, (G + 1) N_a 64 bytes per
 *    PA, G = 4 N_f, up to 96 MB, else K1) and the Gram in closed form; FP64 evaluations run the segmented Horner
 *    correlation (K1); PLANAR_NB in FP32 runs its correlation on the tensor cores (tcgen05, error-free fp16
 *    split) with a closed-form Gram.  All engines meet the same parity tolerances.
 *    Environment knobs read at cdms_create, for A/B measurements only: CDMS_TAYLOR=0 (K1 instead of K1T),
 *    CDMS_TAYLOR_GRAM=k1 (K1T's off-diagonal Gram from K1's Horner-free variant), CDMS_TAY_LANES=0/1 (force
 *    K1T's thread-per-particle / lane-group kernel; default by P J), CDMS_TAY_PREP=direct (direct-sum tables
 *    instead of the FFT), CDMS_STEP_FUSED=1 (single-rank bp_step O(P) phases in one cooperative kernel; results
 *    identical), CDMS_NB_TENSOR=0 keeps PLANAR_NB on the FP32 pipe, CDMS_NB_ATMEM=0 keeps the tensor path's A
 *    operand in shared memory.
 */
#ifndef CDMS_H_
#define CDMS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cdms_ctx_s* cdms_ctx;
typedef struct cdms_loopback_s* cdms_loopback;

typedef enum {
  CDMS_OK = 0,
  CDMS_EINVAL = 1,
  CDMS_EDEGENERATE = 2,
  CDMS_EZEROMASS = 3,
  CDMS_ENOMEM = 4,
  CDMS_ECUDA = 5,
  CDMS_ENCCL = 6,
  CDMS_EUNSUPPORTED = 7
} cdms_status;

/* Array-response model (C-amb-5): spherical wideband (default), planar wideband
 * (P:L118-143), planar narrowband Kronecker. */
typedef enum { CDMS_SPHERICAL = 0, CDMS_PLANAR_WB = 1, CDMS_PLANAR_NB = 2 } cdms_wavefront;

/* Inner-loop precision of the correlation / Gram (C-amb-18): FP32 (default, fp64 geometry and
 * assembly) or FP64 end to end. */
typedef enum { CDMS_FP32 = 0, CDMS_FP64 = 1 } cdms_precision;

/* Scene: J PAs with identical N_y x N_v URAs (template P~ in the local yz-plane, column
 * m = iy*nv + iv), K walls (S = K+1 propagation components, s = 0 LOS), N_f subcarriers
 * f_pb[k] = fc + (k - (nf-1)/2) * df.  Limits: 1 <= J <= 8,
 * 0 <= K <= 8, 1 <= nf <= 65536, 1 <= ny*nv <= 4096. */
typedef struct {
  int32_t J, K;
  int32_t ny, nv;
  int32_t nf;
  int32_t wavefront;     /* cdms_wavefront */
  int32_t pathloss;      /* 1: psi = lambda/(4 pi ||r'||) psi~ (C-amb-6) */
  int32_t precision;     /* cdms_precision */
  double dy, dv;         /* element spacing (m) */
  double fc, df;         /* carrier and subcarrier spacing (Hz) */
  const double* h_pa_pos;  /* [J][3] PA phase centres p_j (m) */
  const double* h_pa_rot;  /* [J][3][3] row-major R_j in SO(3) (checked to 1e-9) */
} cdms_scene;

/* Per-(PA j, component s) amplitude prior seen by the MT update: mean m, variance v >= 0
 * (moment-matched, reading C-amb-7; cdms_moment_match gives the map). */
typedef struct {
  double m_re, m_im, v;
} cdms_prior;

/* ---- context ------------------------------------------------------------------------------ */

/* Create a context bound to CUDA device `device` and stream `cuda_stream` (a cudaStream_t, may be
 * NULL = legacy default stream).  The context owns its workspaces and (optionally) an NCCL
 * communicator; it is not thread-safe. */
cdms_status cdms_create(cdms_ctx* out, int device, void* cuda_stream);
cdms_status cdms_destroy(cdms_ctx ctx);
/* Re-bind the stream used by subsequent calls (e.g. torch.cuda.current_stream()). */
cdms_status cdms_set_stream(cdms_ctx ctx, void* cuda_stream);
/* Human-readable description of the last error on this context (static storage of the ctx). */
const char* cdms_last_error(cdms_ctx ctx);
/* Synchronize the stream; returns the sticky device flag (see conventions) and clears it. */
cdms_status cdms_sync(cdms_ctx ctx);
/* Pre-size the workspaces for up to P_local particles and the given scene (so that later calls
 * can be captured in a CUDA graph). */
cdms_status cdms_reserve(cdms_ctx ctx, const cdms_scene* scene, int64_t P_local);
/* Number of library kernel launches enqueued by this context so far (for launch accounting). */
int64_t cdms_launch_count(cdms_ctx ctx);
/* Kernel timing: while enabled, every launch of the likelihood kernel (rows A2-A5) is bracketed by CUDA
 * events on the context's stream.  cdms_timing_read synchronizes those events and returns the summed
 * kernel time (ms) and the number of launches since the last enable; it does not disable timing. */
cdms_status cdms_timing_enable(cdms_ctx ctx, int on);
cdms_status cdms_timing_read(cdms_ctx ctx, double* loglik_ms, int64_t* n_launches);
/* The same events split by kernel: ms[0] the correlation kernel (row A3), ms[1] the Gram kernel (row A4; 0 when the
 * engine computes both in one kernel), ms[2] the S x S assembly (row A5), summed over *n_launches batches. */
cdms_status cdms_timing_read_stages(cdms_ctx ctx, double ms[3], int64_t* n_launches);

/* NCCL bootstrap: rank 0 calls cdms_get_unique_id, broadcasts the 128 bytes (e.g. through
 * torch.distributed), then every rank calls cdms_comm_init.  nranks = 1 is allowed. */
cdms_status cdms_get_unique_id(unsigned char nccl_unique_id_out[128]);
cdms_status cdms_comm_init(cdms_ctx ctx, const unsigned char nccl_unique_id[128], int rank,
                           int nranks);

/* TEST backend for the multi-rank path on one GPU: nranks contexts of ONE process, each driven by its
 * own host thread, form a group whose collectives are host barriers plus device copies (instead of NCCL) and whose
 * peer buffers are the other contexts' device buffers.  Every collective entry point (cdms_weights_normalize,
 * cdms_moments, cdms_resample, cdms_bp_step, cdms_bp_update, cdms_reserve) then runs exactly the device code of the
 * NCCL path.  The group must outlive its contexts; a context takes either NCCL or a loopback group, once. */
cdms_status cdms_loopback_create(int nranks, cdms_loopback* out);
cdms_status cdms_loopback_destroy(cdms_loopback group);
cdms_status cdms_comm_init_loopback(cdms_ctx ctx, cdms_loopback group, int rank);

/* ---- row A1: anchor geometry ----------------------------------------------------------------- */

/* Householder matrices H_s = I - 2 s s^T/||s||^2 (H_0 = I), VA phase centres
 * p_VA,js = p_j - (2 p_j^T s/||s||^2 - 1) s (p_VA,j0 = p_j) and VA layouts
 * P_{j,s} = p_VA,js 1^T + H_s R_j P~, computed on the device with the same functions the
 * likelihood kernel uses.  d_sfv [K][3] (fp64).  Outputs (device, fp64): d_layout [J][S][3][Na],
 * d_va [J][S][3], d_H [S][3][3].  ||sfv_k|| = 0 -> CDMS_EINVAL. */
cdms_status cdms_layout(cdms_ctx ctx, const cdms_scene* scene, const double* d_sfv,
                        double* d_layout, double* d_va, double* d_H);

/* ---- rows A2-A5: coherent log-likelihood ----------------------------------------------------- */

/* For every particle p: l_p = log w_beta(p) + sum_j log iota~(x_p; z^(j)) with the
 * low-rank evaluation of the MT update message (Supplement S-V-C):
 *   log iota~ = -Nz ln(pi eta_j) - ln det(I + M^H M/eta_j) - ||e||^2/eta_j
 *               + ||(I + M^H M/eta_j)^{-1/2} M^H e||^2 / eta_j^2,
 * M = Psi_j(x_p) V_j^{1/2}, e = z^(j) - Psi_j(x_p) m_j, Psi_j = [psi_j,0 .. psi_j,K] the unit-modulus
 * responses of the scene's wavefront model, which equals log CN(z; Psi m, eta I + Psi V Psi^H)
 * (P:L2217-2224).
 *   d_particles [P][pstride] fp64, position = first 3 entries (velocity does not enter, C-amb-21).
 *   d_sfv       fp64 [K][3] (sfv_per_particle = 0) or [P][K][3] (= 1, C-amb-8).
 *   d_y         complex64 [J][nf][Na]: z^(j) in the paper's vec order, n = k*Na + m (C-amb-1).
 *   h_f_pb      [nf] passband grid; must equal the scene grid to 1e-9 relative (uniformity check).
 *   h_prior     [J][S]; h_eta [J] noise variances eta_j > 0 (C-amb-10).
 *   d_logw_prior [P] fp64 or NULL (= 0).
 *   d_loglik    out [P] fp64.
 *   d_amp       out complex128 [P][J][S] LMMSE amplitudes m + V^1/2 K^-1 M^H e / eta, or NULL.
 * Purely local (no communication).  Degenerate particles: l = -inf + CDMS_EDEGENERATE at sync.
 * PLANAR_NB in FP32: correlation on the tensor cores (see Conventions, "Engines"). */
cdms_status cdms_loglik(cdms_ctx ctx, const cdms_scene* scene, const double* d_particles,
                        int64_t P, int32_t pstride, const double* d_sfv, int32_t sfv_per_particle,
                        const void* d_y, const double* h_f_pb, const cdms_prior* h_prior,
                        const double* h_eta, const double* d_logw_prior, double* d_loglik,
                        void* d_amp);

/* Sufficient statistics of rows A3/A4 as the likelihood kernel computes them (same launch, same
 * arithmetic): the correlation c_s = psi_s^H z^(j) ("M^H e" with e = z) and the Gram
 * G_ab = psi_a^H psi_b (P:L769 fn), path-loss gains applied.  Arguments as cdms_loglik,
 * plus d_c out complex128 [P][J][S] and d_G out complex128 [P][J][S][S] (full Hermitian).  Test entry:
 * it lets the parity tests check A3 and A4 separately from the assembly A5. */
cdms_status cdms_loglik_terms(cdms_ctx ctx, const cdms_scene* scene, const double* d_particles, int64_t P,
                              int32_t pstride, const double* d_sfv, int32_t sfv_per_particle,
                              const void* d_y, const double* h_f_pb, const cdms_prior* h_prior,
                              const double* h_eta, double* d_loglik, void* d_c, void* d_G);

/* F3: the efficient birth proposal of one new PF.
 *   1. residual z~_j = (I - Psi_j Psi_j^dagger) z_j, Psi_j = [psi(x_hat, LOS) psi(x_hat, sfv_1) ...
 *      psi(x_hat, sfv_L)] the steering vectors at the predicted MMSE MT position h_x_hat [3] for the LOS and the
 *      L legacy PFs' MMSE SFVs h_sfv_legacy [L][3] (L in [0, 8], h_sfv_legacy may be NULL if 0);
 *   2. N_g candidates p_i uniform in the partition P_q = the axis-aligned box h_box [6] = (lo[3], hi[3])
 *      (reading C-amb-F3a), p_i = lo + u (hi - lo), u_a = (x_a + 1/2) 2^-32 from the Philox4x32-10 block
 *      (key; i, i >> 32, counter, 7), words 0..2 (C-amb-F3b);
 *   3. coherent Bartlett spectrum P_B,i = | sum_j z~_j^H psi(x_hat, p_i) / N_z |^2;
 *   4. mode mu = p_{i*}, i* = the first argmax, and C = sum_i w_i (p_i - mu)(p_i - mu)^T, w_i = P_B,i / sum P_B
 *      (P:L3332-3340).
 * Uses the scene's arrays, wavefront, path loss and precision (K is ignored); d_y complex64 [J][nf][Na] as for
 * cdms_loglik.  Outputs (device, caller-owned): d_out double [13] = mu[3], C[9] row-major, i* (as a double);
 * optional d_pb double [N_g] (P_B) and d_cand double [N_g][3] (candidates), NULL to skip.  The correlations run
 * on the likelihood engine (K1, or the tensor cores for PLANAR_NB in FP32) at the candidate walls' mirror images
 * of x_hat.  Errors: CDMS_EINVAL for bad arguments (immediately) or a singular Psi^H Psi (at sync);
 * CDMS_EZEROMASS when the residual has no power (at sync); CDMS_EDEGENERATE for a degenerate response.
 * Purely local.  Workspaces O(J (L+1) N_z + N_g) are kept in the context. */
cdms_status cdms_birth_proposal(cdms_ctx ctx, const cdms_scene* scene, const double* h_f_pb,
                                const double* h_x_hat, const double* h_sfv_legacy, int32_t L,
                                const void* d_y, const double* h_box, int64_t N_g, uint64_t key,
                                uint64_t counter, double* d_out, double* d_pb, double* d_cand);

/* F1: the approximate PF update message kappa~ of one PF s at its particles and the PF weights with the
 * normalization constant M_{y,s,n} (Supplement S-V "PF State Update Message" P:L660-834, PF weights P:L3392-3432,
 * Supplement S-IV P:L527-632).  Per PA j, C^kappa(phi_p, r) = r q_p psi_p psi_p^H + eta_j I + M_j M_j^H and
 * mu^kappa(phi_p, r) = r zeta_j mu_p psi_p + mu3_j with q_p = (gamma_p + |mu_p|^2 (1 - zeta_j)) zeta_j, psi_p the
 * response of PA j at the paired MT particle x_p (d_particles row p, reading C-amb-8 / C-amb-F1a) through the wall of
 * SFV phi_p (d_phi [P][3]; d_phi = NULL: the PF is the LOS s = 0, psi_p the LOS response).  det A and
 * pi^Nz cancel against the H0 branch, so:
 *   d_logr out [P] = log w_alpha,p + sum_j [log kappa~(phi_p, 1; z_j) - log kappa~(., 0; z_j)],
 *   d_out  out [2] = (log M_y in units of prod_j kappa~(., 0; z_j), posterior existence sum_p w_p),
 *   d_w    out [P] or NULL: PF weights w_p = e^{logr_p} / M_y  (sum_p w_p + (1 - sum w_alpha) / M_y = 1).
 * Inputs: d_particles [P][pstride] fp64 (xyz first), d_walpha [P] fp64 (the PF prediction weights, sum <= 1),
 * d_mu complex128 [P], d_gamma [P] fp64 (particle amplitude mean / variance), h_zeta [J] (zeta_j(1) of the PF's PPRs),
 * h_eta [J] > 0, d_y complex64 [J][nf][Na] (as cdms_loglik), d_mu3 complex64 [J][nf][Na] (the other features' summed
 * mean sum_{s' != s} mu~_3), d_mcols complex64 [J][L][nf][Na] (the columns m_{s'} of M, L <= 8), both particle-
 * independent and formed by the caller (reading C-amb-F1b).  The scene's K is ignored (the PF is component 1).
 * Engine: the correlations psi_p^H (z - mu3) and psi_p^H m_l on K1T tables of the L + 1 snapshots (FP32 spherical /
 * planar WB; other modes CDMS_EUNSUPPORTED), the rest in fp64.  Purely local.  Degenerate particles: logr = -inf +
 * CDMS_EDEGENERATE at sync; sum of everything zero -> CDMS_EZEROMASS. */
cdms_status cdms_pf_update(cdms_ctx ctx, const cdms_scene* scene, const double* h_f_pb, const double* d_particles,
                           int64_t P, int32_t pstride, const double* d_phi, const double* d_walpha, const void* d_mu,
                           const double* d_gamma, const double* h_zeta, const double* h_eta, const void* d_y,
                           const void* d_mu3, const void* d_mcols, int32_t L, double* d_logr, double* d_w,
                           double* d_out);

/* F4 parts: the noise variance update message nu~ (Supplement S-V) at the noise particles
 * eta_p^(j) of every PA and the normalized noise weights:
 *   log nu~ = -Nz ln(pi eta_p) - ln det(I + M^H M/eta_p) - |e|^2/eta_p + |(I + M^H M/eta_p)^{-1/2} M^H e|^2/eta_p^2,
 *   e = z_j - mu_nu,j, M = the S feature columns of PA j.
 * d_eta, d_wxi [J][P] fp64 (noise particles and their prediction weights), d_y, d_mu complex64 [J][nf][Na] (mu_nu =
 * sum_s mu~_3), d_mcols complex64 [J][S][nf][Na] (S <= 9).  Outputs: d_logw [J][P] = log w_xi + log nu~, d_w [J][P]
 * normalized weights per PA (or NULL), d_lognorm [J] = log sum_p w_xi nu~.  Engine: fp64 dot products of the S + 1
 * vectors per PA, an eigendecomposition of M^H M per PA, then O(S) per (particle, PA).  The scene supplies J, N_a, N_f
 * (its K, wavefront and precision are not used). */
cdms_status cdms_noise_update(cdms_ctx ctx, const cdms_scene* scene, const double* d_eta, const double* d_wxi,
                              int64_t P, const void* d_y, const void* d_mu, const void* d_mcols, int32_t S,
                              double* d_logw, double* d_w, double* d_lognorm);

/* F4 parts: the PPR update message omega~ of one PF s at every PA (Supplement S-V) and the PPR existence
 * with revival (Supplement S-VI): C^omega(r) = r m_omega m_omega^H + eta_j I + M M^H, mu^omega(r) =
 * r mu~_4 + mu3; out [J][3] = (log omega~(1) - log omega~(0), u = log(zeta/(1 - zeta)) + that, sigma(u)).
 * d_y, d_mu3, d_momega, d_mu4 complex64 [J][nf][Na]; d_mcols complex64 [J][L][nf][Na] (L <= 9); h_zeta in (0, 1),
 * h_eta > 0 [J]. */
cdms_status cdms_ppr_update(cdms_ctx ctx, const cdms_scene* scene, const double* h_zeta, const double* h_eta,
                            const void* d_y, const void* d_mu3, const void* d_mcols, int32_t L, const void* d_momega,
                            const void* d_mu4, double* d_out);

/* ---- F4: the synthetic SLAM step (driver) ------------------------------------------------------ */

/* Constants of the F4 step (Experiment 1). */
typedef struct {
  double T, sigma_v;        /* NCV time step (s) and process noise (m/s^2) */
  double c_eta;             /* noise variance transition G(eta; c_eta, eta_{n-1}/c_eta), P:L3783-3784 (>= 1) */
  double c_gamma;           /* amplitude variance transition G(gamma; c_gamma, gamma_{n-1}/c_gamma), P:L3788 (>= 1) */
  double sigma_mu;          /* amplitude mean transition CN(mu; mu_{n-1}, sigma_mu^2) */
  double sigma_sfv;         /* SFV transition N(phi; phi_{n-1}, sigma_sfv^2 I) */
  double p_s, p_s_pr, p_rev_pr, p_b_pr;  /* PF survival, PPR survival / revival / birth */
  double mu_b;              /* Poisson birth mean (Q = 1: p_B = mu_b / (1 + mu_b)) */
  double gamma_max, mu_max; /* birth hyperpriors U(0, gamma_max), U(|mu| <= mu_max) */
  double T_dec, T_pru;      /* declaration / pruning thresholds */
  double box[6];            /* SFV birth box (lo[3], hi[3]) = [2 p_min, 2 p_max] */
  int64_t N_g;              /* birth-proposal candidates (F3) */
  int32_t P_m;              /* belief-average sample size (reading F4c) */
  int32_t regularize;       /* MT and PF-SFV regularization */
  uint64_t key;             /* Philox key of every draw (stream map: DESIGN.md, reading F4i) */
  int32_t keep_debug;       /* 1: keep the step's intermediate messages for cdms_slam_get_view (parity tests) */
  int32_t pad_;
} cdms_slam_params;

typedef struct cdms_slam_s* cdms_slam;

#define CDMS_SLAM_MAXS 9   /* slots: the LOS s = 0 and up to 8 PFs (the likelihood's component limit) */

/* What one step estimated.  Per slot i < n_feat (the slots after the birth, before pruning, in slot
 * order): ident (0 = LOS, then birth order), posterior existence (eq. existenceProb), MMSE SFV (LOS: 0), amplitude
 * mean / variance, PPR probabilities zeta [J], declared (exist > T_dec), pruned (exist < T_pru, never the LOS).  est: the
 * MT belief's moments as cdms_moments; eta_hat: MMSE noise variances; eta_bar / x_pred_hat: the prediction messages'
 * means the step used. */
typedef struct {
  int64_t n;
  int32_t n_feat, n_slots;
  int32_t ident[CDMS_SLAM_MAXS], declared[CDMS_SLAM_MAXS], pruned[CDMS_SLAM_MAXS];
  double exist[CDMS_SLAM_MAXS];
  double phi_hat[CDMS_SLAM_MAXS][3];
  double mu_hat[CDMS_SLAM_MAXS][2];
  double gamma_hat[CDMS_SLAM_MAXS];
  double zeta[CDMS_SLAM_MAXS][8];
  double est[28];
  double lse;
  double eta_hat[8], eta_bar[8];
  double x_pred_hat[3];
} cdms_slam_report;

/* Device arrays of a SLAM state (owned by the library; valid until cdms_slam_destroy).  Slot-major PF arrays: slot i
 * at offset i P (phi at i P 3); slot 0 is the LOS (phi unused).  Debug arrays (keep_debug = 1, else NULL) hold the last
 * step's prediction messages (x_pred, eta_pred) and prior PF arrays after the birth (phi/mu/gamma/w_prior), the MT
 * log-likelihood, the noise weights w_eta [J][P], the PF log-ratios logr and posterior weights w_post [slot][P], the
 * complex64 columns m_cols [J][n_feat][Nz] and mu_nu [J][Nz], the fp64 belief sums u/m/mw_sums complex128
 * [J][n_feat][Nz], pf_out [slot][2] (log M_y, existence) and ppr_out [slot][8][3] (cdms_ppr_update's rows). */
typedef struct {
  int64_t P;
  int32_t J, n_slots, n_feat, pad_;
  double *x, *eta, *phi;
  void* mu;
  double *gamma, *w;
  double *x_pred, *eta_pred, *phi_prior;
  void* mu_prior;
  double *gamma_prior, *w_prior;
  double *loglik, *w_eta, *logr, *w_post;
  void *m_cols, *mu_nu, *u_sums, *m_sums, *mw_sums;
  double *pf_out, *ppr_out;
  /* host side of the state (copies): the next time index, the next birth id, per slot the id, the PPR probabilities
   * and the previous MMSE SFV -- with the device arrays above, everything a checkpoint needs (restore through
   * cdms_slam_set_slots; the step is deterministic, so a restored state continues bit for bit) */
  int64_t n;
  int32_t next_id, pad2_;
  int32_t ident[CDMS_SLAM_MAXS];
  double zeta[CDMS_SLAM_MAXS][8];
  double phi_hat[CDMS_SLAM_MAXS][3];
} cdms_slam_view;

/* Create a SLAM state of P paired particles (MT, noise per PA, every PF slot) on a single-rank context.  The scene's K
 * is ignored (the slots set it per step); its precision selects the MT likelihood's engine (the PF updates always run
 * in FP32 on K1T tables).  Errors: CDMS_EINVAL, CDMS_EUNSUPPORTED (a communicator is attached), CDMS_ENOMEM. */
cdms_status cdms_slam_create(cdms_ctx ctx, const cdms_scene* scene, const double* h_f_pb, int64_t P,
                             const cdms_slam_params* prm, cdms_slam* out);
cdms_status cdms_slam_destroy(cdms_slam slam);
/* Initial state: d_x0 [P][6] MT particles, d_eta0 [J][P] noise particles (device, copied), only the
 * LOS slot with its hyperprior amplitudes (Philox stream 0x601 at n = 0), weights p_B / P, zeta = p_B^PR; n = 1. */
cdms_status cdms_slam_init(cdms_slam slam, const double* d_x0, const double* d_eta0);
/* Test / restart entry: the host side of a state whose device arrays the caller wrote through cdms_slam_get_view --
 * n_slots (>= 1, slot 0 the LOS), h_ident [n_slots], h_zeta [n_slots][J] PPR probabilities, h_phi_hat [n_slots][3]
 * the previous MMSE SFVs (the birth proposal's legacy SFVs; may be NULL), the next time index n and birth id. */
cdms_status cdms_slam_set_slots(cdms_slam slam, int32_t n_slots, const int32_t* h_ident, const double* h_zeta,
                                const double* h_phi_hat, int64_t n, int32_t next_id);
cdms_status cdms_slam_get_view(cdms_slam slam, cdms_slam_view* out);
/* One time step n on the measurement d_y (complex64 [J][nf][Na], as cdms_loglik), in the schedule of P:L2494-2508:
 *  (i)  prediction messages: NCV MT draw, Gamma noise draws, legacy PFs (p_s w, SFV / amplitude jitter, Gamma
 *       amplitude variance), PPRs zeta = p_s^PR zeta~ + p_rev (1 - zeta~); birth of one PF (Q = 1) from the F3
 *       proposal at the predicted MMSE position and the previous MMSE SFVs, importance weights
 *       normalized to p_B (reading F4h), zeta = p_B^PR;
 *  (ii) belief-averaged columns u, m, m_omega of every slot over P_m paired particles (reading F4c);
 *  (iii) iota~ (cdms_loglik with the moment-matched priors and the paired SFVs), nu~ (cdms_noise_update), kappa~ and
 *       omega~ of every slot (cdms_pf_update, cdms_ppr_update) -- all from the prediction messages;
 *  beliefs: MT normalize / estimate / resample / regularize (cdms_bp_update), systematic resampling of the noise per PA
 *  and of every kept PF (weights -> existence / P) with the SFV particles regularized like the MT's (P:L3447-3450,
 *  d = 3, reading F4k), PPR zeta~ = sigma(u); MMSE estimates, declaration (exist > T_dec)
 *  and pruning (exist < T_pru, slots compacted in order).  h_report (host, may be NULL) gets the step's estimates.
 *  Synchronizes the context's stream four times.  On an error return the state is undefined (restore a checkpoint:
 *  cdms_slam_get_view + cdms_slam_set_slots). */
cdms_status cdms_slam_step(cdms_slam slam, const void* d_y, cdms_slam_report* h_report);

/* ---- row A6: weight normalization ------------------------------------------------------------ */

/* w_p = exp((l_p - M) - ln S), M = max_p l_p, S = sum_p exp(l_p - M), lse = M + ln S over ALL ranks'
 * particles (log domain with max subtraction).  d_logw [P_local] fp64,
 * d_w out [P_local] fp64, d_lse out [1] fp64 (same value on every rank).  All l = -inf ->
 * CDMS_EZEROMASS at sync, d_lse = -inf, d_w untouched. */
cdms_status cdms_weights_normalize(cdms_ctx ctx, const double* d_logw, int64_t P_local,
                                   double* d_w, double* d_lse);

/* ---- row A7: belief moments ------------------------------------------------------------------ */

/* MMSE moments of the weighted MT belief and its second central moment
 * (regularization kernel covariance), two-pass over all ranks:
 * d_est out [28] fp64 = [sum w, mean(6), cov upper triangle row-major (21)], cov = sum w (x-mean)
 * (x-mean)^T / sum w.  d_particles [P_local][6], d_w [P_local]. */
cdms_status cdms_moments(cdms_ctx ctx, const double* d_particles, const double* d_w,
                         int64_t P_local, double* d_est);

/* ---- row A8: systematic resampling ----------------------------------------------------------- */

/* Systematic resampling [Arulampalam et al., Alg. 2] in integer form (C-amb-15):
 * q_p = rint(ldexp(w_p / w_max, 36)) (w_max over all ranks), C = inclusive scan of q over the
 * GLOBAL particle order, Q = C_last, t_i = floor((u + i 2^32) Q / (P_total 2^32)), ancestor
 * a_i = min{p : C_p > t_i}.  d_ancestors out [P_local] int64: GLOBAL ancestor indices of this
 * rank's output slots i = rank*P_local + [0, P_local).  P_total <= 2^26.  Bit-exact. */
cdms_status cdms_resample(cdms_ctx ctx, const double* d_w, int64_t P_local, uint32_t u_bits,
                          int64_t* d_ancestors);

/* ---- row A9 + the whole step ----------------------------------------------------------------- */

typedef struct {
  double T;            /* NCV time step (s), C-amb-17 */
  double sigma_v;      /* process-noise std (m/s^2) */
  uint64_t philox_key; /* counter-based RNG key: Philox4x32-10, counter (p_lo, p_hi, step, stream) */
  uint64_t step;       /* time index n (RNG counter) */
  int32_t regularize;  /* 1: Gaussian regularization kernel after resampling */
  int32_t pad_;
} cdms_step_params;

/* One MT BP time step on the device (message schedule P:L2494-2508, MT belief only):
 *  predict x <- F x + Gamma a, a ~ N(0, sigma_v^2 I3) (stream 0) ->
 *  l = loglik (uniform w_beta) -> normalize (lse) -> moments (d_est) -> systematic resampling with
 *  u = first word of Philox(key, (0, 0, step, 3)) and redistribution of the ancestors' states so that
 *  every rank again holds P_local particles -> optional regularization x += h_opt chol(Sigma) n
 *  (streams 1, 2 of the slot index; h_opt = (4/(8 P_total))^(1/10), C-amb-16).
 * d_particles [P_local][6] fp64 in/out.  d_est out [28] (pre-resampling moments), d_lse out [1]. */
cdms_status cdms_bp_step(cdms_ctx ctx, const cdms_scene* scene, double* d_particles,
                         int64_t P_local, const double* d_sfv, const void* d_y,
                         const double* h_f_pb, const cdms_prior* h_prior, const double* h_eta,
                         const cdms_step_params* params, double* d_est, double* d_lse);

/* Rows A6-A9 on given log-weights: the part of cdms_bp_step after the likelihood (P:L3409-3410, P:L2367-2371,
 * P:L3446) with the same kernels -- normalize d_loglik [P_local] (log w~_x, any finite offset), MMSE
 * moments of the weighted particles (d_est out [28]), lse (d_lse out [1]), systematic resampling of the masses
 * e^{l - M} (C-amb-23) with u = first word of Philox(key, (0, 0, step, 3)), the ancestors' states written back into
 * d_particles [P_local][6] (in/out) so that every rank again holds P_local particles, and (prm->regularize) the
 * regularization x += h_opt chol(Sigma) n.  d_ancestors out [P_local] int64 (GLOBAL ancestor index of each of this
 * rank's output slots) or NULL.  prm->T and prm->sigma_v are not used (no prediction).  Collective with a
 * communicator.  Errors as cdms_bp_step (all l = -inf: CDMS_EZEROMASS at sync, particles untouched). */
cdms_status cdms_bp_update(cdms_ctx ctx, const double* d_loglik, double* d_particles, int64_t P_local,
                           const cdms_step_params* params, double* d_est, double* d_lse, int64_t* d_ancestors);

/* ---- test / helper entries ------------------------------------------------------------------- */

/* Materialize psi for n (position, PA j, component s) items with the SAME device functions and
 * phase recurrences as cdms_loglik (parity of |d phase| per element).  d_pos [n][3] fp64,
 * d_js [n][2] int32 (j, s), d_sfv [K][3] fp64, d_psi out complex128 [n][Nz] (n = k*Na + m order). */
cdms_status cdms_response(cdms_ctx ctx, const cdms_scene* scene, const double* d_pos, int64_t n,
                          const int32_t* d_js, const double* d_sfv, void* d_psi);

/* Moment matching of a PF amplitude prior into the (m, v) the MT update consumes (Prop. 1,
 * P:L2818-3165, reading C-amb-7): exist = eps * zeta, m = exist mu, v = exist (gamma + |mu|^2 (1 -
 * exist)).  Host function. */
cdms_status cdms_moment_match(double mu_re, double mu_im, double gamma, double exist,
                              cdms_prior* out);

/* Host-side plan of the distributed resampling (pure function, no device): given every rank's
 * integer mass Q_r (h_Q [nranks]) and u_bits for P_total = nranks * P_local output slots, rank
 * `rank`'s CDF range [O_r, O_r + Q_r) covers the contiguous slot range
 * [*slot_lo, *slot_hi) = [I(O_r), I(O_r + Q_r)), I(x) = #{i : t_i < x}.  h_send_counts [nranks]
 * gets how many of those slots belong to each destination rank (slot i lives on rank i / P_local). */
cdms_status cdms_resample_plan(const uint64_t* h_Q, int nranks, int rank, int64_t P_local,
                               uint32_t u_bits, int64_t* slot_lo, int64_t* slot_hi,
                               int64_t* h_send_counts);

#ifdef __cplusplus
}
#endif
#endif /* CDMS_H_ */
