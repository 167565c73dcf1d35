"""Thin ctypes binding of libcdms (include/cdms.h): argument marshalling only.

Every step of the path runs in libcdms's CUDA kernels; torch tensors provide device memory and the
stream.  There is no CPU fallback: a missing library or device raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CDMS_LIB", os.path.join(HERE, "libcdms.so"))

OK, EINVAL, EDEGENERATE, EZEROMASS, ENOMEM, ECUDA, ENCCL, EUNSUPPORTED = range(8)
STATUS_NAMES = ["OK", "EINVAL", "EDEGENERATE", "EZEROMASS", "ENOMEM", "ECUDA", "ENCCL", "EUNSUPPORTED"]
WAVEFRONTS = {"spherical": 0, "planar_wb": 1, "planar_nb": 2}
PRECISIONS = {"fp32": 0, "fp64": 1}


class CdmsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 8 else status}: {msg}")
        self.status = status


class SceneC(C.Structure):
    _fields_ = [("J", C.c_int32), ("K", C.c_int32), ("ny", C.c_int32), ("nv", C.c_int32), ("nf", C.c_int32),
                ("wavefront", C.c_int32), ("pathloss", C.c_int32), ("precision", C.c_int32),
                ("dy", C.c_double), ("dv", C.c_double), ("fc", C.c_double), ("df", C.c_double),
                ("h_pa_pos", C.POINTER(C.c_double)), ("h_pa_rot", C.POINTER(C.c_double))]


class PriorC(C.Structure):
    _fields_ = [("m_re", C.c_double), ("m_im", C.c_double), ("v", C.c_double)]


class StepParamsC(C.Structure):
    _fields_ = [("T", C.c_double), ("sigma_v", C.c_double), ("philox_key", C.c_uint64), ("step", C.c_uint64),
                ("regularize", C.c_int32), ("pad_", C.c_int32)]


class SlamParamsC(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("T", "sigma_v", "c_eta", "c_gamma", "sigma_mu", "sigma_sfv", "p_s", "p_s_pr",
                                          "p_rev_pr", "p_b_pr", "mu_b", "gamma_max", "mu_max", "T_dec", "T_pru")] + [
        ("box", C.c_double * 6), ("N_g", C.c_int64), ("P_m", C.c_int32), ("regularize", C.c_int32),
        ("key", C.c_uint64), ("keep_debug", C.c_int32), ("pad_", C.c_int32)]


SLAM_MAXS = 9


class SlamReportC(C.Structure):
    _fields_ = [("n", C.c_int64), ("n_feat", C.c_int32), ("n_slots", C.c_int32),
                ("ident", C.c_int32 * SLAM_MAXS), ("declared", C.c_int32 * SLAM_MAXS), ("pruned", C.c_int32 * SLAM_MAXS),
                ("exist", C.c_double * SLAM_MAXS), ("phi_hat", C.c_double * (3 * SLAM_MAXS)),
                ("mu_hat", C.c_double * (2 * SLAM_MAXS)), ("gamma_hat", C.c_double * SLAM_MAXS),
                ("zeta", C.c_double * (8 * SLAM_MAXS)), ("est", C.c_double * 28), ("lse", C.c_double),
                ("eta_hat", C.c_double * 8), ("eta_bar", C.c_double * 8), ("x_pred_hat", C.c_double * 3)]


class SlamViewC(C.Structure):
    _fields_ = [("P", C.c_int64), ("J", C.c_int32), ("n_slots", C.c_int32), ("n_feat", C.c_int32), ("pad_", C.c_int32)] + [
        (n, C.c_void_p) for n in ("x", "eta", "phi", "mu", "gamma", "w", "x_pred", "eta_pred", "phi_prior", "mu_prior",
                                  "gamma_prior", "w_prior", "loglik", "w_eta", "logr", "w_post", "m_cols", "mu_nu",
                                  "u_sums", "m_sums", "mw_sums", "pf_out", "ppr_out")] + [
        ("n", C.c_int64), ("next_id", C.c_int32), ("pad2_", C.c_int32), ("ident", C.c_int32 * SLAM_MAXS),
        ("zeta", C.c_double * (8 * SLAM_MAXS)), ("phi_hat", C.c_double * (3 * SLAM_MAXS))]


_lib = None


def lib() -> C.CDLL:
    """Load libcdms.so (built in-tree by paper_2604_19723_b200.build); raise if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2604_19723_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i64, i32, dp = C.c_void_p, C.c_int64, C.c_int32, C.POINTER(C.c_double)
        sig = {
            "cdms_create": ([C.POINTER(vp), C.c_int, vp], C.c_int),
            "cdms_destroy": ([vp], C.c_int),
            "cdms_set_stream": ([vp, vp], C.c_int),
            "cdms_last_error": ([vp], C.c_char_p),
            "cdms_sync": ([vp], C.c_int),
            "cdms_reserve": ([vp, C.POINTER(SceneC), i64], C.c_int),
            "cdms_launch_count": ([vp], i64),
            "cdms_timing_enable": ([vp, C.c_int], C.c_int),
            "cdms_timing_read": ([vp, C.POINTER(C.c_double), C.POINTER(i64)], C.c_int),
            "cdms_timing_read_stages": ([vp, C.POINTER(C.c_double), C.POINTER(i64)], C.c_int),
            "cdms_get_unique_id": ([C.c_char_p], C.c_int),
            "cdms_comm_init": ([vp, C.c_char_p, C.c_int, C.c_int], C.c_int),
            "cdms_layout": ([vp, C.POINTER(SceneC), vp, vp, vp, vp], C.c_int),
            "cdms_loglik": ([vp, C.POINTER(SceneC), vp, i64, i32, vp, i32, vp, dp, C.POINTER(PriorC), dp, vp, vp, vp],
                            C.c_int),
            "cdms_loglik_terms": ([vp, C.POINTER(SceneC), vp, i64, i32, vp, i32, vp, dp, C.POINTER(PriorC), dp, vp,
                                   vp, vp], C.c_int),
            "cdms_weights_normalize": ([vp, vp, i64, vp, vp], C.c_int),
            "cdms_moments": ([vp, vp, vp, i64, vp], C.c_int),
            "cdms_resample": ([vp, vp, i64, C.c_uint32, vp], C.c_int),
            "cdms_bp_step": ([vp, C.POINTER(SceneC), vp, i64, vp, vp, dp, C.POINTER(PriorC), dp,
                              C.POINTER(StepParamsC), vp, vp], C.c_int),
            "cdms_response": ([vp, C.POINTER(SceneC), vp, i64, vp, vp, vp], C.c_int),
            "cdms_bp_update": ([vp, vp, vp, i64, C.POINTER(StepParamsC), vp, vp, vp], C.c_int),
            "cdms_noise_update": ([vp, C.POINTER(SceneC), vp, vp, i64, vp, vp, vp, i32, vp, vp, vp], C.c_int),
            "cdms_ppr_update": ([vp, C.POINTER(SceneC), dp, dp, vp, vp, vp, i32, vp, vp, vp], C.c_int),
            "cdms_pf_update": ([vp, C.POINTER(SceneC), dp, vp, i64, i32, vp, vp, vp, vp, dp, dp, vp, vp, vp, i32, vp,
                                vp, vp], C.c_int),
            "cdms_loopback_create": ([C.c_int, C.POINTER(vp)], C.c_int),
            "cdms_loopback_destroy": ([vp], C.c_int),
            "cdms_comm_init_loopback": ([vp, vp, C.c_int], C.c_int),
            "cdms_birth_proposal": ([vp, C.POINTER(SceneC), dp, dp, dp, i32, vp, dp, i64, C.c_uint64, C.c_uint64,
                                     vp, vp, vp], C.c_int),
            "cdms_moment_match": ([C.c_double, C.c_double, C.c_double, C.c_double, C.POINTER(PriorC)], C.c_int),
            "cdms_slam_create": ([vp, C.POINTER(SceneC), dp, i64, C.POINTER(SlamParamsC), C.POINTER(vp)], C.c_int),
            "cdms_slam_destroy": ([vp], C.c_int),
            "cdms_slam_init": ([vp, vp, vp], C.c_int),
            "cdms_slam_set_slots": ([vp, i32, C.POINTER(C.c_int32), dp, dp, i64, i32], C.c_int),
            "cdms_slam_get_view": ([vp, C.POINTER(SlamViewC)], C.c_int),
            "cdms_slam_step": ([vp, vp, C.POINTER(SlamReportC)], C.c_int),
            "cdms_resample_plan": ([C.POINTER(C.c_uint64), C.c_int, C.c_int, i64, C.c_uint32, C.POINTER(i64),
                                    C.POINTER(i64), C.POINTER(i64)], C.c_int),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def exported_symbols() -> list[str]:
    return [n for n in ["cdms_create", "cdms_destroy", "cdms_set_stream", "cdms_last_error", "cdms_sync",
                        "cdms_reserve", "cdms_launch_count", "cdms_timing_enable", "cdms_timing_read",
                        "cdms_timing_read_stages",
                        "cdms_get_unique_id", "cdms_comm_init", "cdms_layout",
                        "cdms_loglik", "cdms_loglik_terms", "cdms_weights_normalize", "cdms_moments", "cdms_resample", "cdms_bp_step",
                        "cdms_response", "cdms_moment_match", "cdms_resample_plan", "cdms_birth_proposal",
                        "cdms_bp_update", "cdms_loopback_create", "cdms_loopback_destroy",
                        "cdms_comm_init_loopback", "cdms_pf_update", "cdms_noise_update",
                        "cdms_ppr_update", "cdms_slam_create", "cdms_slam_destroy", "cdms_slam_init",
                        "cdms_slam_set_slots", "cdms_slam_get_view", "cdms_slam_step"]]


def _ptr(t) -> Optional[int]:
    return None if t is None else C.c_void_p(t.data_ptr())


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Scene:
    """Host-side scene (cdms_scene).  Keeps the numpy arrays alive for the C struct."""

    def __init__(self, pa_pos, pa_rot, ny, nv, dy, dv, nf, fc, df, K, wavefront="spherical", pathloss=False,
                 precision="fp32"):
        self.pa_pos = np.ascontiguousarray(pa_pos, dtype=np.float64).reshape(-1, 3)
        self.pa_rot = np.ascontiguousarray(pa_rot, dtype=np.float64).reshape(-1, 3, 3)
        self.J = self.pa_pos.shape[0]
        self.K, self.S = int(K), int(K) + 1
        self.ny, self.nv, self.nf = int(ny), int(nv), int(nf)
        self.Na = self.ny * self.nv
        self.Nz = self.Na * self.nf
        self.fc, self.df = float(fc), float(df)
        self.c = SceneC(self.J, self.K, self.ny, self.nv, self.nf, WAVEFRONTS[wavefront], int(bool(pathloss)),
                        PRECISIONS[precision], float(dy), float(dv), self.fc, self.df, _dp(self.pa_pos),
                        _dp(self.pa_rot))

    @classmethod
    def from_synthetic(cls, scene, wavefront="spherical", pathloss=False, precision="fp32"):
        cfg = scene.cfg
        return cls(scene.pa_pos, scene.pa_rot, cfg.ny, cfg.nv, scene.dy, scene.dv, cfg.nf, cfg.fc, cfg.df, cfg.K,
                   wavefront=wavefront, pathloss=pathloss, precision=precision)

    def f_pb(self) -> np.ndarray:
        k = np.arange(self.nf, dtype=np.float64)
        return self.fc + (k - (self.nf - 1) / 2.0) * self.df


def priors_c(m, v) -> C.Array:
    m = np.asarray(m, dtype=np.complex128).reshape(-1)
    v = np.asarray(v, dtype=np.float64).reshape(-1)
    arr = (PriorC * len(m))()
    for i in range(len(m)):
        arr[i] = PriorC(float(m[i].real), float(m[i].imag), float(v[i]))
    return arr


class Context:
    """cdms_ctx bound to one CUDA device and stream (default: torch's current stream)."""

    def __init__(self, device: int = 0, stream=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("libcdms needs a CUDA device (no CPU fallback)")
        self.device = device
        self.torch = torch
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        h = C.c_void_p()
        st = lib().cdms_create(C.byref(h), device, C.c_void_p(stream.cuda_stream))
        if st != OK:
            raise CdmsError(st, "cdms_create failed")
        self.h = h
        self.rank, self.nranks = 0, 1

    def close(self):
        if self.h:
            lib().cdms_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, st: int):
        if st != OK:
            raise CdmsError(st, lib().cdms_last_error(self.h).decode())

    def set_stream(self, stream):
        self.stream = stream
        self.check(lib().cdms_set_stream(self.h, C.c_void_p(stream.cuda_stream)))

    def sync(self, raise_on_error: bool = True) -> int:
        st = lib().cdms_sync(self.h)
        if raise_on_error:
            self.check(st)
        return st

    def launch_count(self) -> int:
        return int(lib().cdms_launch_count(self.h))

    def timing_enable(self, on: bool = True):
        self.check(lib().cdms_timing_enable(self.h, int(bool(on))))

    def timing_read(self) -> tuple[float, int]:
        """(summed likelihood-kernel time in ms, number of launches) since timing_enable."""
        ms, n = C.c_double(), C.c_int64()
        self.check(lib().cdms_timing_read(self.h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def timing_read_stages(self) -> tuple[list[float], int]:
        """([correlation, Gram, assembly] kernel ms summed, number of likelihood batches) since timing_enable."""
        ms, n = (C.c_double * 3)(), C.c_int64()
        self.check(lib().cdms_timing_read_stages(self.h, ms, C.byref(n)))
        return [ms[0], ms[1], ms[2]], n.value

    def reserve(self, scene: Scene, P_local: int):
        self.check(lib().cdms_reserve(self.h, C.byref(scene.c), int(P_local)))

    def comm_init_loopback(self, group: "LoopbackGroup", rank: int):
        """Attach the TEST collective backend (cdms_comm_init_loopback): this context becomes rank `rank` of a group of
        contexts in this process; drive each rank's collective calls from its own thread."""
        self.check(lib().cdms_comm_init_loopback(self.h, group.h, int(rank)))
        self.rank, self.nranks = int(rank), group.nranks

    def comm_init_from_torch(self, rank: int, world: int):
        """NCCL bootstrap: rank 0 creates the unique id, torch.distributed broadcasts it."""
        import torch.distributed as dist
        buf = C.create_string_buffer(128)
        if rank == 0:
            self.check(lib().cdms_get_unique_id(buf))
        t = self.torch.tensor(list(buf.raw), dtype=self.torch.uint8,
                              device=f"cuda:{self.device}" if dist.get_backend() == "nccl" else "cpu")
        dist.broadcast(t, 0)
        raw = bytes(t.cpu().tolist())
        self.check(lib().cdms_comm_init(self.h, raw, rank, world))
        self.rank, self.nranks = rank, world


class LoopbackGroup:
    """cdms_loopback: the test-only collective backend of nranks contexts in one process (include/cdms.h)."""

    def __init__(self, nranks: int):
        h = C.c_void_p()
        st = lib().cdms_loopback_create(int(nranks), C.byref(h))
        if st != OK:
            raise CdmsError(st, "cdms_loopback_create")
        self.h, self.nranks = h, int(nranks)

    def close(self):
        if self.h:
            lib().cdms_loopback_destroy(self.h)
            self.h = None


# ---------------------------------------------------------------------------- entry points
def layout(ctx: Context, scene: Scene, sfv):
    torch = ctx.torch
    dev = f"cuda:{ctx.device}"
    sfv = torch.as_tensor(np.asarray(sfv, dtype=np.float64).reshape(-1, 3), device=dev).contiguous()
    lay = torch.empty((scene.J, scene.S, 3, scene.Na), dtype=torch.float64, device=dev)
    va = torch.empty((scene.J, scene.S, 3), dtype=torch.float64, device=dev)
    H = torch.empty((scene.S, 3, 3), dtype=torch.float64, device=dev)
    ctx.check(lib().cdms_layout(ctx.h, C.byref(scene.c), _ptr(sfv), _ptr(lay), _ptr(va), _ptr(H)))
    return lay, va, H


def loglik(ctx: Context, scene: Scene, particles, sfv, y, prior_m, prior_v, eta, logw_prior=None,
           sfv_per_particle: bool = False, want_amp: bool = False, out=None):
    """particles: float64 cuda tensor [P][pstride]; sfv: float64 cuda [K][3] or [P][K][3];
    y: complex64 cuda [J][nf][Na]; prior_m/prior_v: [J][S]; eta: [J].  Returns l [P] (and amp)."""
    torch = ctx.torch
    P, pstride = particles.shape
    assert particles.dtype == torch.float64 and particles.is_contiguous()
    assert y.dtype == torch.complex64 and y.is_contiguous()
    l = out if out is not None else torch.empty(P, dtype=torch.float64, device=particles.device)
    amp = torch.empty((P, scene.J, scene.S), dtype=torch.complex128, device=particles.device) if want_amp else None
    f_pb = scene.f_pb()
    pr = priors_c(prior_m, prior_v)
    et = np.ascontiguousarray(eta, dtype=np.float64).reshape(-1)
    ctx.check(lib().cdms_loglik(ctx.h, C.byref(scene.c), _ptr(particles), int(P), int(pstride), _ptr(sfv),
                                int(bool(sfv_per_particle)), _ptr(y), _dp(f_pb), pr, _dp(et), _ptr(logw_prior),
                                _ptr(l), _ptr(amp)))
    return (l, amp) if want_amp else l


def loglik_terms(ctx: Context, scene: Scene, particles, sfv, y, prior_m, prior_v, eta, sfv_per_particle=False):
    """(l [P], c complex128 [P][J][S], G complex128 [P][J][S][S]) from one likelihood-kernel launch."""
    torch = ctx.torch
    P, pstride = particles.shape
    l = torch.empty(P, dtype=torch.float64, device=particles.device)
    c = torch.empty((P, scene.J, scene.S), dtype=torch.complex128, device=particles.device)
    G = torch.empty((P, scene.J, scene.S, scene.S), dtype=torch.complex128, device=particles.device)
    ctx.check(lib().cdms_loglik_terms(ctx.h, C.byref(scene.c), _ptr(particles), int(P), int(pstride), _ptr(sfv),
                                      int(bool(sfv_per_particle)), _ptr(y), _dp(scene.f_pb()),
                                      priors_c(prior_m, prior_v),
                                      _dp(np.ascontiguousarray(eta, dtype=np.float64).reshape(-1)), _ptr(l),
                                      _ptr(c), _ptr(G)))
    return l, c, G


def birth_proposal(ctx: Context, scene: Scene, x_hat, sfv_legacy, y, box, N_g: int, key: int, counter: int,
                   want_pb: bool = True, want_cand: bool = True):
    """F3 birth proposal (cdms_birth_proposal): (out [13] = mu[3], C[9], i*; P_B [N_g] or None; candidates
    [N_g][3] or None), device tensors on y's device."""
    torch = ctx.torch
    dev = y.device
    sl = np.ascontiguousarray(np.asarray(sfv_legacy, dtype=np.float64).reshape(-1, 3))
    out = torch.empty(13, dtype=torch.float64, device=dev)
    pb = torch.empty(N_g, dtype=torch.float64, device=dev) if want_pb else None
    cand = torch.empty((N_g, 3), dtype=torch.float64, device=dev) if want_cand else None
    ctx.check(lib().cdms_birth_proposal(ctx.h, C.byref(scene.c), _dp(scene.f_pb()),
                                        _dp(np.ascontiguousarray(x_hat, dtype=np.float64)),
                                        _dp(sl) if sl.shape[0] else None, int(sl.shape[0]), _ptr(y),
                                        _dp(np.ascontiguousarray(box, dtype=np.float64)), int(N_g), int(key),
                                        int(counter), _ptr(out), _ptr(pb), _ptr(cand)))
    return out, pb, cand


def weights_normalize(ctx: Context, logw):
    torch = ctx.torch
    w = torch.empty_like(logw)
    lse = torch.empty(1, dtype=torch.float64, device=logw.device)
    ctx.check(lib().cdms_weights_normalize(ctx.h, _ptr(logw), int(logw.shape[0]), _ptr(w), _ptr(lse)))
    return w, lse


def moments(ctx: Context, particles, w):
    torch = ctx.torch
    est = torch.empty(28, dtype=torch.float64, device=w.device)
    ctx.check(lib().cdms_moments(ctx.h, _ptr(particles), _ptr(w), int(w.shape[0]), _ptr(est)))
    return est


def resample(ctx: Context, w, u_bits: int):
    torch = ctx.torch
    anc = torch.empty(w.shape[0], dtype=torch.int64, device=w.device)
    ctx.check(lib().cdms_resample(ctx.h, _ptr(w), int(w.shape[0]), C.c_uint32(u_bits), _ptr(anc)))
    return anc


def bp_step(ctx: Context, scene: Scene, particles, sfv, y, prior_m, prior_v, eta, T: float, sigma_v: float,
            philox_key: int, step: int, regularize: bool = True, est=None, lse=None):
    torch = ctx.torch
    est = est if est is not None else torch.empty(28, dtype=torch.float64, device=particles.device)
    lse = lse if lse is not None else torch.empty(1, dtype=torch.float64, device=particles.device)
    prm = StepParamsC(float(T), float(sigma_v), int(philox_key), int(step), int(bool(regularize)), 0)
    ctx.check(lib().cdms_bp_step(ctx.h, C.byref(scene.c), _ptr(particles), int(particles.shape[0]), _ptr(sfv),
                                 _ptr(y), _dp(scene.f_pb()), priors_c(prior_m, prior_v),
                                 _dp(np.ascontiguousarray(eta, dtype=np.float64).reshape(-1)), C.byref(prm),
                                 _ptr(est), _ptr(lse)))
    return est, lse


def bp_update(ctx: Context, loglik, particles, philox_key: int, step: int, regularize: bool = True, est=None,
              lse=None, want_ancestors: bool = False):
    """Rows A6-A9 on given log-weights (cdms_bp_update): particles [P][6] updated in place; returns (est, lse,
    ancestors or None)."""
    torch = ctx.torch
    dev = particles.device
    est = est if est is not None else torch.empty(28, dtype=torch.float64, device=dev)
    lse = lse if lse is not None else torch.empty(1, dtype=torch.float64, device=dev)
    anc = torch.empty(particles.shape[0], dtype=torch.int64, device=dev) if want_ancestors else None
    prm = StepParamsC(0.0, 0.0, int(philox_key), int(step), int(bool(regularize)), 0)
    ctx.check(lib().cdms_bp_update(ctx.h, _ptr(loglik), _ptr(particles), int(particles.shape[0]), C.byref(prm),
                                   _ptr(est), _ptr(lse), _ptr(anc)))
    return est, lse, anc


def pf_update(ctx: Context, scene: Scene, particles, phi, walpha, mu, gamma, zeta, eta, y, mu3, mcols=None):
    """F1 (cdms_pf_update): (logr [P], w [P], out [2] = (log M_y, existence)) for one PF at its particles.
    particles float64 cuda [P][pstride] (paired MT particles), phi [P][3], walpha [P], mu complex128 [P], gamma [P];
    y, mu3 complex64 cuda [J][nf][Na]; mcols complex64 cuda [J][L][nf][Na] or None (L = 0)."""
    torch = ctx.torch
    P, pstride = particles.shape
    dev = particles.device
    L = 0 if mcols is None else int(mcols.shape[1])
    logr = torch.empty(P, dtype=torch.float64, device=dev)
    w = torch.empty(P, dtype=torch.float64, device=dev)
    out = torch.empty(2, dtype=torch.float64, device=dev)
    ctx.check(lib().cdms_pf_update(ctx.h, C.byref(scene.c), _dp(scene.f_pb()), _ptr(particles), int(P), int(pstride),
                                   _ptr(phi), _ptr(walpha), _ptr(mu), _ptr(gamma),
                                   _dp(np.ascontiguousarray(zeta, dtype=np.float64).reshape(-1)),
                                   _dp(np.ascontiguousarray(eta, dtype=np.float64).reshape(-1)), _ptr(y), _ptr(mu3),
                                   _ptr(mcols), int(L), _ptr(logr), _ptr(w), _ptr(out)))
    return logr, w, out


def noise_update(ctx: Context, scene: Scene, eta, wxi, y, mu, mcols=None):
    """F4 nu~ (cdms_noise_update): (logw [J][P], w [J][P], lognorm [J]).  eta, wxi float64 cuda [J][P]; y, mu
    complex64 cuda [J][nf][Na]; mcols complex64 cuda [J][S][nf][Na] or None."""
    torch = ctx.torch
    J, P = eta.shape
    S = 0 if mcols is None else int(mcols.shape[1])
    logw = torch.empty((J, P), dtype=torch.float64, device=eta.device)
    w = torch.empty((J, P), dtype=torch.float64, device=eta.device)
    ln = torch.empty(J, dtype=torch.float64, device=eta.device)
    ctx.check(lib().cdms_noise_update(ctx.h, C.byref(scene.c), _ptr(eta), _ptr(wxi), int(P), _ptr(y), _ptr(mu),
                                      _ptr(mcols), int(S), _ptr(logw), _ptr(w), _ptr(ln)))
    return logw, w, ln


def ppr_update(ctx: Context, scene: Scene, zeta, eta, y, mu3, momega, mu4, mcols=None):
    """F4 omega~ (cdms_ppr_update): out [J][3] = (log ratio, u, existence)."""
    torch = ctx.torch
    L = 0 if mcols is None else int(mcols.shape[1])
    out = torch.empty((scene.J, 3), dtype=torch.float64, device=y.device)
    ctx.check(lib().cdms_ppr_update(ctx.h, C.byref(scene.c), _dp(np.ascontiguousarray(zeta, dtype=np.float64)),
                                    _dp(np.ascontiguousarray(eta, dtype=np.float64)), _ptr(y), _ptr(mu3), _ptr(mcols),
                                    int(L), _ptr(momega), _ptr(mu4), _ptr(out)))
    return out


def response(ctx: Context, scene: Scene, pos, js, sfv):
    """psi for n (position, (j, s)) items: complex128 cuda [n][Nz] (n = k*Na + m order)."""
    torch = ctx.torch
    dev = f"cuda:{ctx.device}"
    pos = torch.as_tensor(np.asarray(pos, dtype=np.float64).reshape(-1, 3), device=dev).contiguous()
    js = torch.as_tensor(np.asarray(js, dtype=np.int32).reshape(-1, 2), device=dev).contiguous()
    sfv = torch.as_tensor(np.asarray(sfv, dtype=np.float64).reshape(-1, 3), device=dev).contiguous()
    n = pos.shape[0]
    psi = torch.empty((n, scene.Nz), dtype=torch.complex128, device=dev)
    ctx.check(lib().cdms_response(ctx.h, C.byref(scene.c), _ptr(pos), int(n), _ptr(js), _ptr(sfv), _ptr(psi)))
    return psi


def moment_match(mu: complex, gamma: float, exist: float):
    out = PriorC()
    st = lib().cdms_moment_match(float(np.real(mu)), float(np.imag(mu)), float(gamma), float(exist), C.byref(out))
    if st != OK:
        raise CdmsError(st, "cdms_moment_match")
    return complex(out.m_re, out.m_im), out.v


def resample_plan(Q: Sequence[int], rank: int, P_local: int, u_bits: int):
    """Host-side distributed resampling plan (no device): (slot_lo, slot_hi, send_counts)."""
    R = len(Q)
    q = (C.c_uint64 * R)(*[int(x) for x in Q])
    lo, hi = C.c_int64(), C.c_int64()
    counts = (C.c_int64 * R)()
    st = lib().cdms_resample_plan(q, R, rank, int(P_local), C.c_uint32(u_bits), C.byref(lo), C.byref(hi), counts)
    if st != OK:
        raise CdmsError(st, "cdms_resample_plan")
    return lo.value, hi.value, [int(x) for x in counts]


# -- F4: the SLAM step driver ----------------------------------------------------------------------------------------
class _DevArray:
    """A device pointer with __cuda_array_interface__ (zero-copy torch view of library-owned memory)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(int(d) for d in shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 2, "strides": None}


def _view(torch, ptr, shape, typestr):
    if not ptr:
        return None
    return torch.as_tensor(_DevArray(ptr, shape, typestr), device="cuda")


SLAM_DEFAULTS = dict(T=0.1, sigma_v=0.5, c_eta=10.0, c_gamma=1000.0, sigma_mu=0.03, sigma_sfv=0.004, p_s=0.8,
                     p_s_pr=0.9, p_rev_pr=0.1, p_b_pr=0.9, mu_b=0.5, gamma_max=5.0, mu_max=0.001, T_dec=0.5, T_pru=0.1,
                     box=(-7.0, -2.0, -2.0, 9.0, 9.0, 2.0), N_g=4096, P_m=256, regularize=1, key=1234, keep_debug=0)


class Slam:
    """F4 driver state (cdms_slam_*): create, init or set a state, step on measurements, read the estimates."""

    def __init__(self, ctx: Context, scene: Scene, P: int, **params):
        self.ctx = ctx
        self.scene = scene
        self.P = int(P)
        prm = dict(SLAM_DEFAULTS)
        prm.update(params)
        c = SlamParamsC()
        for k, v in prm.items():
            if k == "box":
                c.box = (C.c_double * 6)(*[float(b) for b in v])
            else:
                setattr(c, k, v)
        self.params = prm
        self._f_pb = np.ascontiguousarray(scene.f_pb(), dtype=np.float64)
        h = C.c_void_p()
        ctx.check(lib().cdms_slam_create(ctx.h, C.byref(scene.c), _dp(self._f_pb), self.P, C.byref(c), C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            lib().cdms_slam_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def init(self, x0, eta0):
        """x0 float64 cuda [P][6], eta0 float64 cuda [J][P]."""
        self.ctx.check(lib().cdms_slam_init(self.h, _ptr(x0), _ptr(eta0)))

    def set_slots(self, ident, zeta, phi_hat=None, n=1, next_id=1):
        ident = np.ascontiguousarray(ident, dtype=np.int32)
        zeta = np.ascontiguousarray(zeta, dtype=np.float64)
        ph = None if phi_hat is None else np.ascontiguousarray(phi_hat, dtype=np.float64)
        self.ctx.check(lib().cdms_slam_set_slots(self.h, int(ident.shape[0]), ident.ctypes.data_as(C.POINTER(C.c_int32)),
                                                 _dp(zeta), None if ph is None else _dp(ph), int(n), int(next_id)))

    def view(self) -> dict:
        """Zero-copy torch views of the state (and, with keep_debug, the last step's messages)."""
        torch = self.ctx.torch
        v = SlamViewC()
        self.ctx.check(lib().cdms_slam_get_view(self.h, C.byref(v)))
        P, J, S, Sf = v.P, v.J, SLAM_MAXS, max(1, v.n_feat)
        Nz = self.scene.Nz
        f8, c16, c8 = "<f8", "<c16", "<c8"
        ns = v.n_slots
        return dict(
            n_slots=v.n_slots, n_feat=v.n_feat, n=v.n, next_id=v.next_id, ident=list(v.ident[:ns]),
            zeta=np.array(v.zeta[:8 * ns]).reshape(ns, 8)[:, :v.J], phi_hat=np.array(v.phi_hat[:3 * ns]).reshape(ns, 3),
            x=_view(torch, v.x, (P, 6), f8), eta=_view(torch, v.eta, (J, P), f8),
            phi=_view(torch, v.phi, (S, P, 3), f8), mu=_view(torch, v.mu, (S, P), c16),
            gamma=_view(torch, v.gamma, (S, P), f8), w=_view(torch, v.w, (S, P), f8),
            x_pred=_view(torch, v.x_pred, (P, 6), f8), eta_pred=_view(torch, v.eta_pred, (J, P), f8),
            phi_prior=_view(torch, v.phi_prior, (S, P, 3), f8), mu_prior=_view(torch, v.mu_prior, (S, P), c16),
            gamma_prior=_view(torch, v.gamma_prior, (S, P), f8), w_prior=_view(torch, v.w_prior, (S, P), f8),
            loglik=_view(torch, v.loglik, (P,), f8), w_eta=_view(torch, v.w_eta, (J, P), f8),
            logr=_view(torch, v.logr, (S, P), f8), w_post=_view(torch, v.w_post, (S, P), f8),
            m_cols=_view(torch, v.m_cols, (J, Sf, Nz), c8), mu_nu=_view(torch, v.mu_nu, (J, Nz), c8),
            u_sums=_view(torch, v.u_sums, (J, Sf, Nz), c16), m_sums=_view(torch, v.m_sums, (J, Sf, Nz), c16),
            mw_sums=_view(torch, v.mw_sums, (J, Sf, Nz), c16), pf_out=_view(torch, v.pf_out, (S, 2), f8),
            ppr_out=_view(torch, v.ppr_out, (S, 8, 3), f8))

    def checkpoint(self) -> dict:
        """Host copy of the whole state (device arrays + the host side); restore() continues bit for bit."""
        v = self.view()
        keys = ("x", "eta", "phi", "mu", "gamma", "w")
        ck = {k: v[k].clone() for k in keys}
        ck.update({k: v[k] for k in ("n", "next_id", "ident", "zeta", "phi_hat")})
        return ck

    def restore(self, ck: dict):
        v = self.view()
        for k in ("x", "eta", "phi", "mu", "gamma", "w"):
            v[k].copy_(ck[k])
        self.set_slots(ck["ident"], ck["zeta"], ck["phi_hat"], n=ck["n"], next_id=ck["next_id"])

    def step(self, y) -> dict:
        """One time step on y (complex64 cuda [J][nf][Na]); returns the step's report as numpy arrays."""
        r = SlamReportC()
        self.ctx.check(lib().cdms_slam_step(self.h, _ptr(y), C.byref(r)))
        nf = r.n_feat
        J = self.scene.J
        return dict(n=r.n, n_feat=nf, n_slots=r.n_slots, ident=list(r.ident[:nf]),
                    declared=[bool(d) for d in r.declared[:nf]], pruned=[bool(d) for d in r.pruned[:nf]],
                    exist=np.array(r.exist[:nf]), phi_hat=np.array(r.phi_hat[:3 * nf]).reshape(nf, 3),
                    mu_hat=np.array(r.mu_hat[:2 * nf]).reshape(nf, 2) @ np.array([1.0, 1j]),
                    gamma_hat=np.array(r.gamma_hat[:nf]), zeta=np.array(r.zeta[:8 * nf]).reshape(nf, 8)[:, :J],
                    est=np.array(r.est[:]), lse=r.lse, eta_hat=np.array(r.eta_hat[:J]),
                    eta_bar=np.array(r.eta_bar[:J]), x_pred_hat=np.array(r.x_pred_hat[:]))
