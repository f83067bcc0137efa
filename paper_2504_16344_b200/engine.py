"""Online subset of the reference's ``InferenceEngine`` over libltb.so.

Mirrors ``proj/include/ltibayes/bayes_engine.hpp:83-107``: ``set_factor``,
``solve_k_inplace``, ``infer_map`` (the timed region of
bayes_engine.cpp:307-320: copy d, K^{-1} via the Cholesky pair, G* apply) and
the F_q forecast of ``m_map`` (acceptance_main.cpp:243-264).  The offline
phases (form_K, factorize, form_Q, ...) are out of scope; their artifacts --
the factor and the G*/F_q kernels -- are inputs here.
"""
import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .matvec import (Layout, MatvecPlan, ObsSeries, QoISeries, SpaceTimeField, StateError,
                     DimensionError, LayoutError, _buffer, _opts, check)


def _kernel_data(k, what):
    """(data, (rows, cols, nt)) of a BlockToeplitzKernel, a 3-D numpy array or
    a 3-D CUDA tensor."""
    if hasattr(k, "data") and hasattr(k, "n_time") and not hasattr(k, "dtype"):
        return np.ascontiguousarray(k.data, dtype=np.float64).ravel(), (k.rows_out, k.n_cols, k.n_time)
    if len(k.shape) != 3:
        raise DimensionError("%s: kernel must be [rows][cols][nt]" % what)
    shape = tuple(int(s) for s in k.shape)
    if type(k).__module__.startswith("torch"):
        return k.contiguous().view(-1), shape
    return np.ascontiguousarray(k, dtype=np.float64).ravel(), shape


@dataclass
class MapResult:
    """bayes_engine.hpp MapResult: m_map, the device seconds of the timed
    region, the untimed normal-equation residual (None without a residual
    model) and, optionally, the forecast."""
    m_map: SpaceTimeField
    seconds: float
    q_map: QoISeries = None
    smw_rel_residual: float = None


@dataclass
class QoIPrediction:
    """bayes_engine.hpp:101-104"""
    q_map: QoISeries
    ci_lower: QoISeries
    ci_upper: QoISeries
    seconds: float


def normal_quantile(p):
    """bayes_engine.cpp:39-75 (ConfigError unless 0 < p < 1)."""
    out = C.c_double()
    check(_lib.load().ltb_normal_quantile(float(p), C.byref(out)))
    return out.value


class InferenceEngine:
    """Device-resident online engine: factor of K, G* plan, optional F_q plan."""

    def __init__(self, plan_gstar, plan_fq=None, device=None, world=1, rank=0, stream=None):
        """``world`` > 1: distributed K^{-1} (one process per GPU, torch.distributed
        initialised); the plans are then this rank's column shards and the
        factor must be set with ``set_factor_generated`` (collective)."""
        self.plan_g = plan_gstar
        self.plan_fq = plan_fq
        self.world, self.rank = int(world), int(rank)
        h = C.c_void_p()
        opts = _opts(device)
        check(_lib.load().ltb_engine_create(plan_gstar._h, plan_fq._h if plan_fq else None,
                                            C.byref(opts), C.byref(h)))
        self._h = h
        if self.world > 1:
            check(_lib.load().ltb_engine_set_world(self._h, self.world, self.rank))
        self._scratch = MatvecPlan.Scratch(plan_gstar, stream=stream)
        self.n_sensors = plan_gstar.rows_out()
        self.n_space = plan_gstar.n_cols()
        self.n_time = plan_gstar.n_time()
        self.n_qoi = plan_fq.rows_out() if plan_fq else 0

    def n_data(self):
        return self.n_sensors * self.n_time

    def close(self):
        if getattr(self, "_h", None):
            # the engine's internal F_q scratch borrows this scratch's stream:
            # destroy the engine first
            _lib.load().ltb_engine_destroy(self._h)
            self._h = None
            self._scratch.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_factor(self, chol_lower):
        """bayes_engine.cpp:211-217.  ``chol_lower`` is the (n, n) factor;
        only its lower triangle is read."""
        L = np.asarray(chol_lower, dtype=np.float64)
        n = L.shape[0]
        if L.shape != (n, n):
            raise DimensionError("set_factor: wrong factor dims")
        Lf = np.asfortranarray(L)  # the ABI takes column-major (Eigen) storage
        check(_lib.load().ltb_engine_set_factor(self._h, C.c_void_p(Lf.ctypes.data), n, n, 0))

    def set_factor_generated(self, seed, group=None):
        """Synthetic factor (oracle ``orc_gen_factor``) built on the device.
        Distributed: every rank builds its block rows, then the ranks
        exchange CUDA IPC handles of their receive buffers over
        ``torch.distributed`` (collective)."""
        L = _lib.load()
        check(L.ltb_engine_set_factor_generated(self._h, self.n_data(), seed))
        self._connect(group)

    def _connect(self, group=None):
        """Distributed K^{-1}: swap the CUDA IPC handles of the ranks' receive
        buffers (collective)."""
        if self.world == 1:
            return
        import torch.distributed as dist
        L = _lib.load()
        mine = (C.c_char * 64)()
        check(L.ltb_engine_ipc_handle(self._h, mine))
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(mine), group=group)
        blob = (C.c_char * (64 * self.world)).from_buffer_copy(b"".join(handles))
        check(L.ltb_engine_connect(self._h, blob))

    def _ensure_comm(self, group=None):
        """NCCL communicator of the distributed offline phase: rank 0's id
        broadcast over ``torch.distributed`` (collective, once)."""
        if self.world == 1 or getattr(self, "_comm", False):
            return
        import torch.distributed as dist
        L = _lib.load()
        buf = (C.c_char * 128)()
        if self.rank == 0:
            check(L.ltb_nccl_unique_id(buf))
        obj = [bytes(buf) if self.rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        blob = (C.c_char * 128).from_buffer_copy(obj[0])
        check(L.ltb_engine_set_comm(self._h, blob))
        self._comm = True

    # ---- offline phase 2 on the device (bayes_engine.cpp:136-209) ----
    def form_K(self, f_kernel, g_kernel=None, prior=None, sigma2=0.0):
        """K = F G* + sigma2 I from the time-domain kernels (BlockToeplitzKernel,
        numpy [rows][cols][nt] or CUDA tensor).  ``g_kernel`` None: G is the
        Gamma_x premultiplied F, ``prior`` = (h_x, gamma, delta)."""
        f, shape = _kernel_data(f_kernel, "form_K f")
        g = None
        if g_kernel is not None:
            g, gshape = _kernel_data(g_kernel, "form_K g")
            if gshape != shape:
                raise DimensionError("form_K: F and G kernel dims differ")
        elif prior is None:
            raise ValueError("form_K: need g_kernel or prior=(h_x, gamma, delta)")
        rows, cols, nt = shape
        pf, kind, _a = _buffer(f, rows * cols * nt, "form_K f")
        pg = None
        if g is not None:
            pg, kind_g, _b = _buffer(g, rows * cols * nt, "form_K g")
            if kind_g != kind:
                raise ValueError("form_K: f and g must both be host or both be device arrays")
        p3 = (C.c_double * 3)(*prior) if prior is not None else None
        check(_lib.load().ltb_engine_form_k(self._h, pf, pg, p3, rows, cols, nt, float(sigma2), kind))

    def form_K_generated(self, seed, stream, prior, sigma2, nm_total=None, distributed=None, group=None):
        """form_K of the generated kernel (ltb_plan_create_generated's) and its
        premultiplied G; prior = (h_x, gamma, delta).  Distributed engines
        (world > 1, or ``distributed=True`` to run that code path on one GPU)
        form their block rows of K collectively; ``nm_total`` is the global
        N_m of the generated kernel (default: this engine's plan columns)."""
        h_x, gamma, delta = prior
        dist_path = self.world > 1 if distributed is None else bool(distributed)
        if dist_path:
            self._ensure_comm(group)
            nm = self.n_space if nm_total is None else int(nm_total)
            check(_lib.load().ltb_engine_form_k_generated_dist(self._h, nm, int(seed), int(stream), float(h_x),
                                                               float(gamma), float(delta), float(sigma2)))
            self._dist_k = True
            return
        check(_lib.load().ltb_engine_form_k_generated(self._h, int(seed), int(stream), float(h_x),
                                                      float(gamma), float(delta), float(sigma2)))
        self._dist_k = False

    def factorize(self, group=None):
        """In-place Cholesky of K (bayes_engine.cpp:176-209); after a
        distributed form_K, the distributed factorisation (collective) and the
        IPC hand-shake of the distributed K^{-1}."""
        if getattr(self, "_dist_k", False):
            check(_lib.load().ltb_engine_factorize_dist(self._h))
            self._dist_k = False
            self._connect(group)
            return
        check(_lib.load().ltb_engine_factorize(self._h))

    def offline_ms(self):
        """(form_K, factorize) device milliseconds of the last calls."""
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        check(_lib.load().ltb_engine_offline_ms(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value

    def form_Q_ms(self):
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        check(_lib.load().ltb_engine_offline_ms(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return c.value

    def form_Q(self, f_kernel, fq_kernel, gq_kernel=None, prior=None):
        """form_Q + form_qoi_cov (bayes_engine.cpp:242-285) on the device; needs
        the factor.  Installs the Phase-3 operator used by predict_qoi."""
        f, fshape = _kernel_data(f_kernel, "form_Q f")
        fq, qshape = _kernel_data(fq_kernel, "form_Q fq")
        nd, nm, nt = fshape
        nq = qshape[0]
        if qshape[1:] != fshape[1:]:
            raise DimensionError("form_Q: F and F_q kernel dims are inconsistent")
        pf, kind, _a = _buffer(f, nd * nm * nt, "form_Q f")
        pq, kind_q, _b = _buffer(fq, nq * nm * nt, "form_Q fq")
        pg = None
        if gq_kernel is not None:
            gq, gshape = _kernel_data(gq_kernel, "form_Q gq")
            if gshape != qshape:
                raise DimensionError("form_Q: Gq kernel dims differ from F_q")
            pg, kind_g, _c = _buffer(gq, nq * nm * nt, "form_Q gq")
        elif prior is None:
            raise ValueError("form_Q: need gq_kernel or prior=(h_x, gamma, delta)")
        if kind_q != kind or (pg is not None and kind_g != kind):
            raise ValueError("form_Q: kernels must all be host or all be device arrays")
        p3 = (C.c_double * 3)(*prior) if prior is not None else None
        check(_lib.load().ltb_engine_form_q(self._h, pf, pq, pg, p3, nd, nq, nm, nt, kind))
        if not self.n_qoi:
            self.n_qoi = nq

    def form_Q_generated(self, seed, nq, prior, stream_f=1, stream_fq=2):
        """form_Q of the generated F / F_q kernels (ltb_plan_create_generated's
        streams: F = 1, F_q = 2) and the premultiplied Gq."""
        h_x, gamma, delta = prior
        check(_lib.load().ltb_engine_form_q_generated(self._h, int(seed), int(stream_f), int(stream_fq),
                                                      int(nq), float(h_x), float(gamma), float(delta)))
        if not self.n_qoi:
            self.n_qoi = nq

    def _phase3(self, which):
        m = self.n_qoi * self.n_time
        n = self.n_data()
        Q = np.empty((m, n), order="F") if which == "Q" else None
        G = np.empty((m, m), order="F") if which != "Q" else None
        gp = G if which == "gpost" else None
        pc = G if which == "prior" else None
        check(_lib.load().ltb_engine_export_phase3(
            self._h, C.c_void_p(Q.ctypes.data) if Q is not None else None, m,
            C.c_void_p(gp.ctypes.data) if gp is not None else None,
            C.c_void_p(pc.ctypes.data) if pc is not None else None, m, 0))
        return Q if Q is not None else G

    def Q(self):
        """The Phase-3 operator Q (N_q N_t x N_d N_t)."""
        return self._phase3("Q")

    def gamma_post_q(self):
        return self._phase3("gpost")

    def prior_qoi_cov(self):
        return self._phase3("prior")

    def _export(self):
        n = self.n_data()
        out = np.empty((n, n), dtype=np.float64, order="F")
        check(_lib.load().ltb_engine_export_lower(self._h, C.c_void_p(out.ctypes.data), n, 0))
        return out

    def K_lower(self):
        """Lower triangle of K after form_K (zeros above)."""
        return self._export()

    def K(self):
        """Symmetric K (bayes_engine.hpp K() accessor)."""
        L = self._export()
        return L + np.tril(L, -1).T

    def chol_lower(self):
        """The Cholesky factor (after factorize / set_factor)."""
        return self._export()

    def solve_k_inplace(self, y, scratch=None):
        """bayes_engine.cpp:236-240: y <- K^{-1} y (numpy or CUDA tensor)."""
        p, kind, keep = _buffer(y, self.n_data(), "solve_k_inplace", writable=True)
        check(_lib.load().ltb_engine_solve_k(self._h, (scratch or self._scratch)._h, p, kind))
        return y

    def _check_obs(self, d, what):
        d.check_consistent(what)
        if d.layout != Layout.SpaceMajorRows:
            raise LayoutError("%s: requires SpaceMajorRows" % what)
        if d.n_rows != self.n_sensors or d.n_time != self.n_time:
            raise DimensionError("%s: dims do not match engine" % what)

    def infer_map(self, d_obs, with_forecast=False):
        """m_map = G* K^{-1} d_obs (+ q_map = F_q m_map); ``seconds`` is the
        device time of the call."""
        self._check_obs(d_obs, "infer_map")
        m = SpaceTimeField(self.n_space, self.n_time, Layout.SpaceMajorRows)
        q = QoISeries(self.n_qoi, self.n_time, Layout.SpaceMajorRows) if with_forecast else None
        secs = C.c_double()
        check(_lib.load().ltb_engine_infer_and_forecast(
            self._h, self._scratch._h, C.c_void_p(d_obs.values.ctypes.data),
            C.c_void_p(m.values.ctypes.data), C.c_void_p(q.values.ctypes.data) if q else None,
            C.byref(secs), 0))
        res = MapResult(m, secs.value, q)
        if getattr(self, "_resid_plan", None) is not None:
            r = C.c_double()
            check(_lib.load().ltb_engine_map_residual(self._h, self._scratch._h,
                                                      C.c_void_p(d_obs.values.ctypes.data),
                                                      C.c_void_p(m.values.ctypes.data), C.byref(r), 0))
            res.smw_rel_residual = r.value
        return res

    def set_residual_model(self, plan_f, sigma2, prior):
        """Enable infer_map's untimed normal-equation residual
        (bayes_engine.cpp:322-336): the F plan, sigma2 and (h_x, gamma, delta)."""
        h_x, gamma, delta = prior
        check(_lib.load().ltb_engine_set_residual_model(self._h, plan_f._h, float(sigma2), float(h_x),
                                                        float(gamma), float(delta)))
        self._resid_plan = plan_f

    @staticmethod
    def integrate_displacement(m, dt_obs):
        """bayes_engine.cpp:411-419: dt * sum over time of every row of m."""
        m.check_consistent("integrate_displacement")
        vals = np.ascontiguousarray(m.values, dtype=np.float64)
        if m.layout != Layout.SpaceMajorRows:  # SpaceTimeField::at() is layout aware
            from .matvec import reindex as _re
            vals = _re(m, Layout.SpaceMajorRows).values
        out = np.empty(m.n_rows)
        check(_lib.load().ltb_integrate_displacement(C.c_void_p(vals.ctypes.data), m.n_rows, m.n_time,
                                                     float(dt_obs), C.c_void_p(out.ctypes.data), 0))
        return out

    def infer_raw(self, d, m_map, q=None, scratch=None):
        """Raw-pointer variant (numpy host arrays or CUDA tensors); returns the
        device seconds."""
        pd, kd, _a = _buffer(d, self.n_data(), "infer d")
        pm, km, _b = _buffer(m_map, self.n_space * self.n_time, "infer m_map", writable=True)
        pq = None
        if q is not None:
            pq, kq, _c = _buffer(q, self.n_qoi * self.n_time, "infer q", writable=True)
        secs = C.c_double()
        check(_lib.load().ltb_engine_infer_and_forecast(self._h, (scratch or self._scratch)._h,
                                                        pd, pm, pq, C.byref(secs), kd))
        return secs.value

    def set_phase3(self, Q, gamma_post_q_diag):
        """Online part of set_phase3 (bayes_engine.cpp:218-234): Q
        (Nq*Nt x Nd*Nt) and diag(Gamma_post_q)."""
        Qf = np.asfortranarray(np.asarray(Q, dtype=np.float64))
        rows, cols = Qf.shape
        if rows != self.n_qoi * self.n_time or cols != self.n_data():
            raise DimensionError("set_phase3: wrong artifact dims")
        g = np.ascontiguousarray(gamma_post_q_diag, dtype=np.float64)
        if g.size != rows:
            raise DimensionError("set_phase3: wrong artifact dims")
        check(_lib.load().ltb_engine_set_phase3(self._h, C.c_void_p(Qf.ctypes.data), rows,
                                                C.c_void_p(g.ctypes.data), 0))

    def load_factor(self, path):
        """set_factor from a DNSM1 archive (chol.dnsm, io.cpp:102-136)."""
        check(_lib.load().ltb_engine_load_factor_dnsm(self._h, str(path).encode()))

    def load_phase3(self, q_path, gamma_post_q_path):
        """set_phase3 from Q.dnsm / Gamma_post_q.dnsm (workflow.cpp:325-330)."""
        check(_lib.load().ltb_engine_load_phase3_dnsm(self._h, str(q_path).encode(),
                                                      str(gamma_post_q_path).encode()))

    def predict_qoi(self, d_obs, level=0.95):
        """bayes_engine.cpp:340-362: q_map = Q d_obs with credible intervals
        q_map -/+ z sqrt(diag Gamma_post_q)."""
        self._check_obs(d_obs, "predict_qoi")
        n = self.n_qoi * self.n_time
        q, lo, hi = (QoISeries(self.n_qoi, self.n_time, Layout.SpaceMajorRows) for _ in range(3))
        secs = C.c_double()
        check(_lib.load().ltb_engine_predict_qoi(
            self._h, self._scratch._h, C.c_void_p(d_obs.values.ctypes.data), float(level),
            C.c_void_p(q.values.ctypes.data), C.c_void_p(lo.values.ctypes.data),
            C.c_void_p(hi.values.ctypes.data), C.byref(secs), 0))
        assert q.values.size == n
        return QoIPrediction(q, lo, hi, secs.value)

    def forecast(self, m_map):
        """q = F_q m (the F_q route pinned to Q d by acceptance criterion 5)."""
        if self.plan_fq is None:
            raise StateError("engine: no F_q plan (forecast unavailable)")
        q = QoISeries(self.n_qoi, self.n_time, Layout.SpaceMajorRows)
        check(_lib.load().ltb_engine_forecast(self._h, self._scratch._h,
                                              C.c_void_p(np.ascontiguousarray(m_map.values).ctypes.data),
                                              C.c_void_p(q.values.ctypes.data), 0))
        return q
