"""ctypes front end for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Two libraries, both built by oracle/Makefile:

* ``liboracle.so`` -- our C restatement of the reference hot path
  (oracle/ltb_oracle.c; every function cites the reference file:line);
* ``_ref/libltibayes_ref.so`` -- the reference's own ``fft_matvec.cpp`` and
  ``core.cpp`` compiled verbatim against oracle/shim, exposed through
  oracle/ref_capi.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  The product package
(paper_2504_16344_b200) never does.
"""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_dp = C.POINTER(C.c_double)

_lib = None
_ref = None


def _ptr(a):
    return a.ctypes.data_as(_dp)


def build():
    import subprocess
    subprocess.check_call(["make", "-s", "-C", HERE], stdout=subprocess.DEVNULL)


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.orc_plan_create.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.orc_plan_destroy.argtypes = [C.c_void_p]
        L.orc_plan_dims.argtypes = [C.c_void_p] + [C.POINTER(C.c_int)] * 5
        L.orc_plan_khat.argtypes = [C.c_void_p]
        L.orc_plan_khat.restype = _dp
        L.orc_apply_raw.argtypes = [C.c_void_p, _dp, _dp]
        L.orc_apply_adjoint_raw.argtypes = [C.c_void_p, _dp, _dp]
        L.orc_kernel_hat_sqnorm.argtypes = [C.c_void_p]
        L.orc_kernel_hat_sqnorm.restype = C.c_double
        L.orc_dense_apply.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp, C.c_int,
                                      C.c_uint64, _dp]
        L.orc_reindex.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp]
        L.orc_gen_uniform.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.orc_gen_uniform.restype = C.c_double
        L.orc_gen_fill.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_size_t, _dp]
        L.orc_gen_kernel.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int,
                                     C.c_int, C.c_int, _dp]
        L.orc_gen_factor_entry.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int]
        L.orc_gen_factor_entry.restype = C.c_double
        L.orc_gen_factor.argtypes = [C.c_uint64, C.c_int, _dp]
        L.orc_trsv_lower.argtypes = [_dp, C.c_int, C.c_size_t, _dp]
        L.orc_trsv_lower_t.argtypes = [_dp, C.c_int, C.c_size_t, _dp]
        L.orc_solve_k.argtypes = [_dp, C.c_int, C.c_size_t, _dp]
        L.orc_solve_k_gen.argtypes = [C.c_uint64, C.c_int, _dp]
        L.orc_solve_k_gen_mt.argtypes = [C.c_uint64, C.c_int, _dp, C.c_int]
        L.orc_prior_premultiply.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_double,
                                            C.c_double, C.c_double, _dp]
        L.orc_prior_apply_precision.argtypes = [_dp, C.c_int, C.c_int, C.c_double,
                                                C.c_double, C.c_double, _dp]
        L.orc_form_k.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                 _dp, _dp]
        L.orc_cholesky.argtypes = [_dp, C.c_int, C.c_size_t]
        L.orc_form_q.argtypes = [_dp, _dp, _dp, C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _dp]
        L.orc_fft_create.argtypes = [C.c_int]
        L.orc_fft_create.restype = C.c_void_p
        L.orc_fft_destroy.argtypes = [C.c_void_p]
        L.orc_rfft.argtypes = [C.c_void_p, _dp, _dp]
        L.orc_irfft.argtypes = [C.c_void_p, _dp, _dp]
        L.orc_fft_exec.argtypes = [C.c_void_p, _dp, _dp, C.c_int]
        _lib = L
    return _lib


def ref_available():
    return os.path.exists(os.path.join(HERE, "_ref", "libltibayes_ref.so"))


def ref():
    """The reference's own MatvecPlan (oracle/_ref)."""
    global _ref
    if _ref is None:
        R = C.CDLL(os.path.join(HERE, "_ref", "libltibayes_ref.so"))
        R.ref_plan_create.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int,
                                      C.POINTER(C.c_void_p)]
        R.ref_plan_destroy.argtypes = [C.c_void_p]
        R.ref_apply_raw.argtypes = [C.c_void_p, _dp, _dp]
        R.ref_apply_adjoint_raw.argtypes = [C.c_void_p, _dp, _dp]
        R.ref_kernel_hat_sqnorm.argtypes = [C.c_void_p]
        R.ref_kernel_hat_sqnorm.restype = C.c_double
        R.ref_last_error.restype = C.c_char_p
        R.ref_bench.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_ulonglong, C.c_int,
                                C.c_int, _dp, _dp, _dp]
        _ref = R
    return _ref


# ----------------------------------------------------------------------------
# numpy-level helpers
# ----------------------------------------------------------------------------

class OraclePlan:
    """Restated ``MatvecPlan`` (fft_matvec.cpp:73-217) on host memory."""

    def __init__(self, kernel_rck):
        k = np.ascontiguousarray(kernel_rck, dtype=np.float64)
        rows, cols, nt = k.shape
        h = C.c_void_p()
        st = lib().orc_plan_create(_ptr(k), rows, cols, nt, C.byref(h))
        if st != 0:
            raise RuntimeError("orc_plan_create status %d" % st)
        self._h = h
        self.rows, self.cols, self.nt = rows, cols, nt
        self.nf = nt + 1

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_plan_destroy(self._h)
            self._h = None

    def apply(self, m):
        m = np.ascontiguousarray(m, dtype=np.float64)
        out = np.empty(self.rows * self.nt)
        lib().orc_apply_raw(self._h, _ptr(m), _ptr(out))
        return out

    def apply_adjoint(self, d):
        d = np.ascontiguousarray(d, dtype=np.float64)
        out = np.empty(self.cols * self.nt)
        lib().orc_apply_adjoint_raw(self._h, _ptr(d), _ptr(out))
        return out

    def kernel_hat_sqnorm(self):
        return lib().orc_kernel_hat_sqnorm(self._h)

    def khat(self):
        p = lib().orc_plan_khat(self._h)
        n = 2 * self.nf * self.rows * self.cols
        a = np.ctypeslib.as_array(p, shape=(n,)).copy()
        return a.view(np.complex128).reshape(self.nf, self.cols, self.rows)


class RefPlan:
    """The reference's own ``MatvecPlan`` (oracle/_ref, verbatim sources)."""

    def __init__(self, kernel_rck, tag=0):
        k = np.ascontiguousarray(kernel_rck, dtype=np.float64)
        rows, cols, nt = k.shape
        h = C.c_void_p()
        st = ref().ref_plan_create(_ptr(k), rows, cols, nt, tag, C.byref(h))
        if st != 0:
            raise RuntimeError("ref_plan_create: %s" % ref().ref_last_error())
        self._h = h
        self.rows, self.cols, self.nt = rows, cols, nt

    def __del__(self):
        if getattr(self, "_h", None) and _ref is not None:
            _ref.ref_plan_destroy(self._h)
            self._h = None

    def apply(self, m):
        m = np.ascontiguousarray(m, dtype=np.float64)
        out = np.empty(self.rows * self.nt)
        ref().ref_apply_raw(self._h, _ptr(m), _ptr(out))
        return out

    def apply_adjoint(self, d):
        d = np.ascontiguousarray(d, dtype=np.float64)
        out = np.empty(self.cols * self.nt)
        ref().ref_apply_adjoint_raw(self._h, _ptr(d), _ptr(out))
        return out

    def kernel_hat_sqnorm(self):
        return ref().ref_kernel_hat_sqnorm(self._h)


def dense_apply(kernel_rck, v, adjoint, cap=2 << 30):
    """FFT-free time-domain product (fft_matvec.cpp:267-315).  Returns None
    on CapacityError."""
    k = np.ascontiguousarray(kernel_rck, dtype=np.float64)
    rows, cols, nt = k.shape
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = np.empty((cols if adjoint else rows) * nt)
    st = lib().orc_dense_apply(_ptr(k), rows, cols, nt, _ptr(v), int(adjoint), cap, _ptr(out))
    if st == 4:
        return None
    if st != 0:
        raise RuntimeError("orc_dense_apply status %d" % st)
    return out


def gen_fill(seed, stream, n, index0=0):
    out = np.empty(n)
    lib().orc_gen_fill(seed, stream, index0, n, _ptr(out))
    return out


def gen_kernel(seed, rows, nm_total, nt, c0=0, cols=None, stream=1):
    cols = nm_total - c0 if cols is None else cols
    out = np.empty((rows, cols, nt))
    lib().orc_gen_kernel(seed, stream, rows, nm_total, c0, cols, nt, _ptr(out))
    return out


def gen_factor(seed, n):
    """Dense column-major synthetic factor as an (n, n) C-order array L with
    L[i, j] the entry (row i, col j)."""
    buf = np.empty(n * n)
    lib().orc_gen_factor(seed, n, _ptr(buf))
    return buf.reshape(n, n).T  # buffer is column-major


def solve_k(L, y):
    """y <- L^{-T} L^{-1} y with L an (n, n) array (only the lower triangle
    is read)."""
    Lc = np.asfortranarray(L, dtype=np.float64)
    y = np.array(y, dtype=np.float64, copy=True)
    n = y.size
    lib().orc_solve_k(Lc.ctypes.data_as(_dp), n, n, _ptr(y))
    return y


def solve_k_gen(seed, y, threads=None):
    """K^{-1} y with the synthetic factor; threads > 1 (default: all host
    cores for n >= 20000) runs the blocked multi-threaded sweeps."""
    y = np.array(y, dtype=np.float64, copy=True)
    if threads is None:
        threads = (os.cpu_count() or 1) if y.size >= 20000 else 1
    if threads > 1:
        lib().orc_solve_k_gen_mt(seed, y.size, _ptr(y), int(threads))
    else:
        lib().orc_solve_k_gen(seed, y.size, _ptr(y))
    return y


def rfft(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    n = x.size
    h = lib().orc_fft_create(n)
    out = np.empty(2 * (n // 2 + 1))
    lib().orc_rfft(h, _ptr(x), _ptr(out))
    lib().orc_fft_destroy(h)
    return out.view(np.complex128)


def irfft(X, n):
    X = np.ascontiguousarray(X, dtype=np.complex128).view(np.float64)
    h = lib().orc_fft_create(n)
    out = np.empty(n)
    lib().orc_irfft(h, _ptr(X), _ptr(out))
    lib().orc_fft_destroy(h)
    return out


def prior_premultiply(f_rck, h_x, gamma, delta):
    f = np.ascontiguousarray(f_rck, dtype=np.float64)
    rows, nm, nt = f.shape
    g = np.empty_like(f)
    st = lib().orc_prior_premultiply(_ptr(f), rows, nm, nt, h_x, gamma, delta, _ptr(g))
    if st != 0:
        raise RuntimeError("orc_prior_premultiply status %d" % st)
    return g


def prior_apply_precision(v_tm, nm, nt, h_x, gamma, delta):
    v = np.ascontiguousarray(v_tm, dtype=np.float64)
    out = np.empty_like(v)
    st = lib().orc_prior_apply_precision(_ptr(v), nm, nt, h_x, gamma, delta, _ptr(out))
    if st != 0:
        raise RuntimeError("orc_prior_apply_precision status %d" % st)
    return out


def reindex(v, rows, nt, to_time_major):
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = np.empty_like(v)
    lib().orc_reindex(_ptr(v), rows, nt, int(to_time_major), _ptr(out))
    return out


def form_k(f_rck, g_rck, sigma2, mode=0):
    """(K, asymmetry): bayes_engine.cpp:136-172 restated (mode 0
    ColumnByColumn, 1 FusedBatched); K is an (n, n) array."""
    f = np.ascontiguousarray(f_rck, dtype=np.float64)
    g = np.ascontiguousarray(g_rck, dtype=np.float64)
    rows, nm, nt = f.shape
    n = rows * nt
    K = np.empty(n * n)
    asym = C.c_double()
    st = lib().orc_form_k(_ptr(f), _ptr(g), rows, nm, nt, float(sigma2), int(mode), _ptr(K),
                          C.byref(asym))
    if st != 0:
        raise RuntimeError("orc_form_k status %d" % st)
    return K.reshape(n, n).T.copy(), asym.value


def cholesky(A):
    """Lower Cholesky factor (zeros above); raises ValueError on a
    non-positive pivot (bayes_engine.cpp:195-206 NumericalError)."""
    L = np.array(A, dtype=np.float64, order="F", copy=True)
    n = L.shape[0]
    st = lib().orc_cholesky(L.ctypes.data_as(_dp), n, n)
    if st != 0:
        raise ValueError("factorize: K not positive definite (column %d)" % (st - 1))
    return np.ascontiguousarray(L)


def form_q(f_rck, fq_rck, gq_rck, L):
    """(Q, Gamma_post_q, prior_qoi_cov) of form_Q + form_qoi_cov
    (bayes_engine.cpp:242-285) restated; L is the (n, n) factor."""
    f = np.ascontiguousarray(f_rck, dtype=np.float64)
    fq = np.ascontiguousarray(fq_rck, dtype=np.float64)
    gq = np.ascontiguousarray(gq_rck, dtype=np.float64)
    nd, nm, nt = f.shape
    nq = fq.shape[0]
    n, m = nd * nt, nq * nt
    Lc = np.asfortranarray(L, dtype=np.float64)
    Q = np.empty(m * n)
    gp = np.empty(m * m)
    pc = np.empty(m * m)
    st = lib().orc_form_q(_ptr(f), _ptr(fq), _ptr(gq), nd, nq, nm, nt, Lc.ctypes.data_as(_dp),
                          _ptr(Q), _ptr(gp), _ptr(pc))
    if st == 2:
        raise ValueError("form_qoi_cov: negative posterior QoI variance beyond tolerance")
    if st != 0:
        raise RuntimeError("orc_form_q status %d" % st)
    return (Q.reshape(n, m).T.copy(), gp.reshape(m, m).T.copy(), pc.reshape(m, m).T.copy())


def rel_err(a, b):
    """Relative l2 error as the reference tests define it
    (test_fft_matvec.cpp:35-42)."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return float(np.sqrt(np.sum((a - b) ** 2) / max(np.sum(b * b), 1e-300)))
