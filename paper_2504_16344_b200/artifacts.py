"""Artifact writers mirroring the reference's io.hpp (write_kernel,
write_dense; io.cpp:40-115) over the C ABI, so artifacts built on the device
(F / F_q / G* kernels, K, the factor, Q, Gamma_post_q, the prior QoI
covariance) can be handed to the reference's own CLI, and read back here by
MatvecPlan.load / InferenceEngine.load_factor / load_phase3."""
import ctypes as C
import os

import numpy as np

from . import _lib
from .matvec import BlockToeplitzKernel, _buffer, check


def write_kernel(path, kernel):
    """BTPZ1 (io.cpp:71-85): header rows, cols, N_t, tag, then [row][col][lag]."""
    if isinstance(kernel, BlockToeplitzKernel):
        data, rows, cols, nt, tag = kernel.data, kernel.rows_out, kernel.n_cols, kernel.n_time, int(kernel.tag)
    else:
        raise TypeError("write_kernel: expects a BlockToeplitzKernel")
    p, kind, _k = _buffer(np.ascontiguousarray(data).ravel(), rows * cols * nt, "write_kernel")
    check(_lib.load().ltb_write_btpz(os.fsencode(str(path)), p, rows, cols, nt, tag, kind))


def write_dense(path, m, symmetric=False):
    """DNSM1 (io.cpp:102-115): header rows, cols, symmetric flag, row-major
    doubles.  ``m`` is a 2-D numpy array (any order) or CUDA tensor."""
    if type(m).__module__.startswith("torch"):
        rows, cols = m.shape
        mt = m.t().contiguous()  # column-major storage of m
        check(_lib.load().ltb_write_dnsm(os.fsencode(str(path)), C.c_void_p(mt.data_ptr()), rows, cols, rows,
                                         int(bool(symmetric)), 1))
        return
    a = np.asfortranarray(np.asarray(m, dtype=np.float64))
    rows, cols = a.shape
    check(_lib.load().ltb_write_dnsm(os.fsencode(str(path)), C.c_void_p(a.ctypes.data), rows, cols, rows,
                                     int(bool(symmetric)), 0))


def write_engine_artifacts(directory, engine, f_kernel=None, fq_kernel=None, K=None):
    """The dense part of the reference's artifact set (workflow.cpp:256-264)
    from an engine after form_K / factorize / form_Q: chol.dnsm, Q.dnsm,
    gamma_post_q.dnsm, prior_qoi_cov.dnsm, plus K.dnsm when the caller kept
    K (``engine.K()`` before factorize) and f.btpz / fq.btpz when given."""
    os.makedirs(directory, exist_ok=True)
    if f_kernel is not None:
        write_kernel(os.path.join(directory, "f.btpz"), f_kernel)
    if fq_kernel is not None:
        write_kernel(os.path.join(directory, "fq.btpz"), fq_kernel)
    if K is not None:
        write_dense(os.path.join(directory, "K.dnsm"), K, True)
    write_dense(os.path.join(directory, "chol.dnsm"), engine.chol_lower(), False)
    write_dense(os.path.join(directory, "Q.dnsm"), engine.Q(), False)
    write_dense(os.path.join(directory, "gamma_post_q.dnsm"), engine.gamma_post_q(), True)
    write_dense(os.path.join(directory, "prior_qoi_cov.dnsm"), engine.prior_qoi_cov(), True)
