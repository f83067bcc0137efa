"""Host mirror of the reference's ``ltibayes`` matvec API over libltb.so.

Mirrors ``proj/include/ltibayes/core.hpp`` (series, kernel tensor, layout,
error taxonomy) and ``proj/include/ltibayes/fft_matvec.hpp`` (``MatvecPlan``
with ``Scratch``, ``apply_raw``/``apply_adjoint_raw``, typed ``apply``/
``apply_adjoint``, ``kernel_hat_sqnorm``), so code written against the
reference reads the same.  Every compute call goes through the C ABI
(include/ltb.h) into the sm_100a kernels; there is no CPU path.

Buffers may be numpy arrays (host; synchronous, the reference semantics) or
CUDA ``torch.Tensor``s (device pointers; asynchronous on the scratch's
stream).
"""
import ctypes as C
import enum

import numpy as np

from . import _lib

PTR_HOST, PTR_DEVICE = 0, 1


# ---------------------------------------------------------------------------
# error taxonomy (core.hpp:12-35)
# ---------------------------------------------------------------------------
class LtbError(RuntimeError):
    pass


class DimensionError(LtbError):
    pass


class LayoutError(LtbError):
    pass


class NumericalError(LtbError):
    pass


class CapacityError(LtbError):
    pass


class StateError(LtbError):
    pass


class CudaError(LtbError):
    pass


class ConfigError(LtbError):
    pass


class IoError(LtbError):
    pass


_ERRORS = {1: DimensionError, 2: LayoutError, 3: NumericalError, 4: CapacityError,
           5: StateError, 6: CudaError, 7: ValueError, 8: ConfigError, 9: IoError}


def check(status):
    if status != 0:
        raise _ERRORS.get(status, LtbError)(_lib.last_error())


# ---------------------------------------------------------------------------
# core types (core.hpp:50-140)
# ---------------------------------------------------------------------------
class Layout(enum.IntEnum):
    TimeMajorBlocks = 0
    SpaceMajorRows = 1


class KernelTag(enum.IntEnum):
    F = 0
    Fq = 1
    Gstar = 2
    Gqstar = 3


class BlockSeries:
    """Stacked space-time vector; ``values.size == n_rows * n_time``."""

    def __init__(self, n_rows, n_time, layout=Layout.TimeMajorBlocks, values=None):
        self.n_rows = int(n_rows)
        self.n_time = int(n_time)
        self.layout = Layout(layout)
        if values is None:
            values = np.zeros(self.n_rows * self.n_time)
        self.values = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)

    def index(self, r, j):  # core.hpp:73-77
        if self.layout == Layout.SpaceMajorRows:
            return r * self.n_time + j
        return j * self.n_rows + r

    def check_consistent(self, what):  # core.cpp:29-38
        if self.n_rows < 1 or self.n_time < 1 or self.values.size != self.n_rows * self.n_time:
            raise DimensionError("%s: length %d does not match n_rows*n_time = %d*%d"
                                 % (what, self.values.size, self.n_rows, self.n_time))


class SpaceTimeField(BlockSeries):
    """Parameter vector m, n_rows == N_m."""


class ObsSeries(BlockSeries):
    """Stacked sensor data d, n_rows == N_d."""


class QoISeries(BlockSeries):
    """QoI forecasts q, n_rows == N_q."""


def reindex(v, target):
    """Bijective layout permutation (core.cpp:40-51), on the device through
    ltb_reindex (a tiled transpose of the host values); bit exact."""
    v.check_consistent("reindex")
    target = Layout(target)
    n = v.n_rows * v.n_time
    out = np.empty(n)
    check(_lib.load().ltb_reindex(C.c_void_p(v.values.ctypes.data), v.n_rows, v.n_time, int(v.layout),
                                  int(target), C.c_void_p(out.ctypes.data), PTR_HOST, None))
    return type(v)(v.n_rows, v.n_time, target, out)


def reindex_device(values, n_rows, n_time, layout, target, out=None):
    """reindex of a CUDA float64 tensor (asynchronous on torch's current
    stream); returns the permuted tensor."""
    import torch
    n = int(n_rows) * int(n_time)
    out = torch.empty_like(values) if out is None else out
    pi, _k1, _a = _buffer(values, n, "reindex input")
    po, _k2, _b = _buffer(out, n, "reindex output", writable=True)
    check(_lib.load().ltb_reindex(pi, int(n_rows), int(n_time), int(layout), int(target), po, PTR_DEVICE,
                                  C.c_void_p(torch.cuda.current_stream().cuda_stream or 1)))
    return out


class BlockToeplitzKernel:
    """First block column of a block lower-triangular Toeplitz map,
    ``data[r, c, k]`` with the lag axis contiguous (core.hpp:114-140)."""

    def __init__(self, rows_out, n_cols, n_time, tag=KernelTag.F, data=None):
        self.rows_out, self.n_cols, self.n_time = int(rows_out), int(n_cols), int(n_time)
        self.tag = KernelTag(tag)
        if data is None:
            data = np.zeros((self.rows_out, self.n_cols, self.n_time))
        self.data = np.ascontiguousarray(data, dtype=np.float64).reshape(
            self.rows_out, self.n_cols, self.n_time)

    def lag_series(self, r, c):
        return self.data[r, c]


# ---------------------------------------------------------------------------
# buffers
# ---------------------------------------------------------------------------
def _buffer(x, n, what, writable=False):
    """Returns (pointer, ptr_kind, keepalive) for a numpy array or CUDA
    torch tensor of n float64 values."""
    mod = type(x).__module__
    if mod.startswith("torch"):
        import torch
        if not x.is_cuda or x.dtype != torch.float64 or not x.is_contiguous():
            raise ValueError("%s: torch tensor must be a contiguous CUDA float64 tensor" % what)
        if x.numel() != n:
            raise DimensionError("%s: length %d, expected %d" % (what, x.numel(), n))
        return C.c_void_p(x.data_ptr()), PTR_DEVICE, x
    a = np.asarray(x)
    if a.dtype != np.float64 or not a.flags.c_contiguous or (writable and not a.flags.writeable):
        if writable:
            raise ValueError("%s: output must be a writable C-contiguous float64 array" % what)
        a = np.ascontiguousarray(a, dtype=np.float64)
    if a.size != n:
        raise DimensionError("%s: length %d, expected %d" % (what, a.size, n))
    return C.c_void_p(a.ctypes.data), PTR_HOST, a


def _opts(device, unit_cols=0):
    return _lib.LtbOpts(-1 if device is None else int(device), int(unit_cols))


# ---------------------------------------------------------------------------
# MatvecPlan (fft_matvec.hpp:29-78)
# ---------------------------------------------------------------------------
class MatvecPlan:
    """Reusable fast-apply plan for a block lower-triangular Toeplitz map.

    F-hat lives in HBM in the reference's [f][c][r] layout.  Immutable once
    built; concurrent applies need one ``Scratch`` each."""

    class Scratch:
        """Workspace (device buffers + CUDA stream) for one apply at a time."""

        def __init__(self, plan, stream=None):
            h = C.c_void_p()
            if stream is not None and not isinstance(stream, int):
                # torch.cuda.Stream; its default stream has handle 0, which the
                # ABI reads as "private stream" -- pass cudaStreamLegacy (1)
                stream = stream.cuda_stream or 1
            check(_lib.load().ltb_scratch_create(plan._h, C.c_void_p(stream or 0), C.byref(h)))
            self._h = h
            self.plan = plan

        def sync(self):
            check(_lib.load().ltb_scratch_sync(self._h))

        def timing(self, enable=True):
            """Start (and clear) / stop per-stage CUDA-event timing."""
            check(_lib.load().ltb_scratch_timing(self._h, int(bool(enable))))

        def stage_ms(self):
            """Accumulated device ms per stage since timing(True):
            {"F": [r2c, gemv_n, c2r], "Fstar": [r2c, gemv_h, c2r],
            "calls": [n_F, n_Fstar]}."""
            ms = (C.c_double * 6)()
            calls = (C.c_int * 2)()
            check(_lib.load().ltb_scratch_stage_ms(self._h, ms, calls))
            return {"F": list(ms[0:3]), "Fstar": list(ms[3:6]), "calls": list(calls)}

        @property
        def stream_handle(self):
            return _lib.load().ltb_scratch_stream(self._h)

        def close(self):
            if getattr(self, "_h", None):
                _lib.load().ltb_scratch_destroy(self._h)
                self._h = None

        def __del__(self):
            try:
                self.close()
            except Exception:
                pass

    def __init__(self, kernel, device=None, unit_cols=0):
        if not isinstance(kernel, BlockToeplitzKernel):
            raise TypeError("MatvecPlan expects a BlockToeplitzKernel")
        L = _lib.load()
        h = C.c_void_p()
        opts = _opts(device, unit_cols)
        check(L.ltb_plan_create(C.c_void_p(kernel.data.ctypes.data), kernel.rows_out,
                                kernel.n_cols, kernel.n_time, int(kernel.tag), PTR_HOST,
                                C.byref(opts), C.byref(h)))
        self._h = h
        self._dims()

    @classmethod
    def generated(cls, rows, cols, nt, seed, tag=KernelTag.F, nm_total=None, c0=0,
                  stream=None, device=None, unit_cols=0):
        """Plan over the device-generated kernel k(r, c, t) = U(seed, stream,
        (r nm_total + c0 + c) nt + t) (a column shard of an rows x nm_total
        kernel); ``stream`` defaults to the tag's stream id."""
        self = cls.__new__(cls)
        h = C.c_void_p()
        opts = _opts(device, unit_cols)
        nm_total = cols if nm_total is None else nm_total
        stream = int(tag) + 1 if stream is None else stream
        check(_lib.load().ltb_plan_create_generated(rows, cols, nt, int(tag), seed, stream,
                                                    nm_total, c0, C.byref(opts), C.byref(h)))
        self._h = h
        self._dims()
        return self

    @classmethod
    def premultiplied(cls, kernel, prior, device=None, unit_cols=0):
        """G* plan from an F kernel: PriorOp::premultiply_kernel
        (prior.cpp:108-134) on the device, then the transform.
        ``prior`` = (h_x, gamma, delta) of A_x = delta I - gamma L."""
        self = cls.__new__(cls)
        h = C.c_void_p()
        opts = _opts(device, unit_cols)
        hx, gamma, delta = (float(v) for v in prior)
        check(_lib.load().ltb_plan_create_premultiplied(
            C.c_void_p(kernel.data.ctypes.data), kernel.rows_out, kernel.n_cols, kernel.n_time,
            int(kernel.tag), PTR_HOST, hx, gamma, delta, C.byref(opts), C.byref(h)))
        self._h = h
        self._dims()
        return self

    @classmethod
    def generated_premultiplied(cls, rows, cols, nt, seed, prior, tag=KernelTag.F, stream=None,
                                device=None, unit_cols=0, nm_total=None, c0=0):
        """G* plan of the device-generated F kernel: all columns, or (with
        ``nm_total``) the column shard [c0, c0 + cols) of a rows x nm_total
        kernel (premultiplied over all of its columns)."""
        self = cls.__new__(cls)
        h = C.c_void_p()
        opts = _opts(device, unit_cols)
        stream = int(tag) + 1 if stream is None else stream
        hx, gamma, delta = (float(v) for v in prior)
        if nm_total is None:
            check(_lib.load().ltb_plan_create_generated_premultiplied(
                rows, cols, nt, int(tag), seed, stream, hx, gamma, delta, C.byref(opts), C.byref(h)))
        else:
            check(_lib.load().ltb_plan_create_generated_premultiplied_shard(
                rows, cols, nt, int(tag), seed, stream, int(nm_total), int(c0), hx, gamma, delta, C.byref(opts),
                C.byref(h)))
        self._h = h
        self._dims()
        return self

    @classmethod
    def load(cls, path, prior=None, device=None, unit_cols=0):
        """Plan from a BTPZ1 kernel archive (io.cpp:71-100), optionally
        premultiplied by the prior on the way."""
        self = cls.__new__(cls)
        h = C.c_void_p()
        opts = _opts(device, unit_cols)
        p3 = (C.c_double * 3)(*[float(v) for v in prior]) if prior is not None else None
        check(_lib.load().ltb_plan_load_btpz(str(path).encode(), p3, C.byref(opts), C.byref(h)))
        self._h = h
        self._dims()
        return self

    def _dims(self):
        v = [C.c_int() for _ in range(6)]
        check(_lib.load().ltb_plan_dims(self._h, *[C.byref(x) for x in v]))
        self._rows, self._cols, self._nt, self._npad, self._nf, self._tag = (x.value for x in v)

    def close(self):
        if getattr(self, "_h", None):
            _lib.load().ltb_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # fft_matvec.hpp:38-43
    def rows_out(self):
        return self._rows

    def n_cols(self):
        return self._cols

    def n_time(self):
        return self._nt

    def padded_len(self):
        return self._npad

    def n_freq(self):
        return self._nf

    def tag(self):
        return KernelTag(self._tag)

    def device_bytes(self):
        n = C.c_size_t()
        check(_lib.load().ltb_plan_bytes(self._h, C.byref(n)))
        return n.value

    def kernel_hat_sqnorm(self):
        out = C.c_double()
        check(_lib.load().ltb_kernel_hat_sqnorm(self._h, C.byref(out)))
        return out.value

    def kernel_hat(self, f0=0, nfreq=None):
        """F-hat frequencies [f0, f0+nfreq) as a complex (nfreq, cols, rows) array."""
        nfreq = self._nf - f0 if nfreq is None else nfreq
        out = np.empty(2 * nfreq * self._cols * self._rows)
        check(_lib.load().ltb_plan_copy_kernel_hat(self._h, f0, nfreq,
                                                   out.ctypes.data_as(_lib._dp)))
        return out.view(np.complex128).reshape(nfreq, self._cols, self._rows)

    # fft_matvec.hpp:60-65
    def apply_raw(self, inp, out, scratch):
        pi, ki, _a = _buffer(inp, self._cols * self._nt, "apply_raw input")
        po, ko, _b = _buffer(out, self._rows * self._nt, "apply_raw output", writable=True)
        if ki != ko:
            raise ValueError("apply_raw: input and output must both be host or both be device")
        check(_lib.load().ltb_apply(self._h, scratch._h, pi, po, ki))

    def apply_adjoint_raw(self, inp, out, scratch):
        pi, ki, _a = _buffer(inp, self._rows * self._nt, "apply_adjoint_raw input")
        po, ko, _b = _buffer(out, self._cols * self._nt, "apply_adjoint_raw output", writable=True)
        if ki != ko:
            raise ValueError("apply_adjoint_raw: input and output must both be host or both be device")
        check(_lib.load().ltb_apply_adjoint(self._h, scratch._h, pi, po, ki))

    # fft_matvec.cpp:221-265 (typed, with layout / dims contract)
    def apply(self, m, scratch=None):
        m.check_consistent("MatvecPlan::apply")
        s = scratch or MatvecPlan.Scratch(self)
        d = ObsSeries(self._rows, self._nt, Layout.SpaceMajorRows)
        check(_lib.load().ltb_apply_series(self._h, s._h, C.c_void_p(m.values.ctypes.data),
                                           m.n_rows, m.n_time, int(m.layout),
                                           C.c_void_p(d.values.ctypes.data), PTR_HOST))
        return d

    def apply_adjoint(self, d, scratch=None):
        d.check_consistent("MatvecPlan::apply_adjoint")
        s = scratch or MatvecPlan.Scratch(self)
        m = SpaceTimeField(self._cols, self._nt, Layout.SpaceMajorRows)
        check(_lib.load().ltb_apply_adjoint_series(self._h, s._h, C.c_void_p(d.values.ctypes.data),
                                                   d.n_rows, d.n_time, int(d.layout),
                                                   C.c_void_p(m.values.ctypes.data), PTR_HOST))
        return m


class ShardedMatvecPlan:
    """One MatvecPlan with its N_m columns sharded over several GPUs of this
    process (include/ltb.h ltb_plan_create_sharded): same apply_raw /
    apply_adjoint_raw contract as MatvecPlan; device buffers live on the home
    device ``devices[0]``.  Devices may repeat (shards on one GPU)."""

    class Scratch:
        def __init__(self, plan, stream=None):
            h = C.c_void_p()
            if stream is not None and not isinstance(stream, int):
                stream = stream.cuda_stream or 1
            check(_lib.load().ltb_sscratch_create(plan._h, C.c_void_p(stream or 0), C.byref(h)))
            self._h = h
            self.plan = plan

        def sync(self):
            check(_lib.load().ltb_sscratch_sync(self._h))

        def close(self):
            if getattr(self, "_h", None):
                _lib.load().ltb_sscratch_destroy(self._h)
                self._h = None

        def __del__(self):
            try:
                self.close()
            except Exception:
                pass

    def __init__(self, kernel, devices, unit_cols=0):
        devs = (C.c_int * len(devices))(*[int(d) for d in devices])
        h = C.c_void_p()
        opts = _opts(None, unit_cols)
        check(_lib.load().ltb_plan_create_sharded(C.c_void_p(kernel.data.ctypes.data), kernel.rows_out,
                                                  kernel.n_cols, kernel.n_time, int(kernel.tag), len(devices),
                                                  devs, C.byref(opts), C.byref(h)))
        self._h = h
        self._dims()

    @classmethod
    def generated(cls, rows, cols, nt, seed, devices, tag=KernelTag.F, stream=None, unit_cols=0):
        """Sharded plan of the device-generated kernel (ltb_plan_create_generated
        per shard, each its own column range of the rows x cols kernel)."""
        self = cls.__new__(cls)
        devs = (C.c_int * len(devices))(*[int(d) for d in devices])
        h = C.c_void_p()
        opts = _opts(None, unit_cols)
        stream = int(tag) + 1 if stream is None else stream
        check(_lib.load().ltb_plan_create_generated_sharded(rows, cols, nt, int(tag), seed, stream, len(devices),
                                                            devs, C.byref(opts), C.byref(h)))
        self._h = h
        self._dims()
        return self

    def _dims(self):
        r, c, t, n = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        check(_lib.load().ltb_splan_dims(self._h, C.byref(r), C.byref(c), C.byref(t), C.byref(n)))
        self._r, self._c, self._t, self._n = r.value, c.value, t.value, n.value

    def shards(self):
        """[(device, c0, c1, peer)] per shard."""
        out = []
        for k in range(self._n):
            d, a, b, p = C.c_int(), C.c_longlong(), C.c_longlong(), C.c_int()
            check(_lib.load().ltb_splan_shard(self._h, k, C.byref(d), C.byref(a), C.byref(b), C.byref(p)))
            out.append((d.value, a.value, b.value, bool(p.value)))
        return out

    def close(self):
        if getattr(self, "_h", None):
            _lib.load().ltb_splan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def rows_out(self):
        return self._r

    def n_cols(self):
        return self._c

    def n_time(self):
        return self._t

    def kernel_hat_sqnorm(self):
        out = C.c_double()
        check(_lib.load().ltb_splan_kernel_hat_sqnorm(self._h, C.byref(out)))
        return out.value

    def apply_raw(self, inp, out, scratch):
        pi, ki, _a = _buffer(inp, self._c * self._t, "apply_raw input")
        po, ko, _b = _buffer(out, self._r * self._t, "apply_raw output", writable=True)
        if ki != ko:
            raise ValueError("apply_raw: input and output must both be host or both device")
        check(_lib.load().ltb_apply_sharded(self._h, scratch._h, pi, po, ki))

    def apply_adjoint_raw(self, inp, out, scratch):
        pi, ki, _a = _buffer(inp, self._r * self._t, "apply_adjoint_raw input")
        po, ko, _b = _buffer(out, self._c * self._t, "apply_adjoint_raw output", writable=True)
        if ki != ko:
            raise ValueError("apply_adjoint_raw: input and output must both be host or both device")
        check(_lib.load().ltb_apply_adjoint_sharded(self._h, scratch._h, pi, po, ki))


def dense_apply(kernel, v, adjoint=False, mem_cap_bytes=2 << 30):
    """fft_matvec.hpp:80-87 / fft_matvec.cpp:267-315: the FFT-free time-domain
    block-Toeplitz product on the device (the reference's test oracle, kept for
    the drop-in).  ``kernel`` is a BlockToeplitzKernel (host data); ``v`` has
    n_cols*N_t values (rows_out*N_t for the adjoint) on the host; the result
    is a new host array.  CapacityError when the implied dense operator
    exceeds ``mem_cap_bytes`` (0: no cap)."""
    k = kernel
    kp, _kk, _a = _buffer(k.data.ravel(), k.rows_out * k.n_cols * k.n_time, "dense_apply kernel")
    nin = (k.rows_out if adjoint else k.n_cols) * k.n_time
    nout = (k.n_cols if adjoint else k.rows_out) * k.n_time
    if type(v).__module__.startswith("torch"):
        raise ValueError("dense_apply: host arrays only (the kernel is host data)")
    vp, vk, _b = _buffer(v, nin, "dense_apply input")
    out = np.empty(nout)
    check(_lib.load().ltb_dense_apply(kp, k.rows_out, k.n_cols, k.n_time, vp, int(bool(adjoint)),
                                      int(mem_cap_bytes), C.c_void_p(out.ctypes.data), vk))
    return out


def algorithmic_bytes(rows, cols, nt):
    """Bytes one F or F* matvec must move: F-hat once plus
    the input and output series."""
    return 16 * (nt + 1) * rows * cols + 8 * nt * (cols + rows)
