"""Artifact writers mirroring the reference's io.hpp (write_kernel,
write_dense; io.cpp:40-115) over the C ABI, so artifacts built on the device
(F / F_q / G* kernels, K, the factor, Q, Gamma_post_q, the prior QoI
covariance) can be handed to the reference's own CLI, and read back here by
MatvecPlan.load / InferenceEngine.load_factor / load_phase3."""
import ctypes as C
import os

import numpy as np

from . import _lib
from .matvec import BlockToeplitzKernel, IoError, _buffer, check


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


# ---------------------------------------------------------------------------
# manifest (io.cpp:221-299): "artifact <name> <bytes> <fnv1a64 hex>",
# "phase <name> <seconds>", "meta <key> <value>" lines after a comment header
# ---------------------------------------------------------------------------
def fnv1a64_file(path):
    """FNV-1a 64 of a file's bytes (io.cpp:198-219), through the native library."""
    h = C.c_uint64()
    check(_lib.load().ltb_fnv1a64_file(os.fsencode(str(path)), C.byref(h)))
    return h.value


class Manifest:
    """ltibayes::Manifest (io.hpp): artifact entries (name, bytes, hash),
    phase timings and free-form meta key/values, in file order."""

    def __init__(self, artifacts=None, phases=None, meta=None):
        self.artifacts = list(artifacts or [])  # (name, bytes, hash)
        self.phases = list(phases or [])        # (name, seconds)
        self.meta = list(meta or [])            # (key, value)

    def add_artifact(self, directory, name):
        p = os.path.join(directory, name)
        self.artifacts.append((name, os.path.getsize(p), fnv1a64_file(p)))

    def find(self, name):
        for e in self.artifacts:
            if e[0] == name:
                return e
        return None

    def meta_value(self, key):
        for k, v in self.meta:
            if k == key:
                return v
        raise IoError("manifest: missing meta key " + key)


def write_manifest(path, m):
    """write_manifest (io.cpp:245-263), atomically."""
    lines = ["# ltibayes artifact manifest"]
    lines += ["artifact %s %d %016x" % (n, b, h) for n, b, h in m.artifacts]
    lines += ["phase %s %.6f" % (n, sec) for n, sec in m.phases]
    lines += ["meta %s %s" % (k, v) for k, v in m.meta]
    _atomic_bytes(str(path), ("\n".join(lines) + "\n").encode())


def read_manifest(path):
    """read_manifest (io.cpp:265-291); unknown line kinds raise IOError."""
    m = Manifest()
    with open(path) as fh:
        for line in fh.read().split("\n"):
            if not line or line[0] == "#":
                continue
            kind, _, rest = line.partition(" ")
            if kind == "artifact":
                name, nbytes, hexv = rest.split()[:3]
                m.artifacts.append((name, int(nbytes), int(hexv, 16)))
            elif kind == "phase":
                name, sec = rest.split()[:2]
                m.phases.append((name, float(sec)))
            elif kind == "meta":
                k, _, v = rest.partition(" ")
                m.meta.append((k, v))
            else:
                raise IoError("unknown manifest line: " + line)
    return m


def verify_manifest(directory, m):
    """verify_manifest (io.cpp:293-303): the first artifact that is missing,
    has another size or fails its hash, else None."""
    for name, nbytes, h in m.artifacts:
        p = os.path.join(directory, name)
        if not os.path.exists(p) or os.path.getsize(p) != nbytes or fnv1a64_file(p) != h:
            return name
    return None


def write_engine_artifacts(directory, engine, f_kernel=None, fq_kernel=None, K=None, meta=None, phases=None):
    """The dense part of the reference's artifact set (workflow.cpp:256-264)
    from an engine after form_K / factorize / form_Q: chol.dnsm, Q.dnsm,
    gamma_post_q.dnsm, prior_qoi_cov.dnsm, plus K.dnsm when the caller kept
    K (``engine.K()`` before factorize) and f.btpz / fq.btpz when given;
    then manifest.txt with the size and FNV-1a hash of every artifact present
    (+ the caller's meta / phase entries, e.g. ("sigma2", "0.01"))."""
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
    # manifest over what was written, in the reference's artifact order
    # (workflow.cpp:240-244,266-284); meta / phases as the caller supplies
    man = Manifest(phases=phases, meta=meta)
    for name in ("f.btpz", "fq.btpz", "gstar.btpz", "gqstar.btpz", "K.dnsm", "chol.dnsm", "Q.dnsm",
                 "gamma_post_q.dnsm", "prior_qoi_cov.dnsm"):
        if os.path.exists(os.path.join(directory, name)):
            man.add_artifact(directory, name)
    write_manifest(os.path.join(directory, "manifest.txt"), man)
    return man


# ---------------------------------------------------------------------------
# series files (io.cpp:138-188): raw little-endian doubles + a ".hdr" sidecar
# "rows=R nt=T layout=SpaceMajorRows|TimeMajorBlocks"
# ---------------------------------------------------------------------------
def write_series(path, series):
    """write_series (io.cpp:138-150)."""
    from .matvec import Layout
    series.check_consistent("write_series")
    path = str(path)
    _atomic_bytes(path, np.ascontiguousarray(series.values, dtype="<f8").tobytes())
    _atomic_bytes(path + ".hdr", ("rows=%d nt=%d layout=%s\n" % (
        series.n_rows, series.n_time, Layout(series.layout).name)).encode())


def read_series(path, cls):
    """read_series (io.cpp:152-180) into ``cls`` (ObsSeries, SpaceTimeField,
    QoISeries); IoError on a missing / malformed sidecar or short data."""
    import re
    from .matvec import IoError, Layout
    path = str(path)
    try:
        with open(path + ".hdr") as fh:
            line = fh.readline()
    except OSError:
        raise IoError("missing series sidecar %s.hdr" % path)
    mt = re.match(r"rows=(\d+) nt=(\d+) layout=(\S+)", line)
    if not mt or int(mt.group(1)) < 1 or int(mt.group(2)) < 1:
        raise IoError("malformed series sidecar %s.hdr" % path)
    if mt.group(3) not in ("TimeMajorBlocks", "SpaceMajorRows"):
        raise IoError("unknown layout in sidecar %s.hdr" % path)
    rows, nt = int(mt.group(1)), int(mt.group(2))
    try:
        data = np.fromfile(path, dtype="<f8")
    except OSError:
        raise IoError("cannot open series %s" % path)
    if data.size < rows * nt:
        raise IoError("truncated archive while reading series data")
    return cls(rows, nt, Layout[mt.group(3)], data[:rows * nt].astype(np.float64))


def _atomic_bytes(path, payload):
    d = os.path.dirname(path)
    if d:
        os.makedirs(d, exist_ok=True)
    tmp = "%s.tmp%d.%d" % (path, id(payload) & 0xFFFF, os.getpid())
    with open(tmp, "wb") as fh:
        fh.write(payload)
    os.replace(tmp, path)


def infer_from_artifacts(directory, d_obs_path, sigma2, prior, dt_obs, h_x=None, level=0.95, device=None):
    """cmd_infer (workflow.cpp:300-380) over this library: the artifact set
    (f.btpz, fq.btpz, gstar.btpz if present -- else F premultiplied by the
    prior --, chol.dnsm, Q.dnsm, gamma_post_q.dnsm) and d_obs (a series file)
    -> infer_map + predict_qoi + integrate_displacement on the device; writes
    m_map.f64 (+ .hdr), map_displacement.csv (std = nan: no Hutchinson
    probes), qoi_forecast.csv and latency.txt next to the artifacts.  The
    artifacts are checked against manifest.txt when it exists (a missing or
    altered file raises StateError, as workflow.cpp:317-320); the config
    digest check of the CLI is out of scope: sigma2 (None: the manifest's
    "sigma2" meta), the prior (h_x, gamma, delta) and dt_obs are arguments."""
    import time
    from .engine import InferenceEngine
    from .matvec import Layout, MatvecPlan, ObsSeries, reindex
    from .matvec import StateError
    t0 = time.perf_counter()
    mpath = os.path.join(directory, "manifest.txt")
    if os.path.exists(mpath):
        man = read_manifest(mpath)
        bad = verify_manifest(directory, man)
        if bad is not None:
            raise StateError("stale artifacts: %s is missing or fails its manifest hash; rerun offline" % bad)
        if sigma2 is None:
            sigma2 = float(man.meta_value("sigma2"))
    if sigma2 is None:
        raise StateError("infer_from_artifacts: sigma2 not given and no manifest to read it from")
    f_plan = MatvecPlan.load(os.path.join(directory, "f.btpz"), device=device)
    gpath = os.path.join(directory, "gstar.btpz")
    g_plan = (MatvecPlan.load(gpath, device=device) if os.path.exists(gpath)
              else MatvecPlan.load(os.path.join(directory, "f.btpz"), prior=prior, device=device))
    fq_plan = MatvecPlan.load(os.path.join(directory, "fq.btpz"), device=device)
    eng = InferenceEngine(g_plan, fq_plan, device=device)
    eng.load_factor(os.path.join(directory, "chol.dnsm"))
    eng.load_phase3(os.path.join(directory, "Q.dnsm"), os.path.join(directory, "gamma_post_q.dnsm"))
    eng.set_residual_model(f_plan, sigma2, prior)
    d_obs = read_series(d_obs_path, ObsSeries)
    if d_obs.layout != Layout.SpaceMajorRows:
        d_obs = reindex(d_obs, Layout.SpaceMajorRows)
    load_s = time.perf_counter() - t0
    t1 = time.perf_counter()
    res = eng.infer_map(d_obs)
    qoi = eng.predict_qoi(d_obs, level)
    disp = InferenceEngine.integrate_displacement(res.m_map, dt_obs)
    compute_s = time.perf_counter() - t1
    write_series(os.path.join(directory, "m_map.f64"), res.m_map)
    hx = prior[0] if h_x is None else h_x
    lines = ["x,mean,std"] + ["%r,%r,nan" % (float(x * hx), float(disp[x])) for x in range(eng.n_space)]
    _atomic_bytes(os.path.join(directory, "map_displacement.csv"), ("\n".join(lines) + "\n").encode())
    q, lo, hi = (v.values.reshape(eng.n_qoi, eng.n_time) for v in (qoi.q_map, qoi.ci_lower, qoi.ci_upper))
    lines = ["qoi_id,t,mean,ci_lo,ci_hi"] + [
        "%d,%r,%r,%r,%r" % (s, (j + 1) * dt_obs, float(q[s, j]), float(lo[s, j]), float(hi[s, j]))
        for s in range(eng.n_qoi) for j in range(eng.n_time)]
    _atomic_bytes(os.path.join(directory, "qoi_forecast.csv"), ("\n".join(lines) + "\n").encode())
    _atomic_bytes(os.path.join(directory, "latency.txt"), (
        "load_seconds %g\ncompute_seconds %g\nsmw_rel_residual %g\nwave_solver_invocations 0\n"
        % (load_s, compute_s, res.smw_rel_residual)).encode())
    out = {"load_seconds": load_s, "compute_seconds": compute_s, "device_seconds": res.seconds,
           "smw_rel_residual": res.smw_rel_residual, "m_map": res.m_map, "qoi": qoi, "displacement": disp}
    eng.close()
    return out
