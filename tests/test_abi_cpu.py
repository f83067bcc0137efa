"""CPU-side checks of the drop-in boundary (no GPU calls): the C-ABI library
builds, loads and exports every symbol include/ltb.h declares; the host
mirror's pure-host logic (layout permutation, series contracts) behaves like
the reference's core.cpp."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ltb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ltb_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2504_16344_b200 import _lib
    _lib.build()
    L = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.SIGNATURES), "ctypes table out of sync with include/ltb.h"
    assert L.ltb_version().decode().startswith("ltb")


def test_library_is_sm100a():
    """The shared object carries sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess
    from paper_2504_16344_b200 import _lib
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_series_contract():
    from paper_2504_16344_b200 import DimensionError, ObsSeries
    d = ObsSeries(3, 4)
    d.check_consistent("x")
    d.values = np.zeros(11)
    with pytest.raises(DimensionError):
        d.check_consistent("x")


def test_no_product_import_of_oracle():
    """The product package never imports the oracle (test infrastructure)."""
    pkg = os.path.join(ROOT, "paper_2504_16344_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "ltb_oracle.h" not in txt and "liboracle" not in txt, f
                assert "_ref/" not in txt and "libltibayes_ref" not in txt, f


def test_artifact_writers_match_the_reference_byte_layout(tmp_path):
    """ltb_write_btpz / ltb_write_dnsm (host pointers: no GPU involved) write
    exactly io.cpp's bytes (write_kernel :71-85, write_dense :102-115),
    restated here independently with struct; atomic_write leaves no temp."""
    import struct
    import paper_2504_16344_b200 as ltb
    rng = np.random.default_rng(4)
    k = rng.standard_normal((3, 5, 7))
    ltb.write_kernel(tmp_path / "sub" / "f.btpz", ltb.BlockToeplitzKernel(3, 5, 7, tag=ltb.KernelTag.Fq, data=k))
    want = b"BTPZ1" + struct.pack("<4Q", 3, 5, 7, 1) + np.ascontiguousarray(k, dtype="<f8").tobytes()
    assert (tmp_path / "sub" / "f.btpz").read_bytes() == want
    m = rng.standard_normal((6, 4))
    ltb.write_dense(tmp_path / "m.dnsm", m, symmetric=False)
    want = b"DNSM1" + struct.pack("<3Q", 6, 4, 0) + np.ascontiguousarray(m, dtype="<f8").tobytes()
    assert (tmp_path / "m.dnsm").read_bytes() == want
    ltb.write_dense(tmp_path / "s.dnsm", np.asfortranarray(m @ m.T), symmetric=True)
    assert (tmp_path / "s.dnsm").read_bytes()[5:29] == struct.pack("<3Q", 6, 6, 1)
    assert sorted(p.name for p in tmp_path.iterdir()) == ["m.dnsm", "s.dnsm", "sub"]
    with pytest.raises(ltb.NumericalError):
        bad = k.copy()
        bad[0, 0, 0] = np.nan
        ltb.write_kernel(tmp_path / "bad.btpz", ltb.BlockToeplitzKernel(3, 5, 7, data=bad))
    with pytest.raises(ltb.IoError):
        ltb.write_dense("/proc/forbidden/x.dnsm", m)


def test_series_files_roundtrip(tmp_path):
    """io.cpp:138-180 series format: raw doubles + the "rows= nt= layout="
    sidecar; bit-exact round trip, IoError contract."""
    import paper_2504_16344_b200 as ltb
    rng = np.random.default_rng(8)
    s = ltb.ObsSeries(3, 5, ltb.Layout.TimeMajorBlocks, rng.standard_normal(15))
    ltb.write_series(tmp_path / "d.f64", s)
    assert (tmp_path / "d.f64.hdr").read_text() == "rows=3 nt=5 layout=TimeMajorBlocks\n"
    assert (tmp_path / "d.f64").read_bytes() == s.values.astype("<f8").tobytes()
    r = ltb.read_series(tmp_path / "d.f64", ltb.ObsSeries)
    assert r.layout == ltb.Layout.TimeMajorBlocks and np.array_equal(r.values, s.values)
    with pytest.raises(ltb.IoError):
        ltb.read_series(tmp_path / "missing.f64", ltb.ObsSeries)
    (tmp_path / "bad.f64.hdr").write_text("rows=3 nt=5 layout=Diagonal\n")
    with pytest.raises(ltb.IoError):
        ltb.read_series(tmp_path / "bad.f64", ltb.ObsSeries)
    (tmp_path / "short.f64.hdr").write_text("rows=30 nt=5 layout=SpaceMajorRows\n")
    (tmp_path / "short.f64").write_bytes(b"\0" * 64)
    with pytest.raises(ltb.IoError):
        ltb.read_series(tmp_path / "short.f64", ltb.ObsSeries)


def _fnv1a64(data, h=0xcbf29ce484222325):
    # io.cpp:198-206, restated independently
    for b in data:
        h = ((h ^ b) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def test_fnv1a64_known_answers(tmp_path):
    """ltb_fnv1a64_file (io.cpp:208-219) on the published FNV-1a 64 test
    strings and on a file longer than the reference's 64 KB read buffer."""
    import paper_2504_16344_b200 as ltb
    for text, want in ((b"", 0xcbf29ce484222325), (b"a", 0xaf63dc4c8601ec8c), (b"foobar", 0x85944171f73967e8)):
        (tmp_path / "t").write_bytes(text)
        assert ltb.fnv1a64_file(tmp_path / "t") == want
    blob = np.random.default_rng(3).integers(0, 256, 70000, dtype=np.uint8).tobytes()
    (tmp_path / "b").write_bytes(blob)
    assert ltb.fnv1a64_file(tmp_path / "b") == _fnv1a64(blob)
    with pytest.raises(ltb.IoError):
        ltb.fnv1a64_file(tmp_path / "missing")


def test_manifest_roundtrip_and_verify(tmp_path):
    """io.cpp:221-303: write_manifest's line format, read_manifest (meta values
    with spaces, unknown kinds rejected), verify_manifest reporting the first
    missing / resized / altered artifact."""
    import paper_2504_16344_b200 as ltb
    rng = np.random.default_rng(5)
    ltb.write_dense(tmp_path / "Q.dnsm", rng.standard_normal((4, 3)))
    ltb.write_kernel(tmp_path / "f.btpz", ltb.BlockToeplitzKernel(2, 3, 4, data=rng.standard_normal((2, 3, 4))))
    m = ltb.Manifest(phases=[("phase2_form_K", 1.25)], meta=[("sigma2", "0.01"), ("note", "two words")])
    for name in ("f.btpz", "Q.dnsm"):
        m.add_artifact(tmp_path, name)
    ltb.write_manifest(tmp_path / "manifest.txt", m)
    lines = (tmp_path / "manifest.txt").read_text().splitlines()
    fb = (tmp_path / "f.btpz").read_bytes()
    assert lines[0] == "# ltibayes artifact manifest"
    assert lines[1] == "artifact f.btpz %d %016x" % (len(fb), _fnv1a64(fb))
    assert lines[3] == "phase phase2_form_K 1.250000"
    assert lines[5] == "meta note two words"
    r = ltb.read_manifest(tmp_path / "manifest.txt")
    assert r.artifacts == m.artifacts and r.phases == m.phases and r.meta == m.meta
    assert r.meta_value("sigma2") == "0.01" and r.find("Q.dnsm")[1] == (tmp_path / "Q.dnsm").stat().st_size
    assert ltb.verify_manifest(tmp_path, r) is None
    q = bytearray((tmp_path / "Q.dnsm").read_bytes())
    q[40] ^= 1  # same size, different bytes
    (tmp_path / "Q.dnsm").write_bytes(bytes(q))
    assert ltb.verify_manifest(tmp_path, r) == "Q.dnsm"
    (tmp_path / "f.btpz").unlink()
    assert ltb.verify_manifest(tmp_path, r) == "f.btpz"
    (tmp_path / "bad.txt").write_text("# x\nbogus line\n")
    with pytest.raises(ltb.IoError):
        ltb.read_manifest(tmp_path / "bad.txt")
    with pytest.raises(ltb.IoError):
        r.meta_value("missing")
