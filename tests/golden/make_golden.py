"""Regenerate tests/golden/golden.npz from the reference's own sources.

Compiles tests/golden/make_golden.cpp against the reference headers and the
objects oracle/Makefile builds verbatim from /root/reference/proj/src
(fft_matvec.cpp, core.cpp + shims), runs it, and packs its output into a
compressed .npz.  Needs /root/reference (this container only); the .npz is
committed so the GPU box never needs the reference.

    python tests/golden/make_golden.py
"""
import os
import struct
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
ORACLE = os.path.join(ROOT, "oracle")
REF = os.environ.get("LTB_REFERENCE", "/root/reference/proj")


def read_container(path):
    out = {}
    with open(path, "rb") as fh:
        data = fh.read()
    pos = 0
    while pos < len(data):
        (nl,) = struct.unpack_from("<I", data, pos)
        pos += 4
        name = data[pos:pos + nl].decode()
        pos += nl
        (nd,) = struct.unpack_from("<I", data, pos)
        pos += 4
        shape = struct.unpack_from("<%dq" % nd, data, pos)
        pos += 8 * nd
        n = int(np.prod(shape))
        arr = np.frombuffer(data, dtype="<f8", count=n, offset=pos).reshape(shape)
        pos += 8 * n
        out[name] = arr.copy()
    return out


def main():
    subprocess.check_call(["make", "-C", ORACLE, "ref"])
    exe = os.path.join(ORACLE, "_ref", "make_golden")
    objs = [os.path.join(ORACLE, "_ref", "obj", o)
            for o in ("ltb_oracle.o", "fftw_shim.o", "fft_matvec.o", "core.o")]
    subprocess.check_call(
        ["g++", "-std=c++20", "-O2", "-ffp-contract=off",
         "-I", os.path.join(ORACLE, "shim"), "-I", os.path.join(REF, "include"),
         "-I", ORACLE, os.path.join(HERE, "make_golden.cpp")] + objs +
        ["-o", exe, "-lm"])
    raw = os.path.join(ORACLE, "_ref", "golden.bin")
    subprocess.check_call([exe, raw])
    arrays = read_container(raw)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    print("golden.npz: %d arrays" % len(arrays))


if __name__ == "__main__":
    sys.exit(main())
