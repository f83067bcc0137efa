#!/bin/bash
# Builds tests/cpp/_build/dropin_test: the reference's MatvecPlan tests
# (restated in dropin_main.cpp) linked against the DROP-IN
# paper_2504_16344_b200/cpp/fft_matvec_b200.cpp over libltb.so, with the
# reference's UNCHANGED headers and its own core.cpp (oracle/_ref/obj/core.o).
# Needs /root/reference (headers) -- run here; the binary travels to the GPU box.
set -e
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(cd "$HERE/../.." && pwd)"
REF="${LTB_REFERENCE:-/root/reference/proj}"
[ -f "$REF/include/ltibayes/fft_matvec.hpp" ] || { echo "reference headers absent; keeping prebuilt binary"; exit 0; }
make -s -C "$ROOT/oracle" ref
make -s -C "$ROOT/paper_2504_16344_b200"
mkdir -p "$HERE/_build"
g++ -std=c++20 -O2 -I"$REF/include" -I"$ROOT/oracle/shim" -I"$ROOT/include" \
    "$HERE/dropin_main.cpp" "$ROOT/paper_2504_16344_b200/cpp/fft_matvec_b200.cpp" \
    "$ROOT/oracle/_ref/obj/core.o" \
    -L"$ROOT/paper_2504_16344_b200/lib" -lltb -Wl,-rpath,'$ORIGIN/../../../paper_2504_16344_b200/lib' \
    -o "$HERE/_build/dropin_test"
echo "built $HERE/_build/dropin_test"
