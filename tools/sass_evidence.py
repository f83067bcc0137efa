"""SASS evidence for profiles/ (dev tool): per kernel of libltb.so, counts of
the instructions that show the B200 paths -- TMA bulk copies (UBLKCP, also
the L2 bulk prefetch UBLKPF), mbarrier / async-proxy ops (SYNCS), cp.async
(LDGSTS), 128/256-bit global loads / stores, distributed-shared-memory
stores (st.async -> STAS), FP64 tensor-core MMAs (DMMA) and FP64 FMAs.

    python tools/sass_evidence.py > profiles/r01_sass_evidence.txt
"""
import collections
import os
import re
import subprocess
import sys

here = os.path.dirname(os.path.abspath(__file__))
lib = os.path.join(here, "..", "paper_2504_16344_b200", "lib", "libltb.so")
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
PATS = [("UBLKCP", r"\bUBLKCP\b"), ("UBLKPF", r"\bUBLKPF\b"), ("SYNCS", r"\bSYNCS\."), ("LDGSTS", r"\bLDGSTS\b"),
        ("LDG128", r"\bLDG\.E[^ ]*\.128\b"), ("LDG256", r"\bLDG\.E[^ ]*\.256\b"), ("STG256", r"\bSTG\.E[^ ]*\.256\b"),
        ("STAS", r"\bSTAS\b"), ("DMMA", r"\bDMMA\b"), ("DFMA", r"\bDFMA\b")]
counts = collections.OrderedDict()
fn = None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        fn = m.group(1)
        counts[fn] = collections.Counter()
        continue
    if fn is None:
        continue
    for name, pat in PATS:
        if re.search(pat, line):
            counts[fn][name] += 1
print("# SASS evidence: cuobjdump -sass paper_2504_16344_b200/lib/libltb.so (tools/sass_evidence.py)")
print("# per kernel: " + ", ".join(n for n, _ in PATS) + " (static instruction counts)")
for f, c in counts.items():
    short = re.sub(r"_ZN3ltb\d+_GLOBAL__N__[0-9a-f]+_\d+_", "", f)
    print("%-90s %s" % (short[:90], " ".join("%s=%d" % (n, c[n]) for n, _ in PATS if c[n])))
