"""The drop-in fft_matvec_b200.cpp (reference header unchanged) passes the
reference's own MatvecPlan test cases on the B200 (tests/cpp/dropin_main.cpp,
built by tests/cpp/build.sh)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
EXE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_build", "dropin_test")


def test_dropin_reference_cases():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(EXE):
        pytest.skip("dropin_test not built (needs the reference headers at build time)")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "checks passed" in r.stdout


def test_dropin_reference_cases_sharded():
    """The same reference cases with every MatvecPlan sharded over GPUs by
    the drop-in (LTB_DEVICES): two real GPUs when present, else two shards on
    device 0 -- same interface, same bars."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(EXE):
        pytest.skip("dropin_test not built (needs the reference headers at build time)")
    devs = "0,1" if torch.cuda.device_count() >= 2 else "0,0"
    env = dict(os.environ, LTB_DEVICES=devs)
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=300, env=env)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "checks passed" in r.stdout
