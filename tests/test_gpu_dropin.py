"""The integration a reference maintainer would do, run end to end: a C++
program using the reference's OWN CsrMatrix / McConfig / ApproxInverse /
SplitError types and generators calls include/mcmi/mcspai_compat.hpp and the
unmodified reference side by side and requires CsrMatrix::operator== equality
(oracle/dropin_demo.cpp, built by `make -C oracle dropin`)."""
import os
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(REPO, "oracle", "_ref", "dropin_demo")


@pytest.mark.gpu
def test_dropin_demo_byte_identical():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(DEMO):
        pytest.skip("oracle/_ref/dropin_demo not built")
    r = subprocess.run([DEMO], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[FAIL]" not in r.stdout


def test_dropin_demo_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available() or not os.path.exists(DEMO):
        pytest.skip("needs the built demo and no GPU")
    r = subprocess.run([DEMO], capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "mcmi:" in r.stderr


@pytest.mark.gpu
def test_dropin_demo_sharded_via_env():
    """The drop-in's GPU count comes from MCMI_GPUS without a code change; the
    demo's byte-for-byte comparison against the reference must still hold
    (three row shards, all on this box's one GPU via MCMI_SHARD_WRAP)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(DEMO):
        pytest.skip("oracle/_ref/dropin_demo not built")
    env = dict(os.environ, MCMI_GPUS="3", MCMI_SHARD_WRAP="1")
    r = subprocess.run([DEMO], capture_output=True, text=True, timeout=600, env=env)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[FAIL]" not in r.stdout
