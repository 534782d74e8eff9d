"""Debug builds bound every mbarrier wait (-DHRKAN_HANG_GUARD=1, tc_ptx.cuh): with no compute-sanitizer on
this pool, a barrier-phase bug must surface as a launch failure, not a hung GPU.

* the guarded variant passes tensor-core parity (the guard never fires on a correct pipeline);
* a deliberate deadlock (HRKAN_TC_DBG bit 6: the forward MMA issuer waits for its own first commit)
  traps after HRKAN_HANG_CYCLES (2^31 here, ~1 s) and the call fails with HRKAN_ECUDA, in a subprocess
  (the trap poisons that process's CUDA context) bounded by an outer timeout."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VARIANT = os.path.join(ROOT, "paper_2409_14248_b200", "_lib", "variants", "hangguard", "libhrkan.so")

CHILD = r"""
import os, sys
sys.path.insert(0, os.path.join(ROOT, "tests")); sys.path.insert(0, ROOT)
import numpy as np, torch
import hrkan_inputs as HI
from test_gpu_parity import _make, _loss_grad_gpu, _loss_grad_oracle, _check_loss_grad, _points
w = HI.WORKLOADS["C3"]
ps = _points(w).subset(4, 2)
net, params = _make(w)
if MODE == "parity":
    out = _loss_grad_gpu(torch, net, w, ps)
    _check_loss_grad(out, w, *_loss_grad_oracle(w, params, ps))
    print("PARITY_OK")
else:
    try:
        _loss_grad_gpu(torch, net, w, ps)
        torch.cuda.synchronize()
        print("NO_ERROR")
    except Exception as e:
        print("RAISED", type(e).__name__, str(e)[:200])
"""


@pytest.fixture(scope="module")
def variant():
    if not os.path.exists(VARIANT):
        r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "build_variant.py"), "hangguard",
                            "-DHRKAN_HANG_GUARD=1", "-DHRKAN_HANG_CYCLES=(1ll<<31)"], cwd=ROOT, capture_output=True,
                           text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-2000:]
    return VARIANT


def _run(mode, variant, extra_env=None):
    env = dict(os.environ, HRKAN_LIB=variant, **(extra_env or {}))
    code = f"ROOT = {ROOT!r}\nMODE = {mode!r}\n" + CHILD
    return subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)


def test_guarded_build_passes_parity(variant):
    r = _run("parity", variant)
    assert "PARITY_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_deliberate_deadlock_traps_instead_of_hanging(variant):
    r = _run("hang", variant, {"HRKAN_TC_DBG": "64"})
    out = r.stdout + r.stderr
    assert "hang guard" in out, out[-3000:]
    assert "RAISED" in r.stdout or r.returncode != 0, out[-3000:]
