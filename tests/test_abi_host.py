"""CPU-side checks of the C ABI boundary: libhrkan.so loads, exports every symbol include/hrkan.h
declares, and rejects invalid arguments before touching a device (no compute calls here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hrkan.h")


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hrkan_[a-z_]+)\s*\(", src)))


def _lib():
    from paper_2409_14248_b200 import hrkan
    if not os.path.exists(hrkan.LIB_PATH):
        pytest.skip("libhrkan.so not built (run __graft_entry__.build())")
    return hrkan.load_library()


def test_header_declares_the_boundary():
    names = _declared_functions()
    for required in ["hrkan_create", "hrkan_forward_jet", "hrkan_pinn_loss_grad", "hrkan_adam_step", "hrkan_free"]:
        assert required in names


def test_library_exports_every_declared_symbol():
    lib = _lib()
    for name in _declared_functions():
        assert hasattr(lib, name), name
    # and the binding wraps exactly the declared set
    from paper_2409_14248_b200 import hrkan
    assert sorted(s[0] for s in hrkan.SYMBOLS) == _declared_functions()


def test_exported_symbols_are_c_linkage():
    so = os.path.join(ROOT, "paper_2409_14248_b200", "_lib", "libhrkan.so")
    if not os.path.exists(so):
        pytest.skip("not built")
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(l.split()[-1] for l in out.splitlines() if " T " in l)
    for name in _declared_functions():
        assert name in exported


def test_invalid_arguments_rejected_without_device():
    lib = _lib()
    from paper_2409_14248_b200 import hrkan
    h = ctypes.c_void_p()

    def create(widths, G=5, k=3, m=4, lo=-1.0, hi=1.0):
        w = (ctypes.c_int32 * len(widths))(*widths)
        return lib.hrkan_create(w, len(widths), G, k, m, lo, hi, 1, 0, ctypes.byref(h))

    EINVAL = 1
    assert create([2]) == EINVAL                     # < 2 widths
    assert create([2, 0, 1]) == EINVAL               # width < 1
    assert create([4, 5, 1]) == EINVAL               # D not in {1,2,3}
    assert create([2, 5, 2]) == EINVAL               # scalar output required
    assert create([2, 5, 1], G=0) == EINVAL
    assert create([2, 5, 1], k=0) == EINVAL
    assert create([2, 5, 1], m=1) == EINVAL          # jets need m >= 2
    assert create([2, 5, 1], m=9) == EINVAL
    assert create([2, 5, 1], lo=1.0, hi=1.0) == EINVAL
    assert create([2, 5, 1], lo=float("nan")) == EINVAL
    assert b"width" in lib.hrkan_last_error() or len(lib.hrkan_last_error()) > 0
    assert lib.hrkan_create(None, 0, 5, 3, 4, -1.0, 1.0, 1, 0, None) == EINVAL
    assert lib.hrkan_num_params(None) == -1
    assert lib.hrkan_launch_count(None) == -1
    lib.hrkan_free(None)                              # no-op
    assert lib.hrkan_set_engine(None, 0) == EINVAL
    assert lib.hrkan_forward_jet(None, None, 0, None, None, None, None) == EINVAL
    pde = hrkan.pde_struct("poisson")
    assert lib.hrkan_pinn_loss_grad(None, ctypes.byref(pde), None, None, 0, None, None, 0, None, None, 0,
                                    0, 0, None, None) == EINVAL


def test_execution_widths_padding_rule(monkeypatch):
    """hrkan_execution_widths (host-only): hidden widths in (32, 256] are padded to 64 / 128 / 256 when the
    net has at least two hidden layers, all in that range, and G + k >= 8; otherwise unchanged."""
    lib = _lib()

    def ew(widths, G=10, k=3):
        w = (ctypes.c_int32 * len(widths))(*widths)
        out = (ctypes.c_int32 * len(widths))()
        assert lib.hrkan_execution_widths(w, len(widths), G, k, out) == 0
        return list(out)

    assert ew([2, 100, 100, 1]) == [2, 128, 128, 1]
    assert ew([2, 48, 200, 72, 1]) == [2, 64, 256, 128, 1]
    assert ew([3, 33, 256, 1]) == [3, 64, 256, 1]
    assert ew([2, 64, 64, 1]) == [2, 64, 64, 1]                   # already tensor-core widths
    assert ew([2, 100, 1]) == [2, 100, 1]                         # one hidden layer: no hidden->hidden contraction
    assert ew([2, 100, 20, 1]) == [2, 100, 20, 1]                 # a thin hidden layer keeps the SIMT engine
    assert ew([2, 100, 300, 1]) == [2, 100, 300, 1]               # wider than the tensor-core kernels take
    assert ew([2, 5, 5, 1]) == [2, 5, 5, 1]                       # tiny nets: the one-launch kernel
    assert ew([2, 100, 100, 1], G=3, k=3) == [2, 100, 100, 1]     # G + k < 8: no tensor-core path
    monkeypatch.setenv("HRKAN_PAD_WIDTHS", "0")
    assert ew([2, 100, 100, 1]) == [2, 100, 100, 1]
    monkeypatch.delenv("HRKAN_PAD_WIDTHS")
    out = (ctypes.c_int32 * 2)()
    assert lib.hrkan_execution_widths(None, 2, 5, 3, out) == 1
    w = (ctypes.c_int32 * 2)(2, 1)
    assert lib.hrkan_execution_widths(w, 1, 5, 3, out) == 1
    assert lib.hrkan_execution_widths(w, 2, 0, 3, out) == 1
