"""ctypes binding of libhrkan.so (include/hrkan.h).  Argument marshalling only: every step of the
hot path runs in the library's CUDA kernels.  There is no CPU fallback: if the shared library is
missing or the device is not a B200, the calls raise.

Tensors may be torch CUDA tensors (fast path) or CPU tensors / numpy arrays (host buffers: the
library stages them with cudaMemcpyAsync on the stream, see include/hrkan.h)."""
from __future__ import annotations

import ctypes
import math
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libhrkan.so")
if os.environ.get("HRKAN_LIB"):             # experiment variants only (scripts/build_variant.py)
    LIB_PATH = os.environ["HRKAN_LIB"]

HRKAN_POISSON = 0
HRKAN_BURGERS = 1
HRKAN_KAWAHARA = 2
HRKAN_ANISO = 3
JET_TAYLOR5, JET_HESSIAN = 1, 2
ENGINE_AUTO, ENGINE_SIMT, ENGINE_TC = 0, 1, 2

KERNEL_CLASSES = ["fwd_first", "fwd_hidden", "fwd_last", "loss", "wgrad_first", "wgrad_hidden", "wgrad_last",
                  "dgrad_hidden", "dgrad_last", "reduce", "adam", "other", "fused_step"]   # hrkan_kernel_class order

_STATUS = {0: "OK", 1: "EINVAL", 2: "EUNSUPPORTED", 3: "ENOMEM", 4: "ECUDA", 5: "ENONFINITE"}

# (name, restype, argtypes): every symbol include/hrkan.h declares
_P = ctypes.c_void_p
_I32, _I64, _F, _U64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_uint64
SYMBOLS = [
    ("hrkan_create", ctypes.c_int, [ctypes.POINTER(_I32), _I32, _I32, _I32, _I32, _F, _F, _U64, _I32, ctypes.POINTER(_P)]),
    ("hrkan_execution_widths", ctypes.c_int, [ctypes.POINTER(_I32), _I32, _I32, _I32, ctypes.POINTER(_I32)]),
    ("hrkan_num_params", _I64, [_P]),
    ("hrkan_get_params", ctypes.c_int, [_P, _P, _P]),
    ("hrkan_set_params", ctypes.c_int, [_P, _P, _P]),
    ("hrkan_init_params", ctypes.c_int, [_P, _U64, _P]),
    ("hrkan_forward_jet", ctypes.c_int, [_P, _P, _I64, _P, _P, _P, _P]),
    ("hrkan_forward_jet_ex", ctypes.c_int, [_P, _I32, _P, _I64, _P, _P]),
    ("hrkan_pinn_loss_grad", ctypes.c_int, [_P, _P, _P, _P, _I64, _P, _P, _I64, _P, _P, _I64, _I64, _I64, _P, _P]),
    ("hrkan_adam_step", ctypes.c_int, [_P, _P, _F, _F, _F, _F, _P]),
    ("hrkan_set_chunk_points", ctypes.c_int, [_P, _I64]),
    ("hrkan_set_engine", ctypes.c_int, [_P, _I32]),
    ("hrkan_set_graph_mode", ctypes.c_int, [_P, _I32]),
    ("hrkan_launch_count", _I64, [_P]),
    ("hrkan_profile_enable", ctypes.c_int, [_P, _I32]),
    ("hrkan_profile_read", ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_I64)]),
    ("hrkan_free", None, [_P]),
    ("hrkan_last_error", ctypes.c_char_p, []),
]


class HrkanPde(ctypes.Structure):
    _fields_ = [("kind", _I32), ("alpha", _F), ("adv", _F), ("visc", _F), ("disp3", _F), ("disp5", _F),
                ("aniso", _F * 6)]


class HrkanError(RuntimeError):
    pass


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libhrkan.so (raises if it has not been built: `python __graft_entry__.py build`)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise HrkanError(f"libhrkan.so not built at {path}; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    for name, res, args in SYMBOLS:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(status: int, what: str):
    if status != 0:
        msg = _lib.hrkan_last_error().decode(errors="replace")
        raise HrkanError(f"{what} failed: {_STATUS.get(status, status)}: {msg}")


def _ptr(x) -> Optional[int]:
    """Raw pointer of a contiguous float32 torch tensor or numpy array (None -> NULL)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        if x.dtype != np.float32 or not x.flags["C_CONTIGUOUS"]:
            raise TypeError("numpy buffers must be contiguous float32")
        return x.ctypes.data
    import torch
    if not isinstance(x, torch.Tensor):
        raise TypeError(f"unsupported buffer type {type(x)}")
    if x.dtype != torch.float32 or not x.is_contiguous():
        raise TypeError("tensors must be contiguous float32")
    return x.data_ptr()


def _numel(x) -> int:
    if x is None:
        return 0
    return int(x.size if isinstance(x, np.ndarray) else x.numel())


def _stream(stream) -> Optional[int]:
    if stream is not None:
        return int(stream)
    import torch
    if torch.cuda.is_available():
        return torch.cuda.current_stream().cuda_stream
    return None


def pde_struct(kind: str, alpha: float = 0.05, adv: float = 1.0, visc: float = 0.01 / math.pi,
               disp3: float = 0.0, disp5: float = 0.0, aniso=None) -> HrkanPde:
    """kind: "poisson" | "burgers" (adv, visc) | "kawahara" (adv, disp3, disp5) | "aniso" (aniso = the
    upper-triangle coefficients of u_ab, D=2: xx, xy, yy; D=3: xx, xy, xz, yy, yz, zz)."""
    k = {"poisson": HRKAN_POISSON, "burgers": HRKAN_BURGERS, "kawahara": HRKAN_KAWAHARA, "aniso": HRKAN_ANISO}[kind]
    K = (_F * 6)(*(list(aniso or []) + [0.0] * (6 - len(aniso or []))))
    return HrkanPde(k, alpha, adv if k in (HRKAN_BURGERS, HRKAN_KAWAHARA) else 0.0,
                    visc if k == HRKAN_BURGERS else 0.0, disp3 if k == HRKAN_KAWAHARA else 0.0,
                    disp5 if k == HRKAN_KAWAHARA else 0.0, K)


def jet_channels(kind: int, D: int) -> int:
    """Channels of hrkan_forward_jet_ex: TAYLOR5 [u, u_x .. u_xxxxx, u_t]; HESSIAN [u, u_a, u_ab (a <= b)]."""
    return 7 if kind == JET_TAYLOR5 else 1 + D + D * (D + 1) // 2


class HRKANNet:
    """One network on one device (see include/hrkan.h for every call's contract)."""

    def __init__(self, widths, G: int, k: int, m: int, lo: float = -1.0, hi: float = 1.0,
                 seed: int = 1, device: int = 0):
        lib = load_library()
        w = (ctypes.c_int32 * len(widths))(*widths)
        h = ctypes.c_void_p()
        _check(lib.hrkan_create(w, len(widths), G, k, m, lo, hi, seed, device, ctypes.byref(h)), "hrkan_create")
        self._h = h
        self.widths = list(widths)
        self.D = widths[0]
        self.G, self.k, self.m, self.B = G, k, m, G + k
        self.device = device
        self.n_params = int(lib.hrkan_num_params(h))

    # ------------------------------------------------------------------ lifecycle
    def close(self):
        if getattr(self, "_h", None):
            _lib.hrkan_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ parameters
    def get_params(self, out=None, stream=None):
        import torch
        if out is None:
            out = torch.empty(self.n_params, dtype=torch.float32, device=f"cuda:{self.device}")
        assert _numel(out) == self.n_params
        _check(_lib.hrkan_get_params(self._h, _ptr(out), _stream(stream)), "hrkan_get_params")
        return out

    def set_params(self, src, stream=None):
        assert _numel(src) == self.n_params
        _check(_lib.hrkan_set_params(self._h, _ptr(src), _stream(stream)), "hrkan_set_params")

    def init_params(self, seed: int, stream=None):
        _check(_lib.hrkan_init_params(self._h, seed, _stream(stream)), "hrkan_init_params")

    def set_chunk_points(self, n: int):
        _check(_lib.hrkan_set_chunk_points(self._h, n), "hrkan_set_chunk_points")

    def set_engine(self, mode: int):
        _check(_lib.hrkan_set_engine(self._h, mode), "hrkan_set_engine")

    def set_graph_mode(self, on: bool = True):
        """CUDA-graph replay of pinn_loss_grad for repeated calls with the same device buffers."""
        _check(_lib.hrkan_set_graph_mode(self._h, 1 if on else 0), "hrkan_set_graph_mode")

    def launch_count(self) -> int:
        return int(_lib.hrkan_launch_count(self._h))

    def profile_enable(self, on: bool = True):
        _check(_lib.hrkan_profile_enable(self._h, 1 if on else 0), "hrkan_profile_enable")

    def profile_read(self):
        """{class name: (total device ms, launches)} since the last read (synchronises the events)."""
        ms = (ctypes.c_double * len(KERNEL_CLASSES))()
        n = (_I64 * len(KERNEL_CLASSES))()
        _check(_lib.hrkan_profile_read(self._h, ms, n), "hrkan_profile_read")
        return {name: (ms[i], int(n[i])) for i, name in enumerate(KERNEL_CLASSES)}

    # ------------------------------------------------------------------ hot path
    def forward_jet(self, pts, u=None, du=None, d2u=None, stream=None):
        """u[P], du[P,D], d2u[P,D] at pts[P,D] (allocated on the device if not given)."""
        import torch
        P = _numel(pts) // self.D
        dev = f"cuda:{self.device}"
        if u is None:
            u = torch.empty(P, dtype=torch.float32, device=dev)
        if du is None:
            du = torch.empty(P, self.D, dtype=torch.float32, device=dev)
        if d2u is None:
            d2u = torch.empty(P, self.D, dtype=torch.float32, device=dev)
        _check(_lib.hrkan_forward_jet(self._h, _ptr(pts), P, _ptr(u), _ptr(du), _ptr(d2u), _stream(stream)),
               "hrkan_forward_jet")
        return u, du, d2u

    def forward_jet_ex(self, kind: int, pts, jet=None, stream=None):
        """Higher-order / mixed jet jet[P, C] (JET_TAYLOR5 or JET_HESSIAN, see include/hrkan.h)."""
        import torch
        P = _numel(pts) // self.D
        if jet is None:
            jet = torch.empty(P, jet_channels(kind, self.D), dtype=torch.float32, device=f"cuda:{self.device}")
        _check(_lib.hrkan_forward_jet_ex(self._h, kind, _ptr(pts), P, _ptr(jet), _stream(stream)), "hrkan_forward_jet_ex")
        return jet

    def pinn_loss_grad(self, pde: HrkanPde, interior, boundary, g_boundary, initial=None, g_initial=None,
                       forcing=None, n_int_global: Optional[int] = None, n_bi_global: Optional[int] = None,
                       out=None, stream=None):
        """Returns out[num_params + 4] = [dL/dtheta | alpha*L_pde | L_bi | nonfinite flag | 0]."""
        import torch
        D = self.D
        Ni = _numel(interior) // D
        Nb = _numel(boundary) // D
        N0 = _numel(initial) // D
        if n_int_global is None:
            n_int_global = Ni
        if n_bi_global is None:
            n_bi_global = Nb + N0
        if out is None:
            out = torch.empty(self.n_params + 4, dtype=torch.float32, device=f"cuda:{self.device}")
        assert _numel(out) == self.n_params + 4
        _check(_lib.hrkan_pinn_loss_grad(self._h, ctypes.byref(pde), _ptr(interior), _ptr(forcing), Ni,
                                         _ptr(boundary), _ptr(g_boundary), Nb, _ptr(initial), _ptr(g_initial), N0,
                                         n_int_global, n_bi_global, _ptr(out), _stream(stream)),
               "hrkan_pinn_loss_grad")
        return out

    def adam_step(self, grad, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, stream=None):
        _check(_lib.hrkan_adam_step(self._h, _ptr(grad), lr, beta1, beta2, eps, _stream(stream)), "hrkan_adam_step")
