"""ctypes binding of the C ABI in include/swsdc_b200.h.

The library `libswsdc_b200.so` is built in-tree by `__graft_entry__.build()`
(or `make -C paper_1805_07923_b200/csrc`).  There is no fallback: if the
library is missing or no CUDA device is present, every GPU entry point raises.
Status codes map to the reference's exceptions: 1 -> ValueError (usage),
2 -> RuntimeError (numerics), 3 -> RuntimeError (CUDA).
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SWSDC_LIB: load another build of the library (same-box A/B of kernel changes)
LIB_PATH = os.environ.get("SWSDC_LIB") or os.path.join(_HERE, "libswsdc_b200.so")

_lib = None


class SwsdcCudaError(RuntimeError):
    """A CUDA runtime failure inside the B200 library."""


class Params(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("radius", "omega", "gravity", "nu", "h_bar")]


_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double
_LL = ctypes.c_longlong

_SIGNATURES = {
    "swsdc_last_error": ([], ctypes.c_char_p),
    "swsdc_version": ([], ctypes.c_char_p),
    "swsdc_plan_create": ([_I, _I, _I, _P, _P, ctypes.POINTER(_P)], _I),
    "swsdc_plan_destroy": ([_P], _I),
    "swsdc_plan_reserve": ([_P, _I], _I),
    "swsdc_plan_config": ([_P, _I, _I], _I),
    "swsdc_synthesize": ([_P, _P, _I, _I, _P, _P], _I),
    "swsdc_analyze": ([_P, _P, _I, _P, _P], _I),
    "swsdc_synthesize_uv": ([_P, _P, _P, _I, _I, _P, _P, _P], _I),
    "swsdc_analyze_divcurl": ([_P, _P, _P, _I, _P, _P, _P], _I),
    "swsdc_eval_fe": ([_P, ctypes.POINTER(Params), _I, _P, _I, _P, _P], _I),
    "swsdc_eval_fi": ([_I, ctypes.POINTER(Params), _P, _I, _P, _P], _I),
    "swsdc_set_row_filter": ([_I, _I], _I),
    "swsdc_fe_layout": ([_P, _I, _I, ctypes.POINTER(_LL), ctypes.POINTER(_LL), ctypes.POINTER(_I),
                         ctypes.POINTER(_I)], _I),
    "swsdc_fe_synthesis": ([_P, ctypes.POINTER(Params), _P, _I, _P, _P], _I),
    "swsdc_fe_grid": ([_P, ctypes.POINTER(Params), _I, _P, _I, _I, _I, _P, _P], _I),
    "swsdc_fe_analysis": ([_P, ctypes.POINTER(Params), _I, _P, _I, _P, _P], _I),
    "swsdc_solve_implicit": ([_I, ctypes.POINTER(Params), _D, _P, _I, _P, _P], _I),
    "swsdc_combine": ([_I, ctypes.POINTER(_P), ctypes.POINTER(_D), _LL, _P, _P], _I),
    "swsdc_resize": ([_P, _I, _P, _I, _LL, _P], _I),
    "swsdc_laplacian": ([_P, _P, _I, _LL, _D, _I, _P], _I),
    "swsdc_upload_coeffs": ([_P, _I, _LL, _P, _P], _I),
    "swsdc_pack_triangles": ([_P, _I, _LL, _P], _I),
    "swsdc_spec_combine_multi": ([_I, _P, _P, _P, _P, _I, _LL, _P, _P, _P], _I),
    "swsdc_copy_finite": ([_P, _P, _LL, _P, _P], _I),
    "swsdc_exchange_blocks": ([_P, _LL, _LL, _LL, _LL, _I, _P, _P, _P, _P, _P, _P, _I, _P], _I),
    "swsdc_download_coeffs": ([_P, _I, _LL, _P, _I, _P], _I),
    "swsdc_spec_combine": ([_I, ctypes.POINTER(_P), ctypes.POINTER(_D), ctypes.POINTER(_I), _I, _LL,
                            _P, _P], _I),
    "swsdc_sweep_node": ([_I, ctypes.POINTER(Params), _D, _I, ctypes.POINTER(_P),
                          ctypes.POINTER(_D), _I, _P, _P, _P], _I),
    "swsdc_launch_count": ([], _LL),
    "swsdc_profile_enable": ([_I], _I),
    "swsdc_profile_collect": ([ctypes.c_char_p, _I], _I),
    "swsdc_probe_fp64": ([_I, ctypes.POINTER(_D)], _I),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)


def load(path: str = LIB_PATH):
    """Load (once) and return the library; raises ImportError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = ctypes.CDLL(path)
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def check(status: int) -> None:
    """Raise the reference's exception type for a non-zero status."""
    if status == 0:
        return
    msg = load().swsdc_last_error().decode(errors="replace")
    if status == 1:
        raise ValueError(msg)
    if status == 2:
        raise RuntimeError(msg)
    raise SwsdcCudaError(msg)


def params_struct(p) -> Params:
    return Params(p.radius, p.omega, p.gravity, p.nu, p.h_bar)


def launch_count() -> int:
    return int(load().swsdc_launch_count())


def profile_enable(on: bool) -> None:
    load().swsdc_profile_enable(1 if on else 0)


def profile_collect() -> dict:
    """{stage: (launches, total_ms)} of the events recorded since profile_enable."""
    lib = load()
    need = lib.swsdc_profile_collect(None, 0)
    buf = ctypes.create_string_buffer(max(need, 1))
    lib.swsdc_profile_collect(buf, len(buf))
    out = {}
    for line in buf.value.decode().splitlines():
        name, n, ms = line.split("\t")
        out[name] = (int(n), float(ms))
    return out


def probe_fp64(reps: int = 20) -> float:
    """Measured FP64 FMA peak of the current device, TFLOP/s."""
    out = ctypes.c_double()
    check(load().swsdc_probe_fp64(reps, ctypes.byref(out)))
    return float(out.value)
