"""ctypes binding of ``libbfq.so`` (the C ABI declared in ``include/bfq.h``).

The shared library is built in-tree by ``__graft_entry__.build()``.  There is
no fallback: if the library is missing every entry point raises, so a GPU
code path can never silently degrade to a CPU implementation.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import _build

_HERE = os.path.dirname(os.path.abspath(__file__))
# BFQ_LIB=checked selects the self-checking build (libbfq_checked.so),
# BFQ_LIB=timing the timing-experiment build (libbfq_timing.so)
VARIANT = os.environ.get("BFQ_LIB", "")
CHECKED = VARIANT == "checked"
LIB_SEL = VARIANT if VARIANT in ("checked", "timing", "exp") else False
LIB_PATH = _build.lib_path(LIB_SEL)

BFQ_OK = 0
BFQ_EINVAL = -1
BFQ_EUNSORTED = -2
BFQ_ECUDA = -3
BFQ_ENOMEM = -4
BFQ_ESMEM = -5
BFQ_EIO = -6
BFQ_EFORMAT = -7
BFQ_EINTEGRITY = -8
BFQ_EDIVERGED = -9

# every symbol include/bfq.h declares (checked by tests/test_abi.py)
EXPORTED_SYMBOLS = (
    "bfq_plan_create",
    "bfq_plan_create_bfct",
    "bfq_plan_destroy",
    "bfq_plan_get_info",
    "bfq_plan_work",
    "bfq_eval",
    "bfq_eval_host",
    "bfq_rk4_step",
    "bfq_moments",
    "bfq_host_plan_info",
    "bfq_project_maxwellians",
    "bfq_projector_create",
    "bfq_project_samples",
    "bfq_projector_destroy",
    "bfq_projector_work",
    "bfq_projector_kernel",
    "bfq_strerror",
    "bfq_last_error",
    "bfq_build_id",
)
# every symbol include/bfr.h declares
EXPORTED_SYMBOLS_BFR = ("bfr_assemble",)

_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)


class BfqDesc(ctypes.Structure):
    _fields_ = [
        ("k_max", ctypes.c_int32),
        ("l_max", ctypes.c_int32),
        ("gamma", ctypes.c_double),
        ("n_t", ctypes.c_int32),
        ("n_g", ctypes.c_int64),
        ("n_s", ctypes.c_int64),
        ("triplets", _i32p),
        ("q1", _i32p),
        ("q2", _i32p),
        ("q3", _i32p),
        ("tau", _i32p),
        ("g", _f64p),
        ("slice_starts", _i64p),
        ("slice_tau", _i32p),
        ("slice_q1", _i32p),
        ("r", _f64p),
        ("conservation", ctypes.c_int32),
        ("detailed_balance", ctypes.c_int32),
    ]


class BfqPlanInfo(ctypes.Structure):
    _fields_ = [
        ("n_k", ctypes.c_int32),
        ("n_q", ctypes.c_int32),
        ("n_t", ctypes.c_int32),
        ("n_g", ctypes.c_int64),
        ("n_s", ctypes.c_int64),
        ("folded", ctypes.c_int32),
        ("cells_per_cta", ctypes.c_int32),
        ("warps_per_cta", ctypes.c_int32),
        ("stages", ctypes.c_int32),
        ("smem_bytes", ctypes.c_int32),
        ("items_per_tile", ctypes.c_int32),
        ("exec_macs_per_cell", ctypes.c_double),
        ("operator_bytes", ctypes.c_double),
        ("useful_macs_per_cell", ctypes.c_double),
    ]


class BfrDesc(ctypes.Structure):
    """include/bfr.h bfr_desc."""

    _fields_ = [
        ("k_max", ctypes.c_int32),
        ("l_max", ctypes.c_int32),
        ("gamma", ctypes.c_double),
        ("kernel_scale", ctypes.c_double),
        ("n_t", ctypes.c_int32),
        ("triplets", _i32p),
        ("swap", _i32p),
        ("w3j", _f64p),
        ("chan_scale", _f64p),
        ("n_e", ctypes.c_int32),
        ("e_x", _f64p),
        ("e_w", _f64p),
        ("n_chi", ctypes.c_int32),
        ("chi_x", _f64p),
        ("chi_w", _f64p),
        ("n_eps", ctypes.c_int32),
        ("eps_x", _f64p),
        ("eps_w", _f64p),
        ("n_outer", ctypes.c_int32 * 2),
        ("n_inner", ctypes.c_int32 * 2),
        ("outer_x", _f64p * 2),
        ("outer_w", _f64p * 2),
        ("inner_x", _f64p * 2),
        ("inner_w", _f64p * 2),
        ("mono", _f64p),
        ("norms", _f64p),
    ]


class BfrStats(ctypes.Structure):
    _fields_ = [
        ("ms_total", ctypes.c_double),
        ("ms_contract", ctypes.c_double),
        ("contract_macs", ctypes.c_double),
        ("alg_macs", ctypes.c_double),
        ("x_bytes", ctypes.c_double),
        ("n_points", ctypes.c_int64 * 2),
        ("launches", ctypes.c_int64),
    ]


class EngineUnavailable(RuntimeError):
    """The CUDA engine library is not built or cannot be loaded."""


_lib = None
_lock = threading.Lock()


def _declare(lib):
    vp = ctypes.c_void_p
    lib.bfq_plan_create.argtypes = [ctypes.POINTER(BfqDesc), ctypes.c_int, ctypes.POINTER(vp)]
    lib.bfq_plan_create_bfct.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(vp)]
    lib.bfq_plan_destroy.argtypes = [vp]
    lib.bfq_plan_get_info.argtypes = [vp, ctypes.POINTER(BfqPlanInfo)]
    lib.bfq_plan_work.argtypes = [vp, _f64p, _f64p]
    lib.bfq_eval.argtypes = [vp, vp, vp, vp, ctypes.c_int64, vp]
    lib.bfq_eval_host.argtypes = [vp, vp, vp, vp, ctypes.c_int64]
    lib.bfq_rk4_step.argtypes = [vp, vp, vp, ctypes.c_int64, ctypes.c_double, vp, vp]
    lib.bfq_moments.argtypes = [vp, vp, vp, ctypes.c_int64, vp]
    lib.bfq_host_plan_info.argtypes = [ctypes.POINTER(BfqDesc), ctypes.c_int, ctypes.POINTER(BfqPlanInfo)]
    lib.bfq_strerror.argtypes = [ctypes.c_int]
    lib.bfq_strerror.restype = ctypes.c_char_p
    lib.bfq_last_error.argtypes = []
    lib.bfq_last_error.restype = ctypes.c_char_p
    lib.bfq_build_id.argtypes = []
    lib.bfq_build_id.restype = ctypes.c_char_p
    lib.bfq_project_maxwellians.argtypes = [ctypes.c_int32, ctypes.c_int32, _f64p, _f64p, ctypes.c_int32, vp, vp, vp,
                                            vp, ctypes.c_int64, vp]
    lib.bfq_projector_create.argtypes = [ctypes.c_int32] * 5 + [_f64p, _f64p, _f64p, ctypes.c_int,
                                                                 ctypes.POINTER(ctypes.c_void_p)]
    lib.bfq_project_samples.argtypes = [vp, vp, vp, ctypes.c_int64, vp]
    lib.bfq_projector_destroy.argtypes = [vp]
    lib.bfq_projector_work.argtypes = [vp, _f64p, _f64p]
    lib.bfq_projector_kernel.argtypes = [vp]
    lib.bfr_assemble.argtypes = [ctypes.POINTER(BfrDesc), ctypes.c_int, vp, vp, ctypes.POINTER(BfrStats)]
    for name in EXPORTED_SYMBOLS + EXPORTED_SYMBOLS_BFR:
        if name not in ("bfq_strerror", "bfq_last_error", "bfq_build_id"):
            getattr(lib, name).restype = ctypes.c_int


def _ensure_current(path: str) -> None:
    """The library must be built from the sources next to it (provenance).
    A stale or missing binary is rebuilt in place (nvcc is part of the image);
    BFQ_NO_AUTOBUILD=1 turns that into an error instead."""
    if _build.is_current(LIB_SEL):
        return
    if os.environ.get("BFQ_NO_AUTOBUILD"):
        raise EngineUnavailable(
            f"{path} is missing or was not built from these sources "
            f"(embedded {_build.embedded_hash(path)}, sources {_build.source_hash(LIB_SEL)}): "
            "rebuild with `python -c 'import __graft_entry__ as g; g.build()'`")
    import fcntl
    import sys

    os.makedirs(_build.BUILD, exist_ok=True)
    with open(os.path.join(_build.BUILD, ".lock"), "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        if not _build.is_current(LIB_SEL):
            sys.stderr.write(f"[bfq] {os.path.basename(path)} stale or missing: rebuilding from source\n")
            try:
                _build.build(checked=LIB_SEL)
            except (RuntimeError, OSError) as exc:
                raise EngineUnavailable(f"cannot build {path}: {exc}") from exc


def lib():
    """Load (once) and return the engine library; raise if it is absent."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None and os.environ.get("BFQ_AB_LIB"):
                # A/B tooling only (tools/gpu/ablib.sh): load a library built from
                # another revision, without the source-hash check
                handle = ctypes.CDLL(os.environ["BFQ_AB_LIB"])
                _declare(handle)
                _lib = handle
                return _lib
            if _lib is None:
                _ensure_current(LIB_PATH)
                if not os.path.exists(LIB_PATH):
                    raise EngineUnavailable(
                        f"{LIB_PATH} is missing: build the CUDA engine with "
                        "`python -c 'import __graft_entry__ as g; g.build()'`"
                    )
                try:
                    handle = ctypes.CDLL(LIB_PATH)
                except OSError as exc:  # pragma: no cover - environment specific
                    raise EngineUnavailable(f"cannot load {LIB_PATH}: {exc}") from exc
                _declare(handle)
                got = handle.bfq_build_id().decode()
                if got != _build.source_hash(LIB_SEL):
                    raise EngineUnavailable(f"{LIB_PATH} build id {got} does not match the sources")
                _lib = handle
    return _lib


def check(code: int) -> None:
    """Map a BFQ_E* code to the reference's exception types."""
    if code == BFQ_OK:
        return
    l = lib()
    msg = f"{l.bfq_strerror(code).decode()}: {l.bfq_last_error().decode()}"
    if code in (BFQ_EINVAL, BFQ_EUNSORTED, BFQ_ESMEM):
        raise ValueError(msg)
    if code == BFQ_EFORMAT:
        from .operator import CacheFormatError

        raise CacheFormatError(msg)
    if code == BFQ_EINTEGRITY:
        from .operator import CacheIntegrityError

        raise CacheIntegrityError(msg)
    if code == BFQ_EIO:
        raise OSError(msg)
    raise RuntimeError(msg)
