"""ctypes binding of libpfx.so (include/pfx.h) — the only route to the compute.

There is no CPU fallback: if the library is missing, or no CUDA device is
present, every compute entry point raises PfexpmError.  Device buffers and
streams come from PyTorch (plumbing only); host arrays may also be passed
directly (PFX_MEM_HOST), in which case the library stages them itself.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import BadSpec, PfexpmError, raise_for_status

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libpfx.so")
PFX_MEM_DEVICE = 0
PFX_MEM_HOST = 1

_lib = None
_lock = threading.Lock()

_dp = ctypes.POINTER(ctypes.c_double)
_fp = ctypes.POINTER(ctypes.c_float)
_i64 = ctypes.c_int64
_int = ctypes.c_int
_vp = ctypes.c_void_p

# name -> (restype, argtypes), mirrors include/pfx.h
SIGNATURES = {
    "pfx_version": (_int, []),
    "pfx_last_error": (ctypes.c_char_p, []),
    "pfx_release": (_int, []),
    "pfx_pole_table": (_int, [_int, _dp, _dp]),
    "pfx_expm_dense": (
        _int,
        [_int, _vp, _int, _i64, _i64, _vp, _int, _i64, ctypes.c_double, _dp, _dp, _int, _vp, _int, _fp, _vp],
    ),
    "pfx_expm_dense_cols": (
        _int,
        [_int, _vp, _int, _i64, ctypes.c_double, _dp, _dp, _int, ctypes.POINTER(_i64), _vp, _int, _int, _vp],
    ),
    "pfx_expm_tridiag": (
        _int,
        [_int, _vp, _vp, _i64, _vp, _i64, ctypes.c_double, _dp, _dp, _int, _vp, _fp, _vp],
    ),
    "pfx_expm_banded": (
        _int,
        [_int, _vp, _i64, _i64, _vp, _i64, ctypes.c_double, _dp, _dp, _int, _vp, _fp, _vp],
    ),
    "pfx_tridiag_shard_rows": (_int, [_i64, _i64, _int, _int, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "pfx_expm_tridiag_shard": (
        _int,
        [_vp, _vp, _i64, _vp, _i64, ctypes.c_double, _dp, _dp, _int, _vp, _int, _int, _vp, _vp, _vp],
    ),
    "pfx_prof_enable": (_int, [_int]),
    "pfx_prof_read": (_int, [ctypes.c_char_p, _int]),
    "pfx_set_pivot_mode": (_int, [_int]),
    "pfx_get_pivot_mode": (_int, []),
    "pfx_pivot_fallbacks": (ctypes.c_longlong, []),
    "pfx_shifted_solve": (
        _int,
        [_int, _vp, _int, _i64, ctypes.c_double, ctypes.c_double, _vp, _i64, _vp, _vp],
    ),
}


def lib():
    """Load libpfx.so once (raises PfexpmError if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise PfexpmError(
                    f"native library {LIB_PATH} is missing; run `python -m paper_2306_16778_b200.build`"
                )
            handle = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def available() -> bool:
    return os.path.exists(LIB_PATH)


def last_error() -> str:
    return lib().pfx_last_error().decode()


def _check(status: int, what: str) -> None:
    if status != 0:
        raise_for_status(status, what, last_error())


def _f64p(arr: np.ndarray):
    return arr.ctypes.data_as(_dp)


def prof_enable(on: bool) -> None:
    lib().pfx_prof_enable(1 if on else 0)


def prof_read() -> dict:
    """{kernel name: (launches, total_ms, total_flops)} since the last read (synchronises the events)."""
    buf = ctypes.create_string_buffer(1 << 16)
    lib().pfx_prof_read(buf, len(buf))
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, tot, fl = line.split()
        out[name] = (int(cnt), float(tot), float(fl))
    return out


PIVOT_MODES = {"checked": 0, "always": 1, "none": 2}


def set_pivot_mode(mode: str) -> None:
    """Dense pivoting policy (include/pfx.h pfx_set_pivot_mode): 'checked' (default: partial
    pivoting semantics, interchange-free kernels verified column by column, redone with
    interchanges when a check fails), 'always' (getrf interchanges), 'none' (unchecked)."""
    if mode not in PIVOT_MODES:
        raise BadSpec(f"pivot mode must be one of {sorted(PIVOT_MODES)}, got {mode!r}")
    _check(lib().pfx_set_pivot_mode(PIVOT_MODES[mode]), "pfx_set_pivot_mode")


def get_pivot_mode() -> str:
    m = lib().pfx_get_pivot_mode()
    return {v: k for k, v in PIVOT_MODES.items()}[m]


def pivot_fallbacks() -> int:
    """Dense calls whose checked interchange-free factorisation was redone with interchanges."""
    return int(lib().pfx_pivot_fallbacks())


def pole_table(n: int):
    theta2 = np.zeros(n, dtype=np.float64)
    coef2 = np.zeros(n, dtype=np.float64)
    _check(lib().pfx_pole_table(n, _f64p(theta2), _f64p(coef2)), f"pfx_pole_table(n={n})")
    return theta2, coef2


# ---- device plumbing (torch) --------------------------------------------------

_torch_ok = None


def _torch():
    global _torch_ok
    if _torch_ok is None:
        import torch

        if not torch.cuda.is_available():
            raise PfexpmError("no CUDA device: the B200 engine has no CPU fallback")
        _torch_ok = torch
    return _torch_ok


def _stream_ptr(stream=None) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _as_device(x: np.ndarray, torch, device):
    t = torch.from_numpy(np.ascontiguousarray(x))
    return t.to(device, non_blocking=False)


def _f64_view(t):
    """Raw float64 storage of a real or complex128 tensor (contiguous)."""
    import torch

    if not isinstance(t, torch.Tensor) or t.device.type != "cuda":
        raise BadSpec("expected a tensor on the CUDA device")
    t = t.contiguous()
    if t.dtype == torch.complex128:
        return t
    if t.dtype != torch.float64:
        raise BadSpec(f"expected float64/complex128 tensor, got {t.dtype}")
    return t


def _real_dev(t, name: str, shape=None):
    """A float64 CUDA tensor argument, contiguous.  The caller keeps the returned tensor
    referenced until the call has returned (a temporary .contiguous() copy freed early would
    hand the library a dangling pointer).  Wrong dtype / device / shape -> BadSpec (never an
    out-of-bounds read of misinterpreted memory)."""
    import torch

    if not isinstance(t, torch.Tensor):
        raise BadSpec(f"{name} must be a torch tensor on the CUDA device")
    if t.dtype != torch.float64:
        raise BadSpec(f"{name} must be float64, got {t.dtype}")
    if t.device.type != "cuda":
        raise BadSpec(f"{name} must live on a CUDA device, got {t.device}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise BadSpec(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    return t.contiguous()


def _ptr(t) -> int:
    return int(t.data_ptr()) if t is not None else 0


# ---- dense ---------------------------------------------------------------------

def expm_dense_device(A, V, theta2, coef2, shift_c: float, out=None, per_pair_ms=None, stream=None):
    """Device-tensor entry: A (batch,d,d) or (d,d); V (batch,d,nrhs)/(d,nrhs)/(d,) or None (full)."""
    torch = _torch()
    A = _f64_view(A)
    if A.dim() not in (2, 3) or A.shape[-1] != A.shape[-2]:
        raise BadSpec(f"A must be (d, d) or (batch, d, d), got {tuple(A.shape)}")
    squeeze_batch = A.dim() == 2
    if squeeze_batch:
        A = A.unsqueeze(0)
    batch, d = A.shape[0], A.shape[1]
    a_complex = A.dtype == torch.complex128
    full = V is None
    v_complex = False
    nrhs = 0
    squeeze_vec = False
    if not full:
        V = _f64_view(V)
        if squeeze_batch:
            V = V.unsqueeze(0)
        if V.dim() == 2:
            V = V.unsqueeze(-1)
            squeeze_vec = True
        if V.shape[0] != batch or V.shape[1] != d:
            raise BadSpec(f"V shape {tuple(V.shape)} does not match A {tuple(A.shape)}")
        nrhs = V.shape[2]
        v_complex = V.dtype == torch.complex128
    real_path = (not a_complex) and (full or not v_complex)
    ncols = d if full else nrhs
    odt = torch.float64 if real_path else torch.complex128
    if out is None:
        out = torch.empty((batch, d, ncols), dtype=odt, device=A.device)
    elif out.dtype != odt or out.numel() != batch * d * ncols or not out.is_contiguous() or out.device != A.device:
        raise BadSpec(f"out must be a contiguous {odt} tensor with {batch * d * ncols} elements on {A.device}")
    npairs = len(theta2) // 2
    ms = (ctypes.c_float * npairs)() if per_pair_ms is not None else None
    st = lib().pfx_expm_dense(
        PFX_MEM_DEVICE, _ptr(A), int(a_complex), d, batch, _ptr(V) if not full else None, int(v_complex), nrhs,
        float(shift_c), _f64p(theta2), _f64p(coef2), npairs, _ptr(out), int(not real_path),
        ctypes.cast(ms, _fp) if ms is not None else None, _stream_ptr(stream),
    )
    _check(st, "pfx_expm_dense")
    if per_pair_ms is not None:
        per_pair_ms[:] = list(ms)
    res = out
    if squeeze_vec:
        res = res.squeeze(-1)
    if squeeze_batch:
        res = res.squeeze(0)
    return res


def expm_dense_host(A: np.ndarray, V, theta2, coef2, shift_c: float, per_pair_ms=None, out=None):
    """Host-array entry through PFX_MEM_HOST (the library stages H2D/D2H itself)."""
    _torch()  # asserts a device exists
    A = np.ascontiguousarray(A)
    squeeze_batch = A.ndim == 2
    if squeeze_batch:
        A = A[None]
    batch, d = A.shape[0], A.shape[1]
    a_complex = np.iscomplexobj(A)
    A = A.astype(np.complex128 if a_complex else np.float64, copy=False)
    full = V is None
    nrhs, v_complex, squeeze_vec = 0, False, False
    if not full:
        V = np.ascontiguousarray(V)
        if squeeze_batch:
            V = V[None]
        if V.ndim == 2:
            V = V[..., None]
            squeeze_vec = True
        nrhs = V.shape[2]
        v_complex = np.iscomplexobj(V)
        V = np.ascontiguousarray(V.astype(np.complex128 if v_complex else np.float64, copy=False))
    real_path = (not a_complex) and (full or not v_complex)
    ncols = d if full else nrhs
    odt = np.float64 if real_path else np.complex128
    if out is None or out.dtype != odt or out.size != batch * d * ncols:
        out = np.empty((batch, d, ncols), dtype=odt)
    out = out.reshape(batch, d, ncols)
    npairs = len(theta2) // 2
    ms = (ctypes.c_float * npairs)() if per_pair_ms is not None else None
    st = lib().pfx_expm_dense(
        PFX_MEM_HOST, A.ctypes.data, int(a_complex), d, batch, V.ctypes.data if not full else None, int(v_complex),
        nrhs, float(shift_c), _f64p(theta2), _f64p(coef2), npairs, out.ctypes.data, int(not real_path),
        ctypes.cast(ms, _fp) if ms is not None else None, None,
    )
    _check(st, "pfx_expm_dense")
    if per_pair_ms is not None:
        per_pair_ms[:] = list(ms)
    if squeeze_vec:
        out = out[..., 0]
    if squeeze_batch:
        out = out[0]
    return out


def expm_dense_cols_device(A, theta2, coef2, col_ranges, shift_c: float = 0.0, out=None, accumulate=False,
                           stream=None):
    """Column split of the full mode (include/pfx.h pfx_expm_dense_cols): pair k contributes the
    columns [col_ranges[k][0], col_ranges[k][1]) of its inverse.  A (d, d) device tensor, d > 512;
    returns / updates the (d, d) partial whose sum over a partition of the columns is exp(A)."""
    torch = _torch()
    A = _f64_view(A)
    if A.dim() != 2 or A.shape[0] != A.shape[1]:
        raise BadSpec(f"A must be (d, d), got {tuple(A.shape)}")
    d = A.shape[0]
    a_complex = A.dtype == torch.complex128
    odt = torch.complex128 if a_complex else torch.float64
    npairs = len(theta2) // 2
    rg = np.ascontiguousarray(np.asarray(col_ranges, dtype=np.int64).reshape(-1))
    if rg.size != 2 * npairs:
        raise BadSpec(f"col_ranges needs one (c0, c1) per pair: {npairs} pairs, got {rg.size // 2} ranges")
    if out is None:
        if accumulate:
            raise BadSpec("accumulate needs an out tensor")
        out = torch.empty((d, d), dtype=odt, device=A.device)
    elif out.dtype != odt or tuple(out.shape) != (d, d) or not out.is_contiguous() or out.device != A.device:
        raise BadSpec(f"out must be a contiguous ({d}, {d}) {odt} tensor on {A.device}")
    st = lib().pfx_expm_dense_cols(
        PFX_MEM_DEVICE, _ptr(A), int(a_complex), d, float(shift_c), _f64p(theta2), _f64p(coef2), npairs,
        rg.ctypes.data_as(ctypes.POINTER(_i64)), _ptr(out), int(a_complex), int(bool(accumulate)), _stream_ptr(stream),
    )
    _check(st, "pfx_expm_dense_cols")
    return out


def expm_dense_cols_host(A: np.ndarray, theta2, coef2, col_ranges, shift_c: float = 0.0, out=None, accumulate=False):
    """Host-array form of expm_dense_cols_device (PFX_MEM_HOST)."""
    _torch()
    A = np.ascontiguousarray(A)
    if A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise BadSpec(f"A must be (d, d), got {A.shape}")
    d = A.shape[0]
    a_complex = np.iscomplexobj(A)
    A = A.astype(np.complex128 if a_complex else np.float64, copy=False)
    odt = np.complex128 if a_complex else np.float64
    npairs = len(theta2) // 2
    rg = np.ascontiguousarray(np.asarray(col_ranges, dtype=np.int64).reshape(-1))
    if rg.size != 2 * npairs:
        raise BadSpec(f"col_ranges needs one (c0, c1) per pair: {npairs} pairs, got {rg.size // 2} ranges")
    if out is None:
        if accumulate:
            raise BadSpec("accumulate needs an out array")
        out = np.empty((d, d), dtype=odt)
    elif out.dtype != odt or out.shape != (d, d) or not out.flags.c_contiguous:
        raise BadSpec(f"out must be a C-contiguous ({d}, {d}) {odt} array")
    st = lib().pfx_expm_dense_cols(
        PFX_MEM_HOST, A.ctypes.data, int(a_complex), d, float(shift_c), _f64p(theta2), _f64p(coef2), npairs,
        rg.ctypes.data_as(ctypes.POINTER(_i64)), out.ctypes.data, int(a_complex), int(bool(accumulate)), None,
    )
    _check(st, "pfx_expm_dense_cols")
    return out


# ---- tridiagonal / banded ------------------------------------------------------

def _out_dev(out, shape, like):
    import torch

    if out is None:
        return torch.empty(shape, dtype=torch.float64, device=like.device)
    if out.dtype != torch.float64 or tuple(out.shape) != tuple(shape) or not out.is_contiguous() \
            or out.device != like.device:
        raise BadSpec(f"out must be a contiguous float64 tensor of shape {tuple(shape)} on {like.device}")
    return out


def expm_tridiag_device(diag, off, V, theta2, coef2, shift_c: float, out=None, per_pair_ms=None, stream=None):
    torch = _torch()
    squeeze = V.dim() == 1
    if squeeze:
        V = V.unsqueeze(-1)
    if V.dim() != 2:
        raise BadSpec(f"V must be (N,) or (N, nrhs), got {tuple(V.shape)}")
    N, nrhs = V.shape
    V = _real_dev(V, "V")
    diag = _real_dev(diag, "diag", (N,))
    off = _real_dev(off, "off", (N - 1,))
    out = _out_dev(out, (N, nrhs), V)
    npairs = len(theta2) // 2
    ms = (ctypes.c_float * npairs)() if per_pair_ms is not None else None
    st = lib().pfx_expm_tridiag(
        PFX_MEM_DEVICE, _ptr(diag), _ptr(off) if N > 1 else None, N, _ptr(V), nrhs, float(shift_c),
        _f64p(theta2), _f64p(coef2), npairs, _ptr(out), ctypes.cast(ms, _fp) if ms is not None else None,
        _stream_ptr(stream),
    )
    _check(st, "pfx_expm_tridiag")
    if per_pair_ms is not None:
        per_pair_ms[:] = list(ms)
    return out.squeeze(-1) if squeeze else out


# pfx_allgather_fn: int (*)(void* ctx, double* buf, int64_t count)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, _dp, ctypes.c_int64)


def tridiag_shard_rows(N: int, nrhs: int, rank: int, nranks: int):
    """Rows [r0, r1) that rank `rank` of `nranks` owns in pfx_expm_tridiag_shard."""
    r0, r1 = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().pfx_tridiag_shard_rows(N, nrhs, rank, nranks, ctypes.byref(r0), ctypes.byref(r1)),
           "pfx_tridiag_shard_rows")
    return r0.value, r1.value


def expm_tridiag_shard(diag, off, V, theta2, coef2, shift_c: float, rank: int, nranks: int, allgather, out=None,
                       stream=None):
    """Row-sharded tridiagonal exp(A)V (include/pfx.h pfx_expm_tridiag_shard): this rank's
    rows [r0, r1) of `out` (N x nrhs, device) are written, final.  `allgather(mine)` takes this
    rank's float64 block and returns all ranks' blocks concatenated in rank order."""
    torch = _torch()
    squeeze = V.dim() == 1
    if squeeze:
        V = V.unsqueeze(-1)
    if V.dim() != 2:
        raise BadSpec(f"V must be (N,) or (N, nrhs), got {tuple(V.shape)}")
    N, nrhs = V.shape
    V = _real_dev(V, "V")
    diag = _real_dev(diag, "diag", (N,))
    off = _real_dev(off, "off", (N - 1,))
    if out is None:
        out = torch.zeros((N, nrhs), dtype=torch.float64, device=V.device)
    out = _out_dev(out, (N, nrhs), V)
    failure = []

    def _cb(ctx, buf, count):
        try:
            full = np.ctypeslib.as_array(buf, shape=(nranks * count,))
            mine = full[rank * count:(rank + 1) * count].copy()
            got = np.asarray(allgather(mine), dtype=np.float64).reshape(-1)
            if got.size != nranks * count:
                raise ValueError(f"allgather returned {got.size} values, expected {nranks * count}")
            full[:] = got
            return 0
        except Exception as exc:  # reported through the status below
            failure.append(exc)
            return 1

    cb = ALLGATHER_FN(_cb)
    st = lib().pfx_expm_tridiag_shard(
        _ptr(diag), _ptr(off) if N > 1 else None, N, _ptr(V), nrhs, float(shift_c), _f64p(theta2),
        _f64p(coef2), len(theta2) // 2, _ptr(out), rank, nranks, ctypes.cast(cb, _vp), None, _stream_ptr(stream),
    )
    if failure:
        raise failure[0]
    _check(st, "pfx_expm_tridiag_shard")
    return out.squeeze(-1) if squeeze else out


def expm_tridiag_host(diag, off, V, theta2, coef2, shift_c: float, per_pair_ms=None, out=None):
    _torch()
    diag = np.ascontiguousarray(diag, dtype=np.float64)
    off = np.ascontiguousarray(off, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    squeeze = V.ndim == 1
    V = np.ascontiguousarray(V[:, None] if squeeze else V)
    N, nrhs = V.shape
    if out is None or out.size != N * nrhs:
        out = np.empty((N, nrhs), dtype=np.float64)
    out = out.reshape(N, nrhs)
    npairs = len(theta2) // 2
    ms = (ctypes.c_float * npairs)() if per_pair_ms is not None else None
    st = lib().pfx_expm_tridiag(
        PFX_MEM_HOST, diag.ctypes.data, off.ctypes.data if N > 1 else None, N, V.ctypes.data, nrhs, float(shift_c),
        _f64p(theta2), _f64p(coef2), npairs, out.ctypes.data, ctypes.cast(ms, _fp) if ms is not None else None, None,
    )
    _check(st, "pfx_expm_tridiag")
    if per_pair_ms is not None:
        per_pair_ms[:] = list(ms)
    return out[:, 0] if squeeze else out


def expm_banded_host(band, V, theta2, coef2, shift_c: float, per_pair_ms=None, out=None):
    _torch()
    band = np.ascontiguousarray(band, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    squeeze = V.ndim == 1
    V = np.ascontiguousarray(V[:, None] if squeeze else V)
    N, nrhs = V.shape
    kb = band.shape[0] - 1
    if out is None or out.size != N * nrhs:
        out = np.empty((N, nrhs), dtype=np.float64)
    out = out.reshape(N, nrhs)
    npairs = len(theta2) // 2
    ms = (ctypes.c_float * npairs)() if per_pair_ms is not None else None
    st = lib().pfx_expm_banded(
        PFX_MEM_HOST, band.ctypes.data, N, kb, V.ctypes.data, nrhs, float(shift_c), _f64p(theta2), _f64p(coef2),
        npairs, out.ctypes.data, ctypes.cast(ms, _fp) if ms is not None else None, None,
    )
    _check(st, "pfx_expm_banded")
    if per_pair_ms is not None:
        per_pair_ms[:] = list(ms)
    return out[:, 0] if squeeze else out


def expm_banded_device(band, V, theta2, coef2, shift_c: float, out=None, per_pair_ms=None, stream=None):
    torch = _torch()
    squeeze = V.dim() == 1
    if squeeze:
        V = V.unsqueeze(-1)
    if V.dim() != 2 or band.dim() != 2:
        raise BadSpec(f"V must be (N,) or (N, nrhs) and band (kb + 1, N), got {tuple(V.shape)}, {tuple(band.shape)}")
    N, nrhs = V.shape
    kb = band.shape[0] - 1
    V = _real_dev(V, "V")
    band = _real_dev(band, "band", (kb + 1, N))
    out = _out_dev(out, (N, nrhs), V)
    npairs = len(theta2) // 2
    ms = (ctypes.c_float * npairs)() if per_pair_ms is not None else None
    st = lib().pfx_expm_banded(
        PFX_MEM_DEVICE, _ptr(band), N, kb, _ptr(V), nrhs, float(shift_c), _f64p(theta2),
        _f64p(coef2), npairs, _ptr(out), ctypes.cast(ms, _fp) if ms is not None else None, _stream_ptr(stream),
    )
    _check(st, "pfx_expm_banded")
    if per_pair_ms is not None:
        per_pair_ms[:] = list(ms)
    return out.squeeze(-1) if squeeze else out


def shifted_solve(A, theta: complex, V: np.ndarray) -> np.ndarray:
    """Host entry for linalg.shifted_solve: Y = (A + theta I)^{-1} V, complex128."""
    _torch()
    a = A.entries
    a_complex = not A.is_real()
    a = np.ascontiguousarray(a if a_complex else a.real)
    V = np.asarray(V, dtype=np.complex128)
    squeeze = V.ndim == 1
    Vc = np.ascontiguousarray(V[:, None] if squeeze else V)
    d, nrhs = Vc.shape
    if d != A.d:
        raise BadSpec(f"V has {d} rows, A is {A.d} x {A.d}")
    Y = np.empty_like(Vc)
    st = lib().pfx_shifted_solve(
        PFX_MEM_HOST, a.ctypes.data, int(a_complex), d, theta.real, theta.imag, Vc.ctypes.data, nrhs, Y.ctypes.data,
        None,
    )
    _check(st, "pfx_shifted_solve")
    return Y[:, 0] if squeeze else Y
