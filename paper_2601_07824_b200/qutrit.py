"""Pure-state qutrit mana (NEXT-3) -- thin ctypes binding over the C ABI (include/sre.h,
``sre_mana*``).  Argument marshalling only: every step runs in libsre_b200.so (csrc/mana.cu).

    m, norm2 = mana(psi)                       # P:869-884 Alg. 5; log2(sum |chi| / 3^N), Eq. (10)
    sums = partial_sums(psi, a0, a1)           # device [2] = (sum |chi|, sum chi) over X-strings [a0, a1)
    m, tr = mana_mixed(rho)                    # P:1059-1087 Alg. 6 (mixed states, NEXT-4)
    sums = mixed_sums_(rho_flat_cuda, n)       # in place: rho overwritten; device [2] = (sum |w|, sum w)

psi: complex128 of length 3^N (qutrit j = ternary digit j of the index), numpy or torch.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import SreError, _bind_stream, _check, load

_ready = False


def _lib():
    global _ready
    lib = load()
    if not _ready:
        vp, dp, i, u64 = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.c_uint64
        lib.sre_mana_workspace_size.argtypes = [i]
        lib.sre_mana_workspace_size.restype = ctypes.c_size_t
        lib.sre_mana_partial_sums.argtypes = [vp, i, u64, u64, vp, ctypes.c_size_t, vp, vp]
        lib.sre_mana_partial_sums.restype = i
        lib.sre_mana.argtypes = [vp, i, dp, dp]
        lib.sre_mana.restype = i
        lib.sre_mana_finalize.argtypes = [dp, i, dp, dp]
        lib.sre_mana_finalize.restype = i
        lib.sre_mana_mixed_workspace_size.argtypes = [i]
        lib.sre_mana_mixed_workspace_size.restype = ctypes.c_size_t
        lib.sre_mana_mixed_sums.argtypes = [vp, i, vp, ctypes.c_size_t, vp, vp]
        lib.sre_mana_mixed_sums.restype = i
        lib.sre_mana_mixed.argtypes = [vp, i, dp, dp]
        lib.sre_mana_mixed.restype = i
        _ready = True
    return lib


def n_qutrits(dim: int) -> int:
    n, d = 0, 1
    while d < dim:
        d *= 3
        n += 1
    if d != dim or dim < 3:
        raise SreError(2, f"state length {dim} is not 3^N with N >= 1")
    return n


def _ptr(psi):
    try:
        import torch
        if isinstance(psi, torch.Tensor):
            if psi.dtype != torch.complex128 or psi.dim() != 1:
                raise SreError(1, "psi must be a 1-D complex128 tensor")
            t = psi.contiguous()
            return t.data_ptr(), n_qutrits(t.numel()), t
    except ImportError:
        pass
    a = np.ascontiguousarray(np.asarray(psi))
    if a.dtype != np.complex128 or a.ndim != 1:
        raise SreError(1, "psi must be a 1-D complex128 array")
    return a.ctypes.data, n_qutrits(a.size), a


def workspace_size(n: int) -> int:
    return int(_lib().sre_mana_workspace_size(n))


def mana(psi):
    """(mana, ||psi||^2) of a host or cuda state via sre_mana (synchronous)."""
    lib = _lib()
    ptr, n, keep = _ptr(psi)
    m = ctypes.c_double(0.0)
    n2 = ctypes.c_double(0.0)
    _check(lib.sre_mana(ctypes.c_void_p(ptr), n, ctypes.byref(m), ctypes.byref(n2)))
    del keep
    return m.value, n2.value


def finalize(sums, n: int):
    """(mana, ||psi||^2) from complete sums (S_abs, S_sum) over all 3^n X-strings, through the
    library's host-side sre_mana_finalize (Eq. (10); no GPU needed)."""
    import numpy as np
    s = np.ascontiguousarray(np.asarray(sums.cpu() if hasattr(sums, "cpu") else sums, dtype=np.float64).reshape(-1)[:2])
    lib = _lib()
    m, n2 = ctypes.c_double(), ctypes.c_double()
    _check(lib.sre_mana_finalize(s.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), int(n), ctypes.byref(m),
                                 ctypes.byref(n2)))
    return m.value, n2.value


def partial_sums(psi, a_begin: int, a_end: int, out=None, workspace=None, stream=None):
    """Device float64[2] = (sum |chi_b(a)|, sum chi_b(a)) over X-strings a in [a_begin, a_end),
    enqueued on ``stream`` (default: torch's current stream).  psi must be a cuda tensor."""
    import torch
    lib = _lib()
    if not (isinstance(psi, torch.Tensor) and psi.is_cuda):
        raise SreError(1, "partial_sums needs a cuda complex128 tensor")
    ptr, n, keep = _ptr(psi)
    dev = psi.device
    if out is None:
        out = torch.empty(2, dtype=torch.float64, device=dev)
    need = workspace_size(n)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=dev)
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    _bind_stream(st, psi, keep, out, workspace)
    _check(lib.sre_mana_partial_sums(ctypes.c_void_p(ptr), n, int(a_begin), int(a_end),
                                     ctypes.c_void_p(workspace.data_ptr()), workspace.numel(),
                                     ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st.cuda_stream)))
    del keep
    return out


def _mixed_flat(rho):
    """(pointer, N, keepalive) of a column-major flat complex128 buffer (rho[r + c 3^N]).
    2-D inputs are transposed into column-major order; 1-D inputs are taken as already flat."""
    try:
        import torch
        if isinstance(rho, torch.Tensor):
            if rho.dtype != torch.complex128:
                raise SreError(1, "rho must be complex128")
            t = rho.t().contiguous() if rho.dim() == 2 else rho.contiguous()
            d = rho.shape[0] if rho.dim() == 2 else int(round(t.numel() ** 0.5))
            return t.data_ptr(), n_qutrits(d), t
    except ImportError:
        pass
    a = np.asarray(rho)
    if a.dtype != np.complex128:
        raise SreError(1, "rho must be complex128")
    if a.ndim == 2:
        if a.shape[0] != a.shape[1]:
            raise SreError(1, "rho must be square")
        d = a.shape[0]
        a = np.ascontiguousarray(a.flatten(order="F"))
    else:
        a = np.ascontiguousarray(a)
        d = int(round(a.size ** 0.5))
    return a.ctypes.data, n_qutrits(d), a


def mana_mixed(rho):
    """(mana, Tr rho) of a density matrix (host or cuda; 2-D, or 1-D column-major flat) via
    sre_mana_mixed (Alg. 6; synchronous; rho is not modified)."""
    lib = _lib()
    ptr, n, keep = _mixed_flat(rho)
    m = ctypes.c_double(0.0)
    tr = ctypes.c_double(0.0)
    _check(lib.sre_mana_mixed(ctypes.c_void_p(ptr), n, ctypes.byref(m), ctypes.byref(tr)))
    del keep
    return m.value, tr.value


def mixed_sums_(rho_flat, n: int, out=None, workspace=None, stream=None):
    """IN PLACE on a cuda column-major flat rho (length 9^n): device float64[2] = (sum |w_u|,
    sum w_u); rho's contents are unspecified afterwards.  Enqueued on ``stream``."""
    import torch
    lib = _lib()
    if not (isinstance(rho_flat, torch.Tensor) and rho_flat.is_cuda and rho_flat.is_contiguous()):
        raise SreError(1, "mixed_sums_ needs a contiguous cuda complex128 tensor")
    if rho_flat.numel() != 9 ** n:
        raise SreError(2, f"rho has {rho_flat.numel()} entries, 9^{n} expected")
    dev = rho_flat.device
    if out is None:
        out = torch.empty(2, dtype=torch.float64, device=dev)
    need = int(lib.sre_mana_mixed_workspace_size(n))
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=dev)
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    _bind_stream(st, rho_flat, rho_flat, out, workspace)
    _check(lib.sre_mana_mixed_sums(ctypes.c_void_p(rho_flat.data_ptr()), n, ctypes.c_void_p(workspace.data_ptr()),
                                   workspace.numel(), ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st.cuda_stream)))
    return out
