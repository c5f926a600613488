"""paper_2601_07824_b200 -- exact stabilizer Renyi entropy of N-qubit state vectors on B200.

Thin Python face of ``libsre_b200.so`` (C ABI in ``include/sre.h``): argument marshalling
only.  Every step of the hot path (Alg. 2 of arXiv:2601.07824) runs in
the library's sm_100a kernels; PyTorch supplies device memory, streams and process groups.
There is no CPU fallback: importing works anywhere, but every call needs the built library
and an sm_100 device and raises ``SreError`` otherwise.

    import torch, paper_2601_07824_b200 as sre
    m, lost_norm = sre.exact(psi_cuda_complex128, [2.0])      # (SRE(psi, 2) -> (m, l))
"""
from __future__ import annotations

import ctypes
import os
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsre_b200.so")

__all__ = ["SreError", "load", "exact", "exact_batched", "partial_sums", "x_string_sums", "finalize", "workspace_size",
           "chi", "norm2", "launch_count", "profile_begin", "profile_end", "LIB_PATH"]

PRECISION = {"fp64": 0, "fp32": 1}   # sre_precision (include/sre.h)

_STATUS = {0: "SRE_OK", 1: "SRE_EINVAL", 2: "SRE_ERANGE", 3: "SRE_ENOTNORM", 4: "SRE_EWORKSPACE",
           5: "SRE_ENOMEM", 6: "SRE_ECUDA", 7: "SRE_EINTERNAL", 8: "SRE_ENODEV"}


class SreError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_STATUS.get(code, code)}: {msg}")
        self.code = code


_lib = None


def load():
    """Load libsre_b200.so (raises if it has not been built: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SreError(-1, f"{LIB_PATH} missing: run `python -m paper_2601_07824_b200._build` "
                               "or __graft_entry__.build()")
        lib = ctypes.CDLL(LIB_PATH)
        vp, dp, i, u64 = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.c_uint64
        sig = {
            "sre_status_string": ([i], ctypes.c_char_p),
            "sre_last_error": ([], ctypes.c_char_p),
            "sre_version": ([], i),
            "sre_exact": ([vp, i, dp, i, dp, dp], i),
            "sre_exact_batched": ([vp, i, i, dp, i, dp, dp], i),
            "sre_workspace_size": ([i, i, i], ctypes.c_size_t),
            "sre_partial_sums": ([vp, i, i, u64, u64, dp, i, vp, ctypes.c_size_t, vp, vp], i),
            "sre_finalize": ([dp, i, i, dp, i, dp, dp], i),
            "sre_norm2": ([vp, i, i, vp, vp], i),
            "sre_chi": ([vp, i, u64, vp, vp], i),
            "sre_workspace_size_ex": ([i, i, i, i], ctypes.c_size_t),
            "sre_exact_ex": ([vp, i, i, dp, i, i, dp, dp], i),
            "sre_partial_sums_ex": ([vp, i, i, u64, u64, dp, i, i, vp, ctypes.c_size_t, vp, vp], i),
            "sre_x_string_sums": ([vp, i, ctypes.POINTER(u64), i, dp, i, vp, ctypes.c_size_t, vp, vp], i),
            "sre_pauli_spectrum": ([vp, i, u64, u64, vp, vp, ctypes.c_size_t, vp], i),
            "sre_launch_count": ([], u64),
            "sre_profile_begin": ([i], i),
            "sre_profile_end": ([dp, ctypes.POINTER(u64), ctypes.POINTER(u64)], i),
        }
        for name, (args, res) in sig.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = res
        _lib = lib
    return _lib


def _check(rc: int):
    if rc != 0:
        raise SreError(rc, _lib.sre_last_error().decode())


def _alphas(alphas: Sequence[float]) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(list(alphas), dtype=np.float64))
    if a.ndim != 1 or a.size == 0:
        raise SreError(1, "alphas must be a non-empty sequence")
    return a


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _nqubits(dim: int) -> int:
    n = int(dim).bit_length() - 1
    if dim < 2 or (1 << n) != dim:
        raise SreError(2, f"state length {dim} is not 2^N with N >= 1")
    return n


def _psi_ptr(psi):
    """(pointer, N, B, keepalive) for a torch tensor (cuda or cpu) or numpy array, complex128."""
    try:
        import torch
        if isinstance(psi, torch.Tensor):
            if psi.dtype != torch.complex128:
                raise SreError(1, f"psi dtype {psi.dtype}; complex128 required")
            t = psi.contiguous()
            b = 1 if t.dim() == 1 else t.shape[0]
            return t.data_ptr(), _nqubits(t.shape[-1]), b, t
    except ImportError:
        pass
    a = np.ascontiguousarray(np.asarray(psi))
    if a.dtype != np.complex128:
        raise SreError(1, f"psi dtype {a.dtype}; complex128 required")
    b = 1 if a.ndim == 1 else a.shape[0]
    return a.ctypes.data, _nqubits(a.shape[-1]), b, a


def _bind_stream(st, psi, keep, *tensors):
    """Make the tensors a call enqueues on ``st`` safe when ``st`` is not torch's current stream: a
    contiguous copy of psi (made on the current stream) is waited for, and every tensor the kernels use
    is recorded on ``st`` so the caching allocator cannot recycle it before they finish."""
    import torch
    cur = torch.cuda.current_stream(st.device)
    if st == cur:
        return
    if keep is not psi:
        st.wait_stream(cur)
    for t in (keep,) + tensors:
        if isinstance(t, torch.Tensor) and t.is_cuda:
            t.record_stream(st)


def _prec(precision: str) -> int:
    if precision not in PRECISION:
        raise SreError(1, f"precision {precision!r}: one of {sorted(PRECISION)}")
    return PRECISION[precision]


def exact(psi, alphas: Sequence[float] = (2.0,), precision: str = "fp64"):
    """M_alpha (bits) and lost_norm of one state -- Eq. (2) via Alg. 2 over all 2^N X-strings.
    Synchronous; runs on the legacy default stream (which waits for torch's blocking streams).
    psi: complex128 torch tensor (cuda: no copy; cpu) or numpy array (host: copied by the call).
    precision "fp32" selects the optional FP32 transform (FP64 accumulation, ~1e-4 relative)."""
    lib = load()
    ptr, n, b, keep = _psi_ptr(psi)
    if b != 1:
        raise SreError(1, "exact() takes one state; use exact_batched()")
    al = _alphas(alphas)
    out = np.zeros(al.size)
    ln = ctypes.c_double(0.0)
    if precision == "fp64":
        _check(lib.sre_exact(ctypes.c_void_p(ptr), n, _dp(al), al.size, _dp(out), ctypes.pointer(ln)))
    else:
        _check(lib.sre_exact_ex(ctypes.c_void_p(ptr), n, 1, _dp(al), al.size, _prec(precision), _dp(out),
                                ctypes.pointer(ln)))
    del keep
    return [float(x) for x in out], ln.value


def exact_batched(psi, alphas: Sequence[float] = (2.0,), precision: str = "fp64"):
    """[B][n_alpha] M values and [B] lost_norms for a batch psi[B, 2^N]."""
    lib = load()
    ptr, n, b, keep = _psi_ptr(psi)
    al = _alphas(alphas)
    out = np.zeros((b, al.size))
    ln = np.zeros(b)
    _check(lib.sre_exact_ex(ctypes.c_void_p(ptr), n, b, _dp(al), al.size, _prec(precision), _dp(out), _dp(ln)))
    del keep
    return out, ln


def workspace_size(n: int, b: int = 1, n_alpha: int = 1, precision: str = "fp64") -> int:
    return int(load().sre_workspace_size_ex(n, b, n_alpha, _prec(precision)))


def partial_sums(psi, a_begin: int, a_end: int, alphas: Sequence[float], out=None, workspace=None, stream=None,
                 precision: str = "fp64"):
    """Raw sums [B, n_alpha+2] (S_alpha..., S_1, sum t ln t) over X-strings a in [a_begin, a_end),
    enqueued on ``stream`` (default: torch's current stream).  psi must be a cuda tensor."""
    import torch
    lib = load()
    if not (isinstance(psi, torch.Tensor) and psi.is_cuda):
        raise SreError(1, "partial_sums needs a cuda complex128 tensor")
    ptr, n, b, keep = _psi_ptr(psi)
    al = _alphas(alphas)
    dev = psi.device
    if out is None:
        out = torch.empty((b, al.size + 2), dtype=torch.float64, device=dev)
    ws_need = workspace_size(n, b, al.size, precision)
    if workspace is None or workspace.numel() < ws_need:
        workspace = torch.empty(ws_need, dtype=torch.uint8, device=dev)
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    _bind_stream(st, psi, keep, out, workspace)
    _check(lib.sre_partial_sums_ex(ctypes.c_void_p(ptr), n, b, int(a_begin), int(a_end), _dp(al), al.size,
                                   _prec(precision), ctypes.c_void_p(workspace.data_ptr()), workspace.numel(),
                                   ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st.cuda_stream)))
    del keep
    return out


def x_string_sums(psi, a_list, alphas: Sequence[float] = (2.0,), out=None, workspace=None, stream=None):
    """Per-X-string raw sums [len(a_list), n_alpha+2] (row i = sums over the Z-strings of X-string
    a_list[i]) -- the energy evaluations of the thermodynamic-integration sampler (Alg. 3)."""
    import torch
    lib = load()
    if not (isinstance(psi, torch.Tensor) and psi.is_cuda):
        raise SreError(1, "x_string_sums needs a cuda complex128 tensor")
    ptr, n, b, keep = _psi_ptr(psi)
    if b != 1:
        raise SreError(1, "x_string_sums takes one state")
    al = _alphas(alphas)
    a = np.ascontiguousarray(np.asarray(a_list, dtype=np.uint64).ravel())
    if out is None:
        out = torch.empty((a.size, al.size + 2), dtype=torch.float64, device=psi.device)
    ws_need = workspace_size(n, 1, al.size)
    if workspace is None or workspace.numel() < ws_need:
        workspace = torch.empty(ws_need, dtype=torch.uint8, device=psi.device)
    st = stream if stream is not None else torch.cuda.current_stream(psi.device)
    _bind_stream(st, psi, keep, out, workspace)
    _check(lib.sre_x_string_sums(ctypes.c_void_p(ptr), n, a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                 a.size, _dp(al), al.size, ctypes.c_void_p(workspace.data_ptr()), workspace.numel(),
                                 ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st.cuda_stream)))
    del keep
    return out


def finalize(sums, n: int, alphas: Sequence[float]):
    """Host Eq. (2) from complete sums [B, n_alpha+2] -> (M [B][n_alpha], lost_norm [B])."""
    lib = load()
    al = _alphas(alphas)
    s = np.ascontiguousarray(np.asarray(sums.cpu() if hasattr(sums, "cpu") else sums, dtype=np.float64))
    s = s.reshape(-1, al.size + 2)
    b = s.shape[0]
    m = np.zeros((b, al.size))
    ln = np.zeros(b)
    _check(lib.sre_finalize(_dp(s), n, b, _dp(al), al.size, _dp(m), _dp(ln)))
    return m, ln


def norm2(psi):
    """||psi_s||^2 per state on the device (FP64) -> torch tensor [B]."""
    import torch
    lib = load()
    ptr, n, b, keep = _psi_ptr(psi)
    out = torch.empty(b, dtype=torch.float64, device=psi.device)
    _check(lib.sre_norm2(ctypes.c_void_p(ptr), n, b, ctypes.c_void_p(out.data_ptr()),
                         ctypes.c_void_p(torch.cuda.current_stream(psi.device).cuda_stream)))
    del keep
    return out


def chi(psi, a: int):
    """chi_b(a) = <psi|X_a Z_b|psi> for all b (complex128 cuda tensor, natural b order), computed by
    the same kernels as the sums (verification entry)."""
    import torch
    lib = load()
    ptr, n, b, keep = _psi_ptr(psi)
    out = torch.zeros(2 << n, dtype=torch.float64, device=psi.device)
    _check(lib.sre_chi(ctypes.c_void_p(ptr), n, int(a), ctypes.c_void_p(out.data_ptr()),
                       ctypes.c_void_p(torch.cuda.current_stream(psi.device).cuda_stream)))
    torch.cuda.current_stream(psi.device).synchronize()
    del keep
    return torch.view_as_complex(out.view(-1, 2))


def spectrum(psi, a_begin: int = 0, a_end: int | None = None, workspace=None, stream=None) -> np.ndarray:
    """Histogram (numpy int64[64]) of t = |<P>|^2 over the Pauli strings of X-strings
    [a_begin, a_end) (default all 4^N strings): bin k = round(-log2 t) for k <= 62, bin 63 = t below
    2^-62.5 or zero (NEXT-2 spectrum epilogue, any N).  psi: cuda complex128 [2^N]."""
    import torch
    lib = load()
    if not (isinstance(psi, torch.Tensor) and psi.is_cuda):
        raise SreError(1, "spectrum needs a cuda complex128 tensor")
    ptr, n, b, keep = _psi_ptr(psi)
    if b != 1:
        raise SreError(1, "spectrum takes one state")
    a_end = (1 << n) if a_end is None else a_end
    hist = torch.empty(64, dtype=torch.int64, device=psi.device)
    ws_need = workspace_size(n, 1, 1) + 256
    if workspace is None or workspace.numel() < ws_need:
        workspace = torch.empty(ws_need, dtype=torch.uint8, device=psi.device)
    st = stream if stream is not None else torch.cuda.current_stream(psi.device)
    _bind_stream(st, psi, keep, hist, workspace)
    _check(lib.sre_pauli_spectrum(ctypes.c_void_p(ptr), n, int(a_begin), int(a_end), ctypes.c_void_p(hist.data_ptr()),
                                  ctypes.c_void_p(workspace.data_ptr()), workspace.numel(),
                                  ctypes.c_void_p(st.cuda_stream)))
    st.synchronize()                                  # the histogram is complete on st before the copy
    del keep
    return hist.cpu().numpy()


KINDS = ("single_pass", "pass_a", "pass_b", "aux", "fused")


def launch_count() -> int:
    """Cumulative number of kernels libsre_b200 launched in this process."""
    return int(load().sre_launch_count())


def profile_begin(stride: int = 1) -> None:
    """Sample every stride-th launch of each kernel kind with CUDA events on its stream."""
    _check(load().sre_profile_begin(int(stride)))


def profile_end() -> dict:
    """{kind: {"ms_sum", "timed", "launched"}} for the launches since profile_begin()."""
    lib = load()
    ms = np.zeros(len(KINDS))
    nt = (ctypes.c_uint64 * len(KINDS))()
    nl = (ctypes.c_uint64 * len(KINDS))()
    _check(lib.sre_profile_end(_dp(ms), nt, nl))
    return {k: {"ms_sum": float(ms[i]), "timed": int(nt[i]), "launched": int(nl[i])} for i, k in enumerate(KINDS)}
