"""Checkpointed exact SRE over long X-string sweeps.

The chunks of the Alg. 2 loop are independent: the sweep over a in [lo, hi) is split into
fixed chunks; after each chunk the raw sums (S_alpha..., S_1, sum t ln t) are appended to a JSON
journal.  On restart, chunks already in the journal are skipped and the stored sums are reused,
so an interrupted N = 24..26 run loses at most one chunk.  Sums of chunks are combined in chunk
order (deterministic, same as one call over the union up to FP64 reassociation).
"""
from __future__ import annotations

import json
import os
from typing import Callable, Sequence

import numpy as np


def _load(path):
    if not path or not os.path.exists(path):
        return {}
    with open(path) as f:
        return json.load(f)


def _save(path, journal):
    tmp = path + ".tmp"
    with open(tmp, "w") as f:
        json.dump(journal, f)
    os.replace(tmp, path)


def state_fingerprint(psi) -> str:
    """sha256 of the state's amplitudes (host bytes of the complex128 vector): the journal key that
    stops a restart with another state from reusing stored chunk sums."""
    import hashlib
    a = psi.detach().cpu().numpy() if hasattr(psi, "detach") else np.asarray(psi)
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def chunked_sums(n: int, alphas: Sequence[float], partial_fn: Callable, lo: int = 0, hi: int | None = None,
                 chunk: int = 1 << 16, journal_path: str | None = None, max_chunks: int | None = None,
                 state_id: str = "", precision: str = "fp64"):
    """Sum partial_fn(a0, a1) -> array[n_alpha+2] over [lo, hi) in chunks, journaled.
    Returns (sums, complete) where complete is False if max_chunks stopped the sweep early.
    The journal is keyed by (n, alphas, range, chunk, state_id, precision); a mismatch raises."""
    hi = (1 << n) if hi is None else hi
    key = {"n": n, "alphas": list(map(float, alphas)), "lo": lo, "hi": hi, "chunk": chunk, "state": state_id,
           "precision": precision}
    journal = _load(journal_path)
    if journal and journal.get("key") != key:
        raise ValueError(f"journal {journal_path} belongs to a different run: {journal.get('key')}")
    done = journal.get("done", {}) if journal else {}
    total = np.zeros(len(alphas) + 2)
    ran = 0
    complete = True
    for a0 in range(lo, hi, chunk):
        a1 = min(hi, a0 + chunk)
        k = str(a0)
        if k not in done:
            if max_chunks is not None and ran >= max_chunks:
                complete = False
                continue
            done[k] = [float(x) for x in np.asarray(partial_fn(a0, a1), dtype=np.float64).ravel()]
            ran += 1
            if journal_path:
                _save(journal_path, {"key": key, "done": done})
    if complete:
        for a0 in range(lo, hi, chunk):
            total += np.asarray(done[str(a0)])
    return total, complete


def exact_resumable(psi, alphas: Sequence[float] = (2.0,), chunk: int = 1 << 16, journal_path: str | None = None,
                    max_chunks: int | None = None, precision: str = "fp64"):
    """M_alpha and lost_norm of a cuda state through journaled chunks of sre_partial_sums.
    Returns (M list, lost_norm) when complete, else None (call again to continue)."""
    import torch

    from . import finalize, partial_sums, workspace_size
    n = psi.shape[-1].bit_length() - 1
    ws = torch.empty(workspace_size(n, 1, len(alphas), precision), dtype=torch.uint8, device=psi.device)

    def part(a0, a1):
        out = partial_sums(psi, a0, a1, alphas, workspace=ws, precision=precision)
        return out.cpu().numpy()[0]

    sid = state_fingerprint(psi) if journal_path else ""
    sums, complete = chunked_sums(n, alphas, part, chunk=chunk, journal_path=journal_path, max_chunks=max_chunks,
                                  state_id=sid, precision=precision)
    if not complete:
        return None
    m, ln = finalize(sums, n, alphas)
    return [float(x) for x in m[0]], float(ln[0])
