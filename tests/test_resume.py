"""Journaled chunked sweeps (resume after interruption) -- host logic on CPU with oracle chunks."""
import json

import numpy as np

import sre_inputs as si


def test_resume_equals_single_sweep(oracle_lib, tmp_path):
    from paper_2601_07824_b200.resume import chunked_sums
    n, al = 7, [1.0, 2.0]
    psi = si.haar(n, 3)
    calls = []

    def part(a0, a1):
        calls.append((a0, a1))
        return oracle_lib.sums_fwht(psi, al, a_range=(a0, a1))

    j = str(tmp_path / "journal.json")
    s1, done1 = chunked_sums(n, al, part, chunk=16, journal_path=j, max_chunks=3)   # "interrupted"
    assert not done1 and len(calls) == 3
    s2, done2 = chunked_sums(n, al, part, chunk=16, journal_path=j)                 # resumed
    assert done2 and len(calls) == 8                                                 # 3 + remaining 5
    full = oracle_lib.sums_fwht(psi, al)
    assert np.max(np.abs(s2 - full) / np.maximum(np.abs(full), 1e-300)) < 1e-12
    assert len(json.load(open(j))["done"]) == 8


def test_journal_key_mismatch(tmp_path):
    import pytest
    from paper_2601_07824_b200.resume import chunked_sums
    j = str(tmp_path / "j.json")
    chunked_sums(3, [2.0], lambda a0, a1: np.zeros(3), chunk=4, journal_path=j)
    with pytest.raises(ValueError):
        chunked_sums(3, [3.0], lambda a0, a1: np.zeros(3), chunk=4, journal_path=j)


def test_journal_rejects_other_state_or_precision(tmp_path):
    """the key carries a state fingerprint and the precision, so a restart with another psi
    cannot silently mix stored chunk sums of two states."""
    import pytest
    from paper_2601_07824_b200.resume import chunked_sums, state_fingerprint
    a, b = si.haar(3, 1), si.haar(3, 2)
    assert state_fingerprint(a) != state_fingerprint(b) and state_fingerprint(a) == state_fingerprint(a.copy())
    j = str(tmp_path / "j.json")
    chunked_sums(3, [2.0], lambda a0, a1: np.zeros(3), chunk=4, journal_path=j, state_id=state_fingerprint(a))
    with pytest.raises(ValueError):
        chunked_sums(3, [2.0], lambda a0, a1: np.zeros(3), chunk=4, journal_path=j, state_id=state_fingerprint(b))
    with pytest.raises(ValueError):
        chunked_sums(3, [2.0], lambda a0, a1: np.zeros(3), chunk=4, journal_path=j, state_id=state_fingerprint(a),
                     precision="fp32")
