"""Frame decode + RS reconstruct oracle (oracle/codec.py) and the sender-side
workload generators (paper_2604_27441_b200/synth.py) against the golden
outputs of the UNMODIFIED reference (tests/golden/codec_golden.npz).  Also
checks the host half of the C-ABI RS path (nvrec_rs_plan, pure C++) without a
GPU."""

import ctypes

import numpy as np
import pytest

from codec_cases import blob, i_shards, p_body, ref_plane, sha, trials
from oracle import codec as oc
from oracle.lossmask import UndecodableError


def test_pframe_receiver_trials():
    n = 0
    for t in trials("pframe"):
        header, shards, body_len = p_body(t)
        body, zf = oc.finalize_p_body(t["n"], shards, t["L"], body_len)
        plane, grid = oc.decode(header, body, ref_plane(t["ref"]), zf)
        assert sha(plane) == t["digest"]
        assert np.array_equal(grid.reshape(-1), t["grid"])
        n += 1
    assert n >= 100


def test_iframe_receiver_trials_and_parity():
    n = 0
    for t in trials("iframe"):
        data, shards = i_shards(t)
        par = b"".join(s for s in __import__("tools.synth").synth.rs_parity(
            data, t["n"], t["r"], t["L"]))
        assert sha(np.frombuffer(par, np.uint8)) == t["parity_digest"]
        try:
            got = oc.rs_reconstruct(t["n"], t["r"], t["L"], len(data), shards)
        except oc.UnrecoverableError:
            assert t["err"] == "lost"
            continue
        assert got == data
        plane, grid = oc.decode_bytes(got)
        assert t["err"] == ""
        assert sha(plane) == t["digest"]
        assert np.array_equal(grid.reshape(-1), t["grid"])
        n += 1
    assert n >= 10


def test_direct_decode_cases():
    names = set()
    for t in trials("direct"):
        names.add(t["name"])
        try:
            plane, grid = oc.decode(blob(t["header"]), blob(t["payload"]), ref_plane(t["ref"]),
                                    t["ranges"])
        except (UndecodableError, ValueError) as e:
            assert str(e) == t["err"], t["name"]
            continue
        assert t["err"] == "", t["name"]
        assert sha(plane) == t["digest"], t["name"]
        assert np.array_equal(grid.reshape(-1), t["grid"]), t["name"]
    assert {"straddle_shift1", "crafted_q255_k1", "not_whole_records", "bad_count",
            "inverted_offsets", "bad_kind", "p_without_ref"} <= names


def test_decode_bytes_header_overlap():
    for t in trials("bytes"):
        with pytest.raises(UndecodableError, match=t["err"]):
            oc.decode_bytes(blob(t["data"]), zero_fill_ranges=t["ranges"])


def _plan(lib, n, r, present):
    coef = (ctypes.c_uint8 * (r * n + 1))()
    src = (ctypes.c_int32 * n)()
    miss = (ctypes.c_int32 * (r + 1))()
    m = ctypes.c_int32()
    pres = (ctypes.c_uint8 * (n + r))(*[int(bool(p)) for p in present])
    rc = lib.nvrec_rs_plan(n, r, pres, coef, src, miss, ctypes.byref(m))
    return rc, np.frombuffer(coef, np.uint8)[:m.value * n].reshape(m.value, n), \
        list(src), list(miss)[:m.value]


def _apply(coef, src, miss, shards, n, L):
    out = [bytearray(s) if s is not None and i < n else None for i, s in enumerate(shards[:n])]
    for i, row in enumerate(miss):
        acc = np.zeros(L, np.uint8)
        for s_idx, s in enumerate(src):
            if coef[i, s_idx]:
                acc ^= oc.MUL[coef[i, s_idx]][np.frombuffer(shards[s], np.uint8)]
        out[row] = bytearray(acc.tobytes())
    return b"".join(bytes(o) for o in out)


def test_rs_plan_host_matches_reference_reconstruct():
    """nvrec_rs_plan's reduced (m x n) decode coefficients reproduce the
    reference's full Gauss-Jordan reconstruction on every golden erasure
    pattern, plus random patterns up to n + r = 255."""
    from paper_2604_27441_b200 import _native
    from tools import synth
    lib = _native.load_library()
    cases = 0
    for t in trials("iframe"):
        data, shards = i_shards(t)
        n, r, L = t["n"], t["r"], t["L"]
        rc, coef, src, miss = _plan(lib, n, r, [s is not None for s in shards])
        if t["err"]:
            assert rc != 0
            assert "required shards present" in lib.nvrec_last_error().decode()
            continue
        assert rc == 0
        got = _apply(coef, src, miss, shards, n, L)[:len(data)]
        assert got == data
        cases += 1
    rng = np.random.default_rng(5)
    for n, r in ((1, 1), (2, 3), (17, 9), (170, 85), (200, 55)):
        L = 64
        data = rng.integers(0, 256, n * L - 5, dtype=np.uint8).tobytes()
        full = [data[i * L:(i + 1) * L].ljust(L, b"\0") for i in range(n)] + \
            synth.rs_parity(data, n, r, L)
        for _ in range(3):
            lost = rng.choice(n + r, r, replace=False)
            shards = [None if i in lost else s for i, s in enumerate(full)]
            rc, coef, src, miss = _plan(lib, n, r, [s is not None for s in shards])
            assert rc == 0
            want = oc.rs_reconstruct(n, r, L, len(data), shards)
            assert _apply(coef, src, miss, shards, n, L)[:len(data)] == want == data
            cases += 1
    assert cases >= 20
