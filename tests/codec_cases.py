"""Loader for ``tests/golden/codec_golden.npz`` (written by
``tests/golden/make_golden.py gen_codec`` from the UNMODIFIED reference):
encoded frames, reference planes, receiver shard patterns and the decoded
plane digests / grids the reference produced."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

from helpers import GOLDEN_DIR

_Z = None


def _z():
    global _Z
    if _Z is None:
        _Z = dict(np.load(os.path.join(GOLDEN_DIR, "codec_golden.npz")))
    return _Z


def blob(i: int) -> bytes:
    z = _z()
    return z["blobs"][z["blobs_off"][i]:z["blobs_off"][i + 1]].tobytes()


def ref_plane(i: int):
    if i < 0:
        return None
    z = _z()
    a = z["refs"][z["refs_off"][i]:z["refs_off"][i + 1]]
    shp = tuple(int(v) for v in z["refs_shape"][i])
    a = a.reshape(shp)
    return a[:, :, 0] if int(z["refs_ndim"][i]) == 2 else a


def _ragged(key, i, dtype=None):
    z = _z()
    a = z[key][z[key + "_off"][i]:z[key + "_off"][i + 1]]
    return a if dtype is None else a.astype(dtype)


def trials(kind: str | None = None):
    z = _z()
    meta = json.loads(str(z["meta"]))
    for i, m in enumerate(meta):
        if kind is not None and m["kind"] != kind:
            continue
        t = dict(m)
        t["present"] = _ragged("present", i, bool)
        t["grid"] = _ragged("grid", i, bool)
        t["ranges"] = [tuple(int(x) for x in r) for r in _ragged("ranges", i).reshape(-1, 2)]
        yield t


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def p_body(t):
    """Receiver._finalize_p inputs of a ``pframe`` trial: (header, shards
    dict of the received body shards, body_len)."""
    header, payload = blob(t["header"]), blob(t["payload"])
    L = t["L"]
    shards = {i: payload[(i - 1) * L:i * L] for i in range(1, t["n"]) if t["present"][i]}
    return header, shards, t["encoded_len"] - len(header)


def i_shards(t):
    """Receiver._finalize_i inputs of an ``iframe`` trial: the n + r shard
    list (None = lost), padded to shard_len (receiver.py:185-191)."""
    from tools import synth
    data = blob(t["data"])
    n, r, L = t["n"], t["r"], t["L"]
    shards = [data[i * L:(i + 1) * L].ljust(L, b"\0") for i in range(n)]
    shards += synth.rs_parity(data, n, r, L)
    return data, [s if t["present"][i] else None for i, s in enumerate(shards)]
