"""Oracle: restatement of the frame decode that feeds the recovery path.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

SURVEY.md 8(f) rank 4: the steps immediately before ``nvrec`` produce the
corrupted plane (zero-fill P-frame decode) and, for I-frames, the
Reed-Solomon erasure reconstruction.  Each function restates one reference
function with numpy, keeping its integer semantics (int16 wrap-around,
python slicing, error order):

* ``decode``          -- ``codec.decode`` (rgbdstream/codec.py:260-321),
  with ``_rle_decode`` (codec.py:134-138) and ``_unzigzag`` (codec.py:146-148).
* ``decode_bytes``    -- ``codec.decode_bytes`` (codec.py:324-340).
* ``rs_reconstruct``  -- ``fec.rs_reconstruct`` (rgbdstream/fec.py:144-163),
  with the GF(2^8) tables (fec.py:24-41), ``_gf_inv_matrix`` (fec.py:60-75)
  and ``_generator_matrix`` (fec.py:78-88).
* ``finalize_p_body`` -- the body assembly of ``Receiver._finalize_p``
  (rgbdstream/receiver.py:222-237).
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np

from .lossmask import UndecodableError, block_ranges, corrupted_blocks, parse_header

KIND_I, KIND_P = 0, 1            # frames.py FrameKind values
RLE_DTYPE = np.dtype([("run", "u1"), ("val", "<u2")])   # codec.py:25


def rle_decode(buf: bytes) -> np.ndarray:
    """codec.py:134-138."""
    if len(buf) % RLE_DTYPE.itemsize != 0:
        raise UndecodableError("payload range is not whole RLE records")
    rec = np.frombuffer(buf, dtype=RLE_DTYPE)
    return np.repeat(rec["val"].astype(np.uint16), rec["run"])


def unzigzag(u: np.ndarray) -> np.ndarray:
    """codec.py:146-148 (int16 result)."""
    u = u.astype(np.uint16)
    return ((u >> 1).astype(np.int16)) ^ (-(u & 1).astype(np.int16))


def decode(header: bytes, payload: bytes, reference=None, zero_fill_ranges=()):
    """codec.py:260-321: returns (plane, grid)."""
    hdr = parse_header(header)
    if hdr["kind"] == KIND_P and reference is None:
        raise ValueError("P-frame decode requires a reference plane")
    block, c = hdr["block"], hdr["channels"]
    h, w = hdr["height"], hdr["width"]
    bs = block * block * c
    n_blocks = (h // block) * (w // block)
    payload = bytes(payload)
    zr = list(zero_fill_ranges)
    if len(payload) < hdr["payload_len"]:
        zr = zr + [(len(payload), hdr["payload_len"])]
        payload = payload + b"\x00" * (hdr["payload_len"] - len(payload))
    ranges = block_ranges(hdr)
    flagged = corrupted_blocks(ranges, zr)
    present_ids = np.flatnonzero(hdr["present"])
    clean = ~flagged
    clean_buf = b"".join(payload[int(s):int(e)] for s, e in ranges[clean])
    clean_vals = rle_decode(clean_buf)
    if len(clean_vals) != int(clean.sum()) * bs:
        raise UndecodableError("payload sample count disagrees with header")
    hb, wb = h // block, w // block
    clean_ids = present_ids[clean]
    if hdr["kind"] == KIND_I:
        plane3 = np.zeros((h, w, c), dtype=np.uint8)
        patch = np.clip(clean_vals.astype(np.int16) * np.int16(hdr["quant"]),
                        0, 255).astype(np.uint8)
    else:
        base = reference if reference.ndim == 3 else reference[:, :, None]
        plane3 = base.copy()
        deltas = unzigzag(clean_vals).reshape(-1, c, block, block) * np.int16(hdr["quant"])
        view = plane3.reshape(hb, block, wb, block, c)
        by, bx = np.divmod(clean_ids, wb)
        ref_sel = view[by, :, bx, :, :].astype(np.int16)
        patch = np.clip(ref_sel + deltas.transpose(0, 2, 3, 1), 0, 255).astype(np.uint8)
    view = plane3.reshape(hb, block, wb, block, c)
    by, bx = np.divmod(clean_ids, wb)
    view[by, :, bx, :, :] = patch.reshape(-1, c, block, block).transpose(0, 2, 3, 1) \
        if hdr["kind"] == KIND_I else patch
    plane = plane3[:, :, 0] if c == 1 else plane3
    grid = np.zeros(n_blocks, dtype=bool)
    grid[present_ids[flagged]] = True
    return plane, grid.reshape(h // block, w // block)


def decode_bytes(data: bytes, reference=None, zero_fill_ranges=()):
    """codec.py:324-340 (ranges relative to the whole encoded frame)."""
    hdr = parse_header(data)
    hl = hdr["header_len"]
    pr = []
    for z0, z1 in zero_fill_ranges:
        if z0 < hl and z1 > 0 and z1 > z0:
            raise UndecodableError("zero-filled range overlaps codec header")
        pr.append((z0 - hl, z1 - hl))
    return decode(data[:hl], data[hl:], reference, pr)


def finalize_p_body(n_data: int, shards: dict, shard_len: int, body_len: int):
    """receiver.py:222-237: (body bytes, zero_fill ranges)."""
    zero_fill, chunks = [], []
    for i in range(1, n_data):
        lo = (i - 1) * shard_len
        hi = min(lo + shard_len, body_len)
        if i in shards:
            chunks.append(shards[i])
        else:
            chunks.append(b"\x00" * (hi - lo))
            zero_fill.append((lo, hi))
    return b"".join(chunks), zero_fill


# ---- Reed-Solomon over GF(2^8), primitive polynomial 0x11D (fec.py:19-88) ----

def _tables():
    exp = np.zeros(512, dtype=np.uint8)
    log = np.zeros(256, dtype=np.int32)
    x = 1
    for i in range(255):
        exp[i] = x
        log[x] = i
        x <<= 1
        if x & 0x100:
            x ^= 0x11D
    exp[255:510] = exp[:255]
    mul = np.zeros((256, 256), dtype=np.uint8)
    a = np.arange(1, 256)
    mul[1:, 1:] = exp[(log[a][:, None] + log[a][None, :]) % 255]
    return exp, log, mul


EXP, LOG, MUL = _tables()


class UnrecoverableError(Exception):
    """fec.py:91-92."""


def gf_matmul(a, b):
    return np.bitwise_xor.reduce(MUL[a[:, :, None], b[None, :, :]], axis=1)


def gf_inv_matrix(m):
    """fec.py:60-75 (Gauss-Jordan, first non-zero pivot)."""
    n = m.shape[0]
    aug = np.concatenate((m.copy(), np.eye(n, dtype=np.uint8)), axis=1)
    for col in range(n):
        pivot = col + int(np.argmax(aug[col:, col] != 0))
        if aug[pivot, col] == 0:
            raise ValueError("singular matrix")
        if pivot != col:
            aug[[col, pivot]] = aug[[pivot, col]]
        inv = int(EXP[255 - LOG[int(aug[col, col])]])
        aug[col] = MUL[inv, aug[col]]
        for row in range(n):
            if row != col and aug[row, col]:
                aug[row] ^= MUL[int(aug[row, col]), aug[col]]
    return aug[:, n:]


@lru_cache(maxsize=64)
def generator_matrix(n: int, r: int) -> np.ndarray:
    """fec.py:78-88: (n+r) x n systematic Vandermonde-derived generator."""
    points = np.arange(n + r, dtype=np.uint8)
    vand = np.zeros((n + r, n), dtype=np.uint8)
    vand[:, 0] = 1
    for j in range(1, n):
        vand[:, j] = MUL[vand[:, j - 1], points]
    return gf_matmul(vand, gf_inv_matrix(vand[:n]))


def rs_reconstruct(n: int, r: int, shard_len: int, data_len: int, shards) -> bytes:
    """fec.py:144-163; ``shards`` is a length n+r list, None = erased."""
    present = [s is not None for s in shards]
    if sum(present) < n:
        raise UnrecoverableError("only %d of %d required shards present" % (sum(present), n))
    if all(present[:n]):
        return b"".join(shards[:n])[:data_len]
    idx = [i for i in range(n + r) if present[i]][:n]
    inv = gf_inv_matrix(generator_matrix(n, r)[idx])
    received = np.stack([np.frombuffer(shards[i], dtype=np.uint8) for i in idx])
    out = np.zeros((n, shard_len), dtype=np.uint8)
    for i in range(n):
        for j in range(n):
            if inv[i, j]:
                out[i] ^= MUL[inv[i, j]][received[j]]
    return out.reshape(-1).tobytes()[:data_len]
