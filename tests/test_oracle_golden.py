"""Pin the CPU oracle against golden vectors produced by the unmodified
reference (tests/golden/make_golden.py)."""

import os

import numpy as np
import pytest

from golden_cases import MODEL_CASES, RECOVER_CASES, model_case, recover_case
from helpers import GOLDEN_DIR, digest
from oracle import lossmask, nvrec_forward, recover

MODEL = np.load(os.path.join(GOLDEN_DIR, "model_golden.npz"))
RECOV = np.load(os.path.join(GOLDEN_DIR, "recover_golden.npz"))
LMASK = np.load(os.path.join(GOLDEN_DIR, "lossmask_golden.npz"))


@pytest.mark.parametrize("name", sorted(MODEL_CASES))
def test_model_oracle_matches_reference(name):
    arch, c, state, stack, mask = model_case(name)
    assert str(MODEL[name + "__digest"]) == digest(stack, mask, *state.values())
    got = nvrec_forward.forward(state, arch, c, stack, mask).numpy()
    np.testing.assert_allclose(got, MODEL[name], atol=2e-6, rtol=0)


@pytest.mark.parametrize("name", sorted(RECOVER_CASES))
def test_recover_oracle_matches_reference(name):
    arch, c, state, plane, grid, refs = recover_case(name)
    assert str(RECOV[name + "__digest"]) == digest(plane, grid, *refs,
                                                   *state.values())
    got = recover.recover(state, arch, c, plane, grid, refs)
    want = RECOV[name]
    # fp32 re-association can move a value across a .5 quantisation edge
    assert np.abs(got.astype(int) - want.astype(int)).max() <= 1
    assert (got != want).mean() < 1e-3


def lossmask_trials():
    off = {k: LMASK[k + "_off"] for k in ("header", "received", "grid")}
    for i in range(len(LMASK["n_data"])):
        yield dict(
            header=LMASK["header"][off["header"][i]:off["header"][i + 1]].tobytes(),
            received=LMASK["received"][off["received"][i]:off["received"][i + 1]],
            grid=LMASK["grid"][off["grid"][i]:off["grid"][i + 1]].astype(bool),
            n_data=int(LMASK["n_data"][i]), shard_len=int(LMASK["shard_len"][i]),
            encoded_len=int(LMASK["encoded_len"][i]),
            gh=int(LMASK["gh"][i]), gw=int(LMASK["gw"][i]))


def test_lossmask_oracle_matches_reference_receiver():
    n = 0
    for t in lossmask_trials():
        recv = {i for i in range(t["n_data"]) if t["received"][i]}
        g = lossmask.mask_from_shards(t["header"], t["n_data"], recv,
                                      t["shard_len"], t["encoded_len"])
        assert g.shape == (t["gh"], t["gw"])
        assert np.array_equal(g.reshape(-1), t["grid"])
        n += 1
    assert n >= 200


def test_lossmask_oracle_codec_tail_rule():
    off = {k: LMASK["x_" + k + "_off"] for k in ("header", "ranges", "grid")}
    for i in range(len(LMASK["x_received_len"])):
        hdr = LMASK["x_header"][off["header"][i]:off["header"][i + 1]].tobytes()
        rng = LMASK["x_ranges"][off["ranges"][i]:off["ranges"][i + 1]]
        want = LMASK["x_grid"][off["grid"][i]:off["grid"][i + 1]].astype(bool)
        g = lossmask.decode_mask(hdr, int(LMASK["x_received_len"][i]),
                                 [tuple(r) for r in rng.reshape(-1, 2)])
        assert np.array_equal(g.reshape(-1), want)


BASE = np.load(os.path.join(GOLDEN_DIR, "baseline_golden.npz"))


@pytest.mark.parametrize("name", sorted(k for k in BASE.files if "__" not in k))
def test_baseline_oracle_matches_reference(name):
    from golden_cases import baseline_case
    from oracle import baseline
    c, plane, grid, refs = baseline_case(name)
    assert str(BASE[name + "__digest"]) == digest(plane, grid, *refs)
    fn = baseline.baseline_rgb if c == 3 else baseline.baseline_depth
    got, fb = fn(plane, grid, refs)
    assert not fb and np.array_equal(got, BASE[name])
