"""The SSIM restatement (oracle/metrics.py) against values computed by the
UNMODIFIED reference ``rgbdstream.metrics.ssim`` (metrics.py:41-72) in the
build container (tests/golden/make_golden.py gen_ssim)."""

import os

import numpy as np
import pytest

from golden_cases import SSIM_CASES, ssim_case
from helpers import GOLDEN_DIR, digest
from oracle.metrics import ssim

GOLD = np.load(os.path.join(GOLDEN_DIR, "ssim_golden.npz"))


@pytest.mark.parametrize("name", sorted(SSIM_CASES))
def test_ssim_oracle_matches_reference(name):
    a, b = ssim_case(name)
    assert digest(a, b) == str(GOLD[name + "__digest"])
    assert abs(ssim(a, b) - float(GOLD[name])) <= 1e-12


def test_ssim_contract():
    a, _ = ssim_case("s_depth_17x23_odd")
    with pytest.raises(ValueError):
        ssim(a, a[:-1])
    with pytest.raises(ValueError):
        ssim(a[:7], a[:7])
    assert ssim(a, a) == 1.0
