"""Host-side logic that needs no GPU: config mirror, stack slot order, grid
packing, checkpoint round trip, synthetic workload generators."""

import numpy as np
import pytest
import torch

from oracle import lossmask as om
from paper_2604_27441_b200 import Checkpoint, LossWeights, MaskedVideoModel, ModelConfig
from paper_2604_27441_b200.lossmask import PFrameShards, grid_blocks
from paper_2604_27441_b200.recovery import pack_grid, stack_slots
from tools.synth import GilbertElliott, n_data_shards, p_frame_header


def test_config_mirror():
    cfg = ModelConfig()
    assert (cfg.k, cfg.tubelet_t, cfg.patch, cfg.dim, cfg.layers, cfg.heads) == (5, 2, 16, 64, 2, 2)
    assert ModelConfig(k=4, tubelet_t=2).stack_len == 6
    assert ModelConfig(k=3, tubelet_t=1).stack_len == 4
    for kw in ({"k": 0}, {"tubelet_t": 0}, {"dim": 0}, {"lr": 0.0}, {"dim": 30, "heads": 4}):
        with pytest.raises(ValueError):
            ModelConfig(**kw)
    with pytest.raises(ValueError):
        LossWeights(depth_alpha_e=-1.0)


def test_stack_slots_front_pad():
    # refs[-k:] + [plane], front-padded with the oldest (server.py:189, model.py:99-101)
    assert stack_slots(5, 5, 6) == [0, 1, 2, 3, 4, 5]
    assert stack_slots(2, 5, 6) == [0, 0, 0, 0, 1, 2]
    assert stack_slots(7, 5, 6) == [2, 3, 4, 5, 6, 7]
    assert stack_slots(1, 1, 2) == [0, 1]


def test_pack_grid_is_wire_bitset():
    g = np.random.default_rng(0).random((45, 80)) < 0.2
    assert pack_grid(g).tobytes() == om.wire_bits(g)


def test_model_param_layout_and_checkpoint_roundtrip(tmp_path):
    torch.manual_seed(0)
    m = MaskedVideoModel(ModelConfig(), 3)
    from oracle.nvrec_forward import state_keys
    assert list(m.state_dict()) == state_keys(2)
    ck = Checkpoint.random_init(ModelConfig(), 3, seed=0)
    for k, v in m.state_dict().items():
        assert torch.equal(v, ck.state[k])
    ck.save(tmp_path / "c.pt")
    ck2 = Checkpoint.load(tmp_path / "c.pt")
    assert ck2.config == ck.config and ck2.channels == 3
    m2 = ck2.build_model()
    for k, v in m2.state_dict().items():
        assert torch.equal(v, ck.state[k])


def test_synthetic_headers_parse_like_the_codec():
    rng = np.random.default_rng(1)
    for (w, h, c) in ((1280, 720, 3), (320, 240, 1)):
        hdr, plen = p_frame_header(rng, w, h, c, 0.1)
        p = om.parse_header(hdr)
        assert p["width"] == w and p["height"] == h and p["payload_len"] == plen
        assert grid_blocks(hdr) == (w // 16) * (h // 16)
        assert np.all(np.diff(np.append(p["offsets"], plen)) % 3 == 0)
        assert n_data_shards(plen, 1024) == 1 + -(-plen // 1024)


def test_gilbert_elliott_stationary_rate():
    ge = GilbertElliott(seed=0)
    drops = np.mean([ge.drop() for _ in range(200000)])
    assert abs(drops - 0.0155 / (0.0155 + 0.5)) < 0.006


def test_pframe_received_flags():
    fr = PFrameShards(b"", 4, {0, 2}, 1024, 10)
    assert fr.received_flags().tolist() == [1, 0, 1, 0]
    fr = PFrameShards(b"", 3, np.array([True, False, True]), 1024, 10)
    assert fr.received_flags().tolist() == [1, 0, 1]


def test_cyclic_slot_ring_schedule():
    """The serving pipelines' cyclic slot schedule: step t reads references
    t..t+k-1 (mod S, oldest first) and stages its plane in slot t+k, which is
    the newest reference of step t+1; a slot is re-staged only nbuf steps
    after the last step that read it (the pipeline's ev_cmp wait)."""
    from paper_2604_27441_b200.recovery import cyclic_slot_tables
    k, nbuf, n, F = 5, 3, 2, 6
    S = k + nbuf
    tab = cyclic_slot_tables(k, nbuf, n, F, "cpu").numpy()
    assert tab.shape == (S, n, F)
    last_read = {}
    for t in range(40):
        p = t % S
        slots = tab[p] // n
        assert (tab[p] % n == np.arange(n)[:, None]).all()      # stream s reads its own planes
        ring, staged = list(slots[0, :-1]), int(slots[0, -1])
        assert ring == [(t + j) % S for j in range(k)]
        assert staged == (t + k) % S and staged not in ring
        if t > 0:
            prev = tab[(t - 1) % S][0] // n
            assert ring[-1] == prev[-1]                          # last step's plane is newest
        if staged in last_read:
            assert t - last_read[staged] >= nbuf
        for s in ring:
            last_read[s] = t


def test_forward_value_errors_match_reference():
    """pkg/nvrec/tests/test_nvrec_model.py:79-97: the reference raises
    ValueError mentioning "channels", "patch" and "stack" (model.py:93-98),
    before any compute -- so no GPU is needed to check them."""
    import torch
    from paper_2604_27441_b200 import MaskedVideoModel, ModelConfig
    cfg = ModelConfig(k=1, tubelet_t=1, dim=16, layers=1, heads=2)
    model = MaskedVideoModel(cfg, 3)
    mask = torch.zeros(1, 16, 16, dtype=torch.bool)
    with pytest.raises(ValueError, match="channels"):
        model(torch.rand(1, 2, 1, 16, 16), mask)
    with pytest.raises(ValueError, match="patch"):
        model(torch.rand(1, 2, 3, 20, 16), torch.zeros(1, 20, 16, dtype=torch.bool))
    with pytest.raises(ValueError, match="stack"):
        model(torch.rand(1, 3, 3, 16, 16), mask)


def test_u8_path_envelope_and_server_refusal():
    from paper_2604_27441_b200 import Checkpoint, ModelConfig
    from paper_2604_27441_b200.config import u8_path_unsupported
    from paper_2604_27441_b200.server import RecoveryServer
    assert u8_path_unsupported(ModelConfig()) is None
    assert "patch" in u8_path_unsupported(ModelConfig(patch=8))
    assert "dim" in u8_path_unsupported(ModelConfig(dim=24, heads=3))
    ck = Checkpoint.random_init(ModelConfig(patch=8, dim=16, layers=1), 1, seed=0)
    with pytest.raises(ValueError, match="patch"):
        RecoveryServer(("127.0.0.1", 0), checkpoint_depth=ck)


def test_request_size_from_header():
    import struct
    from paper_2604_27441_b200.server import MSG_REQUEST, ProtocolError, _request_bytes
    head = struct.pack("<BBIHHB", MSG_REQUEST, 0, 7, 64, 32, 5)
    assert _request_bytes(head) == 11 + (2 * 4 + 7) // 8 + 64 * 32 * 3 * 6
    with pytest.raises(ProtocolError):
        _request_bytes(struct.pack("<BBIHHB", MSG_REQUEST, 9, 7, 64, 32, 5))
