"""``Checkpoint`` -- the weight source of the recovery path.

Drop-in for ``nvrec.train.Checkpoint`` (reference train.py:20-43): same
fields, the same ``torch.save`` blob layout (so checkpoints written by the
reference load here and vice versa), and ``build_model`` returning the
B200-backed ``MaskedVideoModel``.  Training (``pretrain``/``finetune``) is
outside the recovery path and not provided.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import torch

from .config import ModelConfig
from .model import MaskedVideoModel


@dataclass
class Checkpoint:
    config: ModelConfig
    channels: int
    state: dict
    curve: list = field(default_factory=list)
    stage: str = "init"

    def save(self, path: str | os.PathLike) -> None:
        blob = {"config": vars(self.config), "channels": self.channels,
                "state": self.state, "curve": self.curve, "stage": self.stage}
        torch.save(blob, os.fspath(path))

    @classmethod
    def load(cls, path: str | os.PathLike) -> "Checkpoint":
        blob = torch.load(os.fspath(path), weights_only=False)
        return cls(config=ModelConfig(**blob["config"]), channels=blob["channels"],
                   state=blob["state"], curve=blob["curve"], stage=blob["stage"])

    def build_model(self, precision: str = "fast") -> MaskedVideoModel:
        model = MaskedVideoModel(self.config, self.channels, precision=precision)
        model.load_state_dict(self.state)
        return model

    @classmethod
    def random_init(cls, config: ModelConfig, channels: int, seed: int = 0) -> "Checkpoint":
        """Seeded random-init weights, identical to the reference's
        ``torch.manual_seed(seed); MaskedVideoModel(config, channels)``."""
        torch.manual_seed(seed)
        m = MaskedVideoModel(config, channels)
        return cls(config=config, channels=channels,
                   state={k: v.detach().clone() for k, v in m.state_dict().items()})
