"""B200-native nvrec recovery path (arxiv 2604.27441, ReVo).

Public surface mirrors the reference ``nvrec`` package
(``pkg/nvrec/src/nvrec/__init__.py:7-11``) -- ``ModelConfig``,
``LossWeights``, ``MaskedVideoModel`` -- plus the recovery-path pieces the
reference keeps in ``nvrec.server`` / ``nvrec.train`` / ``rgbdstream``:
``RecoveryServer``, ``Checkpoint``, the batched ``RecoveryEngine`` and the
GPU loss-mask builder.  All compute runs in ``lib/libnvrec_b200.so``
(hand-written sm_100a kernels behind a C-ABI); there is no CPU fallback.
"""

from .config import LossWeights, ModelConfig
from .model import MaskedVideoModel
from .checkpoint import Checkpoint

__all__ = ["LossWeights", "ModelConfig", "MaskedVideoModel", "Checkpoint"]
