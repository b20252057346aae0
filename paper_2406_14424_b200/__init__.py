"""gearserve-b200: B200-native CascadeServe hot paths (arXiv 2406.14424).

Drop-in for the reference package's cascade / gear-plan API
(/root/reference/pkg/src/gearserve): `kernels.evaluate_encoded`, the
`cascades` functions, plus the device-resident full-grid sweep
(`gridsweep.GridSweep`), the online stage step (`stage.stage_step`) and the
engine's batched finish_batch gate (`engine`).  Compute runs in hand-written
sm_100a kernels behind the C ABI in include/gearserve_b200.h; there is no
CPU fallback.
"""

from .types import (  # noqa: F401
    US_PER_S,
    Cascade,
    ModelOutput,
    ModelProfile,
    ProfileSet,
    ValidationArrays,
    ValidationRecord,
    ValidationSet,
)

__version__ = "0.1.0"
