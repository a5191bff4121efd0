"""B200-native batched rigid-body simulation (the Isaac Gym hot path, arXiv 2108.10470).

Drop-in for the reference `batchsim` Scene / SimBuffers / EnvBatch boundary,
backed by hand-written sm_100a CUDA kernels.
"""

from .model import (ArticulationModel, BadLimits, CycleError, MissingLink, ModelError,  # noqa: F401
                    NonPositiveMass, load_model)
from .params import SimParams  # noqa: F401

__version__ = "0.1.0"


def __getattr__(name):
    # torch-dependent pieces load lazily so the host-side modules import without CUDA
    if name in ("Scene", "ContactPoint"):
        from . import scene
        return getattr(scene, name)
    if name == "SimBuffers":
        from .buffers import SimBuffers
        return SimBuffers
    raise AttributeError(name)
