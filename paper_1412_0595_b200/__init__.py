"""B200-native spiking-network step engine (arXiv 1412.0595 hot path).

Drop-in for the reference `synscale` engine's step path: Poisson sources,
conductance-LIF populations, dense and CRS synapse groups, advanced by
hand-written sm_100a kernels behind a C ABI (include/synscale_b200.h).
"""
from .synscale import *  # noqa: F401,F403
from .synscale import (CondLifParams, EngineOptions, NetworkSpec, Simulation, SpecError,  # noqa
                       StorageMode, build_mbody_net, run)

__all__ = [name for name in dir() if not name.startswith("_")]
