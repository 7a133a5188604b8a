"""paper_2604_15765_b200 -- B200-native (sm_100a) implementation of the hot path of arXiv 2604.15765
("Orkan"): single-pass k-local conjugation and Kraus channels on a hermitian operator stored in the
tiled lower-triangle layout.

Layers:
  csrc/engine.cu      CUDA kernels + thin C-ABI (include/hs_cuda.h)
  csrc/host/*.cpp     C++ host API mirroring the reference (include/hermsim_b200/hermsim.hpp) and
                      its C facade (include/hermsim_b200_c.h)
  hermsim.py          Python mirror of the reference API over the C facade (ctypes)
  harness.py          seeded synthetic inputs of the BASELINE.json configs
  multigpu.py         tile-row sharding across GPUs (one process per GPU)
"""
from . import hermsim  # noqa: F401
from .hermsim import (  # noqa: F401
    ApplyOptions, ApplyPlan, ChannelSpec, TiledHermitian, amplitude_damping, apply, bind_channel, depolarising,
    dual_channel, expectation, footprint_bytes, frobenius, make_generic, native_gate, trace, validate_cptni,
)

__version__ = "0.1.0"
