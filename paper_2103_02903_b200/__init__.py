"""B200-native adaptive multiresolution lattice Boltzmann time step (arXiv 2103.02903).

The compute path is hand-written CUDA for sm_100a (csrc/mrlbm_step.cu) behind
the C-ABI in include/mrlbm_gpu.h; this package is the thin host-side mirror.
"""
from .abi import SchemeSpec, RunConfig, StepStats  # noqa: F401
from .schemes import build_config, config_steps, finest_cells, initial_finest, stream_table, CONFIG_NAMES  # noqa: F401
from .solver import Solver, MRLBMError, drag_lift, strouhal  # noqa: F401
