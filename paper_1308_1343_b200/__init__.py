"""B200-native stencil-sweep hot path of the arXiv 1308.1343 reference (`stencilrt`).

Drop-in host API for the reference's loop iterator and stencil kernels
(traverse.py, tuner.py, stencil.py, vlanes.py) over hand-written sm_100a
CUDA kernels reached through the C ABI in include/stencil_b200.h.
"""
from .errors import DeviceError, ResourceError, UsageError  # noqa: F401
from .traverse import (  # noqa: F401
    Block, IndexSpace, Kernel, SplitPlan, Tile, build_plan, execute_plan, index_space_from_bbox,
    index_space_to_bbox, run_loop, run_static,
)
from .tuner import (  # noqa: F401
    ExecParams, LaunchParams, LaunchSpace, LoopSetup, PlanSpace, TopologyConfig, Tuner, TuningCache, device_setup,
)
from .level import Box, Lattice, boxes_of, compact_level  # noqa: F401

__version__ = "0.2.0"
