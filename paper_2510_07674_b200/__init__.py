"""B200-native (sm_100a) two-stage particle optimizer for fixed-skeleton pick-and-place
(SPaSM, arxiv 2510.07674): a drop-in for the reference package's stage-1
``particle_opt.solve`` / ``CostModel`` path and its stage-2 trajectory path, with every
numeric stage in hand-written CUDA kernels behind the C-ABI in include/spasm.h."""

__version__ = "0.1.0"

from .geometry import LINEAR, QUADRATIC  # noqa: F401
