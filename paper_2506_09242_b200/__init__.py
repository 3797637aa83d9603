"""B200-native fused collide-and-stream for the dolb lattice Boltzmann solver
(arXiv 2506.09242 hot path). See DESIGN.md; the C ABI is include/dlb.h."""
from . import _capi  # noqa: F401
from .dolb import *  # noqa: F401,F403
from .cases import (CaseConfig, CaseSetup, build_run, init_cavity, init_porous,  # noqa: F401
                    init_tgv, load_voxels, make_plate_mask, setup_models, sphere_pack)

__version__ = "0.1.0"
