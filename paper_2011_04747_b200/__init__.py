"""B200-native DAETI monodomain hot path (arXiv 2011.04747), drop-in for cardwave's proj/core.

The compute lives in libcwgpu.so (hand-written sm_100a CUDA, C ABI in
include/cwgpu.h); this package is the Python mirror of the reference
interface (see api.py). Importing it loads the library and fails loudly if
it is missing.
"""
from ._lib import lib as _load_lib

_load_lib()

from .api import (  # noqa: E402
    AssembledOperator, CellModel, DeviceError, DiffusionPlan, InstabilityError, IoError, NodeStateArray, Probe,
    Protocol, ProtocolIndex, Scheme, SchemeConfig, ScalarMap, Sheet, SimulationResult, Slab3D, SimulationSetup, Stimulus,
    DeviceSheetOperator, StrangIntegrator, ThresholdOptions, TimingBreakdown, Trace, ValidationError, build_sheet, diastolic_threshold, diffusion_substep, diffusion_substeps,
    k_max_for, make_initial_state, make_model, pace_cells, pace_to_steady_state, PacingResult, reaction_substeps, registered_model_names, run_simulation,
    scheme_from_string, slab_plan,
)

from . import output, postprocess  # noqa: E402
from .postprocess import (  # noqa: E402
    CompareReport, SchemeComparison, align_and_diff, compare_schemes, compute_apd90, compute_cv, nrmse,
)

__all__ = [n for n in dir() if not n.startswith("_")]
