"""curveflow-b200: B200-native (sm_100a) discrete weighted-mean-curvature map and
WMC flow filter of Gong & Goksel, arXiv 1903.07189.

Drop-in for the reference's ``wmc_half_laplace`` / ``mc_flow`` (SPEC.md:171,
:256): C-ABI in include/curveflow/capi.h, C++ API in include/curveflow/wmc.hpp,
this Python mirror in :mod:`.curveflow`.
"""
from .curveflow import (FlowConfig, FlowError, SolveReport, SolverConfig, kernel, kernel_bank,
                        max_sweeps_per_launch, solve, solve_l1_area, solve_l2_area,
                        data_fidelity, wmc_energy, wmc_histogram,
                        mc_flow, mc_flow_image8, mc_flow_u8, merge_channels, split_channels, sweeps_band,
                        synth_image, wmc_half_laplace, workspace_bytes)
from ._lib import LIB_PATH, CurveflowError, CurveflowLibraryError, lib
from .configs import CONFIGS, WmcConfig

__all__ = [
    "FlowConfig", "FlowError", "SolverConfig", "SolveReport", "solve_l2_area", "solve_l1_area", "solve", "data_fidelity",
    "wmc_energy", "wmc_histogram", "kernel", "kernel_bank", "max_sweeps_per_launch", "mc_flow",
    "mc_flow_u8", "mc_flow_image8", "merge_channels", "split_channels", "sweeps_band", "synth_image",
    "wmc_half_laplace", "workspace_bytes", "LIB_PATH", "CurveflowError",
    "CurveflowLibraryError", "lib", "CONFIGS", "WmcConfig",
]
__version__ = "0.1.0"
