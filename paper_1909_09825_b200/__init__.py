"""B200-native SOE fast Gauss transform (arXiv:1909.09825 hot path).

    u_i = sum_j exp(-(x_i - y_j)^2 / (4 delta)) alpha_j

Python mirror of the reference `fgt1d` package surface for the transform path
(proj/python/fgt1d/__init__.py); all compute runs in libfgt1d_b200.so on the
GPU through the C ABI in include/fgt1d_b200.h.
"""
from ._capi import DeviceError, NumericalError
from .soe import (ErrorReport, SoeApprox, SoeForm, cf_soe, error_grid_point, evaluate, fold,
                  load_coefficient_table, max_error, max_error_extended,
                  mode_count_for_tolerance, preset_mode_count, preset_soe,
                  save_coefficient_table, soe_for_tolerance, unfold, validate)
from .transform import (BatchPlan, TransformPlan, TransformRequest, apply_general, apply_same,
                        batch_transform, chebyshev_points, delta_sweep, direct, gen_points,
                        measure_error,
                        direct_transform, gauss_transform, gauss_transform_device, mode_sums, plan,
                        precompute_gap_table, transform_host, uniform_points,
                        uniform_points_array)

__version__ = "0.1.0"

__all__ = [
    "BatchPlan", "DeviceError", "ErrorReport", "NumericalError", "batch_transform", "SoeApprox",
    "SoeForm", "TransformPlan", "TransformRequest", "chebyshev_points", "delta_sweep",
    "error_grid_point", "gen_points", "max_error", "max_error_extended", "measure_error",
    "apply_general", "apply_same", "cf_soe", "direct", "direct_transform", "evaluate", "fold",
    "gauss_transform", "gauss_transform_device", "transform_host", "load_coefficient_table", "mode_count_for_tolerance", "mode_sums", "plan",
    "precompute_gap_table", "preset_mode_count", "preset_soe", "save_coefficient_table",
    "soe_for_tolerance", "unfold", "uniform_points", "uniform_points_array", "validate",
]
