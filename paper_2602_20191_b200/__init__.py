"""B200-native MoBi linear layer (MoBiQuant inference hot path, arXiv 2602.20191).

route -> bucket -> nested residual GEMM (tcgen05) -> un-permute, behind the C ABI in
include/mobi_b200.h.  See DESIGN.md.
"""
from ._lib import MobiError, MobiInvalidArgument, build, lib  # noqa: F401

__all__ = ["MobiError", "MobiInvalidArgument", "build", "lib", "MobiLayer", "permute_by_slice",
           "calibrate_threshold", "decompose", "ratio_from_target_bits", "joint_step", "msb_step", "BudgetSchedule", "share_activations"]


def __getattr__(name):  # lazy: importing the package must not require torch/CUDA
    if name in ("MobiLayer", "permute_by_slice", "calibrate_threshold", "decompose", "ratio_from_target_bits",
                "avg_bits_from_masks", "joint_step", "msb_step", "BudgetSchedule", "share_activations"):
        from . import layer
        return getattr(layer, name)
    raise AttributeError(name)
