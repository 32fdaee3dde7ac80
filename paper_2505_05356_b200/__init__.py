"""B200-native C-ToF Gaussian-splat render/optimise path (drop-in for the
reference tofsplat RenderPass / AdamState hot path).

The compute lives in lib/libtsb.so (hand-written sm_100a CUDA behind the C ABI
of include/tsb.h); this package is the Python mirror of the reference API.
Importing it loads the library and fails loudly if it has not been built.
"""
from ._abi import TsbError, lib as _load_lib

_load_lib()

from .render import (AdamParams, CameraModel, Comm, Context, DeformNet, GaussianScene, LrTable, RenderOptions,  # noqa: E402
                     RenderPass, ToFConfig, frame_for_time, quad_basis, quad_to_depth, read_pfm, unambiguous_range,
                     write_pfm)

__all__ = ["AdamParams", "CameraModel", "Comm", "Context", "DeformNet", "GaussianScene", "LrTable", "RenderOptions", "RenderPass",
           "ToFConfig", "TsbError", "frame_for_time", "quad_basis", "quad_to_depth", "read_pfm", "unambiguous_range",
           "write_pfm"]
