"""B200-native C-ToF Gaussian-splat render/optimise path (drop-in for the
reference tofsplat RenderPass / AdamState hot path).

The compute lives in lib/libtsb.so (hand-written sm_100a CUDA behind the C ABI
of include/tsb.h); this package is the Python mirror of the reference API.
The library is loaded on first use (the first Context, scene, helper call ...),
which raises if it has not been built -- there is no CPU fallback.  Importing
the package alone (e.g. for the seeded input generator in `synthetic`) does not
map it, so bench.py's reference (CPU) arm never loads the product library.
"""
import os as _os

# Render passes run on their own streams (frames overlap on the device).  The default 8
# hardware work queues make streams beyond 8 share a queue (false dependencies between
# frames); 16 queues with 24 passes in flight measured best for the c3 sweep, with and
# without host transfers.  Must be set before the process creates its CUDA context.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "16")

from ._abi import TsbError, lib as load_library  # noqa: E402

from .render import (AdamParams, CameraModel, Comm, Context, DeformNet, GaussianScene, LrTable, RenderOptions,  # noqa: E402
                     RenderPass, ToFConfig, frame_for_time, quad_basis, quad_to_depth, read_pfm, unambiguous_range,
                     write_pfm)

__all__ = ["AdamParams", "CameraModel", "Comm", "Context", "DeformNet", "GaussianScene", "LrTable", "RenderOptions", "RenderPass",
           "ToFConfig", "TsbError", "frame_for_time", "load_library", "quad_basis", "quad_to_depth", "read_pfm", "unambiguous_range",
           "write_pfm"]
