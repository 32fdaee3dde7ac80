"""`_core` (proj/python/bindings.cpp:40-204): the implementation lives in
paper_2505_05356_b200.core and calls the sm_100a kernels of libtsb.so."""
from paper_2505_05356_b200.core import (  # noqa: F401
    builtin_scene_names,
    dataset_info,
    evaluate,
    fit_dataset,
    gradcheck,
    quad_basis,
    quad_to_depth,
    render_timestep,
    simulate_dataset,
    unambiguous_range,
)
