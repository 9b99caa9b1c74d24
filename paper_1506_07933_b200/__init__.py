"""paper_1506_07933_b200 — B200-native distributed 3-D FFT execute path.

A drop-in for the plan / execute / local-size API of the reference dfft
artifact (AccFFT, arXiv 1506.07933), executed by hand-written sm_100a
kernels in libdfftb.so.  See DESIGN.md and INTEGRATION.md.
"""
from .dfft import (  # noqa: F401
    Direction,
    DistTensor,
    Distribution,
    ElementKind,
    Error,
    ExchangePath,
    ExecContext,
    PlanOptions,
    Plan,
    ProcessGrid,
    TimingBreakdown,
    TransformKind,
    block_map,
    execute,
    execute_r2c_c2r_roundtrip,
    execute_world,
    hat_dims,
    kernel_launch_count,
    local_index,
    make_context,
    make_world_contexts,
    plan_general,
    plan_pencil,
    plan_slab,
    workspace_bytes,
)
