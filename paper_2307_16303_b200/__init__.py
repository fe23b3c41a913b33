"""B200-native HODLR3D engine (arXiv 2307.16303): octree + HODLR3D lists +
batched ACA + two-pass streaming matvec on sm_100a, behind a C-ABI
(include/h3d_b200.h). See DESIGN.md."""
from .h3d import (  # noqa: F401
    DegenerateDistributionError,
    DegenerateGeometryError,
    DeviceError,
    GmresOptions,
    GmresResult,
    HMatrixRep,
    HmatOptions,
    IEOperator,
    IeReport,
    KernelSpec,
    MatvecTiming,
    cell_self_integral,
    discretize_ie,
    generate_grid_points,
    generate_points,
    ie_experiment,
    initialize,
    library_path,
    make_kernel,
    matvec,
    nccl_unique_id,
    random_vector,
    reference_error,
    stats,
)
