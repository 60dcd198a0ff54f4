"""dmtk on B200: dense FP64 MTTKRP / Khatri-Rao / CP-ALS (arXiv 1708.08976)
re-built for sm_100a behind the reference's API.

The compute path is libdmtk_gpu.so (CUDA, built in-tree); this package is
the Python mirror of the reference interface over its C ABI. Importing it
without the built library raises: there is no CPU fallback.
"""
from .api import (  # noqa: F401
    DISTS,
    AlsConfig,
    AlsIterRecord,
    AlsResult,
    AlsTrace,
    DenseTensor,
    DeviceError,
    FitResult,
    InvalidArgument,
    KrpStats,
    KruskalModel,
    MttkrpAlgo,
    MttkrpRequest,
    MttkrpResult,
    OutOfRange,
    ShapeOverflow,
    TensorFileError,
    TwoStepOrder,
    als_iterate,
    choose_order,
    cp_als,
    device_count,
    fit,
    fp64_peak_tflops,
    fp64_peak_tflops_sustained,
    generate_factors,
    gram_hadamard,
    krp,
    krp_device,
    krp_naive,
    krp_small,
    launch_count,
    mttkrp,
    mttkrp_baseline,
    mttkrp_device,
    mttkrp_one_step,
    mttkrp_two_step,
    mode_seed,
    solve_psd,
    tensor_norm,
)

__version__ = "0.1.0"
