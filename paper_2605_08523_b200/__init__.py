"""fermiforge-b200: the MLSP2 finite-temperature density-matrix builder on sm_100a.

The product is libfermiforge_b200.so (C ABI in include/fermiforge/ffg.h);
``engine`` mirrors the reference interface over it, ``distributed`` shards
batches across GPUs (one process per GPU, NCCL gather of results).
"""
from .engine import (  # noqa: F401
    PrecisionMode, Mlsp2Model, SpectralBounds, DensityStatistics, Provenance, load_model,
    spectral_bounds, in_region_of_validity, apply_model, mixed_square, density_statistics,
    compute_density_matrix, compute_density_matrices, compute_density_matrices_device,
    algorithmic_flops, kernel_launches, device_available, FermiforgeError, ValidationError,
    OutOfRegionError, DivergedEvaluationError, HalfRangeError, UnsupportedModeError,
    DimensionError, CudaError, lib, LIB_PATH,
)
