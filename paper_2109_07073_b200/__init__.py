"""B200-native (sm_100a) VGICP matching-cost factor evaluation.

Drop-in for the hot path of arxiv 2109.07073's reference (voxel-map build, per-point
linearization with per-factor reduction, error-only evaluation, voxel overlap query); see
DESIGN.md. Compute runs in lib/libvgicp_b200.so (C ABI: include/vgicp_b200.h); there is no CPU
fallback.
"""
from ._lib import KEY_MISS, LINEARIZED_DOUBLES, NoDeviceError, VgicpError
from .vgicp import (
    Context,
    FactorGraph,
    GaussianVoxelMap,
    GicpErrorResult,
    LinearizedFactor,
    MapSet,
    MatchingCostFactor,
    PointCloud,
    Submap,
    as_pose12,
    build_submap,
    cov6_from,
    default_context,
    estimate_covariances,
    estimate_covariances_batch,
    evaluate_matching_cost,
    gicp_error,
    linearize_matching_cost,
    overlap_hits,
    overlap_rate,
    overlap_rates,
    transform_cloud,
    voxel_downsample,
)

__all__ = [
    "KEY_MISS",
    "LINEARIZED_DOUBLES",
    "NoDeviceError",
    "VgicpError",
    "Context",
    "FactorGraph",
    "MapSet",
    "GaussianVoxelMap",
    "GicpErrorResult",
    "LinearizedFactor",
    "MatchingCostFactor",
    "PointCloud",
    "Submap",
    "as_pose12",
    "build_submap",
    "cov6_from",
    "default_context",
    "estimate_covariances",
    "estimate_covariances_batch",
    "evaluate_matching_cost",
    "gicp_error",
    "linearize_matching_cost",
    "overlap_hits",
    "overlap_rate",
    "overlap_rates",
    "transform_cloud",
    "voxel_downsample",
]
