"""B200-native low-synchronization block classical Gram-Schmidt QR (arXiv 2507.21791).

Drop-in for the reference's CPU BCGS QR path (BCGSI+P-1S, BCGSI+P-2S, BCGSI+1S,
BCGSPIPI+, BCGSI+): hand-written sm_100a CUDA kernels behind the C ABI in
include/bgs_gpu.h, mirrored here with the reference's names (see api.py).
"""
from .api import *  # noqa: F401,F403
from .api import (  # noqa: F401
    BcgsOptions, Context, FactorOutcome, SyncStats, VariantId, all_variants, default_context,
    expected_syncs, factor_device, gen_gaussian_device, gen_gaussian_host, gen_matrix, gram,
    loss_and_residual, metrics_device, nccl_unique_id, parse_variant, peer_selftest, run_factor,
    shard_rows,
    tsqr, variant_flops, variant_name,
)

__all__ = [
    "BcgsOptions", "Context", "FactorOutcome", "SyncStats", "VariantId", "all_variants", "default_context",
    "expected_syncs", "factor_device", "gen_gaussian_device", "gen_gaussian_host", "gen_matrix",
    "gram",
    "loss_and_residual", "metrics_device", "nccl_unique_id", "parse_variant", "peer_selftest",
    "run_factor",
    "shard_rows", "tsqr", "variant_flops", "variant_name",
]
