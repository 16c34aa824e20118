"""B200-native hybrid LU-QR hot path (arXiv 1401.5522).

The compute lives in `libhlq.so` (hand-written sm_100a CUDA behind the C ABI in include/hlq.h).
This package is the thin Python binding: argument marshalling only, same names as the C ABI.
There is no CPU fallback: loading fails loudly when the library is missing.
"""
from ._binding import (  # noqa: F401
    CRIT_MAX, CRIT_MUMPS, CRIT_SUM, CRIT_RANDOM, DEC_LU, DEC_QR, LU_A1, LU_A2, PIVOT_TILE, PIVOT_DOMAIN, TREE_GREEDY, TREE_HQR, FLAG_FORCED, FLAG_HINTED, FLAG_NEAR_TIE,
    FLAG_NONFINITE, FLAG_ZERO_PIVOT, HlqError, HlqInfo, HlqOptions, Factors, from_colmajor,
    hlq_abi, hlq_default_options, hlq_factor, hlq_factor_ex, hlq_generate_uniform, hlq_gesv_host,
    hlq_launch_count, hlq_test_schur, hlq_residual, hlq_solve, lib, lib_path, to_colmajor,
    Grid, cyclic_rows, dist_counts, dist_plan, gather_block_cyclic, grid_local, grid_nccl, grid_host, COMM_WORLD, COMM_ROW, COMM_COL, COMM_COL_PANEL, hlq_factor_dist,
    local_shape, nccl_unique_id, scatter_block_cyclic, hlq_generate_uniform_cyclic,
    hlq_residual_dist, _step_vectors)
