"""B200-native Ranky hot path (arXiv 2009.09767): rank check + checker repair,
batched block SVD, UΣ merge and V recovery as sm_100a CUDA kernels behind a
C ABI (include/ranky_b200.h), with a Python mirror of the reference API."""
from .ranky import *  # noqa: F401,F403
from .ranky import (BlockPartition, BlockResultRecord, BlockTask, ColumnRange, ConvergenceError, Context,
                    DeviceMatrix, InvalidArgument, OutOfRange, PipelineResult, ProxyMatrix, RankyRuntimeError,
                    RepairMethod, RepairReport, SparseMatrix, SvdResult, block_svd, block_view, build_proxy,
                    dense_svd, find_lonely_rows, partition_columns, proxy_from_records, proxy_svd,
                    recover_right_vectors, repair, run_block_task, run_block_tasks, run_pipeline, sparse_of,
                    sigma_error, align_signs, left_vector_error, numerical_rank)

__all__ = [
    "BlockPartition", "BlockResultRecord", "BlockTask", "ColumnRange", "ConvergenceError", "Context", "DeviceMatrix",
    "InvalidArgument", "OutOfRange", "PipelineResult", "ProxyMatrix", "RankyRuntimeError", "RepairMethod",
    "RepairReport", "SparseMatrix", "SvdResult", "block_svd", "block_view", "build_proxy", "dense_svd",
    "find_lonely_rows", "partition_columns", "proxy_from_records", "proxy_svd", "recover_right_vectors", "repair",
    "run_block_task", "run_block_tasks", "run_pipeline", "sparse_of",
    "sigma_error", "align_signs", "left_vector_error", "numerical_rank",
]
