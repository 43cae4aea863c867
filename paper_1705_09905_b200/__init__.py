"""B200-native (sm_100a) F-COO sparse tensor hot path of arXiv 1705.09905.

The product is libfcoo.so (C ABI in include/fcoo.h, CUDA sources in csrc/); this package is
its thin Python binding (fcoo.py) plus the in-tree build script (build_lib.py).
"""
from .fcoo import (BUILD_BLOCKED, ERR_ARG, ERR_DUPLICATE, ERR_INDEX_RANGE, ERR_IO, ERR_RANK, ERR_SHAPE, OP_MTTKRP,
                   OP_TTM, Coo, Comm, Fcoo, FcooError, McBuffer, comm_from_process_group, cp_als, fcoo_allreduce_sum,
                   fcoo_build, fcoo_build_sharded, fcoo_comm_init, fcoo_comm_unique_id, fcoo_debug_flip_bit, fcoo_export, fcoo_mttkrp,
                   fcoo_mttkrp_mc, fcoo_set_shard, fcoo_shard_range, fcoo_ttm, fcoo_ttmc, launch_count, load_library,
                   read_tns, write_tns, fcoo_slice_histogram, fcoo_row_partition, fcoo_bucket_rows, fcoo_set_row_shard,
                   fcoo_build_distributed)

__all__ = ["BUILD_BLOCKED", "ERR_ARG", "ERR_DUPLICATE", "ERR_INDEX_RANGE", "ERR_IO", "ERR_RANK", "ERR_SHAPE",
           "OP_MTTKRP", "OP_TTM", "Coo", "Comm", "Fcoo", "FcooError", "McBuffer", "comm_from_process_group", "cp_als",
           "fcoo_allreduce_sum", "fcoo_build", "fcoo_build_sharded", "fcoo_comm_init", "fcoo_comm_unique_id",
           "fcoo_debug_flip_bit", "fcoo_export", "fcoo_mttkrp", "fcoo_mttkrp_mc", "fcoo_set_shard", "fcoo_shard_range", "fcoo_ttm",
           "fcoo_ttmc", "launch_count", "load_library", "read_tns", "write_tns", "fcoo_slice_histogram",
           "fcoo_row_partition", "fcoo_bucket_rows", "fcoo_set_row_shard", "fcoo_build_distributed"]
