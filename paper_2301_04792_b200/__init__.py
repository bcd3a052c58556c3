"""paper_2301_04792_b200: B200-native load-balanced SpMV (atoms / tiles / schedules).

A from-scratch B200 implementation of the load-balancing abstraction of
Osama, Porumbescu & Owens (arXiv 2301.04792) with the public API of the
reference package ``lanework`` for its SpMV path: tile sets, schedules
(thread-mapped, merge-path a.k.a. work-oriented, group-mapped warp/block
tiles) and ``spmv(m, x, cfg)``. The arithmetic runs in hand-written sm_100a
kernels (liblwb200.so, C ABI in include/lw_b200.h); there is no CPU fallback.
"""

from ._backend import (ENV_VAR, NUMBA_AVAILABLE, backend_name, cuda_active, cuda_available,
                       numba_active, use_backend)
from ._lib import BackendUnavailable
from .device import (DeviceCsr, HotColumns, device_group_plan_prefix, device_merge_path_partition,
                     generate_banded_device, generate_rmat_csr,
                     generate_uniform_device)
from .executor import (SENTINEL_TILE, SUM_CARRIES, AtomicMinArray, CarryOut, CarryPolicy,
                       ExecutorConfig, ImbalanceReport, atomic_min_real, device_config,
                       execute_merge_path, execute_tile_major, fixup_combine, imbalance)
from .kernels import (HeuristicConfig, choose_spmv_schedule, spmm, spmv, spmv_auto,
                      spmv_probe)
from .mmio import (MatrixMarketError, load_matrix_market, parse_matrix_market,
                   write_matrix_market)
from .schedules import (GroupMappedSchedule, GroupPlan, MergePathCoord, MergePathSchedule,
                        MergePathSlice, Schedule, ScheduleKind, ThreadMappedSchedule,
                        exclusive_prefix_sum, get_tile, group_plan, make_schedule,
                        merge_path_partition, merge_path_search, merge_path_slices, num_blocks,
                        thread_mapped_tiles)
from .sparse import (CooMatrix, CsrMatrix, Graph, coo_to_csr, csr_to_coo, generate_banded_csr,
                     generate_power_law_csr, generate_random_csr, rmat_thresholds,
                     row_length_stats, transpose_csr, validate_coo, validate_csr)
from .traversal import (UNREACHED, SsspState, bfs, bfs_pass, device_graph, sssp, sssp_init,
                        sssp_pass)
from .work import (TileSet, csr_tile_set, infinite_range, lane_stride_range, step_range,
                   tile_offsets)

__version__ = "0.1.0"

__all__ = [
    "HotColumns",
    "AtomicMinArray", "SsspState", "UNREACHED", "atomic_min_real", "bfs", "bfs_pass",
    "device_graph", "sssp", "sssp_init", "sssp_pass",
    "BackendUnavailable", "NUMBA_AVAILABLE", "CarryOut", "CarryPolicy", "CooMatrix", "CsrMatrix", "Graph",
    "MatrixMarketError", "coo_to_csr", "csr_to_coo", "load_matrix_market", "parse_matrix_market",
    "transpose_csr", "validate_coo", "write_matrix_market", "DeviceCsr", "ENV_VAR",
    "ExecutorConfig", "GroupMappedSchedule", "GroupPlan", "HeuristicConfig", "ImbalanceReport",
    "MergePathCoord", "MergePathSchedule", "MergePathSlice", "SENTINEL_TILE", "SUM_CARRIES",
    "Schedule", "ScheduleKind", "ThreadMappedSchedule", "TileSet", "backend_name",
    "choose_spmv_schedule", "csr_tile_set", "cuda_active", "cuda_available", "device_config",
    "device_group_plan_prefix", "device_merge_path_partition", "exclusive_prefix_sum",
    "execute_merge_path", "execute_tile_major", "fixup_combine", "generate_banded_csr",
    "generate_banded_device", "generate_power_law_csr", "generate_random_csr",
    "generate_rmat_csr", "generate_uniform_device", "get_tile", "group_plan", "imbalance", "infinite_range",
    "lane_stride_range", "make_schedule", "merge_path_partition", "merge_path_search",
    "merge_path_slices", "num_blocks", "numba_active", "rmat_thresholds", "row_length_stats",
    "spmm", "spmv", "spmv_auto", "spmv_probe", "step_range", "thread_mapped_tiles", "tile_offsets",
    "use_backend", "validate_csr",
]
