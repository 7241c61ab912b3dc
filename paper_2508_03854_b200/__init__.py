"""B200-native 2D-sparse-parallel embedding training step (arXiv 2508.03854).

Drop-in for the embedding path of the reference ``sparse2d`` library: table
configs, the 2D mesh planner (``Topology``, ``plan_greedy``) and the
moment-scaled row-wise AdaGrad optimizer keep the reference's names; the step
(input-dist bucketing, pooled lookup, radix-sort dedup, fused AdaGrad, replica
sync) runs as hand-written sm_100a CUDA kernels + NCCL in
``libsparse2d_b200.so`` behind a C ABI (``include/sparse2d_b200.h``).
"""
from .api import (  # noqa: F401
    Trainer,
    TrainerOptions,
    closed_form_ratio,
    estimate_increment_ratio,
    evaluate_ne,
    memory_overhead,
    qps_scaling_factor,
    recommend_c,
    sync_latency,
    LocalHub,
    OptimizerConfig,
    Sparse2DEmbedding,
    TableConfig,
    Topology,
    adagrad_row_step,
    adagrad_rows,
    effective_lr,
    imbalance_ratio,
    launch_count,
    local_mesh,
    nccl_unique_id,
    owner_of,
    plan_greedy,
    run_ranks,
    traces_to_csv,
    train_toy,
    pool_ids,
    lookup_and_pool,
    aggregate_group_gradient,
    validate_plan,
)

__all__ = [
    "Trainer",
    "train_toy",
    "pool_ids",
    "lookup_and_pool",
    "aggregate_group_gradient",
    "TrainerOptions",
    "closed_form_ratio",
    "estimate_increment_ratio",
    "evaluate_ne",
    "memory_overhead",
    "qps_scaling_factor",
    "recommend_c",
    "sync_latency",
    "LocalHub",
    "OptimizerConfig",
    "Sparse2DEmbedding",
    "TableConfig",
    "Topology",
    "adagrad_row_step",
    "adagrad_rows",
    "effective_lr",
    "imbalance_ratio",
    "launch_count",
    "local_mesh",
    "nccl_unique_id",
    "owner_of",
    "plan_greedy",
    "run_ranks",
    "traces_to_csv",
    "validate_plan",
]

__version__ = "0.1.0"
