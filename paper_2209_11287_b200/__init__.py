"""B200-native FP64 epsilon self-join (arXiv 2209.11287, TED-Join).

Drop-in for the self-join path of the reference package `tilejoin`
(/root/reference/pkg/src/tilejoin): same `self_join`, `JoinConfig`,
`JoinResult`, `JoinStats`, errors and grid helpers, computed by hand-written
sm_100a CUDA (libtedjoin.so) behind a C ABI (include/tedjoin.h).
"""

from .datasets import (
    Dataset,
    GenSpec,
    as_dataset,
    generate,
    read_dataset,
    reorder_dims_by_variance,
    write_dataset,
)
from .errors import BoundsError, ParseError, ResourceError, ValidationError
from .join import (
    BatchPlan,
    JoinConfig,
    JoinResult,
    JoinStats,
    join_stats,
    plan_batches,
    plan_from_estimates,
    selectivity,
    self_join,
)

__version__ = "0.1.0"

__all__ = [
    "BatchPlan", "BoundsError", "Dataset", "GenSpec", "JoinConfig", "JoinResult", "JoinStats",
    "ParseError", "ResourceError", "ValidationError", "as_dataset", "generate", "join_stats",
    "plan_batches", "plan_from_estimates", "read_dataset", "reorder_dims_by_variance",
    "selectivity", "self_join", "write_dataset",
]
