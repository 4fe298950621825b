"""B200-native Louver decode hot path (arxiv 2605.06763).

For each decode query: retrieve every cached key with q·k >= tau (zero false
negatives, bit-exact against the reference's normative fp32 dot) and attend
over exactly that set, on sm_100a kernels behind the C ABI in
include/louver_b200.h. See DESIGN.md.
"""
from ._capi import LouverError, LIB_PATH, SYNTH_PATH  # noqa: F401
from .sharding import ShardedLayer, gather_partials, insert_owner, shard_range  # noqa: F401
from .threshold import (  # noqa: F401
    OracleConfig,
    OracleVariant,
    Reservoir,
    estimate_tau,
    estimate_tau_layer,
    parse_oracle,
)
from .snapshot import load_dataset, load_index, save_dataset, save_index  # noqa: F401
from .decode_sim import (DecodeSimConfig, GraphDecodeReport, MetricsReport, ThresholdSource,  # noqa: F401
                         run_decode_graph, run_decode_sim)
from .louver import (  # noqa: F401
    AttentionResult,
    BuildConfig,
    CacheQueryResult,
    CandidateSet,
    FilterAlgo,
    LouverCache,
    LouverLayer,
    QueryRequest,
    QueryStats,
    brute_force_range,
    derive_subspace_thresholds,
    lse_merge,
    query_full_subspace,
    query_ta,
    query_layers_host,
    LayersStep,
    sparse_attention,
    SubspaceIndex,
)

__all__ = [
    "AttentionResult", "BuildConfig", "CacheQueryResult", "FilterAlgo", "LouverCache", "LouverLayer",
    "QueryRequest", "QueryStats", "CandidateSet", "SubspaceIndex", "query_ta", "query_full_subspace",
    "derive_subspace_thresholds", "brute_force_range", "lse_merge", "query_layers_host", "LayersStep", "sparse_attention", "LouverError",
    "ShardedLayer", "gather_partials", "insert_owner", "shard_range",
    "OracleConfig", "OracleVariant", "Reservoir", "estimate_tau", "estimate_tau_layer", "parse_oracle",
    "DecodeSimConfig", "MetricsReport", "ThresholdSource", "run_decode_sim", "GraphDecodeReport", "run_decode_graph",
    "save_dataset", "load_dataset", "save_index", "load_index",
]
