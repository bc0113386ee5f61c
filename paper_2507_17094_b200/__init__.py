"""B200-native batched graph-ANNS search path of PathWeaver (arXiv 2507.17094).

Drop-in for the search path of the reference package ``shardann`` 0.1.0
(``shardann/__init__.py:77-95``): same names, argument meaning and error
behaviour, computed by hand-written sm_100a CUDA kernels behind the C ABI in
``include/pw_b200.h`` (``libpwb200.so``).  There is no CPU fallback: every
compute entry point raises when the CUDA library or device is missing.
"""

from .container import (
    ChecksumError,
    DeviceIndex,
    IndexFormatError,
    VersionError,
    crc32c,
    crc32c_combine,
    crc32c_device,
    deserialize_index,
    index_equal,
    index_file_checksum,
    load_index_device,
    serialize_index,
)
from .data import DataFormatError, Dataset
from .graphs import Index, ShardPack, words_per_vector
from .pipeline import (
    NeighborList,
    PipelineResult,
    StageMessage,
    StageStats,
    build_contexts,
    reduce_topk,
    run_ghost_stage,
    run_pipelined,
    run_sharded_baseline,
)
from .metrics import (
    RunMetrics,
    classify_visits,
    collect_metrics,
    cost_model_report,
    mean_recall,
    read_sweep_csv,
    recall_at_k,
    sweep,
    write_metrics_json,
    write_sweep_csv,
)
from .search import (
    DeviceShard,
    GhostContext,
    SearchCounters,
    SearchParams,
    SearchResult,
    ShardContext,
    device_shard,
    search,
)

__version__ = "0.1.0"
