"""B200-native SSH (Sketch, Shingle & Hash) index-build and query path.

Drop-in for the reference package's hot path (sshts.index: build_index,
query_index).  All compute runs in libsshgpu.so (hand-written
sm_100a CUDA behind the C-ABI in include/sshgpu.h); there is no CPU
fallback.
"""

from .core import (
    ConfigError,
    DataFormatError,
    Dataset,
    IndexLoadError,
    SshError,
    TimeSeries,
    z_normalize,
    z_normalize_dataset,
    z_normalize_rows,
    z_normalize_values,
)
from .index import (
    QueryResult,
    QueryStats,
    RandomFilter,
    SearchStats,
    Float32RoundingWarning,
    SshIndex,
    SshParams,
    WarpingParams,
    SearchResult,
    build_index,
    compute_signatures,
    exact_search,
    exact_search_batch,
    index_from_signatures,
    make_filter,
    num_sketch_bits,
    probe_candidates,
    query_index,
    query_index_batch,
    query_signature,
)

from .dtw import Envelope, build_envelope, dtw_distance, dtw_pairs, lb_keogh, lb_keogh2, lb_kim
from .srp import ndcg_at_k, precision_at_k, srp_matrix, srp_signature, srp_vectors
from .dist import query_index_batch_sharded, shard_range
from .pipeline import extract_subsequences, make_dataset
from .persist import file_checksum, load_dataset, load_index, read_index_file, save_dataset, save_index

__version__ = "0.1.0"
