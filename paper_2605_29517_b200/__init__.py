"""B200-native Flash-MaxSim: a drop-in for the reference `maxsim` operator path on sm_100a.

Same public names as maxsim/__init__.py:9-56 for the hot path (forward, backward, INT8,
varlen, top-K); the compute runs in libmaxsim_b200.so (tcgen05 / TMA / TMEM kernels behind a
C-ABI, include/maxsim_b200.h).  There is no CPU fallback: without the library or a CUDA
device every operator raises.
"""

from .errors import (
    BadTileConfig,
    CudaError,
    DimMismatch,
    EmptyDocument,
    IndexOutOfRange,
    KTooLarge,
    MaxSimError,
    NaNInput,
    ShapeMismatch,
    StaleCsr,
    Unsupported,
    IoError,
    BadMagic,
    VersionUnsupported,
    TruncatedPayload,
    StaleArgmin,
)
from .instrument import TrafficReport
from .types import ArgmaxMap, DEFAULT_TILE, DocBatch, EmbeddingMatrix, ScoreMatrix, TileConfig, validate_pair
from .forward import (
    ForwardStrategy,
    RunningRowState,
    dispatch,
    fused_score_batch,
    fused_score_pair,
    query_chunk_decompose,
    score_dense,
)
from .backward import (
    CsrInverse,
    backward_dispatch,
    build_inverse_csr,
    choose_gradient_path,
    doc_grads_in_layout,
    grad_docs_csr,
    grad_docs_scatter,
    grad_query,
)
from .quant import (
    QuantizedCorpus,
    QuantizedMatrix,
    dequantize,
    fused_score_int8,
    fused_score_int8_batch,
    quantize_corpus,
    quantize_per_token,
    score_int8,
    two_stage_topk,
)
from .varlen import PackedCorpus, fused_score_varlen, pack, score_varlen, unpack
from .topk import TopKHeap, ranked, topk
from .autograd import MaxSimFunction, MaxSimVarlenFunction, maxsim, maxsim_varlen
from .training import contrastive_drift, softmax_ce
from .reference import DenseSimTensor, dense_backward, dense_score, dense_score_batch, finite_diff_grad
from .chamfer import PointSet, chamfer_backward, chamfer_forward, dense_chamfer_backward, dense_chamfer_forward
from .streamio import (
    CorpusReader,
    TrafficModel,
    model_traffic,
    read_embeddings,
    stream_score_host,
    stream_score_topk,
    write_embeddings,
)

__version__ = "0.1.0"

