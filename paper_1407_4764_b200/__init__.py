"""B200 (sm_100a) on-the-fly retrieval hot path — drop-in for otf_retrieval's score/rank/train API.

Re-exports the reference package's hot-path names (otf_retrieval/__init__.py) with GPU
implementations: Repository / score_dense / score_pq / score_binary / top_k / RankedList /
pegasos_step / OnlineTrainer, plus the containers they take. Everything numeric runs in the
hand-written CUDA kernels of ``libotf_b200.so`` through the C ABI in include/otf_b200.h.
"""

__version__ = "0.1.0"

from . import _lib
from ._lib import default_device, launch_count, set_device
from .binary import BinaryCodec, TightFrame, binarize, hamming_distance, unpack_bits
from .errors import (
    ConfigError,
    CorruptionError,
    DegenerateInputError,
    EmptyStoreError,
    FormatError,
    InsufficientDataError,
    NotReadyError,
    RetrievalError,
)
from .model import LinearModel
from .pq import PQCodebook, PQConfig, build_score_lut, learn_pq_codebook, pq_encode, score_codes
from .ranker import RankedList, RankerConfig, Repository, score_binary, score_dense, score_pq, top_k
from .store import FeatureStore
from .trainer import BatchTrainConfig, OnlineTrainer, TrainerConfig, hinge_objective, pegasos_step, train_batch

__all__ = [
    "__version__",
    "BinaryCodec", "TightFrame", "binarize", "hamming_distance", "unpack_bits",
    "ConfigError", "CorruptionError", "DegenerateInputError", "EmptyStoreError", "FormatError",
    "InsufficientDataError", "NotReadyError", "RetrievalError",
    "LinearModel", "PQCodebook", "PQConfig", "build_score_lut", "learn_pq_codebook", "pq_encode", "score_codes",
    "RankedList", "RankerConfig", "Repository", "score_binary", "score_dense", "score_pq", "top_k",
    "FeatureStore", "OnlineTrainer", "TrainerConfig", "pegasos_step",
    "BatchTrainConfig", "train_batch", "hinge_objective",
    "default_device", "set_device", "launch_count",
]
