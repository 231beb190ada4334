"""B200-native factorized linear algebra over normalized matrices (Morpheus, arXiv 1612.07448).

Drop-in for the reference package ``factorla``'s hot path: the normalized-matrix
constructors (normmat.py), the factorized operators (rewrite.py) and the ML drivers
(ml.py), with every arithmetic step in hand-written sm_100a kernels behind the C ABI
``include/factorla_b200.h`` (``libfactorla_b200.so``).
"""

from ._lib import launch_count
from .exceptions import (
    DataError,
    DivergenceError,
    EmptyJoinError,
    ExtensionMissingError,
    FactorlaError,
    NumericError,
    ShapeError,
)
from .kernel import OpCounter
from .normmat import (
    IndicatorMatrix,
    NormalizedMatrix,
    ShapeStats,
    as_normalized,
    build_mn,
    build_multimn,
    build_pkfk,
    build_star,
    materialize,
    stats,
    transpose,
)
from .rewrite import HostCallableWarning, col_sums, crossprod, lmm, rmm, row_sums, scalar_fn, scalar_op, sum_all
from .products import (
    MaterializationWarning,
    dmm,
    dmm_gram,
    elementwise_matrix_op,
    ginv,
    gram_transposed,
    pair_product,
)
from .ml import ModelOutput, TrainConfig, gnmf, kmeans, linreg_gd, linreg_normal, logistic_gd
from . import costmodel
from .costmodel import auto_dispatch
from . import dataio

__version__ = "0.1.0"

__all__ = [
    "DataError",
    "DivergenceError",
    "EmptyJoinError",
    "ExtensionMissingError",
    "FactorlaError",
    "NumericError",
    "ShapeError",
    "OpCounter",
    "IndicatorMatrix",
    "NormalizedMatrix",
    "ShapeStats",
    "as_normalized",
    "build_mn",
    "build_multimn",
    "build_pkfk",
    "build_star",
    "materialize",
    "stats",
    "transpose",
    "col_sums",
    "crossprod",
    "lmm",
    "rmm",
    "row_sums",
    "scalar_fn",
    "scalar_op",
    "sum_all",
    "gram_transposed",
    "ginv",
    "dmm",
    "dmm_gram",
    "elementwise_matrix_op",
    "pair_product",
    "MaterializationWarning",
    "HostCallableWarning",
    "launch_count",
    "costmodel",
    "auto_dispatch",
    "dataio",
    "ModelOutput",
    "TrainConfig",
    "gnmf",
    "kmeans",
    "linreg_gd",
    "linreg_normal",
    "logistic_gd",
]
