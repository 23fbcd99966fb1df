"""B200-native walk-sampling estimator of arXiv 2308.01037 (drop-in for the
reference package ``mcfunm``'s estimator/centrality path).

Host API mirrors the reference; compute runs in
libmcfunm_cuda.so (include/mcfunm_cuda.h) -- sm_100a kernels, no CPU fallback.
"""

from .errors import (ArgumentError, ConvergenceError, DataError, DegenerateInputError, DeviceError,  # noqa: F401
                     McfunmError, ParseError, ResourceError)
from .series import EXPONENTIAL, RESOLVENT, CoefficientStream  # noqa: F401
from .ingest import GraphSource, load_graph, simple_graph_from_edges, symmetrize_digraph  # noqa: F401
from .sparsemat import SparseMatrix, row_abs_sums, scale  # noqa: F401
from .walker import WalkConfig, alpha_diagnostic  # noqa: F401

__version__ = "0.1.0"


def __getattr__(name):
    # torch-dependent parts load lazily so host-only use stays cheap
    if name in ("rand_funm", "rand_funm_diag", "rand_funm_action", "rand_funm_entry", "mc_baseline", "FunmResult"):
        from . import estimators
        return getattr(estimators, name)
    if name in ("subgraph_centrality", "total_communicability", "katz_centrality", "estrada_index",
                "ranking_correlation", "CentralityReport", "gershgorin_gamma"):
        from . import centrality
        return getattr(centrality, name)
    if name == "DeviceGraph":
        from .device import DeviceGraph
        return DeviceGraph
    raise AttributeError(name)
