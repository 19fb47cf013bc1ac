"""B200-native SAGA-NN layer hot path (NGra, arXiv 1810.08403).

Drop-in for the reference's SAGA-NN path: the ``tensor.py`` primitive names
(``ops``), the SAGA-NN front end and model zoo (``program``), the graph store
(``graph``) and the chunk-dataflow executor (``engine``), all running on the
hand-written sm_100a kernels of ``libsagann.so`` (C-ABI: include/sagann.h).
"""

from . import errors
from ._lib import lib as _native  # noqa: F401  (fails loudly if libsagann.so is missing)
from .errors import (BudgetError, ConfigError, EngineError, GraphFormatError, NumericError,
                     ProgramError, ShapeError)
from .graph import (ChunkGrid, Graph, Partition, load_graph, partition_2d, read_features, read_labels,
                    reencode_balance, rmat_graph, synthetic_features, uniform_graph, write_features_bin)
from .program import (FusedGather, LayerProgram, PassReport, build_commnet, build_gcn, build_ggcn,
                      build_ggnn, build_mpgcn,
                      evaluate_expr, fuse_sag, hoist_vertex_computation, make_program, matmul_rows,
                      optimize, trace_udf, validate_program, vertex_form)

__all__ = [
    "errors", "BudgetError", "ConfigError", "EngineError", "GraphFormatError", "NumericError",
    "ProgramError", "ShapeError", "ChunkGrid", "Graph", "Partition", "partition_2d", "load_graph",
    "read_features", "read_labels", "write_features_bin",
    "reencode_balance", "rmat_graph", "synthetic_features", "uniform_graph", "FusedGather",
    "LayerProgram", "PassReport", "build_commnet", "build_gcn", "build_ggcn", "build_mpgcn", "evaluate_expr",
    "fuse_sag", "hoist_vertex_computation", "make_program", "matmul_rows", "optimize", "trace_udf",
    "validate_program", "vertex_form", "SAGAModel", "gcn_model", "ggcn_model", "mpgcn_model", "commnet_model", "run_train",
    "StreamingGCN", "StreamingGGCN", "HostGrid", "GGNNModel", "ggnn_model", "build_ggnn",
    "UnfusedSAGAModel", "unfused_model",
]


def __getattr__(name):
    # the executor needs torch + CUDA; import it lazily so the host-side graph store
    # and front end stay importable on a CPU-only machine
    if name in ("SAGAModel", "gcn_model", "ggcn_model", "mpgcn_model", "commnet_model", "run_train"):
        from . import engine

        return getattr(engine, name)
    if name in ("GGNNModel", "ggnn_model"):
        from . import ggnn

        return getattr(ggnn, name)
    if name in ("UnfusedSAGAModel", "unfused_model"):
        from . import stages

        return getattr(stages, name)
    if name in ("StreamingGCN", "StreamingGGCN", "HostGrid"):
        from . import stream

        return getattr(stream, name)
    raise AttributeError(name)
