"""B200-native partitioned betweenness centrality.

Drop-in for the BC hot path of the reference package ``hybir``
(reference pkg/src/hybir/__init__.py:3-48): same public names for the graph
container, partition / border types, ``RunConfig`` / ``RunResult`` and the
entry point ``run_bc``.  All arithmetic runs in hand-written sm_100a CUDA
behind the C ABI of ``include/bc_b200.h``; importing this package does not
need a GPU, calling ``run_bc`` does (there is no CPU fallback).
"""

from .errors import (ContractViolation, DomainError, EngineError, FormatError, HybirError,
                     InputError, ParseError)
from .graph import (Graph, as_graph, from_edge_arrays, from_edges, graph_stats, load_dimacs_gr,
                    load_edge_list, write_edge_list)
from .partition import (BorderSet, Partition, block_partition, greedy_bipartition, grow_partition,
                        identify_borders, import_partition, mincut_partition, refine_partition,
                        single_partition, strip_partition)
from .engine import (CommTotals, RunConfig, RunResult, border_table_bytes, build_report, choose_mode,
                     pipeline_sources, run_bc, select_sources)

__version__ = "0.1.0"
