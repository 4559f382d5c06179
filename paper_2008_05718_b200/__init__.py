"""B200-native partitioned betweenness centrality (drop-in for ``hybir``'s BC path)."""

from .errors import (ContractViolation, DomainError, EngineError, FormatError, HybirError,
                     InputError, ParseError)
from .graph import Graph, as_graph, from_edge_arrays, from_edges, graph_stats, load_edge_list, write_edge_list

__version__ = "0.1.0"
