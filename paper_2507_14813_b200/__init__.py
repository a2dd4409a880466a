"""mayura-b200: B200-native (sm_100a) MG-Tree temporal motif co-mining.

Paper: "Mayura: Exploiting Similarities in Motifs for Temporal Co-Mining"
(arXiv 2507.14813).  The hot path -- one depth-first co-mining search per root
temporal edge, walking the MG-Tree (Algorithm 3) -- runs in libmayura.so's CUDA
kernels; this package is the ctypes binding of its C ABI (include/mayura.h) plus
the multi-GPU driver (``parallel``).
"""
from .mayura import (Graph, MGTree, MayuraError, comine, comine_stats, mine_independent,  # noqa: F401
                     mayura_build_mgtree, mayura_comine, mayura_comine_ex, mayura_comine_stats, mayura_free_graph,
                     mayura_free_mgtree, mayura_graph_export, mayura_graph_export_succ, mayura_graph_info, mayura_last_error,
                     mayura_load_graph, mayura_mgtree_dump, mayura_mgtree_info, mayura_mine_independent,
                     mayura_partition_roots, mayura_version, mayura_launch_count, STATS_FIELDS,
                     mayura_enumerate, enumerate_matches, split_tuples, mayura_comine_heuristic, mayura_kernel_form,
                     mayura_enum_form)
