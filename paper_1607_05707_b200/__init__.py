"""paper_1607_05707_b200 — B200-native runtime for IrGL's worklist graph hot path.

The compute path is libirgl_rt.so (hand-written sm_100a CUDA behind the C-ABI in
include/irgl/rt.h); this package is its host-side mirror of the IrGL operator API.  Importing the
package loads the shared library and fails loudly if it has not been built.
"""
from .runtime import (  # noqa: F401
    BFS, CC, CC_LP, MST, TEST_ATOMIC, TEST_ATOMIC_ELSE, TEST_EXCLUSIVE, COMB_AND, COMB_OR, COND_NONE, COND_UNTIL, COND_WHILE, INF, MAP_BLOCKED,
    MAP_CONSECUTIVE, PR, RED_ALL, RED_ANY, RED_NONE, SSSP, TC, TEST_COUNTDOWN, TEST_FORALL_MAP,
    TEST_NOPUSH, TEST_PUSHPOP, TEST_REDUCE, TEST_RESPAWN_ODD, TEST_RETRY_ODD, WL_IN, WL_OUT, WL_RETRY,
    BLOCK_ELASTIC, BLOCK_FIXED, BLOCK_SHRINKABLE, EXPORTS, LIB_PATH, Context, Graph, IrglError,
    Module, Pipe, Stats, bfs, cc, cc_lp, launch_count, load_library, mst, nccl_unique_id, pagerank, sssp, t_control,
    triangle_count, STAGE_INVOKE, STAGE_ITERATE, WHEN_ALWAYS, WHEN_PREV_TRUE, WHEN_PREV_FALSE,
)

load_library()
