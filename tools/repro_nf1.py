import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_1607_05707_b200 as irgl
from oracle import oracle as O
ctx = irgl.Context()
og = O.rmat(8, seed=3, wseed=3)
g = ctx.graph_from_csr(og.row_ptr, og.col, og.weight)
seq = [(int(s), delta, ol) for s in og.sources(3) for delta in (64, 264, 1000) for ol in (1, 0)]
print(seq)
for s, delta, ol in seq:
    try:
        d, st = irgl.sssp(ctx, g, s, delta=delta, defer=0, outline=ol)
        print(s, delta, ol, "ok" if np.array_equal(d, O.sssp(og, s)) else "WRONG", st.rounds)
    except irgl.IrglError as e:
        print(s, delta, ol, "ERR", e)
