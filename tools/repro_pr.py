"""PageRank on small random grids vs the oracle: python tools/repro_pr.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1607_05707_b200 as irgl
from oracle import oracle as O

ctx = irgl.Context()
rng = np.random.default_rng(9)
worst = []
for t in range(400):
    W, H = int(rng.integers(2, 40)), int(rng.integers(2, 40))
    og = O.grid(W, H, perc_keep=float(rng.uniform(0.3, 1.0)), perc_seed=int(rng.integers(1, 1000)))
    g = ctx.graph_from_csr(og.row_ptr, og.col, og.weight)
    rl = t % 2
    if rl:
        g.relabel()
    for outline in (1, 0):
        r, st = irgl.pagerank(ctx, g, outline=outline)
        ref, it = O.pagerank(og)
        err = np.abs(r - ref).sum() / max(np.abs(ref).sum(), 1e-300)
        if err > 1e-6:
            worst.append((err, W, H, og.n, og.m, rl, outline, st.rounds, it, float(np.abs(r - ref).max())))
    g.close()
worst.sort(reverse=True)
print(len(worst), "over 1e-6")
for w in worst[:8]:
    print(w)
