"""Near-far SSSP overflow hunt on small RMAT graphs: python tools/repro_nf.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1607_05707_b200 as irgl
from oracle import oracle as O

ctx = irgl.Context()
bad = 0
for seed in range(1, 120):
    for wseed in (1, 2, 3):
        og = O.rmat(8, seed=seed, wseed=wseed)
        for relabel in (0, 1):
            g = ctx.graph_from_csr(og.row_ptr, og.col, og.weight)
            if relabel:
                g.relabel()
            for s in [int(x) for x in og.sources(3)]:
                for delta in (64, 264, 1000):
                    for ol in (1, 0):
                        msg = ""
                        try:
                            d, st = irgl.sssp(ctx, g, s, delta=delta, defer=0, outline=ol)
                            ok = np.array_equal(d, O.sssp(og, s))
                            msg = "WRONG"
                        except irgl.IrglError as e:
                            ok = False
                            msg = str(e)
                        if not ok:
                            bad += 1
                            if bad <= 6:
                                print("BAD", seed, wseed, relabel, s, delta, ol, og.n, og.m, msg, flush=True)
            g.close()
print("done, bad =", bad)
