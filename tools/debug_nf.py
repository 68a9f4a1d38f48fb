import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1607_05707_b200 as irgl
from oracle import oracle as O
for scale in (13, 16):
    og = O.rmat(scale)
    srcs = [int(s) for s in og.sources(3)]
    refs = [O.sssp(og, s) for s in srcs]
    for cfg in [dict(), dict(warp_threshold=1, cta_threshold=1, chunk_edges=5), dict(cta_threshold=1, chunk_edges=64), dict(warp_threshold=1000000, cta_threshold=1000000)]:
        c = irgl.Context(**cfg)
        g = c.graph_from_csr(og.row_ptr, og.col, og.weight)
        for outline in (0, 1):
            for delta in (0, 4, 8, 16):
                bad = 0
                for s, ref in zip(srcs, refs):
                    d, st = irgl.sssp(c, g, s, outline=outline, delta=delta)
                    bad += int((d != ref).sum())
                print(f"s{scale} {cfg} outline={outline} delta={delta}: mismatches={bad}", flush=True)
        c.close()
