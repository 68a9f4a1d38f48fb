"""Fraction of directed edges whose endpoint is among the X highest-degree vertices (degree-ordered
ids: endpoint id < X), RMAT-SCALE.  Sizes a per-CTA shared-memory snapshot of hub state.
python tools/hub_coverage.py [scale]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1607_05707_b200 as irgl

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
ctx = irgl.Context()
g = ctx.generate_rmat(scale)
g.relabel()
rp, col, _ = g.download()
m = len(col)
for X in (4096, 10240, 16384, 32768, 65536, 131072, 262144, 524288, 1 << 20):
    print(f"RMAT-{scale}: endpoints with id < {X:>8d}: {np.count_nonzero(col < X) / m:.3f} of {m} edges", flush=True)
