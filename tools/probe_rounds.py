"""Per-round overhead and near-far sanity: python tools/probe_rounds.py"""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1607_05707_b200 as irgl
from oracle import oracle as O
for bps in (0, 1, 2):
    ctx = irgl.Context(blocks_per_sm=bps)
    g = ctx.generate_grid(1024, 1024)
    for outline in (1, 0):
        lv, st = irgl.bfs(ctx, g, 0, outline=outline)
        print(f"grid1024 BFS bps={bps} outline={outline}: rounds={st.rounds} {st.device_ms:.2f} ms -> {st.device_ms*1e3/st.rounds:.2f} us/round", flush=True)
    ctx.close()
og = O.rmat(18)
ctx = irgl.Context()
g = ctx.graph_from_csr(og.row_ptr, og.col, og.weight)
s = int(og.sources(1)[0])
ref = O.sssp(og, s)
E = int(og.degrees()[ref < O.INF].sum())
for outline in (1, 0):
    for delta in (0, 2, 4, 8, 16):
        d, st = irgl.sssp(ctx, g, s, outline=outline, delta=delta)
        print(f"RMAT-18 SSSP outline={outline} delta={delta}: ok={np.array_equal(d, ref)} scans/E={st.edges/E:.3f} rounds={st.rounds} popped={st.popped} {st.device_ms:.2f} ms", flush=True)
