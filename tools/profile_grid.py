"""One outlined traversal of a W x W grid (latency-bound: one small round per diameter step) for
ncu: python tools/profile_grid.py [bfs|sssp] [W]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1607_05707_b200 as irgl
op = irgl.SSSP if (sys.argv[1] if len(sys.argv) > 1 else "bfs") == "sssp" else irgl.BFS
W = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
ctx = irgl.Context(outline=1)
g = ctx.generate_grid(W, W)
p = ctx.pipe(g.n)
for _ in range(2):
    p.init_scalars([0])
    st = ctx.iterate(op, g, p)
print(f"grid {W}x{W}: rounds={st.rounds} kernel_ms={st.kernel_ms:.3f} us/round={1e3*st.kernel_ms/st.rounds:.2f}")
