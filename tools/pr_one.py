"""One PageRank run for profilers: python tools/pr_one.py OUTLINE [SCALE] [RELABEL] [MAX_ITER]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1607_05707_b200 as irgl

outline = int(sys.argv[1])
scale = int(sys.argv[2]) if len(sys.argv) > 2 else 24
ctx = irgl.Context()
g = ctx.generate_rmat(scale)
if len(sys.argv) > 3 and int(sys.argv[3]):
    g.relabel()
r, st = irgl.pagerank(ctx, g, outline=outline, max_iter=int(sys.argv[4]) if len(sys.argv) > 4 else 2)
print(f"iters={st.rounds} device_ms={st.device_ms:.3f}")
