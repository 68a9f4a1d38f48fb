import sys
sys.path.insert(0, "/root/repo")
import paper_1607_05707_b200 as irgl
ctx = irgl.Context()
g = ctx.generate_rmat(24)
outline = int(sys.argv[1])
r, st = irgl.pagerank(ctx, g, outline=outline, max_iter=2)
