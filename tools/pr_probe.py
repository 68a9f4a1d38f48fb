"""PageRank sweep timing probe: outlined (persistent) vs host loop, original vs degree-ordered ids.
usage: python tools/pr_probe.py SCALE [BPS ...]   (BPS: Context(blocks_per_sm=...), 0 = occupancy)"""
import sys
sys.path.insert(0, "/root/repo")
import paper_1607_05707_b200 as irgl

scale = int(sys.argv[1])
for bps in [int(x) for x in sys.argv[2:]] or [0]:
    for rl in (0, 1):
        ctx = irgl.Context(blocks_per_sm=bps)
        g = ctx.generate_rmat(scale)
        if rl:
            g.relabel()
        for outline in (1, 0):
            r, st = irgl.pagerank(ctx, g, outline=outline)
            r, st = irgl.pagerank(ctx, g, outline=outline)
            print(f"bps={bps} relabel={rl} outline={outline}: {st.rounds} iters, "
                  f"device {st.device_ms / st.rounds:.3f} ms/iter, sum {r.sum():.12f}", flush=True)
        g.close()
        ctx.close()
