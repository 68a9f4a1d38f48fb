"""High-diameter probe (configs[2] shape): BFS and CC-LP on the 4096^2 grid, outlined; mean
kernel ms of 2 runs after a warm-up.  python tools/grid_probe.py [W]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1607_05707_b200 as irgl

W = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
lib = os.path.basename(os.environ.get("IRGL_LIB", "default"))
with irgl.Context() as c:
    g = c.generate_grid(W, W)
    p = c.pipe(g.n)
    t = []
    for rep in range(3):
        lv, st = irgl.bfs(c, g, 0, pipe=p, outline=1)
        if rep:
            t.append(st.kernel_ms)
    r = st.rounds
    t2 = []
    gc = c.generate_grid(W, W, cut_period=512)
    for rep in range(2):
        lab, st2 = irgl.cc_lp(c, gc, outline=1)
        if rep:
            t2.append(st2.kernel_ms)
    print(f"{lib} grid {W}^2: BFS {sum(t)/len(t):.2f} ms ({r} rounds, {1e3*sum(t)/len(t)/r:.2f} us/round); "
          f"CC-LP {sum(t2)/len(t2):.1f} ms ({st2.rounds} rounds)", flush=True)
