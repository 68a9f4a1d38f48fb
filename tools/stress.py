"""Randomised parity stress (rare races): random graphs / sources / operator variants against the
oracle for SECONDS seconds.  python tools/stress.py [SECONDS] [SEED]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1607_05707_b200 as irgl
from oracle import oracle as O  # checker only

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
t_end = time.time() + secs
n_checks = 0
P = int(os.environ.get("STRESS_P", "1"))  # logical partitions (P > 1: BFS / SSSP only)
ctx = irgl.Context(logical_partitions=P) if P > 1 else irgl.Context()
while time.time() < t_end:
    kind = rng.integers(0, 3)
    if kind == 0:
        og = O.rmat(int(rng.integers(6, 19)), seed=int(rng.integers(1, 1000)), wseed=int(rng.integers(1, 1000)))
    elif kind == 1:
        W, H = int(rng.integers(2, 200)), int(rng.integers(2, 200))
        og = O.grid(W, H, perc_keep=float(rng.uniform(0.3, 1.0)), perc_seed=int(rng.integers(1, 1000)))
    else:
        n = int(rng.integers(2, 5000))
        m = int(rng.integers(1, 8 * n))
        og = O.from_edges(n, rng.integers(0, n, m).tolist(), rng.integers(0, n, m).tolist(),
                          w=rng.integers(1, int(rng.choice([2, 16, 256, 100000])), m).tolist())
    g = ctx.graph_from_csr(og.row_ptr, og.col, og.weight)
    relabelled = rng.random() < 0.5
    if relabelled:  # P > 1: block-diagonal degree order
        g.relabel()
    srcs = [int(s) for s in og.sources(3, seed=int(rng.integers(1, 1000)))] or [0]
    for s in srcs:
        ref_l = O.bfs(og, s)[0]
        for direction in (0, 1):  # P > 1: top-down distributed kernel or host rounds; DO host rounds
            ol = int(rng.integers(0, 2)) if (not direction or P > 1) else 1
            lv, _ = irgl.bfs(ctx, g, s, direction=direction, outline=ol)
            assert np.array_equal(lv, ref_l), ("bfs", kind, og.n, s, direction)
        ref_d = O.sssp(og, s)
        for delta, defer in ((0, -1), (0, 0), (int(rng.integers(1, 300)), 0), (0, int(rng.integers(1, 5000)))):
            ol = int(rng.integers(0, 2))
            try:
                d, _ = irgl.sssp(ctx, g, s, delta=delta, defer=defer, outline=ol)
            except irgl.IrglError as e:
                print("FAIL sssp", kind, og.n, og.m, s, delta, defer, ol, g.info.relabeled if hasattr(g.info, "relabeled") else "?",
                      int(og.weight.max()) if og.m else 0, e, flush=True)
                raise
            assert np.array_equal(d, ref_d), ("sssp", kind, og.n, s, delta, defer)
        n_checks += 6
    if P > 1:
        if not relabelled:  # relabelled partitioned graphs return BFS / SSSP results only
            lab2, _ = irgl.cc_lp(ctx, g)
            assert np.array_equal(lab2, O.cc(og)), ("cc_lp P", kind, og.n)
            n_checks += 1
        g.close()
        continue
    p = ctx.pipe(og.n)
    outs = [np.zeros(og.n, dtype=np.int32) for _ in range(2)]
    ctx.traverse_batch(irgl.SSSP, g, p, srcs, outs)
    assert np.array_equal(outs[(len(srcs) - 1) % 2], O.sssp(og, srcs[-1])), ("batch", kind, og.n)
    lab, _ = irgl.cc(ctx, g)
    assert np.array_equal(lab, O.cc(og)), ("cc", kind, og.n)
    lab2, _ = irgl.cc_lp(ctx, g, outline=int(rng.integers(0, 2)))
    assert np.array_equal(lab2, lab), ("cc_lp", kind, og.n)
    r, pst = irgl.pagerank(ctx, g)
    ref_r, it = O.pagerank(og)
    err = np.abs(r - ref_r).sum() / max(np.abs(ref_r).sum(), 1e-300)
    assert err <= 1e-6 and pst.rounds == it, ("pr", kind, og.n, err, pst.rounds, it)
    tc, _ = irgl.triangle_count(ctx, g)
    assert int(tc) == O.tc(og), ("tc", kind, og.n)
    (mw, me), _ = irgl.mst(ctx, g)
    assert (int(mw), int(me)) == O.mst(og), ("mst", kind, og.n)
    n_checks += 6
    p.close()
    g.close()
print(f"stress ok: {n_checks} checks in {secs:.0f} s", flush=True)
