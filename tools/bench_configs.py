"""Secondary measurements for every BASELINE.json config (bench.py measures the headline one).
python tools/bench_configs.py > profiles/<round>_configs.jsonl   (one JSON object per line)

  - BFS (top-down and direction-optimising) / SSSP on RMAT-24 (north-star 1-GPU target), 4 sources
  - PageRank on RMAT-24 (configs[3]), tol 1e-6, <= 100 iterations, outlined, both id orders
  - CC on the 4096^2 grid cut into 8 stripes (known answer: labels k*2^21) and its p=0.5
    percolation; TC on the triangulated 4096^2 grid (known answer 2*4095^2)
  - BFS on the 4096^2 grid from a corner: 8191 rounds, outlined vs host-orchestrated
Algorithmic bytes per SURVEY §8d; peak = MEASURED_PEAKS.json hbm_gbs."""
import ctypes as C, json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import bench
import paper_1607_05707_b200 as irgl

PEAK, _ = bench.load_peaks()


def emit(d):
    print(json.dumps(d), flush=True)


def rowptr(ctx, g):
    rp = np.zeros(g.n + 1, dtype=np.int64)
    ctx._lib.irgl_graph_download(g.handle, rp.ctypes.data_as(C.POINTER(C.c_int64)), None, None)
    return rp


def rmat_traversals(ctx, scale, nsrc=4, relabel=False):
    g = ctx.generate_rmat(scale)
    rp = rowptr(ctx, g)
    srcs = bench.pick_sources(g.n, lambda x: int(rp[x + 1] - rp[x]), count=nsrc)
    tag = ""
    if relabel:
        t0 = time.time()
        g.relabel()
        tag = f" (degree-ordered ids, relabel {time.time() - t0:.2f} s untimed)"
    p = ctx.pipe(g.n)
    for op, name, kw in ((irgl.BFS, "bfs", {}), (irgl.BFS, "bfs-do", {"direction": 1}),
                         (irgl.SSSP, "sssp", {})):
        tms = kms = E = V = X = 0.0
        rounds = []
        for s in srcs:
            p.init_scalars([s]); b = ctx.iterate(irgl.BFS, g, p)
            p.init_scalars([s]); ctx.iterate(op, g, p, **kw)  # warm
            p.init_scalars([s]); st = ctx.iterate(op, g, p, **kw)
            tms += st.device_ms; kms += st.kernel_ms; E += b.edges; V += b.popped; X += st.edges
            rounds.append(st.rounds)
        # direction-optimising BFS: bytes of the edges it actually examined;
        # GTEPS keeps the Graph500 convention (edges of the reached component)
        byts = bench.algorithmic_bytes(name[:3] if name != "sssp" else name, V, X if kw else E)
        row = {"config": f"{name.upper()} RMAT-{scale}{tag}", "n": g.n, "m": g.m, "sources": nsrc,
               "GTEPS": round(E / 2 / (tms * 1e-3) / 1e9, 2), "ms_per_traversal": round(tms / nsrc, 3),
               "rounds": rounds, "roofline_frac": round(byts / (kms * 1e-3) / 1e9 / PEAK, 4),
               "achieved_GBps": round(byts / (kms * 1e-3) / 1e9, 1)}
        if kw:
            row["edges_examined_frac"] = round(X / E, 4)
        emit(row)
    return g


def pagerank(ctx, g, scale, tag=""):
    irgl.pagerank(ctx, g, outline=1)  # first call builds the hub chunk table
    r, st = irgl.pagerank(ctx, g, outline=1)
    it = st.rounds
    byts = (12 * g.m + 36 * g.n) * it
    emit({"config": f"PR RMAT-{scale}{tag}", "iterations": it, "ms_total": round(st.kernel_ms, 3),
          "ms_per_iter": round(st.kernel_ms / it, 4), "sum_rank": float(r.sum()),
          "achieved_GBps": round(byts / (st.kernel_ms * 1e-3) / 1e9, 1),
          "roofline_frac": round(byts / (st.kernel_ms * 1e-3) / 1e9 / PEAK, 4),
          "edges_per_s": round(g.m * it / (st.kernel_ms * 1e-3), 1)})


def grids(ctx):
    W = H = 4096
    g = ctx.generate_grid(W, H, cut_period=512)
    irgl.cc(ctx, g)  # first call allocates the per-graph label state
    lab, st = irgl.cc(ctx, g)
    ok = sorted(set(lab[::4097].tolist())) == [k * 512 * W for k in range(8)] and \
        len(np.unique(lab)) == 8
    emit({"config": "CC cut grid 4096^2 (8 stripes)", "n": g.n, "m": g.m, "rounds": st.rounds,
          "ms": round(st.device_ms, 3), "known_answer_ok": bool(ok),
          "edges_per_s": round(g.m * st.rounds / (st.device_ms * 1e-3), 1)})
    # CC as data-driven label propagation: ~diameter rounds on the cut grid, the
    # iteration-outlining showcase of configs[2]
    for outline in (1, 0):
        irgl.cc_lp(ctx, g, outline=outline)
        lab2, st = irgl.cc_lp(ctx, g, outline=outline)
        emit({"config": f"CC-LP cut grid 4096^2, outline={outline}", "rounds": st.rounds,
              "ms": round(st.device_ms, 3), "us_per_round": round(st.device_ms * 1e3 / st.rounds, 2),
              "same_labels_as_hooking": bool(np.array_equal(lab2, lab))})
    g.close()
    g = ctx.generate_grid(W, H, perc_keep=0.5, perc_seed=5)
    irgl.cc(ctx, g)
    lab, st = irgl.cc(ctx, g)
    emit({"config": "CC percolated grid 4096^2 p=0.5", "n": g.n, "m": g.m, "rounds": st.rounds,
          "ms": round(st.device_ms, 3), "components": int(len(np.unique(lab)))})
    g.close()
    g = ctx.generate_grid(W, H, diag=True)
    t0 = time.time()
    c, st = irgl.triangle_count(ctx, g)
    emit({"config": "TC triangulated grid 4096^2", "n": g.n, "m": g.m, "triangles": c,
          "known_answer_ok": c == 2 * (W - 1) * (H - 1),
          "ms_incl_orientation": round(st.device_ms, 3), "wall_ms_first_call": round((time.time() - t0) * 1e3, 3)})
    c2, st2 = irgl.triangle_count(ctx, g)
    emit({"config": "TC triangulated grid 4096^2 (oriented CSR cached)", "ms": round(st2.device_ms, 3) if st2.device_ms else None})
    g.close()
    g = ctx.generate_grid(W, H)
    for outline in (1, 0):
        lv, st = irgl.bfs(ctx, g, 0, outline=outline)
        emit({"config": f"BFS grid 4096^2 from corner, outline={outline}", "rounds": st.rounds,
              "ms": round(st.device_ms, 3), "us_per_round": round(st.device_ms * 1e3 / st.rounds, 2),
              "known_answer_ok": bool(lv[-1] == (W - 1) + (H - 1))})
    g.close()


def main():
    ctx = irgl.Context()
    scale = int(os.environ.get("IRGL_CFG_SCALE", "24"))
    g = rmat_traversals(ctx, scale)
    pagerank(ctx, g, scale)
    g.close()
    g = rmat_traversals(ctx, scale, relabel=True)
    pagerank(ctx, g, scale, " (degree-ordered ids)")
    g.close()
    grids(ctx)
    ctx.close()


if __name__ == "__main__":
    main()
