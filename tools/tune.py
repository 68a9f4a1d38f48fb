"""SSSP/BFS tuning sweep on device RMAT: python tools/tune.py [scale]"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1607_05707_b200 as irgl
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
def run(ctx, g, srcs, op, **kw):
    p = ctx.pipe(g.n); tms, kms, ed, rnd = 0, 0, 0, 0
    for s in srcs:
        p.init_scalars([s]); st = ctx.iterate(op, g, p, **kw)
        tms += st.device_ms; kms += st.kernel_ms; ed += st.edges; rnd += st.rounds
    return tms / len(srcs), kms / len(srcs), ed / len(srcs), rnd / len(srcs)
CFGS = [dict(), dict(cta_threshold=256), dict(cta_threshold=512, chunk_edges=1024)] if len(sys.argv) < 3 else [dict()]
for cfg in CFGS:
    ctx = irgl.Context(**cfg)
    g = ctx.generate_rmat(scale)
    rp = np.zeros(g.n + 1, dtype=np.int64)
    ctx._lib.irgl_graph_download(g.handle, rp.ctypes.data_as(C.POINTER(C.c_int64)), None, None)
    srcs = bench.pick_sources(g.n, lambda x: int(rp[x + 1] - rp[x]), count=4)
    E = run(ctx, g, srcs, irgl.BFS)[2]
    for outline in (1, 0):
        t, k, e, r = run(ctx, g, srcs, irgl.BFS, outline=outline)
        print(f"{cfg} BFS outline={outline}: {t:.3f} ms (kernel {k:.3f}) GTEPS={E/2/t/1e6:.1f} rounds={r}", flush=True)
        if outline:
            t, k, e, r = run(ctx, g, srcs, irgl.BFS, outline=1, direction=1)
            print(f"{cfg} BFS-DO outline=1: {t:.3f} ms (kernel {k:.3f}) GTEPS={E/2/t/1e6:.1f} rounds={r} scanned/E={e/E:.3f}", flush=True)
        for delta in ([0, 2, 4, 8, 16, 32, 64] if cfg == {} else [8]):
            t, k, e, r = run(ctx, g, srcs, irgl.SSSP, outline=outline, delta=delta)
            print(f"{cfg} SSSP outline={outline} delta={delta}: {t:.3f} ms (kernel {k:.3f}) GTEPS={E/2/t/1e6:.1f} scans/E={e/E:.2f} rounds={r}", flush=True)
    ctx.close()
