"""SSSP deferral-budget sweep on device RMAT: python tools/defer_sweep.py [scale] [K ...]
Prints device ms / GTEPS / scans per reached edge / rounds per K (delta = 0, outlined unless
OUTLINE=0)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1607_05707_b200 as irgl

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
Ks = [int(k) for k in sys.argv[2:]] or [0, 256, 512, 1024, 2048, 4096, 8192, 16384, 65536]
outline = int(os.environ.get("OUTLINE", "1"))
nsrc = int(os.environ.get("NSRC", "8"))
import json
ctx = irgl.Context(**json.loads(os.environ.get("CTX", "{}")))
g = ctx.generate_rmat(scale)
rp = np.zeros(g.n + 1, dtype=np.int64)
ctx._lib.irgl_graph_download(g.handle, rp.ctypes.data_as(C.POINTER(C.c_int64)), None, None)
srcs = bench.pick_sources(g.n, lambda x: int(rp[x + 1] - rp[x]), count=nsrc)
if os.environ.get("RELABEL", "0") == "1":
    g.relabel()
p = ctx.pipe(g.n)
E = 0
for s in srcs:
    p.init_scalars([s])
    E += ctx.iterate(irgl.BFS, g, p).edges
E /= len(srcs)
tb = 0
for s in srcs:
    p.init_scalars([s])
    tb += ctx.iterate(irgl.BFS, g, p).device_ms
print(f"{os.environ.get('CTX', '')} RMAT-{scale} BFS: {tb/len(srcs):.3f} ms GTEPS={E/2/(tb/len(srcs))/1e6:.1f}", flush=True)
ref = None
for K in Ks:
    for s in srcs[:2]:  # warm
        p.init_scalars([s]); ctx.iterate(irgl.SSSP, g, p, outline=outline, delta=0, defer=K)
    t = k = e = r = 0
    for s in srcs:
        p.init_scalars([s])
        st = ctx.iterate(irgl.SSSP, g, p, outline=outline, delta=0, defer=K)
        t += st.device_ms; k += st.kernel_ms; e += st.edges; r += st.rounds
    n = len(srcs)
    p.init_scalars([srcs[0]]); ctx.iterate(irgl.SSSP, g, p, outline=outline, delta=0, defer=K)
    d = ctx.read_result(irgl.SSSP, g)
    if ref is None:
        ref = d
    same = bool(np.array_equal(d, ref))
    print(f"RMAT-{scale} SSSP outline={outline} defer={K}: {t/n:.3f} ms (kernel {k/n:.3f}) "
          f"GTEPS={E/2/(t/n)/1e6:.1f} scans/E={e/n/E:.2f} rounds={r/n:.1f} same_as_K0={same}", flush=True)
ctx.close()
