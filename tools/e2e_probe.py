import os, sys, time, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1607_05707_b200 as irgl, bench
ctx = irgl.Context()
g = ctx.generate_rmat(22)
rp = np.zeros(g.n + 1, dtype=np.int64)
ctx._lib.irgl_graph_download(g.handle, rp.ctypes.data_as(C.POINTER(C.c_int64)), None, None)
srcs = bench.pick_sources(g.n, lambda x: int(rp[x + 1] - rp[x]), count=16)
if os.environ.get("RELABEL", "1") == "1":
    g.relabel()
p = ctx.pipe(g.n)
bufs = [torch.empty(g.n, dtype=torch.int32, pin_memory=True).numpy() for _ in range(2)]
def run(mode, K=32):
    for i in range(3):
        p.init_scalars([srcs[i]]); ctx.iterate(irgl.SSSP, g, p)
    ctx.sync()
    t0 = time.perf_counter()
    km = 0.0
    for i in range(K):
        if mode != "copy":
            p.init_scalars([srcs[i % 16]]); st = ctx.iterate(irgl.SSSP, g, p); km += st.kernel_ms
        if mode in ("async", "copy"):
            ctx.read_result_async(irgl.SSSP, g, bufs[i % 2])
        if mode == "sync":
            ctx.read_result_into(irgl.SSSP, g, bufs[i % 2])
    ctx.results_wait(); ctx.sync()
    return (time.perf_counter() - t0) / K * 1e3, km / K
for m in ("iter", "sync", "async", "copy", "iter", "async", "async", "copy"):
    w, k = run(m)
    print(m, f"{w:.3f} ms/step wall, persistent kernel {k:.3f} ms", flush=True)
