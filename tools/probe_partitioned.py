"""Host-orchestrated multi-partition path on one GPU (P logical partitions, NCCL 1-rank transport
or loopback): per-traversal time and rounds, to size the per-round exchange overhead.
python tools/probe_partitioned.py [scale] [P] [nccl 0|1] [relabel 0|1] [outline -1|0|1]"""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1607_05707_b200 as irgl

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
P = int(sys.argv[2]) if len(sys.argv) > 2 else 2
use_nccl = int(sys.argv[3]) if len(sys.argv) > 3 else 1
relabel = int(sys.argv[4]) if len(sys.argv) > 4 else 0
outline = int(sys.argv[5]) if len(sys.argv) > 5 else -1
kw = dict(logical_partitions=P, outline=outline,
          dense_div=int(os.environ.get("PROBE_DENSE_DIV", "0")))  # -1: no dense rounds
if use_nccl:
    kw["nccl"] = (0, 0, 1, irgl.nccl_unique_id())
ctx = irgl.Context(**kw)
g = ctx.generate_rmat(scale)
rp, _, _ = g.download()
srcs = bench.pick_sources(g.n, lambda x: int(rp[x + 1] - rp[x]), count=4)
if relabel:
    g.relabel()
p = ctx.pipe(max(g.info.local_n, 1))
for op, name, kw2 in ((irgl.BFS, "bfs", {}), (irgl.BFS, "bfs-do", {"direction": 1}), (irgl.SSSP, "sssp", {})):
    for s in srcs[:1]:
        p.init_scalars([s]); ctx.iterate(op, g, p, **kw2)
    t = []; r = []; e = []
    for s in srcs:
        p.init_scalars([s])
        t0 = time.perf_counter(); st = ctx.iterate(op, g, p, **kw2); t.append(time.perf_counter() - t0)
        r.append(st.rounds); e.append(st.edges)
    print(f"RMAT-{scale} P={P} nccl={use_nccl} relabel={relabel} outline={outline} {name}: {1e3*np.mean(t):.2f} ms/traversal, rounds {np.mean(r):.1f}, "
          f"{1e6*np.mean(t)/np.mean(r):.0f} us/round, kernel {st.kernel_ms:.2f} ms, edges {np.mean(e)/1e6:.1f} M "
          f"({np.mean(e)/np.mean(t)/1e9:.1f} G edges/s)", flush=True)
ctx.close()
