"""World-size-2 CPU tests (gloo) of the multi-GPU path's host logic.

1. The 1D vertex-partition exchange protocol the runtime implements in api.cu
   (wl_graph_rounds_dist) and expand.cu (owner routing in wpush<DIST>), restated over
   torch.distributed/gloo: ghost-label send filter, per-owner buckets deduped per round, round
   headers {send counts, |in|} all-gathered (payload sizes + termination in one collective),
   payload all-to-all, owner-side min-reduce.  Checked against the serial oracle on RMAT and grid
   graphs.
2. bench.py's own multi-process plumbing (torchrun launch, rank-0-only reference arm).
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INF = 2147483647


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _partitioned_traversal(rank, world, port, op, graph_spec, src, out_q):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    og = O.rmat(graph_spec[1]) if graph_spec[0] == "rmat" else O.grid(*graph_spec[1:])
    n = og.n
    ps = (n + world - 1) // world          # part_size: owner(v) = v // ps
    lo, hi = rank * ps, min((rank + 1) * ps, n)
    rp, col, w = og.row_ptr, og.col, og.weight
    lab = np.full(n, INF, dtype=np.int64)  # full-size ghost array (send filter)
    stamp = np.zeros(n, dtype=np.int64)
    wl = [src] if lo <= src < hi else []
    if wl:
        lab[src] = 0
    level, rnd = 1, 0
    while True:
        out, buckets = [], [[] for _ in range(world)]
        for u in wl:                        # expand: relax on the ghost array, route by owner
            for e in range(rp[u - 0], rp[u + 1]):
                v = int(col[e])
                nd = level if op == "bfs" else int(lab[u] + w[e])
                better = lab[v] == INF if op == "bfs" else nd < lab[v]
                if better:
                    lab[v] = nd
                    if stamp[v] != rnd + 1:  # per-round push dedupe
                        stamp[v] = rnd + 1
                        (out if v // ps == rank else buckets[v // ps]).append(v)
        # round header {send counts [world], |in|} all-gathered: the sizes of the payload
        # exchange and, folded in, the termination test (wl_graph_rounds_dist: an all-empty round
        # did no work and ends the Iterate)
        hdr = torch.tensor([len(b) for b in buckets] + [len(wl)], dtype=torch.int64)
        hdrs = [torch.zeros_like(hdr) for _ in range(world)]
        dist.all_gather(hdrs, hdr)
        if sum(int(h[world]) for h in hdrs) == 0:
            break
        rnd += 1
        # payload: ids, and for SSSP the ghost value packed after the expansion
        payload = [[(v, int(lab[v])) for v in b] for b in buckets]
        recv = [None] * world
        dist.all_gather_object(recv, payload)
        for p in range(world):              # owner-side min-reduce
            if p == rank:
                continue
            assert len(recv[p][rank]) == int(hdrs[p][rank])
            for v, val in recv[p][rank]:
                nd = level if op == "bfs" else val
                if (op == "bfs" and lab[v] == INF) or (op != "bfs" and nd < lab[v]):
                    lab[v] = nd
                    if stamp[v] != rnd:
                        stamp[v] = rnd
                        out.append(v)
        wl = out
        level += 1
    owned = lab[lo:hi].copy()
    gathered = [None] * world
    dist.all_gather_object(gathered, (lo, owned, rnd))
    if rank == 0:
        out_q.put(gathered)
    dist.destroy_process_group()


@pytest.mark.parametrize("op,spec", [("bfs", ("rmat", 9)), ("sssp", ("rmat", 9)),
                                     ("bfs", ("grid", 12, 9)), ("sssp", ("grid", 12, 9))])
def test_partitioned_protocol_world2(oracle, op, spec):
    import torch.multiprocessing as mp
    og = oracle.rmat(spec[1]) if spec[0] == "rmat" else oracle.grid(*spec[1:])
    src = int(og.sources(1)[0])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_partitioned_traversal, args=(r, 2, port, op, spec, src, q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = np.empty(og.n, dtype=np.int64)
    for lo, owned, rnd in res:
        full[lo:lo + len(owned)] = owned
    if op == "bfs":
        ref, ecc = oracle.bfs(og, src)
        assert res[0][2] == ecc + 1  # rounds = invocations = ecc+1 (App. B1)
    else:
        ref = oracle.sssp(og, src)
    np.testing.assert_array_equal(full, ref)


def test_bench_reference_arm_torchrun_world2():
    """bench.py under torchrun (2 ranks, gloo): rank 0 alone prints the reference line."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "2", "--warmup", "3", "--scale", "12"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"
