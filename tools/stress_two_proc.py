"""Randomised parity stress of the multi-process path: two ranks (processes) on one GPU through the
host transport over gloo, every Iterate in the distributed persistent kernel across the processes
(IRGL_DIST_OUTLINE=2; inboxes and the rendezvous mapped with CUDA IPC) or in host rounds (=0), on
random RMAT graphs / grids / sources, against the oracle for SECONDS seconds.
python tools/stress_two_proc.py [SECONDS] [SEED] [MODE 2|0]"""
import os
import socket
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(rank, port, secs, seed, mode):
    sys.path.insert(0, ROOT)
    os.environ["IRGL_DIST_OUTLINE"] = mode
    import numpy as np
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    import paper_1607_05707_b200 as irgl
    from paper_1607_05707_b200.dist import TorchTransport
    from oracle import oracle as O  # checker only
    rng = np.random.default_rng(seed)  # same stream on both ranks: same graphs and sources
    ctx = irgl.Context(transport=TorchTransport(device=0))
    t_end = time.time() + secs
    checks = 0
    while True:
        go = [time.time() < t_end]
        dist.broadcast_object_list(go, src=0)  # both ranks stop together
        if not go[0]:
            break
        if rng.random() < 0.7:
            sc, gs, ws = int(rng.integers(6, 15)), int(rng.integers(1, 1000)), int(rng.integers(1, 1000))
            og = O.rmat(sc, seed=gs, wseed=ws)
            g = ctx.generate_rmat(sc, seed=gs, wseed=ws)
        else:
            W, H = int(rng.integers(2, 80)), int(rng.integers(2, 80))
            keep, ps = float(rng.uniform(0.4, 1.0)), int(rng.integers(1, 1000))
            og = O.grid(W, H, perc_keep=keep, perc_seed=ps)
            g = ctx.generate_grid(W, H, perc_keep=keep, perc_seed=ps)
        relabel = rng.random() < 0.5
        if relabel:
            g.relabel()
        info = g.info
        lo, hi = info.lo, info.lo + info.local_n
        srcs = [int(s) for s in og.sources(2, seed=int(rng.integers(1, 1000)))] or [0]
        for s in srcs:
            outs = []
            lv, _ = irgl.bfs(ctx, g, s)
            outs.append(("bfs", lv[lo:hi].copy(), O.bfs(og, s)[0]))
            lv, _ = irgl.bfs(ctx, g, s, direction=1)
            outs.append(("bfs-do", lv[lo:hi].copy(), O.bfs(og, s)[0]))
            defer = int(rng.choice([0, -1, 64, 4096]))
            d, _ = irgl.sssp(ctx, g, s, defer=defer)
            outs.append((f"sssp defer={defer}", d[lo:hi].copy(), O.sssp(og, s)))
            for name, mine, ref in outs:
                allp = [None, None]
                dist.all_gather_object(allp, (lo, hi, mine))
                if rank == 0:
                    full = np.full(og.n, -1, dtype=np.int64)
                    for (l0, h0, m) in allp:
                        full[l0:h0] = m
                    assert np.array_equal(full, ref), (name, og.n, og.m, s, relabel)
                checks += 1
        g.close()
    if rank == 0:
        print(f"two-process stress ok (IRGL_DIST_OUTLINE={mode}): {checks} checks in {secs:.0f} s", flush=True)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    import multiprocessing as mp
    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 60
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    mode = sys.argv[3] if len(sys.argv) > 3 else "2"
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    c = mp.get_context("spawn")
    ps = [c.Process(target=main, args=(r, port, secs, seed, mode)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join()
    sys.exit(max(p.exitcode for p in ps))
