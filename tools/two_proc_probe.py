"""Two ranks (processes) on one GPU through the multi-rank path, host transport over gloo: which
orchestration each Iterate took (distributed persistent kernel or host rounds) and its time.
python tools/two_proc_probe.py [kind rmat|grid] [scale or width] [outline -1|0]"""
import os
import socket
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(rank, port, kind, size, outline):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    import paper_1607_05707_b200 as irgl
    from paper_1607_05707_b200.dist import TorchTransport
    ctx = irgl.Context(transport=TorchTransport(device=0))
    g = ctx.generate_rmat(size) if kind == "rmat" else ctx.generate_grid(size, size, perc_keep=0.6)
    for name, fn in (("bfs", lambda s: irgl.bfs(ctx, g, s, outline=outline)),
                     ("sssp", lambda s: irgl.sssp(ctx, g, s, outline=outline))):
        for s in (0, 1, 0):
            t0 = time.perf_counter()
            _, st = fn(s)
            dt = time.perf_counter() - t0
            if rank == 0:
                print(f"{kind}-{size} {name} src={s}: {dt * 1e3:.1f} ms rounds={st.rounds} "
                      f"outlined={st.outlined} launches={st.launches} remote={st.remote_updates}", flush=True)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    import multiprocessing as mp
    kind = sys.argv[1] if len(sys.argv) > 1 else "rmat"
    size = int(sys.argv[2]) if len(sys.argv) > 2 else 14
    outline = int(sys.argv[3]) if len(sys.argv) > 3 else -1
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    c = mp.get_context("spawn")
    ps = [c.Process(target=main, args=(r, port, kind, size, outline)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join()
