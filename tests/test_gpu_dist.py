"""Two real processes through the runtime's multi-rank code path on ONE GPU: each
process is one rank owning half of the vertex range, the rounds run wl_graph_rounds_dist /
exchange_and_apply (api.cu) — local expansion, per-owner buckets, round-header AllGather,
payload all-to-all-v, owner-side min-reduce — with the exchange through the host transport
plugin (irgl_ctx_create_transport) over a torch.distributed gloo group.  NCCL refuses two ranks
on one device, so this is how the multi-process protocol runs on a 1-GPU box; with NCCL
(irgl_ctx_create_nccl) only the byte-moving primitives differ (x_allgather / x_exchange).

Results are gathered from the ranks' owned ranges and checked against the serial oracle."""
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, spec, logical, q, relabel=False, env=None):
    try:
        import torch.distributed as dist
        sys.path.insert(0, ROOT)
        os.environ.update(env or {})
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_1607_05707_b200 as irgl
        from paper_1607_05707_b200.dist import TorchTransport
        ctx = irgl.Context(transport=TorchTransport(device=0), logical_partitions=logical)
        g = ctx.generate_rmat(spec["scale"]) if spec["kind"] == "rmat" else \
            ctx.generate_grid(spec["w"], spec["h"], perc_keep=spec.get("keep", 1.0))
        if relabel:  # block-diagonal degree order (perm blocks exchanged through the transport)
            g.relabel()
        info = g.info
        out = {"n": g.n, "m": g.m, "parts": info.partitions, "lo": info.lo, "local_n": info.local_n}
        res = {}
        outlined = []
        for s in spec["sources"]:
            lv, st = irgl.bfs(ctx, g, s)
            res[("bfs", s)] = (lv, st.rounds, st.exchange_bytes)
            outlined.append(st.outlined)
            lv, st = irgl.bfs(ctx, g, s, direction=1)  # direction-optimising (bitmap exchange)
            res[("bfs-do", s)] = (lv, st.rounds, 0)
            outlined.append(st.outlined)
            for delta, defer in ((0, 0), (0, -1), (8, 0)):
                d, st = irgl.sssp(ctx, g, s, delta=delta, defer=defer)
                res[("sssp", s, delta, defer)] = (d, st.rounds, st.exchange_bytes)
                if delta == 0:
                    outlined.append(st.outlined)
        out["outlined"] = outlined
        if not relabel:
            lab, _ = irgl.cc_lp(ctx, g, outline=0)
            res[("cc_lp",)] = (lab, 0, 0)
        # each rank owns [lo, lo + local_n): keep that slice, gather on rank 0
        lo, hi = info.lo, info.lo + info.local_n
        mine = {k: (v[0][lo:hi].copy(), v[1], v[2]) for k, v in res.items()}
        allr = [None] * world
        dist.all_gather_object(allr, (lo, hi, mine))
        if rank == 0:
            full = {}
            for k in res:
                arr = np.full(g.n, -1, dtype=np.int64)
                for (l0, h0, m) in allr:
                    arr[l0:h0] = m[k][0]
                full[k] = (arr, [m[k][1] for (_, _, m) in allr], sum(m[k][2] for (_, _, m) in allr))
            q.put(("ok", out, full))
        ctx.close()
        dist.destroy_process_group()
    except Exception as e:  # surface the rank's failure to the test
        import traceback
        q.put(("err", rank, traceback.format_exc()))
        raise


def _run(spec, world=2, logical=0, relabel=False, env=None):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_rank_main, args=(r, world, port, spec, logical, q, relabel, env))
          for r in range(world)]
    for p in ps:
        p.start()
    msg = q.get(timeout=600)
    for p in ps:
        p.join(timeout=120)
    assert msg[0] == "ok", msg
    return msg[1], msg[2]


@pytest.mark.parametrize("world,logical", [(2, 0), (2, 2)])
def test_two_process_bfs_sssp_cc_rmat(oracle, world, logical):
    og = oracle.rmat(12)
    srcs = [int(s) for s in og.sources(2)]
    info, res = _run({"kind": "rmat", "scale": 12, "sources": srcs}, world, logical)
    assert info["parts"] == world * max(logical, 1) and info["m"] == og.m
    for s in srcs:
        ref, ecc = oracle.bfs(og, s)
        lv, rounds, xb = res[("bfs", s)]
        np.testing.assert_array_equal(lv, ref)
        assert set(rounds) == {ecc + 1} and xb > 0       # every rank ran ecc+1 rounds; data moved
        lv, rounds, _ = res[("bfs-do", s)]
        np.testing.assert_array_equal(lv, ref)
        assert set(rounds) == {ecc + 1}
        dref = oracle.sssp(og, s)
        for delta, defer in ((0, 0), (0, -1), (8, 0)):
            d, _, xb = res[("sssp", s, delta, defer)]
            np.testing.assert_array_equal(d, dref, err_msg=f"sssp delta={delta} defer={defer}")
    np.testing.assert_array_equal(res[("cc_lp",)][0], oracle.cc(og))


def test_two_process_percolated_grid(oracle):
    og = oracle.grid(64, 48, perc_keep=0.6)
    info, res = _run({"kind": "grid", "w": 64, "h": 48, "keep": 0.6, "sources": [0, 1500]})
    for s in (0, 1500):
        np.testing.assert_array_equal(res[("bfs", s)][0], oracle.bfs(og, s)[0])
        np.testing.assert_array_equal(res[("sssp", s, 0, 0)][0], oracle.sssp(og, s))
    np.testing.assert_array_equal(res[("cc_lp",)][0], oracle.cc(og))


def test_two_process_relabelled(oracle):
    """Block-diagonal degree order across two processes: each rank orders its own range, the
    ranks exchange their new ids through the transport, results come back in the caller's ids."""
    og = oracle.rmat(12)
    srcs = [int(s) for s in og.sources(2)]
    info, res = _run({"kind": "rmat", "scale": 12, "sources": srcs}, 2, 0, relabel=True)
    for s in srcs:
        ref, ecc = oracle.bfs(og, s)
        lv, rounds, _ = res[("bfs", s)]
        np.testing.assert_array_equal(lv, ref)
        assert set(rounds) == {ecc + 1}
        for delta, defer in ((0, 0), (0, -1), (8, 0)):
            np.testing.assert_array_equal(res[("sssp", s, delta, defer)][0], oracle.sssp(og, s))


@pytest.mark.parametrize("logical,relabel", [(0, False), (2, False), (0, True)])
def test_two_process_distributed_persistent_kernel(oracle, logical, relabel):
    # the distributed persistent kernel across processes: inboxes and rank 0's rendezvous mapped
    # with CUDA IPC.  Two ranks on one GPU take turns (time-sliced contexts), so the runtime keeps
    # host rounds for them unless forced (IRGL_DIST_OUTLINE=2); on separate GPUs it is the default.
    og = oracle.rmat(12)
    srcs = [int(s) for s in og.sources(2)]
    info, res = _run({"kind": "rmat", "scale": 12, "sources": srcs}, 2, logical, relabel=relabel,
                     env={"IRGL_DIST_OUTLINE": "2"})
    assert set(info["outlined"]) == {1}, info["outlined"]  # every BFS / DO-BFS / delta=0 SSSP outlined
    for s in srcs:
        ref, ecc = oracle.bfs(og, s)
        for key in ("bfs", "bfs-do"):
            lv, rounds, _ = res[(key, s)]
            np.testing.assert_array_equal(lv, ref)
            assert set(rounds) == {ecc + 1}
        dref = oracle.sssp(og, s)
        for delta, defer in ((0, 0), (0, -1), (8, 0)):
            np.testing.assert_array_equal(res[("sssp", s, delta, defer)][0], dref)
    if not relabel:
        np.testing.assert_array_equal(res[("cc_lp",)][0], oracle.cc(og))


def test_two_process_shared_gpu_keeps_host_rounds(oracle):
    og = oracle.rmat(12)
    srcs = [int(og.sources(1)[0])]
    info, res = _run({"kind": "rmat", "scale": 12, "sources": srcs})
    assert set(info["outlined"]) == {0}  # ranks on one GPU: no time-sliced rendezvous
    np.testing.assert_array_equal(res[("bfs", srcs[0])][0], oracle.bfs(og, srcs[0])[0])
