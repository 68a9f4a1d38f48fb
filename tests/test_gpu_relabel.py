"""Degree-ordered relabelling (irgl_graph_relabel): a data-layout change that must be invisible
through the API — every operator's result, worklist reads and asynchronous reads are in the
caller's vertex ids and equal the oracle's; CC labels stay the smallest ORIGINAL id."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _upload(ctx, og):
    return ctx.graph_from_csr(og.row_ptr, og.col, og.weight)


@pytest.mark.parametrize("gen", ["rmat", "grid"])
def test_relabelled_results_equal_oracle(irgl, oracle, gen):
    og = oracle.rmat(13) if gen == "rmat" else oracle.grid(60, 45, diag=True)
    with irgl.Context() as c:
        g = _upload(c, og)
        g.relabel()
        perm = g.perm()
        assert np.array_equal(np.sort(perm), np.arange(g.n))          # a permutation
        rp, col, w = g.download()                                      # the relabelled CSR
        deg_new = np.diff(rp)
        assert np.all(deg_new[:-1] >= deg_new[1:])                     # degree-ordered
        assert np.array_equal(deg_new[perm], og.degrees())
        srcs = [int(s) for s in og.sources(3)] if gen == "rmat" else [0, 17, g.n - 1]
        for s in srcs:
            ref, ecc = oracle.bfs(og, s)
            for outline in (0, 1):
                lv, st = irgl.bfs(c, g, s, outline=outline)
                np.testing.assert_array_equal(lv, ref)
                assert st.rounds == ecc + 1
            lv, _ = irgl.bfs(c, g, s, direction=1)
            np.testing.assert_array_equal(lv, ref)
            d, _ = irgl.sssp(c, g, s)
            np.testing.assert_array_equal(d, oracle.sssp(og, s))
        lab, _ = irgl.cc(c, g)
        np.testing.assert_array_equal(lab, oracle.cc(og))
        lab, _ = irgl.cc_lp(c, g)
        np.testing.assert_array_equal(lab, oracle.cc(og))
        r, _ = irgl.pagerank(c, g)
        ref, _ = oracle.pagerank(og)
        assert np.abs(r - ref).sum() / np.abs(ref).sum() < 1e-6
        t, _ = irgl.triangle_count(c, g)
        assert t == oracle.tc(og)
        (wsum, ne), _ = irgl.mst(c, g)
        assert (wsum, ne) == oracle.mst(og)


def test_relabelled_pipe_read_and_async(irgl, oracle):
    import torch
    og = oracle.rmat(12)
    with irgl.Context() as c:
        g = _upload(c, og)
        g.relabel()
        s = int(og.sources(1)[0])
        p = c.pipe(g.n)
        p.init_scalars([s])
        c.invoke(irgl.BFS, g, p, round_start=1)       # one round: out = neighbours of s
        got = sorted(p.read(irgl.WL_IN).tolist())     # after the swap they are `in`
        nbrs = sorted(og.col[og.row_ptr[s]:og.row_ptr[s + 1]].tolist())
        assert got == nbrs
        outs = [torch.empty(g.n, dtype=torch.int32, pin_memory=True).numpy() for _ in range(3)]
        srcs = [int(x) for x in og.sources(3)]
        for x, out in zip(srcs, outs):
            p.init_scalars([x])
            c.iterate(irgl.SSSP, g, p)
            c.read_result_async(irgl.SSSP, g, out)
        c.results_wait()
        for x, out in zip(srcs, outs):
            np.testing.assert_array_equal(out, oracle.sssp(og, x))


def test_relabel_partitioned_cc_results_unsupported(irgl, oracle):
    """Relabelled vertex-partitioned graphs return BFS / SSSP results; CC labels (the smallest
    original id per component needs a global reduction) are refused, not wrong."""
    og = oracle.rmat(10)
    with irgl.Context(logical_partitions=2) as c:
        g = _upload(c, og)
        g.relabel()
        with pytest.raises(irgl.IrglError):
            irgl.cc_lp(c, g, outline=0)


@pytest.mark.parametrize("P,nccl", [(2, False), (3, False), (4, True)])
def test_block_diagonal_relabel_partitioned(irgl, oracle, P, nccl):
    """P > 1: every partition renumbers its own vertices by degree inside its own id range
    (block-diagonal order; owners and routing unchanged).  BFS levels, invocation counts and SSSP
    distances stay bit-exact in the caller's ids through the partitioned (exchange) path."""
    og = oracle.rmat(12)
    kw = dict(logical_partitions=P)
    if nccl:
        kw["nccl"] = (0, 0, 1, irgl.nccl_unique_id())
    with irgl.Context(**kw) as c:
        g = c.generate_rmat(12)
        g.relabel()
        perm = g.perm()
        ps = (-(-g.n // P) + 31) // 32 * 32  # partition ranges: multiples of 32 vertices
        assert np.array_equal(np.sort(perm), np.arange(g.n))
        assert np.array_equal(perm // ps, np.arange(g.n) // ps)       # block-diagonal
        rp, col, w = g.download()
        deg_new = np.diff(rp)
        np.testing.assert_array_equal(deg_new[perm], og.degrees())
        for p0 in range(P):                                             # degree-ordered per block
            d = deg_new[p0 * ps:(p0 + 1) * ps]
            assert np.all(d[:-1] >= d[1:])
        for s in og.sources(2):
            s = int(s)
            ref, ecc = oracle.bfs(og, s)
            lv, st = irgl.bfs(c, g, s)
            np.testing.assert_array_equal(lv, ref)
            assert st.rounds == ecc + 1
            for delta, defer in ((0, 0), (0, -1), (8, 0)):
                d, _ = irgl.sssp(c, g, s, delta=delta, defer=defer)
                np.testing.assert_array_equal(d, oracle.sssp(og, s))


@pytest.mark.parametrize("P,nccl,relabel", [(2, False, False), (3, False, True), (4, True, True)])
def test_direction_optimising_bfs_partitioned(irgl, oracle, P, nccl, relabel):
    """F1 on a vertex-partitioned graph: bottom-up rounds test each partition's own unvisited
    vertices against the exchanged partition-blocked frontier bitmap (no remote updates); levels
    and invocation counts equal Listing 2's, on RMAT (both directions happen) and a grid."""
    kw = dict(logical_partitions=P)
    if nccl:
        kw["nccl"] = (0, 0, 1, irgl.nccl_unique_id())
    with irgl.Context(**kw) as c:
        # both graphs exist before the first traversal: a pipe initialised while the grid (the
        # most recent graph) sets the routing is re-routed for the RMAT graph it meets
        for og, g in ((oracle.rmat(13), c.generate_rmat(13)),
                      (oracle.grid(70, 50), c.generate_grid(70, 50))):
            if relabel:
                g.relabel()
            srcs = [int(s) for s in og.sources(2)] if og.n > 4000 else [0, og.n // 2]
            for s in srcs:
                ref, ecc = oracle.bfs(og, s)
                lv, st = irgl.bfs(c, g, s, direction=1)
                np.testing.assert_array_equal(lv, ref, err_msg=f"n={og.n} src={s}")
                assert st.rounds == ecc + 1


@pytest.mark.parametrize("P", [2, 3])
def test_tiny_partitioned_graphs_with_empty_partitions(irgl, oracle, P):
    """Partition ranges are multiples of 32 vertices, so graphs below 32 (P - 1) vertices have
    empty partitions: upload, relabelling, BFS and SSSP stay correct (an empty partition once
    launched a zero-size grid whose sticky error surfaced in the next library call)."""
    rng = np.random.default_rng(5)
    with irgl.Context(logical_partitions=P) as c:
        for n in list(range(2, 70, 3)) + [200]:
            m = int(rng.integers(1, 4 * n))
            og = oracle.from_edges(n, rng.integers(0, n, m).tolist(), rng.integers(0, n, m).tolist())
            g = c.graph_from_csr(og.row_ptr, og.col, og.weight)
            if n % 2:
                g.relabel()
            s = int(og.sources(1)[0]) if og.m else 0
            lv, _ = irgl.bfs(c, g, s)
            np.testing.assert_array_equal(lv, oracle.bfs(og, s)[0])
            d, _ = irgl.sssp(c, g, s)
            np.testing.assert_array_equal(d, oracle.sssp(og, s))
            g.close()
