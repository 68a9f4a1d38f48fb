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


def test_relabel_partitioned_unsupported(irgl, oracle):
    og = oracle.rmat(10)
    with irgl.Context(logical_partitions=2) as c:
        g = _upload(c, og)
        with pytest.raises(irgl.IrglError):
            g.relabel()
