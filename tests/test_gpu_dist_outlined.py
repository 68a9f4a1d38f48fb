"""E3 across partitions: an Iterate on a partitioned graph in one process runs as
one cooperative persistent kernel per partition (dist_persistent_kernel) meeting at a device-side
rendezvous, instead of host-orchestrated rounds (wl_graph_rounds_dist).  The partitions share the
GPU by splitting its co-resident CTAs.

Checked against the serial oracle (queue BFS, Dijkstra, union-find) and against the host rounds
(outline=0) on the same inputs: results, round counts, and that the outlined path really ran
(stats.outlined, one launch per partition)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _upload(ctx, og):
    return ctx.graph_from_csr(og.row_ptr, og.col, og.weight)


@pytest.mark.parametrize("P", [2, 3, 4])
def test_outlined_partitioned_bfs_sssp_cc(irgl, oracle, P):
    og = oracle.rmat(13)
    with irgl.Context(logical_partitions=P) as c:
        g = _upload(c, og)
        for s in [int(x) for x in og.sources(2)]:
            ref, ecc = oracle.bfs(og, s)
            lv, st = irgl.bfs(c, g, s, outline=1)
            np.testing.assert_array_equal(lv, ref)
            assert st.rounds == ecc + 1 and st.outlined == 1 and st.launches == P
            assert st.remote_updates > 0
            dref = oracle.sssp(og, s)
            for defer in (0, -1, 8):
                d, st = irgl.sssp(c, g, s, defer=defer, outline=1)
                np.testing.assert_array_equal(d, dref, err_msg=f"P={P} defer={defer}")
                assert st.outlined == 1
                d0, st0 = irgl.sssp(c, g, s, defer=defer, outline=0)  # host rounds, same answer
                np.testing.assert_array_equal(d0, dref)
                assert st0.outlined == 0
        lab, st = irgl.cc_lp(c, g, outline=1)
        np.testing.assert_array_equal(lab, oracle.cc(og))
        assert st.outlined == 1


@pytest.mark.parametrize("P", [2, 3, 4])
def test_outlined_partitioned_direction_optimising_bfs(irgl, oracle, P):
    # F1 inside the distributed kernel: bottom-up rounds against the frontier bitmap every
    # partition stores into every partition's copy; Listing 2's levels and invocation count
    for relabel in (False, True):
        og = oracle.rmat(14)
        with irgl.Context(logical_partitions=P) as c:
            g = c.generate_rmat(14)
            if relabel:
                g.relabel()
            for s in [int(x) for x in og.sources(3)]:
                ref, ecc = oracle.bfs(og, s)
                lv, st = irgl.bfs(c, g, s, direction=1)
                np.testing.assert_array_equal(lv, ref, err_msg=f"P={P} relabel={relabel} src={s}")
                assert st.rounds == ecc + 1 and st.outlined == 1 and st.launches == P
                lv0, st0 = irgl.bfs(c, g, s, direction=1, outline=0)  # host rounds
                np.testing.assert_array_equal(lv0, ref)
                assert st0.outlined == 0 and st0.rounds == ecc + 1
                assert st.edges < og.m  # bottom-up rounds stopped at the first parent
    og = oracle.grid(64, 48, perc_keep=0.6)
    with irgl.Context(logical_partitions=P) as c:
        g = c.generate_grid(64, 48, perc_keep=0.6)
        for s in (0, 1500):
            ref, ecc = oracle.bfs(og, s)
            lv, st = irgl.bfs(c, g, s, direction=1)
            np.testing.assert_array_equal(lv, ref)
            assert st.rounds == ecc + 1 and st.outlined == 1


def test_outlined_partitioned_relabelled_and_grid(irgl, oracle):
    og = oracle.rmat(14)
    with irgl.Context(logical_partitions=2) as c:
        g = c.generate_rmat(14)
        g.relabel()  # block-diagonal degree order, visited bitmap BFS
        for s in [int(x) for x in og.sources(2)]:
            lv, st = irgl.bfs(c, g, s)
            np.testing.assert_array_equal(lv, oracle.bfs(og, s)[0])
            assert st.outlined == 1
            d, st = irgl.sssp(c, g, s)
            np.testing.assert_array_equal(d, oracle.sssp(og, s))
            assert st.outlined == 1
    og = oracle.grid(64, 48, perc_keep=0.6)  # long diameter: many rendezvous
    with irgl.Context(logical_partitions=3) as c:
        g = c.generate_grid(64, 48, perc_keep=0.6)
        for s in (0, 1500):
            ref, ecc = oracle.bfs(og, s)
            lv, st = irgl.bfs(c, g, s)
            np.testing.assert_array_equal(lv, ref)
            assert st.rounds == ecc + 1 and st.outlined == 1
            np.testing.assert_array_equal(irgl.sssp(c, g, s)[0], oracle.sssp(og, s))


def test_outlined_partitioned_many_and_empty_partitions(irgl, oracle):
    # 16 partitions (kMaxParts) of a graph with fewer than 16 * 32 vertices: most are empty
    og = oracle.rmat(8)
    with irgl.Context(logical_partitions=16) as c:
        g = _upload(c, og)
        for s in [int(x) for x in og.sources(2)]:
            lv, st = irgl.bfs(c, g, s)
            np.testing.assert_array_equal(lv, oracle.bfs(og, s)[0])
            assert st.outlined == 1 and st.launches == 16
            np.testing.assert_array_equal(irgl.sssp(c, g, s)[0], oracle.sssp(og, s))


def test_outlined_partitioned_max_rounds_matches_host_rounds(irgl, oracle):
    og = oracle.rmat(12)
    with irgl.Context(logical_partitions=2) as c:
        g = _upload(c, og)
        s = int(og.sources(1)[0])
        p = c.pipe(g.n)
        out = []
        for outline in (1, 0):
            p.init_scalars([s])
            st = c.iterate(irgl.SSSP, g, p, outline=outline, max_rounds=3, defer=0)
            assert st.rounds == 3 and st.outlined == outline
            out.append((c.read_result(irgl.SSSP, g), sorted(p.read())))
        np.testing.assert_array_equal(out[0][0], out[1][0])  # same labels after 3 rounds
        assert out[0][1] == out[1][1]  # and the same next worklist


def test_outlined_partitioned_overflow_is_reported(irgl, oracle):
    og = oracle.rmat(12)
    with irgl.Context(logical_partitions=2) as c:
        g = _upload(c, og)
        p = c.pipe(64)  # far below one round's pushes
        p.init_scalars([int(og.sources(1)[0])])
        with pytest.raises(irgl.IrglError, match="E_WL_OVERFLOW"):
            c.iterate(irgl.BFS, g, p, outline=1, round_start=1)


def test_outlined_partitioned_opt_out(irgl, oracle, monkeypatch):
    og = oracle.rmat(12)
    monkeypatch.setenv("IRGL_DIST_OUTLINE", "0")  # host rounds (read per Iterate)
    with irgl.Context(logical_partitions=2) as c:
        g = _upload(c, og)
        s = int(og.sources(1)[0])
        lv, st = irgl.bfs(c, g, s)
        assert st.outlined == 0
        np.testing.assert_array_equal(lv, oracle.bfs(og, s)[0])
