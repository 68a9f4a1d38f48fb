"""Parity at every BASELINE.json configuration size (SURVEY §8d C2★, C3, C4, C5), through the
C-ABI on the device graph the bench uses:

  C2★ RMAT-24 : BFS levels and SSSP distances bit-exact against the serial oracle (queue BFS,
                Dijkstra) from 2 sources, in generator ids and in degree-ordered ids (the bench's
                layout); the device CSR equal to the oracle's CSR.
  C4  RMAT-24 : PageRank within 1e-6 L1-relative of the fp64 oracle at the oracle's iteration
                count, both sweep layouts, host loop and outlined.
  C3  4096^2  : CC on the cut grid = 8 row stripes labelled k * 2^21, hooking and
                label propagation; TC on the triangulated grid = 2 * 4095^2 = 33,538,050.
  C5  RMAT-27 : one-GPU BFS and SSSP (4.2G directed edges) checked with the oracle's exact
                certificates (orc_cert_bfs / orc_cert_sssp) on the downloaded CSR — no oracle run
                of that size fits a test budget.

Reference pin for the BFS pattern: /root/reference/SPEC.md:549 (random graphs, bit-exact levels,
rounds = ecc + 1)."""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rmat24(irgl, oracle):
    with ThreadPoolExecutor(1) as ex:  # ctypes releases the GIL: oracle generation overlaps
        fut = ex.submit(oracle.rmat, 24)
        c = irgl.Context()
        g = c.generate_rmat(24)
        og = fut.result()
    yield c, g, og
    c.close()


def _oracle_answers(oracle, og, srcs):
    with ThreadPoolExecutor(2 * len(srcs) + 1) as ex:
        bfs = [ex.submit(oracle.bfs, og, s) for s in srcs]
        sssp = [ex.submit(oracle.sssp, og, s) for s in srcs]
        pr = ex.submit(oracle.pagerank, og)
        return [f.result() for f in bfs], [f.result() for f in sssp], pr.result()


def test_rmat24_bfs_sssp_pagerank_parity(irgl, oracle, rmat24):
    c, g, og = rmat24
    assert (g.n, g.m) == (og.n, og.m)
    rp, col, w = g.download()
    np.testing.assert_array_equal(rp, og.row_ptr)
    np.testing.assert_array_equal(col, og.col)
    np.testing.assert_array_equal(w, og.weight)
    del rp, col, w
    srcs = [int(s) for s in og.sources(2)]
    bfs_ref, sssp_ref, (pr_ref, pr_it) = _oracle_answers(oracle, og, srcs)
    p = c.pipe(g.n)

    def check(tag):
        for s, (lref, ecc), dref in zip(srcs, bfs_ref, sssp_ref):
            for direction in (0, 1):
                lv, st = irgl.bfs(c, g, s, pipe=p, direction=direction)
                np.testing.assert_array_equal(lv, lref, err_msg=f"{tag} bfs src={s} dir={direction}")
                assert st.rounds == ecc + 1
            for outline in (0, 1):
                d, _ = irgl.sssp(c, g, s, pipe=p, outline=outline)
                np.testing.assert_array_equal(d, dref, err_msg=f"{tag} sssp src={s} outline={outline}")
        for outline in (0, 1):
            r, st = irgl.pagerank(c, g, outline=outline)
            err = np.abs(r - pr_ref).sum() / np.abs(pr_ref).sum()
            assert err <= 1e-6, (tag, outline, err)
            assert st.rounds == pr_it, (tag, outline, st.rounds, pr_it)

    check("generator ids")
    g.relabel()  # degree-ordered ids: the bench's layout, byte-weight SSSP, CTA-tile PR
    check("degree-ordered ids")


def test_grid4096_cut_cc_known_answer(irgl):
    with irgl.Context() as c:
        g = c.generate_grid(4096, 4096, cut_period=512)
        expect = (np.arange(g.n, dtype=np.int64) // (512 * 4096) * (1 << 21)).astype(np.int32)
        lab, _ = irgl.cc(c, g)
        np.testing.assert_array_equal(lab, expect)
        for outline in (0, 1):
            lab2, st = irgl.cc_lp(c, g, outline=outline)
            np.testing.assert_array_equal(lab2, expect)


def test_grid4096_triangulated_tc_known_answer(irgl):
    with irgl.Context() as c:
        g = c.generate_grid(4096, 4096, diag=True)
        assert g.m == 100_630_530
        tc, _ = irgl.triangle_count(c, g)
        assert int(tc) == 2 * 4095 * 4095 == 33_538_050


def _host_gb():
    try:
        import psutil
        return psutil.virtual_memory().available / 2**30
    except ImportError:
        return 0.0


@pytest.mark.skipif(_host_gb() < 96, reason="RMAT-27 certificate needs ~60 GB of host memory")
def test_rmat27_one_gpu_certificates(irgl, oracle):
    import bench
    with irgl.Context() as c:
        g = c.generate_rmat(27)
        rp, col, w = g.download()
        deg = np.diff(rp)
        srcs = bench.pick_sources(g.n, lambda x: int(deg[x]), count=2)
        del deg
        p = c.pipe(g.n)
        for relabel in (False, True):
            if relabel:
                g.relabel()
            for s in srcs:
                lv, st = irgl.bfs(c, g, s, pipe=p)
                assert oracle.cert_bfs(rp, col, s, lv) == 0, ("bfs", relabel, s)
                assert st.rounds == int(lv[lv != oracle.INF].max()) + 1
                d, _ = irgl.sssp(c, g, s, pipe=p)
                assert oracle.cert_sssp(rp, col, w, s, d) == 0, ("sssp", relabel, s)
