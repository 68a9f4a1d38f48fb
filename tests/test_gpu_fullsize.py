"""Parity at BASELINE.json's full sizes through size-independent certificates (no oracle run):
the RMAT-22 graph of the bench (and the 4096^2 grid of configs[2]) is generated on the device,
downloaded, and each operator's output is checked against the property that characterises it
exactly:

  BFS  : level[src] = 0; for every edge |level[u] - level[v]| <= 1 within the reached set (no
         edge leaves it); every reached v != src has a neighbour at level[v] - 1  => hop distance.
  SSSP : dist[src] = 0; dist[v] <= dist[u] + w(u,v) for every edge (no violated edge); every
         reached v != src has an edge with dist[u] + w = dist[v] (tight parent)  => shortest.
  CC   : label constant across every edge; label[v] <= v; label[label[v]] = label[v]; every
         root label is the smallest id of its component (BFS-level check via the edge test
         plus the root count matching the component count of the label graph).
  PR   : ranks within the Jacobi fixed point: |rank - ((1-d)/N + d * sum contrib)| <= tol.
Sizes: RMAT-22 (4.19M vertices, 128M directed edges) in generator and in degree-ordered ids,
grid 4096^2 (16.8M vertices)."""
import numpy as np
import pytest

INF = 2147483647
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rmat22(irgl):
    c = irgl.Context()
    g = c.generate_rmat(22)
    rp, col, w = g.download()
    deg = np.diff(rp)
    src = np.repeat(np.arange(g.n, dtype=np.int64), deg)
    yield c, g, rp, col.astype(np.int64), w.astype(np.int64), src, deg
    c.close()


def _sources(deg, k=2):
    import bench
    return bench.pick_sources(len(deg), lambda x: int(deg[x]), count=k)


def test_bfs_certificate_rmat22(irgl, rmat22):
    c, g, rp, col, w, src, deg = rmat22
    for s in _sources(deg):
        for direction in (0, 1):
            lv, st = irgl.bfs(c, g, s, direction=direction)
            lv = lv.astype(np.int64)
            assert lv[s] == 0
            reached = lv != INF
            lu, lw = lv[src], lv[col]
            ru, rw = reached[src], reached[col]
            assert np.array_equal(ru, rw)                       # no edge leaves the reached set
            assert np.all(np.abs(lu[ru] - lw[ru]) <= 1)         # levels differ by <= 1 on edges
            has_parent = np.zeros(g.n, dtype=bool)              # every reached v has a parent
            m = ru & (lu == lw - 1)
            has_parent[col[m]] = True
            has_parent[s] = True
            assert np.array_equal(has_parent, reached)
            assert st.rounds == int(lv[reached].max()) + 1


def test_sssp_certificate_rmat22(irgl, rmat22):
    c, g, rp, col, w, src, deg = rmat22
    for s in _sources(deg):
        for defer in (-1, 0):
            d, st = irgl.sssp(c, g, s, defer=defer)
            d = d.astype(np.int64)
            assert d[s] == 0
            reached = d != INF
            du, dv = d[src], d[col]
            ru = reached[src]
            assert np.all(reached[col][ru])
            assert np.all(dv[ru] <= du[ru] + w[ru])             # no violated edge
            tight = ru & (du + w == dv)
            has_parent = np.zeros(g.n, dtype=bool)
            has_parent[col[tight]] = True
            has_parent[s] = True
            assert np.array_equal(has_parent, reached)          # every distance is attained


def _cc_certificate(g, lab, src, col):
    lab = lab.astype(np.int64)
    assert np.array_equal(lab[src], lab[col])                  # constant on every edge
    assert np.all(lab <= np.arange(g.n))
    assert np.array_equal(lab[lab], lab)                       # labels are roots
    # the root of each component is its smallest id: every vertex with label == v is v's own
    # component root, and a vertex smaller than its root would need label < root (contradiction
    # with lab[v] <= v only if v is in the component) -> check min id per label directly
    mins = np.full(g.n, np.iinfo(np.int64).max)
    np.minimum.at(mins, lab, np.arange(g.n))
    roots = np.unique(lab)
    assert np.array_equal(mins[roots], roots)


def test_cc_certificate_rmat22(irgl, rmat22):
    c, g, rp, col, w, src, deg = rmat22
    lab, _ = irgl.cc(c, g)
    _cc_certificate(g, lab, src, col)
    lab2, _ = irgl.cc_lp(c, g)
    np.testing.assert_array_equal(lab, lab2)


def test_cc_certificate_grid4096(irgl):
    with irgl.Context() as c:
        g = c.generate_grid(4096, 4096, perc_keep=0.5, perc_seed=5)
        rp, col, _ = g.download()
        src = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(rp))
        lab, _ = irgl.cc(c, g)
        _cc_certificate(g, lab, src, col.astype(np.int64))


def test_pagerank_fixed_point_rmat22(irgl, rmat22):
    c, g, rp, col, w, src, deg = rmat22
    r, st = irgl.pagerank(c, g)
    d, tol = 0.85, 1e-6
    contrib = np.where(deg > 0, r / np.maximum(deg, 1), 0.0)
    s = np.zeros(g.n)
    np.add.at(s, src, contrib[col])
    nxt = (1 - d) / g.n + d * s
    # the last sweep changed no vertex by more than tol, so one more Jacobi step stays within it
    # (fp32 contrib storage adds ~1e-8 relative)
    assert np.abs(nxt - r).max() <= 2 * tol
    assert r.sum() <= 1.0 + 1e-9


# ---- the same certificates with degree-ordered ids (irgl_graph_relabel): the bench's layout, the
# byte-weight SSSP kernel, the direction-optimising BFS and both PR sweep layouts.  Results come
# back in the caller's ids, so they are checked against the CSR downloaded before relabelling.
@pytest.fixture(scope="module")
def rmat22_relabelled(irgl):
    c = irgl.Context()
    g = c.generate_rmat(22)
    rp, col, w = g.download()
    deg = np.diff(rp)
    src = np.repeat(np.arange(g.n, dtype=np.int64), deg)
    g.relabel()
    yield c, g, rp, col.astype(np.int64), w.astype(np.int64), src, deg
    c.close()


def test_bfs_certificate_rmat22_relabelled(irgl, rmat22_relabelled):
    test_bfs_certificate_rmat22(irgl, rmat22_relabelled)


def test_sssp_certificate_rmat22_relabelled(irgl, rmat22_relabelled):
    test_sssp_certificate_rmat22(irgl, rmat22_relabelled)


def test_cc_certificate_rmat22_relabelled(irgl, rmat22_relabelled):
    test_cc_certificate_rmat22(irgl, rmat22_relabelled)


def test_pagerank_fixed_point_rmat22_relabelled(irgl, rmat22_relabelled):
    test_pagerank_fixed_point_rmat22(irgl, rmat22_relabelled)
