"""SURVEY §8f F3 on the GPU: IrGL's Atomic / Exclusive constructs and Boruvka MST (Listing 1),
checked against the SPEC's acceptance items 2-4 and the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_atomic_mutual_exclusion(ctx, irgl):
    """256 threads incrementing one counter under blocking Atomic -> 256."""
    for threads in (256, 64, 32 * 148):
        p = ctx.pipe(512)
        p.init_scalars(range(256))
        ctx.invoke(irgl.TEST_ATOMIC, None, p, threads=threads)
        log = ctx.read_result(irgl.TEST_ATOMIC, None, size=2)
        assert log[0] == 256


def test_atomic_else_with_held_lock(ctx, irgl):
    """the Else form with a held lock executes failed stmts in every schedule."""
    p = ctx.pipe(512)
    p.init_scalars(range(256))
    ctx.invoke(irgl.TEST_ATOMIC_ELSE, None, p, guard=1)
    log = ctx.read_result(irgl.TEST_ATOMIC_ELSE, None, size=2)
    assert log[0] == 0 and log[1] == 256
    p.init_scalars(range(256))
    ctx.invoke(irgl.TEST_ATOMIC_ELSE, None, p, guard=0)  # free lock: every item succeeds or fails
    log = ctx.read_result(irgl.TEST_ATOMIC_ELSE, None, size=2)
    assert log[0] + log[1] == 256 and log[0] >= 1


def test_exclusive_protocol_fuzz(ctx, irgl, oracle):
    """random lock sets (<=16 items, <=8 locks): winners' sets pairwise disjoint,
    >= 1 winner whenever >= 1 claimant, fixed-priority winners == protocol oracle."""
    rng = np.random.default_rng(552)
    for case in range(200):
        n = int(rng.integers(1, 17))
        k = 4
        locks = np.full((n, k), -1, dtype=np.int32)
        for x in range(n):
            c = int(rng.integers(0, k + 1))
            locks[x, :c] = rng.choice(8, size=c, replace=False)
        p = ctx.pipe(32)
        p.init_scalars(range(n))
        ctx.invoke(irgl.TEST_EXCLUSIVE, None, p, guard=k, values=locks.reshape(-1))
        won = ctx.read_result(irgl.TEST_EXCLUSIVE, None, size=n)[:n]
        np.testing.assert_array_equal(won, oracle.exclusive(locks))
        sets = [set(locks[x][locks[x] >= 0].tolist()) for x in range(n) if won[x]]
        for i in range(len(sets)):
            for j in range(i + 1, len(sets)):
                assert not (sets[i] & sets[j])
        if (locks >= 0).any():
            assert won.sum() >= 1
    assert oracle.exclusive([[1, 2], [2, 3]]).tolist() == [1, 0]


def test_boruvka_mst_matches_kruskal(ctx, irgl, oracle):
    """MST weight == Kruskal on 20 random weighted graphs (<= 32 nodes)."""
    rng = np.random.default_rng(550)
    for t in range(20):
        n = int(rng.integers(2, 33))
        m = int(rng.integers(n - 1, 3 * n))
        u = rng.integers(0, n, m)
        v = rng.integers(0, n, m)
        w = rng.integers(1, 20, m).astype(np.int32)  # ties on purpose
        og = oracle.from_edges(n, u, v, w=w)
        g = ctx.graph_from_csr(og.row_ptr, og.col, og.weight)
        (wt, ne), st = irgl.mst(ctx, g)
        assert (wt, ne) == oracle.mst(og)


@pytest.mark.parametrize("which", ["rmat12", "rmat15", "grid", "cut_grid"])
def test_boruvka_mst_larger(ctx, irgl, oracle, which):
    og = {"rmat12": lambda: oracle.rmat(12), "rmat15": lambda: oracle.rmat(15),
          "grid": lambda: oracle.grid(60, 50),
          "cut_grid": lambda: oracle.grid(64, 64, cut_period=16)}[which]()
    g = ctx.graph_from_csr(og.row_ptr, og.col, og.weight)
    (wt, ne), st = irgl.mst(ctx, g)
    assert (wt, ne) == oracle.mst(og)
    assert st.rounds >= 2  # Iterate While Any: the last invocation hooks nothing
