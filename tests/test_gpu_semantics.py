"""IrGL orchestration semantics on the GPU runtime, phrased as the reference's own examples
 and checked against the oracle's executor."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_iterate_nonpushing_kernel_one_round(ctx, irgl):
    p = ctx.pipe(16)
    p.init_scalars([1, 2, 3])
    st = ctx.iterate(irgl.TEST_NOPUSH, None, p)
    assert st.rounds == 1
    assert p.size() == 0


def test_countdown_three_invocations(ctx, irgl, oracle):
    p = ctx.pipe(16)
    p.init_scalars([0])
    st = ctx.iterate(irgl.TEST_COUNTDOWN, None, p, guard=3)
    assert st.rounds == 3
    _, ost, _, _ = oracle.iterate(None, oracle.OP_TEST_COUNTDOWN, [0], guard=3, capacity=16)
    assert ost.rounds == st.rounds


def test_retry_odd_two_runs_out_has_all(ctx, irgl, oracle):
    p = ctx.pipe(64)
    p.init_scalars(range(8))
    ctx.op_reset(irgl.TEST_RETRY_ODD)
    _, st = ctx.invoke(irgl.TEST_RETRY_ODD, None, p, guard=1)
    assert st.launches == 2
    assert sorted(p.read().tolist()) == list(range(8))  # after the swap, in == all processed


def test_retry_three_round_trace(ctx, irgl, oracle):
    """SPEC.md:554 golden trace: odd items retried twice -> 3 launches with in<->retry swaps and
    out preserved."""
    p = ctx.pipe(64)
    p.init_scalars(range(8))
    ctx.op_reset(irgl.TEST_RETRY_ODD)
    _, st = ctx.invoke(irgl.TEST_RETRY_ODD, None, p, guard=2)
    _, ost, trace, fin = oracle.iterate(None, oracle.OP_TEST_RETRY_ODD, list(range(8)), guard=2,
                                        capacity=64, max_rounds=1)
    assert trace.tolist() == [[1, 8, 4, 4], [2, 4, 4, 4], [3, 4, 8, 0]]
    assert st.launches == ost.launches == 3
    assert st.retries == ost.retries == 8
    assert sorted(p.read().tolist()) == sorted(fin.tolist()) == list(range(8))


def test_retry_serialisation_after_n_rounds(irgl):
    with irgl.Context(retry_serialize_after=2) as c:
        p = c.pipe(64)
        p.init_scalars([1, 3, 5])
        c.op_reset(irgl.TEST_RETRY_ODD)
        _, st = c.invoke(irgl.TEST_RETRY_ODD, None, p, guard=5)
        assert st.launches == 6
        assert st.serial_launches == 3  # retry rounds 3,4,5 exceed retry_serialize_after=2
        assert sorted(p.read().tolist()) == [1, 3, 5]


@pytest.mark.parametrize("red", ["any", "all"])
def test_reduce_and_return_random(ctx, irgl, oracle, red):
    """random boolean assignments over 1-64 iterations; zero-iteration identities."""
    rng = np.random.default_rng(7)
    R = irgl.RED_ANY if red == "any" else irgl.RED_ALL
    for n in [0, 1, 2, 5, 17, 31, 32, 33, 64]:
        for density in (0.0, 0.05, 0.5, 0.95, 1.0):
            vals = (rng.random(max(n, 1)) < density).astype(np.int32)
            p = ctx.pipe(64)
            p.init_scalars(range(n))
            r, _ = ctx.invoke(irgl.TEST_REDUCE, None, p, reduction=R, values=vals)
            expect = oracle.reduce(vals[:n], oracle.RED_ANY if red == "any" else oracle.RED_ALL)
            assert r == expect, (n, density)
    p = ctx.pipe(4)
    p.init_scalars([])
    r, _ = ctx.invoke(irgl.TEST_REDUCE, None, p, reduction=irgl.RED_ANY, values=[1])
    assert r is False   # Any identity
    r, _ = ctx.invoke(irgl.TEST_REDUCE, None, p, reduction=irgl.RED_ALL, values=[1])
    assert r is True    # All identity


def test_iterate_while_any_until_all(ctx, irgl):
    p = ctx.pipe(8)
    p.init_scalars([0, 1])
    # items never pushed -> worklist empties after one invocation regardless of the cond
    st = ctx.iterate(irgl.TEST_REDUCE, None, p, cond=irgl.COND_WHILE, reduction=irgl.RED_ANY,
                     values=[0, 0])
    assert st.rounds == 1 and st.last_reduced == 0


@pytest.mark.parametrize("blocked", [False, True])
def test_forall_mapping(ctx, irgl, oracle, blocked):
    """100 iterations, 8 threads, consecutive -> thread t runs {t, t+8, ...}."""
    p = ctx.pipe(128)
    p.init_scalars(range(100))
    ctx.op_reset(irgl.TEST_FORALL_MAP)
    ctx.invoke(irgl.TEST_FORALL_MAP, None, p, threads=8,
               mapping=irgl.MAP_BLOCKED if blocked else irgl.MAP_CONSECUTIVE)
    tid = ctx.read_result(irgl.TEST_FORALL_MAP, None, size=100)
    np.testing.assert_array_equal(tid, oracle.forall_assign(100, 8, blocked))


def test_bulk_synchrony_pushes_not_popped_same_launch(ctx, irgl):
    """items pushed in launch e are popped only in launch e+1."""
    p = ctx.pipe(4096)
    p.init_scalars(range(1000))
    ctx.op_reset(irgl.TEST_PUSHPOP)
    st = ctx.iterate(irgl.TEST_PUSHPOP, None, p, guard=1000)
    log = ctx.read_result(irgl.TEST_PUSHPOP, None, size=4096)
    assert st.rounds == 5
    for k in range(5):
        assert (log[k * 1000:(k + 1) * 1000] == k + 1).all()


def test_extra_cond_max_rounds(ctx, irgl):
    p = ctx.pipe(64)
    p.init_scalars([0])
    st = ctx.iterate(irgl.TEST_COUNTDOWN, None, p, guard=50, max_rounds=7, extra_comb=irgl.COMB_OR)
    assert st.rounds == 7
    assert p.read().tolist() == [7]


def test_worklist_overflow_is_an_error(ctx, irgl):
    p = ctx.pipe(4)
    with pytest.raises(irgl.IrglError) as e:
        p.init_scalars(range(5))
    assert e.value.status == 4  # IRGL_E_WL_OVERFLOW


def test_invoke_wl_kernel_without_pipe_is_usage_error(ctx, irgl):
    with pytest.raises(irgl.IrglError) as e:
        ctx.invoke(irgl.TEST_NOPUSH, None, None)
    assert e.value.status == 2


def test_op_plan_fixed_block_and_coresident_grid(ctx, irgl):
    (kind, val), grid_o, grid_f = ctx.op_plan(irgl.BFS)
    assert kind == irgl.BLOCK_FIXED and val in (256, 512)  # this build's kBlock (IRGL_BLOCK)
    assert grid_o > 0 and grid_o % 148 == 0  # occupancy x SMs on B200
    # outlined Pipe of [Elastic, Fixed(kBlock)] -> control kernel at kBlock
    assert irgl.t_control([(irgl.BLOCK_ELASTIC, 0), (kind, val)]) == val


def test_invoke_level_by_level_bfs_matches_iterate(ctx, irgl, oracle):
    """Host-side Iterate written with Invoke + between_rounds (Listing 2 unrolled)."""
    og = oracle.rmat(12)
    g = ctx.graph_from_csr(og.row_ptr, og.col, og.weight)
    s = int(og.sources(1)[0])
    p = ctx.pipe(og.n)
    p.init_scalars([s])
    ctx.op_reset(irgl.BFS, g, p)
    LEVEL = 1
    while p.size() > 0:
        ctx.invoke(irgl.BFS, g, p, round_start=LEVEL)
        LEVEL += 1
    np.testing.assert_array_equal(ctx.read_result(irgl.BFS, g), oracle.bfs(og, s)[0])


def test_looping_pipe_and_pipe_once(ctx, irgl):
    """Listing-3/4 shapes: a looping Pipe repeats its body while `in` is non-empty; Pipe Once
    runs it once; Invokes inside share the pipe context."""
    p = ctx.pipe(64)
    p.init_scalars([0, 1])
    seen = []

    def body(c, pp):
        seen.append(sorted(pp.read().tolist()))
        c.invoke(irgl.TEST_COUNTDOWN, None, pp, guard=4)   # A: pushes x+1 while x+1 < 4
        c.invoke(irgl.TEST_COUNTDOWN, None, pp, guard=4)   # B consumes A's worklist

    n = ctx.run_pipe(p, body)
    # [0,1] -A-> [1,2] -B-> [2,3];  [2,3] -A-> [3] -B-> []
    assert n == 2 and seen == [[0, 1], [2, 3]]
    q = ctx.pipe(8)
    q.init_scalars([5])
    assert ctx.run_pipe(q, lambda c, pp: c.invoke(irgl.TEST_NOPUSH, None, pp), once=True) == 1
    assert q.size() == 0


def test_respawn_is_never_serialised(irgl):
    """Respawn pushes to the retry worklist like Retry but never triggers conflict management
    (SPEC.md:88, :462): same launches, no serial launch."""
    with irgl.Context(retry_serialize_after=2) as c:
        p = c.pipe(64)
        p.init_scalars([1, 3, 5])
        c.op_reset(irgl.TEST_RESPAWN_ODD)
        _, st = c.invoke(irgl.TEST_RESPAWN_ODD, None, p, guard=5)
        assert st.launches == 6 and st.serial_launches == 0
        assert sorted(p.read().tolist()) == [1, 3, 5]
