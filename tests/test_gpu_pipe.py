"""Multi-member Pipe: a Pipe body of several member statements over one pipe
context, host-orchestrated and outlined as ONE cooperative control kernel launched at T_control
(SPEC.md:373-381), against the oracle's restatement (oracle.pipe_run).

Shapes: Listing 3 (a looping Pipe re-dispatching between two kernels, one of them with Retry),
Listing 4 (dynamic piping: the next kernel chosen by the previous invocation's reduced value),
an Iterate member inside a looping Pipe, Pipe Once, Respawn vs Retry serialisation, and the
T_control rules (empty intersection -> IRGL_E_OUTLINE_EMPTY when outlining is forced, the host
fallback when it is not)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

E_OUTLINE_EMPTY = 6


def _cases(irgl, oracle):
    I, T = irgl.STAGE_INVOKE, irgl.STAGE_ITERATE
    vals = (np.arange(64) % 3 == 0).astype(np.int32)
    return [
        # Listing 3: looping Pipe { Invoke refine (Retry); Invoke identify }
        ("listing3", [dict(op=irgl.TEST_RETRY_ODD, kind=I, guard=2),
                      dict(op=irgl.TEST_COUNTDOWN, kind=I, guard=40)],
         [1, 2, 3, 7, 10], False, 0, None),
        # Listing 4: Pipe Once { Any(Invoke A); if (r) Invoke B else Invoke C }
        ("listing4-true", [dict(op=irgl.TEST_REDUCE, reduction=irgl.RED_ANY, guard=0),
                           dict(op=irgl.TEST_PUSHPOP, when=irgl.WHEN_PREV_TRUE, guard=5),
                           dict(op=irgl.TEST_COUNTDOWN, when=irgl.WHEN_PREV_FALSE, guard=9)],
         [0, 1, 2], True, 0, vals),
        ("listing4-false", [dict(op=irgl.TEST_REDUCE, reduction=irgl.RED_ANY),
                            dict(op=irgl.TEST_PUSHPOP, when=irgl.WHEN_PREV_TRUE, guard=5),
                            dict(op=irgl.TEST_COUNTDOWN, when=irgl.WHEN_PREV_FALSE, guard=9)],
         [1, 2, 4], True, 0, vals),
        # looping Pipe { Iterate countdown [max 3]; Invoke pushpop } (nested Iterate inherits)
        ("iterate-member", [dict(op=irgl.TEST_COUNTDOWN, kind=T, guard=30, max_rounds=3),
                            dict(op=irgl.TEST_PUSHPOP, guard=4)],
         [0, 5, 11], False, 0, None),
        # Retry serialised after 4 rounds, Respawn never; bounded looping Pipe
        ("retry-serial", [dict(op=irgl.TEST_RETRY_ODD, guard=6),
                          dict(op=irgl.TEST_RESPAWN_ODD, guard=12)],
         [1, 3, 4, 9], False, 2, None),
        # Any/All cond on an Iterate member: Iterate Until All reduce
        ("until-all", [dict(op=irgl.TEST_REDUCE, kind=T, reduction=irgl.RED_ALL,
                            cond=irgl.COND_UNTIL, max_rounds=5),
                       dict(op=irgl.TEST_NOPUSH)],
         [3, 6, 9], True, 0, vals),
    ]


def _run(irgl, c, stages, init, once, max_rounds, values, outline, cap=64):
    p = c.pipe(cap)
    p.init_scalars(init)
    c.op_reset(irgl.TEST_PUSHPOP)  # test-operator state: launch counter, retry counts, log
    st = [dict(s, values=values) if (values is not None and s["op"] == irgl.TEST_REDUCE) else dict(s)
          for s in stages]
    stats, res = c.pipe_run(p, st, once=once, max_rounds=max_rounds, outline=outline)
    log = c.read_result(irgl.TEST_PUSHPOP, size=cap)
    return stats, res, sorted(p.read().tolist()), np.asarray(log)


@pytest.mark.parametrize("outline", [0, 1])
def test_pipe_matches_oracle(irgl, oracle, outline):
    with irgl.Context() as c:
        for name, stages, init, once, mr, vals in _cases(irgl, oracle):
            st, res, fin, log = _run(irgl, c, stages, init, once, mr, vals, outline)
            ost, ofin, orc, olog, ored = oracle.pipe_run(
                [dict(op=s["op"], kind=s.get("kind", 0), reduction=s.get("reduction", 0),
                      when=s.get("when", 0), cond_mode=s.get("cond", 0),
                      max_rounds=s.get("max_rounds", 0), guard=s.get("guard", 0)) for s in stages],
                init, 64, once=once, max_rounds=mr, values=vals)
            assert res.outlined == outline, name
            assert fin == sorted(ofin.tolist()), name
            assert (st.rounds, st.launches, st.popped, st.pushes, st.retries, st.serial_launches) == \
                (ost.rounds, ost.launches, ost.popped, ost.pushes, ost.retries, ost.serial_launches), name
            assert st.last_reduced == ost.last_reduced, name
            assert list(res.stage_reduced)[: len(stages)] == ored.tolist(), name
            np.testing.assert_array_equal(log[:64], olog, err_msg=name)


def test_outlined_pipe_runs_at_t_control(irgl):
    """The control kernel's block size is T_control of the members: Elastic
    with Shrinkable(256) -> 256; Fixed(96) members -> 96 (a partial-warp block)."""
    with irgl.Context() as c:
        for blocks, want in (([(irgl.BLOCK_ELASTIC, 0), (irgl.BLOCK_SHRINKABLE, 256)], 256),
                             ([(irgl.BLOCK_FIXED, 96), (irgl.BLOCK_SHRINKABLE, 512)], 96),
                             ([(irgl.BLOCK_ELASTIC, 0), (irgl.BLOCK_ELASTIC, 0)], 1024)):
            p = c.pipe(64)
            p.init_scalars([0, 1, 2])
            c.op_reset(irgl.TEST_RETRY_ODD)  # fresh retry counts for each run
            stages = [dict(op=irgl.TEST_COUNTDOWN, guard=10, block=blocks[0]),
                      dict(op=irgl.TEST_RETRY_ODD, guard=1, block=blocks[1])]
            st, res = c.pipe_run(p, stages, outline=1)
            assert res.outlined == 1 and res.block == want
            q = c.pipe(64)
            q.init_scalars([0, 1, 2])
            c.op_reset(irgl.TEST_RETRY_ODD)
            st0, res0 = c.pipe_run(q, stages, outline=0)
            assert (st.rounds, st.launches, st.pushes, st.retries) == \
                (st0.rounds, st0.launches, st0.pushes, st0.retries)


def test_outline_empty_intersection(irgl):
    """Fixed(128) with Fixed(256): T_control is empty -> IRGL_E_OUTLINE_EMPTY when outlining is
    forced, host orchestration with the same results when it is not."""
    with irgl.Context() as c:
        stages = [dict(op=irgl.TEST_COUNTDOWN, guard=6, block=(irgl.BLOCK_FIXED, 128)),
                  dict(op=irgl.TEST_COUNTDOWN, guard=6, block=(irgl.BLOCK_FIXED, 256))]
        p = c.pipe(16)
        p.init_scalars([0])
        with pytest.raises(irgl.IrglError) as e:
            c.pipe_run(p, stages, outline=1)
        assert e.value.status == E_OUTLINE_EMPTY
        st, res = c.pipe_run(p, stages, outline=-1)
        assert res.outlined == 0 and st.rounds == 3 and p.size() == 0  # 0->1->2 ; 2->3->4 ; 4->5->{}


def test_outlined_pipe_rejects_graph_members(irgl, oracle):
    og = oracle.rmat(8)
    with irgl.Context() as c:
        g = c.graph_from_csr(og.row_ptr, og.col, og.weight)
        p = c.pipe(g.n)
        s = int(og.sources(1)[0])
        p.init_scalars([s])
        c.op_reset(irgl.BFS, g, p)
        with pytest.raises(irgl.IrglError):
            c.pipe_run(p, [dict(op=irgl.BFS)], graph=g, outline=1)
        # host-orchestrated Pipe { Invoke BFS } looping until empty == Listing 2 without LEVEL++
        st, res = c.pipe_run(p, [dict(op=irgl.BFS, round_start=1)], graph=g, outline=-1)
        assert res.outlined == 0 and p.size() == 0
        lv = c.read_result(irgl.BFS, g)
        assert lv[s] == 0 and set(np.unique(lv[lv != irgl.INF]).tolist()) <= {0, 1}
