"""IrGL source front end: parse_source + recognition of the
plain kernels as runtime operators + run_host driving the GPU runtime.

CPU tests: parsing, diagnostics with stable rule ids, pretty-print round trip, recognition of the
golden corpus (tests/golden/irgl/*.irgl), the frontend.h exports and the irglc CLI's `check`.
GPU tests: run_host of every corpus program against the oracle, including the SPEC's own example
(Listing 2 on a 5-node path, src = 0 -> [0, 1, 2, 3, 4])."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CORPUS = os.path.join(ROOT, "tests", "golden", "irgl")
IRGLC = os.path.join(ROOT, "paper_1607_05707_b200", "irglc")


def corpus(name):
    with open(os.path.join(CORPUS, name)) as f:
        return f.read()


EXPECT = {  # file -> {kernel: op name or None (not recognised) or "host"}
    "bfs_listing2.irgl": {"BFS": "BFS"},
    "sssp.irgl": {"SSSP": "SSSP"},
    "cc_lp.irgl": {"CC": "CC_LP"},
    "pagerank.irgl": {"PR": "PR"},
    "pipe_bfs.irgl": {"BFS": "BFS", "Helper": None, "main": "host"},
}


def test_frontend_header_exports(irgl):
    src = open(os.path.join(ROOT, "include", "irgl", "frontend.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    syms = sorted(set(re.findall(r"\b(irgl_[a-z0-9_]+)\s*\(", src)))
    assert syms == sorted(irgl.runtime.FRONTEND_EXPORTS)
    out = subprocess.check_output(["nm", "-D", "--defined-only", irgl.LIB_PATH]).decode()
    exported = set(re.findall(r" T (irgl_\w+)", out))
    assert not [s for s in syms if s not in exported]


@pytest.mark.parametrize("name", sorted(EXPECT))
def test_corpus_recognised(irgl, name):
    m = irgl.Module(corpus(name), name)
    ops = {irgl.BFS: "BFS", irgl.SSSP: "SSSP", irgl.CC_LP: "CC_LP", irgl.PR: "PR"}
    got = {k: ("host" if host else ops.get(op)) for k, op, field, host in m.kernels()}
    assert got == EXPECT[name]


@pytest.mark.parametrize("name", sorted(EXPECT))
def test_pretty_print_round_trip(irgl, name):
    """pretty_print / parse_source round trip: a fixed point after one cycle,
    and the recognised roles survive it."""
    m = irgl.Module(corpus(name), name)
    p1 = m.pretty()
    m2 = irgl.Module(p1, name)
    assert m2.pretty() == p1
    assert m2.kernels() == m.kernels()


def test_listing2_fields(irgl):
    m = irgl.Module(corpus("bfs_listing2.irgl"))
    (name, op, field, host), = m.kernels()
    assert (name, op, field, host) == ("BFS", irgl.BFS, "level", False)


@pytest.mark.parametrize("src,rule", [
    # the paper's Listing 2 verbatim lacks the outer ForAll's closing brace
    ("Kernel BFS(graph, LEVEL) {\n ForAll(i In wl) {\n n = wl.pop(i)\n}\nLEVEL=0\n", "E102"),
    ("Kernel f() { }\nKernel f() { }\n", "E007"),
    ("Kernel f() { ForAll(i In wl) { x = wl.top(i) } }", "E103"),
    ("Kernel f() { wl.clear() }", "E103"),
    ("Kernel f() { x = @ }", "E101"),
    ("Iterate While Maybe K(g);", "E102"),
])
def test_diagnostics(irgl, src, rule):
    with pytest.raises(irgl.IrglError) as ei:
        irgl.Module(src, "t.irgl")
    assert f"error[{rule}]" in str(ei.value)
    assert re.search(r"t\.irgl:\d+:\d+: error\[", str(ei.value))


def test_unrecognised_kernel_is_not_silently_run(irgl):
    m = irgl.Module("Kernel K(g) { ForAll(n In g.nodes) { x = 1 } }\nInvoke K(g);\n")
    assert m.kernels() == [("K", -1, "", False)]


def test_irglc_check(irgl):
    out = subprocess.run([IRGLC, "check", os.path.join(CORPUS, "pipe_bfs.irgl")], capture_output=True,
                         text=True, timeout=60)
    assert out.returncode == 0, out.stderr
    assert out.stdout.split("\n")[:3] == ["BFS: BFS", "Helper: plain (not recognised)", "main: host"]
    bad = subprocess.run([IRGLC, "check", "/nonexistent.irgl"], capture_output=True, text=True, timeout=60)
    assert bad.returncode == 2
    usage = subprocess.run([IRGLC], capture_output=True, text=True, timeout=60)
    assert usage.returncode == 2


# ---------------------------------------------------------------------------------------------
# GPU: run_host drives the runtime
def _upload(ctx, og):
    return ctx.graph_from_csr(og.row_ptr, og.col, og.weight)


@pytest.mark.gpu
def test_listing2_path5_spec_example(ctx, irgl, oracle):
    """SPEC.md:438 / :523: Listing 2 on a 5-node path, src = 0 -> levels [0,1,2,3,4]; the Iterate
    made ecc+1 = 5 invocations, so between_rounds ran 5 times (LEVEL = 5)."""
    og = oracle.from_edges(5, [0, 1, 2, 3], [1, 2, 3, 4])
    g = _upload(ctx, og)
    m = irgl.Module(corpus("bfs_listing2.irgl"))
    info = m.run_host(ctx, g, src=0)
    assert info["last_op"] == irgl.BFS and info["invocations"] == 5
    assert ctx.read_result(irgl.BFS, g).tolist() == [0, 1, 2, 3, 4]
    assert m.scalar("LEVEL") == 5


@pytest.mark.gpu
def test_run_host_corpus_parity(ctx, irgl, oracle):
    og = oracle.rmat(12)
    g = _upload(ctx, og)
    s = int(og.sources(1)[0])
    irgl.Module(corpus("bfs_listing2.irgl")).run_host(ctx, g, src=s)
    np.testing.assert_array_equal(ctx.read_result(irgl.BFS, g), oracle.bfs(og, s)[0])
    irgl.Module(corpus("sssp.irgl")).run_host(ctx, g, src=s)
    np.testing.assert_array_equal(ctx.read_result(irgl.SSSP, g), oracle.sssp(og, s))
    irgl.Module(corpus("cc_lp.irgl")).run_host(ctx, g)
    np.testing.assert_array_equal(ctx.read_result(irgl.CC_LP, g), oracle.cc(og))
    info = irgl.Module(corpus("pagerank.irgl")).run_host(ctx, g)
    assert info["last_op"] == irgl.PR
    ref, _ = oracle.pagerank(og)
    r = ctx.read_result(irgl.PR, g)
    assert np.abs(r - ref).sum() / np.abs(ref).sum() < 1e-6


@pytest.mark.gpu
def test_run_host_pipe_entry_two_sources(ctx, irgl, oracle):
    og = oracle.rmat(11)
    g = _upload(ctx, og)
    s1, s2 = (int(x) for x in og.sources(2))
    m = irgl.Module(corpus("pipe_bfs.irgl"))
    info = m.run_host(ctx, g, entry="main", src=s1, src2=s2)
    ref = np.minimum(oracle.bfs(og, s1)[0], oracle.bfs(og, s2)[0])
    np.testing.assert_array_equal(ctx.read_result(irgl.BFS, g), ref)
    assert m.scalar("rounds") == info["invocations"]


@pytest.mark.gpu
def test_run_host_unsupported_kernel(ctx, irgl, oracle):
    g = _upload(ctx, oracle.from_edges(3, [0, 1], [1, 2]))
    m = irgl.Module("Kernel K(g) { ForAll(n In g.nodes) { x = 1 } }\nInvoke K(g);\n", "u.irgl")
    with pytest.raises(irgl.IrglError) as ei:
        m.run_host(ctx, g)
    assert "E_UNSUPPORTED" in str(ei.value) and ei.value.status == irgl.runtime.E_UNSUPPORTED


@pytest.mark.gpu
def test_irglc_run(irgl, oracle, tmp_path):
    og = oracle.from_edges(6, [0, 1, 2, 3, 4], [1, 2, 3, 4, 5])
    el = tmp_path / "path.txt"
    el.write_text("6 5\n" + "".join(f"{u} {u + 1}\n" for u in range(5)))
    out = subprocess.run([IRGLC, "run", os.path.join(CORPUS, "bfs_listing2.irgl"), "--graph", str(el),
                          "--bind", "src=2"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    got = [int(l.split()[1]) for l in out.stdout.strip().split("\n")]
    assert got == oracle.bfs(og, 2)[0].tolist() == [2, 1, 0, 1, 2, 3]
