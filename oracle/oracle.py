"""ctypes view of liboracle.so — the CPU ORACLE.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and ``--impl reference``)
may import this module, and only as the checker / the timed CPU reference arm.  The product
package ``paper_1607_05707_b200`` never imports it.  See oracle.h for the reference anchors
(/root/reference/SPEC.md:423-467).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

INF = 2147483647
OP_BFS, OP_SSSP, OP_CC, OP_PR, OP_TC, OP_CC_LP = 0, 1, 2, 3, 4, 5
OP_TEST_COUNTDOWN, OP_TEST_RETRY_ODD, OP_TEST_REDUCE, OP_TEST_NOPUSH, OP_TEST_PUSHPOP = (
    100, 101, 102, 103, 104)
OP_TEST_RESPAWN_ODD = 106
STAGE_INVOKE, STAGE_ITERATE = 0, 1
WHEN_ALWAYS, WHEN_PREV_TRUE, WHEN_PREV_FALSE = 0, 1, 2
RED_NONE, RED_ANY, RED_ALL = 0, 1, 2
COND_NONE, COND_WHILE, COND_UNTIL = 0, 1, 2
COMB_OR, COMB_AND = 0, 1


class Stats(C.Structure):
    _fields_ = [("rounds", C.c_int64), ("launches", C.c_int64), ("popped", C.c_int64),
                ("pushes", C.c_int64), ("retries", C.c_int64), ("edges", C.c_int64),
                ("serial_launches", C.c_int64), ("last_reduced", C.c_int32),
                ("trace_len", C.c_int32)]


class IterCfg(C.Structure):
    _fields_ = [("op", C.c_int), ("reduction", C.c_int), ("cond_mode", C.c_int),
                ("extra_comb", C.c_int), ("max_rounds", C.c_int64), ("round_start", C.c_int64),
                ("guard", C.c_int64), ("retry_serialize_after", C.c_int), ("threads", C.c_int),
                ("pr_d", C.c_double), ("pr_tol", C.c_double), ("capacity", C.c_int64)]


class PipeStage(C.Structure):
    _fields_ = [("op", C.c_int), ("kind", C.c_int), ("reduction", C.c_int), ("when", C.c_int),
                ("cond_mode", C.c_int), ("max_rounds", C.c_int64), ("guard", C.c_int64)]


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.cpp")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        P = C.c_void_p
        i64p = C.POINTER(C.c_int64)
        i32p = C.POINTER(C.c_int32)
        L.orc_rmat.restype = P
        L.orc_rmat.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_uint64]
        L.orc_grid.restype = P
        L.orc_grid.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64]
        L.orc_from_edges.restype = P
        L.orc_from_edges.argtypes = [C.c_int64, C.c_int64, i64p, i64p, i32p, C.c_int, C.c_uint64]
        L.orc_graph_free.argtypes = [P]
        for f in ("orc_graph_n", "orc_graph_m"):
            getattr(L, f).restype = C.c_int64
            getattr(L, f).argtypes = [P]
        L.orc_graph_row_ptr.restype = i64p
        L.orc_graph_row_ptr.argtypes = [P]
        L.orc_graph_col.restype = i32p
        L.orc_graph_col.argtypes = [P]
        L.orc_graph_weight.restype = i32p
        L.orc_graph_weight.argtypes = [P]
        L.orc_graph_checksum.restype = C.c_uint64
        L.orc_graph_checksum.argtypes = [P]
        L.orc_pick_sources.restype = C.c_int
        L.orc_pick_sources.argtypes = [P, C.c_uint64, C.c_int, i64p]
        L.orc_scramble.restype = C.c_uint64
        L.orc_scramble.argtypes = [C.c_uint64, C.c_int, C.c_uint64]
        L.orc_philox4x32.argtypes = [C.c_uint32] * 6 + [C.POINTER(C.c_uint32)]
        L.orc_bfs_serial.restype = C.c_int64
        L.orc_bfs_serial.argtypes = [P, C.c_int64, i32p]
        L.orc_sssp_dijkstra.argtypes = [P, C.c_int64, i32p]
        L.orc_cc_unionfind.argtypes = [P, i32p]
        L.orc_pagerank.restype = C.c_int
        L.orc_pagerank.argtypes = [P, C.c_double, C.c_double, C.c_int, C.POINTER(C.c_double)]
        L.orc_mst_kruskal.argtypes = [P, C.POINTER(C.c_uint64), i64p]
        L.orc_exclusive.argtypes = [i32p, C.c_int64, C.c_int, i32p]
        L.orc_tc_merge.restype = C.c_uint64
        L.orc_tc_merge.argtypes = [P]
        L.orc_iterate.restype = C.c_int
        L.orc_iterate.argtypes = [P, C.POINTER(IterCfg), i64p, C.c_int64, C.c_int, i32p, P,
                                  C.POINTER(Stats), i64p, C.c_int64, i64p, i64p]
        L.orc_reduce.restype = C.c_int
        L.orc_reduce.argtypes = [i32p, C.c_int64, C.c_int]
        L.orc_forall_assign.argtypes = [C.c_int64, C.c_int64, C.c_int, i64p]
        L.orc_bfs_bsp_omp.restype = C.c_int64
        L.orc_bfs_bsp_omp.argtypes = [P, C.c_int64, i32p, C.c_int, i64p]
        L.orc_sssp_bsp_omp.restype = C.c_int64
        L.orc_sssp_bsp_omp.argtypes = [P, C.c_int64, i32p, C.c_int, i64p]
        L.orc_max_threads.restype = C.c_int
        L.orc_sssp_defer_omp.restype = C.c_int64
        L.orc_sssp_defer_omp.argtypes = [P, C.c_int64, i32p, C.c_int, C.c_int64, i64p]
        L.orc_pipe_run.restype = C.c_int
        L.orc_pipe_run.argtypes = [C.POINTER(PipeStage), C.c_int, C.c_int, C.c_int64, C.c_int64,
                                   i64p, C.c_int64, i32p, C.c_int, i32p, i32p, i32p,
                                   C.POINTER(Stats), i64p, i64p]
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_cert_bfs.restype = C.c_int
        L.orc_cert_bfs.argtypes = [C.c_int64, i64p, i32p, C.c_int64, i32p]
        L.orc_cert_sssp.restype = C.c_int
        L.orc_cert_sssp.argtypes = [C.c_int64, i64p, i32p, i32p, C.c_int64, i32p]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class Graph:
    """Host CSR owned by the oracle (row_ptr int64[n+1], col int32[m], weight int32[m])."""

    def __init__(self, handle):
        if not handle:
            raise ValueError("oracle graph construction failed")
        self._h = handle
        L = lib()
        self.n = L.orc_graph_n(handle)
        self.m = L.orc_graph_m(handle)
        self.row_ptr = np.ctypeslib.as_array(L.orc_graph_row_ptr(handle), (self.n + 1,))
        self.col = np.ctypeslib.as_array(L.orc_graph_col(handle), (max(self.m, 1),))[: self.m]
        self.weight = np.ctypeslib.as_array(L.orc_graph_weight(handle), (max(self.m, 1),))[: self.m]

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_graph_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def checksum(self) -> int:
        return int(lib().orc_graph_checksum(self._h))

    def degrees(self):
        return np.diff(self.row_ptr)

    def sources(self, count=16, seed=7):
        out = np.zeros(count, dtype=np.int64)
        k = lib().orc_pick_sources(self._h, seed, count, _p(out, C.c_int64))
        return out[:k]


def rmat(scale, edge_factor=16, seed=1, wseed=11) -> Graph:
    return Graph(lib().orc_rmat(scale, edge_factor, seed, wseed))


def grid(W, H, diag=False, cut_period=0, perc_keep=1.0, perc_seed=5, wseed=11) -> Graph:
    return Graph(lib().orc_grid(W, H, int(diag), cut_period, int(round(perc_keep * 1e6)),
                                perc_seed, wseed))


def from_edges(n, u, v, w=None, symmetrise=True, wseed=11) -> Graph:
    u = np.ascontiguousarray(u, dtype=np.int64)
    v = np.ascontiguousarray(v, dtype=np.int64)
    wp = None
    if w is not None:
        w = np.ascontiguousarray(w, dtype=np.int32)
        wp = _p(w, C.c_int32)
    return Graph(lib().orc_from_edges(n, len(u), _p(u, C.c_int64), _p(v, C.c_int64), wp,
                                      int(symmetrise), wseed))


def scramble(v, scale, seed):
    return int(lib().orc_scramble(v, scale, seed))


def philox(c, k):
    out = (C.c_uint32 * 4)()
    lib().orc_philox4x32(*(list(c) + list(k)), out)
    return list(out)


def bfs(g: Graph, src: int):
    level = np.empty(g.n, dtype=np.int32)
    ecc = lib().orc_bfs_serial(g.handle, src, _p(level, C.c_int32))
    return level, int(ecc)


def sssp(g: Graph, src: int):
    dist = np.empty(g.n, dtype=np.int32)
    lib().orc_sssp_dijkstra(g.handle, src, _p(dist, C.c_int32))
    return dist


def cc(g: Graph):
    lab = np.empty(g.n, dtype=np.int32)
    lib().orc_cc_unionfind(g.handle, _p(lab, C.c_int32))
    return lab


def pagerank(g: Graph, d=0.85, tol=1e-6, max_iter=100):
    r = np.empty(g.n, dtype=np.float64)
    it = lib().orc_pagerank(g.handle, d, tol, max_iter, _p(r, C.c_double))
    return r, int(it)


def tc(g: Graph) -> int:
    return int(lib().orc_tc_merge(g.handle))


def mst(g: Graph):
    w, n = C.c_uint64(0), C.c_int64(0)
    lib().orc_mst_kruskal(g.handle, C.byref(w), C.byref(n))
    return int(w.value), int(n.value)


def exclusive(locks):
    """locks: int32 [nitems, k] (-1 unused); returns won[nitems] (priority = item index)."""
    lk = np.ascontiguousarray(locks, dtype=np.int32)
    won = np.zeros(lk.shape[0], dtype=np.int32)
    lib().orc_exclusive(_p(lk, C.c_int32), lk.shape[0], lk.shape[1], _p(won, C.c_int32))
    return won


def reduce(values, reduction):
    v = np.ascontiguousarray(values, dtype=np.int32)
    return bool(lib().orc_reduce(_p(v, C.c_int32), len(v), reduction))


def forall_assign(n, threads, blocked=False):
    out = np.zeros(n, dtype=np.int64)
    lib().orc_forall_assign(n, threads, int(blocked), _p(out, C.c_int64))
    return out


def iterate(g: Graph | None, op, init=(), *, reduction=RED_NONE, cond=COND_NONE,
            extra_comb=COMB_OR, max_rounds=0, round_start=1, guard=0, retry_serialize_after=4,
            threads=0, pr_d=0.85, pr_tol=1e-6, capacity=0, values=None, from_array=False,
            trace_cap=64):
    """One standalone Iterate with a fresh pipe context.

    Returns (node_out, Stats, trace[launch, in, out, retry], final_in)."""
    cfg = IterCfg(op, reduction, cond, extra_comb, max_rounds, round_start, guard,
                  retry_serialize_after, threads, pr_d, pr_tol, capacity)
    init = np.ascontiguousarray(np.asarray(init, dtype=np.int64))
    n = g.n if g is not None else 0
    cap = capacity if capacity > 0 else max(n, 1)
    if op == OP_PR:
        out = np.zeros(n, dtype=np.float64)
    elif op == OP_TC:
        out = np.zeros(1, dtype=np.uint64)
    elif op == OP_TEST_PUSHPOP:
        out = np.zeros(cap, dtype=np.int32)
    else:
        out = np.zeros(max(n, 1), dtype=np.int32)
    vals = None
    if values is not None:
        vals = np.ascontiguousarray(values, dtype=np.int32)
    trace = np.zeros((trace_cap, 4), dtype=np.int64)
    fin = np.zeros(cap, dtype=np.int64)
    fin_len = C.c_int64(cap)
    st = Stats()
    rc = lib().orc_iterate(g.handle if g is not None else None, C.byref(cfg), _p(init, C.c_int64),
                           len(init), int(from_array),
                           _p(vals, C.c_int32) if vals is not None else None,
                           out.ctypes.data_as(C.c_void_p), C.byref(st), _p(trace, C.c_int64),
                           trace_cap, _p(fin, C.c_int64), C.byref(fin_len))
    if rc != 0:
        raise RuntimeError(f"orc_iterate failed rc={rc}")
    if op == OP_TC:
        out = int(out[0])
    return out, st, trace[: st.trace_len].copy(), fin[: min(fin_len.value, cap)].copy()


def bfs_bsp_omp(g: Graph, src: int, threads=0):
    level = np.empty(g.n, dtype=np.int32)
    e = C.c_int64(0)
    r = lib().orc_bfs_bsp_omp(g.handle, src, _p(level, C.c_int32), threads, C.byref(e))
    return level, int(r), int(e.value)


def sssp_bsp_omp(g: Graph, src: int, threads=0):
    dist = np.empty(g.n, dtype=np.int32)
    e = C.c_int64(0)
    r = lib().orc_sssp_bsp_omp(g.handle, src, _p(dist, C.c_int32), threads, C.byref(e))
    return dist, int(r), int(e.value)


def sssp_defer_omp(g: Graph, src: int, threads=0, defer_k=1024):
    dist = np.empty(g.n, dtype=np.int32)
    e = C.c_int64(0)
    r = lib().orc_sssp_defer_omp(g.handle, src, _p(dist, C.c_int32), threads, defer_k, C.byref(e))
    return dist, int(r), int(e.value)


def set_threads(t: int):
    lib().orc_set_threads(int(t))


def max_threads() -> int:
    return int(lib().orc_max_threads())


def cert_bfs(row_ptr, col, src: int, level) -> int:
    """0 when `level` is the hop distance from src on the symmetric CSR (see oracle.h)."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    cl = np.ascontiguousarray(col, dtype=np.int32)
    lv = np.ascontiguousarray(level, dtype=np.int32)
    return int(lib().orc_cert_bfs(len(rp) - 1, _p(rp, C.c_int64), _p(cl, C.c_int32), src,
                                  _p(lv, C.c_int32)))


def cert_sssp(row_ptr, col, w, src: int, dist) -> int:
    """0 when `dist` is the shortest-path distance from src (symmetric weights; see oracle.h)."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    cl = np.ascontiguousarray(col, dtype=np.int32)
    ww = np.ascontiguousarray(w, dtype=np.int32)
    d = np.ascontiguousarray(dist, dtype=np.int32)
    return int(lib().orc_cert_sssp(len(rp) - 1, _p(rp, C.c_int64), _p(cl, C.c_int32),
                                   _p(ww, C.c_int32), src, _p(d, C.c_int32)))


def pipe_run(stages, init, cap, *, once=False, max_rounds=0, values=None, retry_serialize_after=4):
    """Multi-member Pipe of test operators (see oracle.h).  stages: dicts with op, kind,
    reduction, when, cond_mode, max_rounds, guard.  Returns (stats, final_in, rcount, log,
    stage_reduced)."""
    n = len(stages)
    arr = (PipeStage * n)(*[PipeStage(d.get("op"), d.get("kind", STAGE_INVOKE),
                                      d.get("reduction", RED_NONE), d.get("when", WHEN_ALWAYS),
                                      d.get("cond_mode", COND_NONE), d.get("max_rounds", 0),
                                      d.get("guard", 0)) for d in stages])
    init = np.ascontiguousarray(np.asarray(init, dtype=np.int64))
    vals = np.ascontiguousarray(values, dtype=np.int32) if values is not None else None
    rc = np.zeros(cap, dtype=np.int32)
    log = np.zeros(cap, dtype=np.int32)
    red = np.zeros(n, dtype=np.int32)
    fin = np.zeros(cap, dtype=np.int64)
    fl = C.c_int64(cap)
    st = Stats()
    r = lib().orc_pipe_run(arr, n, int(once), max_rounds, cap, _p(init, C.c_int64), len(init),
                           _p(vals, C.c_int32) if vals is not None else None, retry_serialize_after,
                           _p(rc, C.c_int32), _p(log, C.c_int32), _p(red, C.c_int32), C.byref(st),
                           _p(fin, C.c_int64), C.byref(fl))
    if r != 0:
        raise RuntimeError(f"orc_pipe_run failed rc={r}")
    return st, fin[: min(fl.value, cap)].copy(), rc, log, red
