"""Python binding of libirgl_rt.so (include/irgl/rt.h) — the host-side mirror of IrGL's operator
API for the worklist graph hot path.

IrGL construct (reference/proj/core/include/irgl/ast.hpp)    here
-----------------------------------------------------------   ------------------------------------
Pipe [Once] { ... }  with WorklistInit (ast.hpp:100-110,206)  Context.pipe(size) + Pipe.init_*
Invoke kernel(args) [Any|All]       (ast.hpp:180-184)         Context.invoke(op, graph, pipe, ...)
Iterate [While|Until Any|All] ... Initial [...] {between}     Context.iterate(op, graph, pipe, ...)
  (ast.hpp:186-204)
ReduceAndReturn / Reduction {Any, All} (ast.hpp:90,176-178)   reduction=ANY|ALL, returned value
Retry / Respawn (ast.hpp:169-174)                             retry worklist inside Invoke
SyncRunningThreads / outlining    outline=True (persistent kernel)
t_control                                  t_control(constraints)

Errors are values in the C-ABI; here they raise IrglError carrying the stable rule id
("E_WL_OVERFLOW: ...").  There is no CPU fallback: if the shared library or a CUDA device is
missing, constructing a Context raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libirgl_rt.so")

INF = 2147483647
# irgl_status_t
OK, E_INVALID, E_USAGE, E_OOM, E_WL_OVERFLOW, E_OCCUPANCY, E_OUTLINE_EMPTY, E_CUDA, E_NCCL, \
    E_UNSUPPORTED = range(10)
STATUS_NAMES = {0: "OK", 1: "E_INVALID", 2: "E_USAGE", 3: "E_OOM", 4: "E_WL_OVERFLOW",
                5: "E_OCCUPANCY", 6: "E_OUTLINE_EMPTY", 7: "E_CUDA", 8: "E_NCCL",
                9: "E_UNSUPPORTED", 10: "E_RANGE"}
# enums
RED_NONE, RED_ANY, RED_ALL = 0, 1, 2
WL_IN, WL_OUT, WL_RETRY = 0, 1, 2
COND_NONE, COND_WHILE, COND_UNTIL = 0, 1, 2
COMB_OR, COMB_AND = 0, 1
MAP_CONSECUTIVE, MAP_BLOCKED = 0, 1
BFS, SSSP, CC, PR, TC, CC_LP, MST = 0, 1, 2, 3, 4, 5, 6
TEST_COUNTDOWN, TEST_RETRY_ODD, TEST_REDUCE, TEST_NOPUSH, TEST_PUSHPOP, TEST_FORALL_MAP = (
    100, 101, 102, 103, 104, 105)
TEST_RESPAWN_ODD = 106
TEST_ATOMIC, TEST_ATOMIC_ELSE, TEST_EXCLUSIVE = 107, 108, 109
GEN_RMAT, GEN_GRID = 0, 1
BLOCK_ELASTIC, BLOCK_SHRINKABLE, BLOCK_FIXED = 0, 1, 2


class IrglError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(message or STATUS_NAMES.get(status, str(status)))
        self.status = status
        self.message = message


class Config(C.Structure):
    _fields_ = [("outline", C.c_int32), ("blocks_per_sm", C.c_int32),
                ("retry_serialize_after", C.c_int32), ("warp_threshold", C.c_int32),
                ("cta_threshold", C.c_int32), ("chunk_edges", C.c_int32),
                ("l2_persist", C.c_int32), ("logical_partitions", C.c_int32),
                ("dense_div", C.c_int32), ("bfs_bitmap_min_n", C.c_int32), ("reserved", C.c_int32 * 6)]


class OpArgs(C.Structure):
    _fields_ = [("round_start", C.c_int64), ("guard", C.c_int64), ("pr_damping", C.c_double),
                ("pr_tol", C.c_double), ("values", C.POINTER(C.c_int32)), ("nvalues", C.c_int64),
                ("mapping", C.c_int32), ("threads", C.c_int32), ("delta", C.c_int32),
                ("direction", C.c_int32), ("defer", C.c_int32), ("reserved", C.c_int32 * 3)]


class IterateOpts(C.Structure):
    _fields_ = [("cond_mode", C.c_int32), ("reduction", C.c_int32), ("extra_comb", C.c_int32),
                ("outline", C.c_int32), ("max_rounds", C.c_int64), ("reset", C.c_int32),
                ("reserved", C.c_int32 * 5)]


class IterStats(C.Structure):
    _fields_ = [("rounds", C.c_int64), ("launches", C.c_int64), ("popped", C.c_int64),
                ("pushes", C.c_int64), ("retries", C.c_int64), ("edges", C.c_int64),
                ("remote_updates", C.c_int64), ("exchange_bytes", C.c_int64),
                ("serial_launches", C.c_int64), ("last_reduced", C.c_int32),
                ("outlined", C.c_int32), ("device_ms", C.c_double), ("kernel_ms", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class GenSpec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("scale", C.c_int32), ("edge_factor", C.c_int32),
                ("width", C.c_int32), ("height", C.c_int32), ("diag", C.c_int32),
                ("cut_period", C.c_int32), ("perc_keep_ppm", C.c_int32), ("seed", C.c_uint64),
                ("wseed", C.c_uint64), ("perc_seed", C.c_uint64), ("reserved", C.c_int32 * 8)]


class GraphInfo(C.Structure):
    _fields_ = [("n", C.c_int64), ("m", C.c_int64), ("local_n", C.c_int64),
                ("local_m", C.c_int64), ("lo", C.c_int64), ("hi", C.c_int64),
                ("partitions", C.c_int32), ("has_weights", C.c_int32), ("max_degree", C.c_int64)]


class BlockConstraint(C.Structure):
    _fields_ = [("kind", C.c_int32), ("value", C.c_int32)]


class PipeStage(C.Structure):
    """irgl_pipe_stage: one member statement of a Pipe body (rt.h)."""
    _fields_ = [("op", C.c_int32), ("kind", C.c_int32), ("reduction", C.c_int32),
                ("when", C.c_int32), ("cond_mode", C.c_int32), ("reserved0", C.c_int32),
                ("max_rounds", C.c_int64), ("block", BlockConstraint), ("args", OpArgs)]


class PipeOpts(C.Structure):
    _fields_ = [("once", C.c_int32), ("outline", C.c_int32), ("max_rounds", C.c_int64),
                ("reserved", C.c_int32 * 4)]


class PipeResult(C.Structure):
    _fields_ = [("outlined", C.c_int32), ("block", C.c_int32), ("last_reduced", C.c_int32),
                ("reserved0", C.c_int32), ("stage_reduced", C.c_int32 * 8)]


STAGE_INVOKE, STAGE_ITERATE = 0, 1
WHEN_ALWAYS, WHEN_PREV_TRUE, WHEN_PREV_FALSE = 0, 1, 2
BLOCK_ELASTIC, BLOCK_SHRINKABLE, BLOCK_FIXED = 0, 1, 2

# every symbol include/irgl/rt.h declares (tests check the .so exports all of them)
EXPORTS = [
    "irgl_ctx_create", "irgl_nccl_unique_id", "irgl_ctx_create_nccl", "irgl_ctx_create_transport",
    "irgl_ctx_destroy",
    "irgl_ctx_sync", "irgl_last_error", "irgl_abi_version", "irgl_graph_create_csr",
    "irgl_graph_generate", "irgl_graph_read_edgelist", "irgl_graph_info_get", "irgl_graph_download", "irgl_graph_destroy",
    "irgl_pipe_create", "irgl_pipe_init_scalars", "irgl_pipe_init_from_array",
    "irgl_pipe_init_range", "irgl_pipe_size", "irgl_pipe_read", "irgl_pipe_destroy",
    "irgl_op_reset", "irgl_invoke", "irgl_iterate", "irgl_read_result", "irgl_t_control",
    "irgl_op_plan", "irgl_event_record", "irgl_event_elapsed", "irgl_launch_count",
    "irgl_read_result_async", "irgl_results_wait", "irgl_graph_relabel", "irgl_graph_perm",
    "irgl_traverse_batch", "irgl_pipe_run",
]

# every symbol include/irgl/frontend.h declares
FRONTEND_EXPORTS = [
    "irgl_module_parse", "irgl_module_destroy", "irgl_module_kernel_count", "irgl_module_kernel_info",
    "irgl_module_print", "irgl_run_host", "irgl_module_scalar",
]

_lib = None


class RunInfo(C.Structure):
    _fields_ = [("last_op", C.c_int32), ("last_reduced", C.c_int32), ("invocations", C.c_int64),
                ("orchestrations", C.c_int64), ("reserved", C.c_int64 * 4)]


def load_library(path: str | None = None):
    """Load libirgl_rt.so.  Raises (no fallback) if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    # IRGL_LIB: load an alternative build (tuning experiments only; same C-ABI)
    path = path or os.environ.get("IRGL_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (there is no CPU fallback for the IrGL GPU runtime)")
    L = C.CDLL(path)
    P, i64, i32 = C.c_void_p, C.c_int64, C.c_int32
    i64p, i32p = C.POINTER(C.c_int64), C.POINTER(C.c_int32)
    pp = C.POINTER(C.c_void_p)
    sig = {
        "irgl_ctx_create": ([C.POINTER(C.c_int), C.c_int, C.POINTER(Config), pp], i32),
        "irgl_nccl_unique_id": ([P], i32),
        "irgl_ctx_create_nccl": ([C.c_int, C.c_int, C.c_int, P, C.POINTER(Config), pp], i32),
        "irgl_ctx_create_transport": ([C.c_int, C.c_int, C.c_int, P, C.POINTER(Config), pp], i32),
        "irgl_ctx_destroy": ([P], i32),
        "irgl_ctx_sync": ([P], i32),
        "irgl_last_error": ([P], C.c_char_p),
        "irgl_abi_version": ([], C.c_int),
        "irgl_graph_create_csr": ([P, i64, i64, i64p, i32p, i32p, pp], i32),
        "irgl_graph_generate": ([P, C.POINTER(GenSpec), pp], i32),
        "irgl_graph_read_edgelist": ([P, C.c_char_p, C.c_int, pp], i32),
        "irgl_graph_info_get": ([P, C.POINTER(GraphInfo)], i32),
        "irgl_graph_download": ([P, i64p, i32p, i32p], i32),
        "irgl_graph_destroy": ([P], i32),
        "irgl_pipe_create": ([P, i64, pp], i32),
        "irgl_pipe_init_scalars": ([P, i64p, i64], i32),
        "irgl_pipe_init_from_array": ([P, i64p, i64], i32),
        "irgl_pipe_init_range": ([P, i64, i64], i32),
        "irgl_pipe_size": ([P, C.c_int, i64p], i32),
        "irgl_pipe_read": ([P, C.c_int, i64p, i64, i64p], i32),
        "irgl_pipe_destroy": ([P], i32),
        "irgl_op_reset": ([P, P, C.c_int, C.POINTER(OpArgs), P], i32),
        "irgl_invoke": ([P, P, P, C.c_int, C.POINTER(OpArgs), C.c_int, i32p,
                         C.POINTER(IterStats)], i32),
        "irgl_iterate": ([P, P, P, C.c_int, C.POINTER(OpArgs), C.POINTER(IterateOpts),
                          C.POINTER(IterStats)], i32),
        "irgl_read_result": ([P, P, C.c_int, P, C.c_size_t], i32),
        "irgl_read_result_async": ([P, P, C.c_int, P, C.c_size_t], i32),
        "irgl_results_wait": ([P], i32),
        "irgl_traverse_batch": ([P, P, P, C.c_int, i64p, C.c_int32, C.POINTER(OpArgs),
                                 C.POINTER(IterateOpts), C.POINTER(C.c_void_p), C.c_size_t,
                                 C.POINTER(IterStats)], i32),
        "irgl_graph_relabel": ([P, P], i32),
        "irgl_graph_perm": ([P, i32p], i32),
        "irgl_t_control": ([C.POINTER(BlockConstraint), C.c_int, i32p], i32),
        "irgl_op_plan": ([P, C.c_int, C.POINTER(BlockConstraint), i32p, i32p], i32),
        "irgl_event_record": ([P, C.c_int], i32),
        "irgl_event_elapsed": ([P, C.c_int, C.c_int, C.POINTER(C.c_double)], i32),
        "irgl_launch_count": ([], i64),
        "irgl_pipe_run": ([P, P, P, C.POINTER(PipeStage), C.c_int32, C.POINTER(PipeOpts),
                           C.POINTER(IterStats), C.POINTER(PipeResult)], i32),
        # IrGL source front end (include/irgl/frontend.h)
        "irgl_module_parse": ([C.c_char_p, C.c_char_p, pp, C.c_char_p, C.c_size_t], i32),
        "irgl_module_destroy": ([P], i32),
        "irgl_module_kernel_count": ([P], C.c_int),
        "irgl_module_kernel_info": ([P, C.c_int, C.c_char_p, C.c_size_t, i32p, C.c_char_p, C.c_size_t,
                                    i32p], i32),
        "irgl_module_print": ([P, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)], i32),
        "irgl_run_host": ([P, P, C.c_char_p, P, C.POINTER(C.c_char_p), C.POINTER(C.c_double), C.c_int,
                           C.POINTER(RunInfo), C.c_char_p, C.c_size_t], i32),
        "irgl_module_scalar": ([P, C.c_char_p, C.POINTER(C.c_double)], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _err(ctx_handle=None) -> str:
    m = load_library().irgl_last_error(ctx_handle)
    return m.decode() if m else ""


def _check(st, ctx_handle=None):
    if st != OK:
        raise IrglError(st, _err(ctx_handle))


def _i64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def _p64(a):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def t_control(constraints) -> int:
    """T_control = max(intersection of T_k) over (kind, value) pairs."""
    arr = (BlockConstraint * len(constraints))(*[BlockConstraint(k, v) for k, v in constraints])
    out = C.c_int32(0)
    _check(load_library().irgl_t_control(arr, len(constraints), C.byref(out)))
    return out.value


def launch_count() -> int:
    """Kernels launched by libirgl_rt.so in this process so far."""
    return int(load_library().irgl_launch_count())


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(load_library().irgl_nccl_unique_id(buf))
    return buf.raw


def _op_args(round_start=0, guard=0, pr_damping=0.0, pr_tol=0.0, values=None, mapping=0,
             threads=0, delta=-1, direction=0, defer=-1):
    a = OpArgs()
    a.delta = delta
    a.defer = defer
    a.direction = direction
    a.round_start = round_start
    a.guard = guard
    a.pr_damping = pr_damping
    a.pr_tol = pr_tol
    a.mapping = mapping
    a.threads = threads
    keep = None
    if values is not None:
        keep = np.ascontiguousarray(values, dtype=np.int32)
        a.values = keep.ctypes.data_as(C.POINTER(C.c_int32))
        a.nvalues = len(keep)
    return a, keep


@dataclass
class Stats:
    rounds: int
    launches: int
    popped: int
    pushes: int
    retries: int
    edges: int
    remote_updates: int
    exchange_bytes: int
    serial_launches: int
    last_reduced: int
    outlined: int
    device_ms: float
    kernel_ms: float


class Context:
    """irgl_ctx: one host thread, one or more vertex partitions."""

    def __init__(self, devices=(0,), *, outline=-1, blocks_per_sm=0, retry_serialize_after=0,
                 warp_threshold=0, cta_threshold=0, chunk_edges=0, logical_partitions=0,
                 dense_div=0, bfs_bitmap_min_n=0, l2_persist=0, nccl=None, transport=None):
        L = load_library()
        cfg = Config()
        cfg.outline = outline
        cfg.blocks_per_sm = blocks_per_sm
        cfg.retry_serialize_after = retry_serialize_after
        cfg.warp_threshold = warp_threshold
        cfg.cta_threshold = cta_threshold
        cfg.chunk_edges = chunk_edges
        cfg.logical_partitions = logical_partitions
        cfg.dense_div = dense_div
        cfg.bfs_bitmap_min_n = bfs_bitmap_min_n
        cfg.l2_persist = l2_persist
        h = C.c_void_p()
        self._transport = transport
        if transport is not None:  # dist.TorchTransport (or any object with .struct/.rank/...)
            _check(L.irgl_ctx_create_transport(transport.device, transport.rank, transport.nranks,
                                               C.byref(transport.struct), C.byref(cfg), C.byref(h)))
        elif nccl is not None:  # (device, rank, nranks, uid)
            dev, rank, nranks, uid = nccl
            _check(L.irgl_ctx_create_nccl(dev, rank, nranks, uid, C.byref(cfg), C.byref(h)))
        else:
            devs = (C.c_int * len(devices))(*devices)
            _check(L.irgl_ctx_create(devs, len(devices), C.byref(cfg), C.byref(h)))
        self._h = h
        self._lib = L

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            self._lib.irgl_ctx_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, st):
        _check(st, self._h)

    def sync(self):
        self._chk(self._lib.irgl_ctx_sync(self._h))

    # ---- graphs ----
    def graph_from_csr(self, row_ptr, col, weight=None) -> "Graph":
        rp = _i64(row_ptr)
        cl = np.ascontiguousarray(col, dtype=np.int32)
        n = len(rp) - 1
        wp = None
        if weight is not None:
            wt = np.ascontiguousarray(weight, dtype=np.int32)
            wp = wt.ctypes.data_as(C.POINTER(C.c_int32))
        h = C.c_void_p()
        self._chk(self._lib.irgl_graph_create_csr(self._h, n, len(cl), _p64(rp),
                                                  cl.ctypes.data_as(C.POINTER(C.c_int32)), wp,
                                                  C.byref(h)))
        return Graph(self, h)

    def generate_rmat(self, scale, edge_factor=16, seed=1, wseed=11) -> "Graph":
        s = GenSpec()
        s.kind, s.scale, s.edge_factor, s.seed, s.wseed = GEN_RMAT, scale, edge_factor, seed, wseed
        return self._generate(s)

    def generate_grid(self, W, H, diag=False, cut_period=0, perc_keep=1.0, perc_seed=5,
                      wseed=11) -> "Graph":
        s = GenSpec()
        s.kind, s.width, s.height, s.diag, s.cut_period = GEN_GRID, W, H, int(diag), cut_period
        s.perc_keep_ppm = int(round(perc_keep * 1e6))
        s.perc_seed, s.wseed = perc_seed, wseed
        return self._generate(s)

    def read_edgelist(self, path, symmetrise=True) -> "Graph":
        """Text edge list: 'N M' then 'u v [w]' lines; CSR built on the device."""
        h = C.c_void_p()
        self._chk(self._lib.irgl_graph_read_edgelist(self._h, str(path).encode(), int(symmetrise),
                                                     C.byref(h)))
        return Graph(self, h)

    def _generate(self, spec) -> "Graph":
        h = C.c_void_p()
        self._chk(self._lib.irgl_graph_generate(self._h, C.byref(spec), C.byref(h)))
        return Graph(self, h)

    # ---- pipe contexts ----
    def pipe(self, capacity) -> "Pipe":
        h = C.c_void_p()
        self._chk(self._lib.irgl_pipe_create(self._h, int(capacity), C.byref(h)))
        return Pipe(self, h, int(capacity))

    # ---- orchestration ----
    def op_reset(self, op, graph=None, pipe=None):
        a, _ = _op_args()
        self._chk(self._lib.irgl_op_reset(self._h, graph.handle if graph else None, op,
                                          C.byref(a), pipe.handle if pipe else None))

    def invoke(self, op, graph=None, pipe=None, *, reduction=RED_NONE, **args):
        """[Any|All(] Invoke op(args) [)] — returns (reduced or None, Stats)."""
        a, _keep = _op_args(**args)
        r = C.c_int32(-1)
        st = IterStats()
        self._chk(self._lib.irgl_invoke(self._h, pipe.handle if pipe else None,
                                        graph.handle if graph else None, op, C.byref(a),
                                        reduction, C.byref(r), C.byref(st)))
        red = None if reduction == RED_NONE else bool(r.value)
        return red, Stats(**st.as_dict())

    def iterate(self, op, graph=None, pipe=None, *, cond=COND_NONE, reduction=RED_NONE,
                extra_comb=COMB_OR, max_rounds=0, outline=-1, reset=True, **args) -> Stats:
        """Iterate [While|Until Any|All] op(args) ... — runs until `in` is empty."""
        a, _keep = _op_args(**args)
        o = IterateOpts()
        o.cond_mode, o.reduction, o.extra_comb = cond, reduction, extra_comb
        o.outline = -1 if outline is None else int(outline)
        o.max_rounds, o.reset = max_rounds, int(bool(reset))
        st = IterStats()
        self._chk(self._lib.irgl_iterate(self._h, pipe.handle if pipe else None,
                                         graph.handle if graph else None, op, C.byref(a),
                                         C.byref(o), C.byref(st)))
        return Stats(**st.as_dict())

    def run_pipe(self, pipe, body, once=False, max_rounds=None):
        """Pipe [Once] { body }: `body(ctx, pipe)` issues the
        Invokes/Iterates of the pipe, which all share the pipe context.  A looping Pipe repeats
        the body while `in` is non-empty at the start of the body; `Pipe Once` runs it once.
        Returns the number of body executions."""
        n = 0
        while True:
            if not once and pipe.size() == 0:
                break
            body(self, pipe)
            n += 1
            if once or (max_rounds is not None and n >= max_rounds):
                break
        return n

    def pipe_run(self, pipe, stages, *, graph=None, once=False, outline=-1, max_rounds=0):
        """Pipe [Once] { member statements } as one call (irgl_pipe_run): `stages` are dicts
        {op, kind=STAGE_INVOKE|STAGE_ITERATE, reduction, when=WHEN_*, cond, max_rounds,
        block=(BLOCK_*, value), **op args}.  outline=1 runs the whole Pipe as one cooperative
        control kernel at T_control (IRGL_E_OUTLINE_EMPTY when the members' block domains do
        not intersect), 0 host-orchestrated, -1 outlined when possible.
        Returns (Stats, PipeResult)."""
        arr = (PipeStage * len(stages))()
        keep = []
        for k, d in enumerate(stages):
            d = dict(d)
            st = arr[k]
            st.op = d.pop("op")
            st.kind = d.pop("kind", STAGE_INVOKE)
            st.reduction = d.pop("reduction", RED_NONE)
            st.when = d.pop("when", WHEN_ALWAYS)
            st.cond_mode = d.pop("cond", COND_NONE)
            st.max_rounds = d.pop("max_rounds", 0)
            bk, bv = d.pop("block", (BLOCK_ELASTIC, 0))
            st.block.kind, st.block.value = bk, bv
            a, kp = _op_args(**d)
            st.args = a
            keep.append(kp)
        o = PipeOpts()
        o.once, o.outline, o.max_rounds = int(bool(once)), int(outline), int(max_rounds)
        stt, res = IterStats(), PipeResult()
        self._chk(self._lib.irgl_pipe_run(self._h, pipe.handle, graph.handle if graph else None,
                                          arr, len(stages), C.byref(o), C.byref(stt), C.byref(res)))
        return Stats(**stt.as_dict()), res

    def read_result(self, op, graph=None, size=None):
        if op == TC:
            out = np.zeros(1, dtype=np.uint64)
        elif op == MST:
            out = np.zeros(2, dtype=np.uint64)
        elif op == PR:
            out = np.zeros(graph.n, dtype=np.float64)
        elif op >= 100:
            out = np.zeros(size, dtype=np.int32)
        else:
            out = np.zeros(graph.n, dtype=np.int32)
        self._chk(self._lib.irgl_read_result(self._h, graph.handle if graph else None, op,
                                             out.ctypes.data_as(C.c_void_p), out.nbytes))
        if op == MST:
            return int(out[0]), int(out[1])
        return int(out[0]) if op == TC else out

    def read_result_into(self, op, graph, out: np.ndarray):
        self._chk(self._lib.irgl_read_result(self._h, graph.handle, op,
                                             out.ctypes.data_as(C.c_void_p), out.nbytes))
        return out

    def read_result_async(self, op, graph, out: np.ndarray):
        """Queue the node result's copy into `out` (pinned to overlap) and return at once; the
        next traversal writes the graph's other label buffer.  Valid after results_wait()."""
        self._chk(self._lib.irgl_read_result_async(self._h, graph.handle, op,
                                                   out.ctypes.data_as(C.c_void_p), out.nbytes))
        return out

    def results_wait(self):
        self._chk(self._lib.irgl_results_wait(self._h))

    def traverse_batch(self, op, graph, pipe, sources, outs=None, *, outline=-1, **args):
        """irgl_traverse_batch: one single-source Iterate per source (Initial [s]); with `outs`
        (numpy arrays, may repeat) each node result is copied asynchronously into outs[i % len]
        and the call returns after the copies landed.  Returns one Stats per source."""
        src = _i64(sources)
        k = len(src)
        a, _keep = _op_args(**args)
        o = IterateOpts()
        o.cond_mode, o.reduction, o.extra_comb = COND_NONE, RED_NONE, COMB_OR
        o.outline, o.max_rounds, o.reset = int(outline), 0, 1
        st = (IterStats * max(k, 1))()
        ptrs = None
        if outs:
            ptrs = (C.c_void_p * k)(*[outs[i % len(outs)].ctypes.data for i in range(k)])
            nbytes = outs[0].nbytes
        self._chk(self._lib.irgl_traverse_batch(self._h, pipe.handle, graph.handle, op, _p64(src), k,
                                                C.byref(a), C.byref(o), ptrs, nbytes if outs else 0, st))
        return [Stats(**st[i].as_dict()) for i in range(k)]

    def event_record(self, slot):
        self._chk(self._lib.irgl_event_record(self._h, slot))

    def event_elapsed(self, a, b) -> float:
        ms = C.c_double(0)
        self._chk(self._lib.irgl_event_elapsed(self._h, a, b, C.byref(ms)))
        return ms.value

    def op_plan(self, op):
        bc = BlockConstraint()
        go, gf = C.c_int32(0), C.c_int32(0)
        self._chk(self._lib.irgl_op_plan(self._h, op, C.byref(bc), C.byref(go), C.byref(gf)))
        return (bc.kind, bc.value), go.value, gf.value


class Graph:
    """irgl_graph: device CSR (reference Value::Graph)."""

    def __init__(self, ctx: Context, handle):
        self.ctx = ctx
        self._h = handle
        info = GraphInfo()
        _check(ctx._lib.irgl_graph_info_get(handle, C.byref(info)), ctx.handle)
        self.info = info
        self.n = info.n
        self.m = info.m

    @property
    def handle(self):
        return self._h

    def relabel(self):
        """Degree-ordered relabelling (irgl_graph_relabel): faster traversals on graphs whose
        per-vertex state leaves L2; ids seen through this API are unchanged."""
        _check(self.ctx._lib.irgl_graph_relabel(self.ctx.handle, self._h), self.ctx.handle)
        return self

    def perm(self):
        out = np.empty(self.n, dtype=np.int32)
        _check(self.ctx._lib.irgl_graph_perm(self._h, out.ctypes.data_as(C.POINTER(C.c_int32))),
               self.ctx.handle)
        return out

    def download(self):
        rp = np.zeros(self.info.local_n + 1, dtype=np.int64) if self.info.partitions > 1 and \
            self.info.local_n != self.n else np.zeros(self.n + 1, dtype=np.int64)
        col = np.zeros(max(self.info.local_m, 1), dtype=np.int32)
        w = np.zeros(max(self.info.local_m, 1), dtype=np.int32)
        _check(self.ctx._lib.irgl_graph_download(self._h, _p64(rp),
                                                 col.ctypes.data_as(C.POINTER(C.c_int32)),
                                                 w.ctypes.data_as(C.POINTER(C.c_int32))),
               self.ctx.handle)
        return rp, col[: self.info.local_m], w[: self.info.local_m]

    def close(self):
        if self._h and self.ctx._h:
            self.ctx._lib.irgl_graph_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Pipe:
    """irgl_pipe: the pipe context {in, out, retry}."""

    def __init__(self, ctx: Context, handle, capacity):
        self.ctx = ctx
        self._h = handle
        self.capacity = capacity

    @property
    def handle(self):
        return self._h

    def init_scalars(self, items):
        a = _i64(items)
        _check(self.ctx._lib.irgl_pipe_init_scalars(self._h, _p64(a), len(a)), self.ctx.handle)

    def init_from_array(self, arr):
        a = _i64(arr)
        _check(self.ctx._lib.irgl_pipe_init_from_array(self._h, _p64(a), len(a)), self.ctx.handle)

    def init_range(self, begin, end):
        _check(self.ctx._lib.irgl_pipe_init_range(self._h, begin, end), self.ctx.handle)

    def size(self, which=WL_IN) -> int:
        out = C.c_int64(0)
        _check(self.ctx._lib.irgl_pipe_size(self._h, which, C.byref(out)), self.ctx.handle)
        return out.value

    def read(self, which=WL_IN):
        n = self.size(which)
        buf = np.zeros(max(n, 1), dtype=np.int64)
        cnt = C.c_int64(0)
        _check(self.ctx._lib.irgl_pipe_read(self._h, which, _p64(buf), len(buf), C.byref(cnt)),
               self.ctx.handle)
        return buf[: cnt.value]

    def close(self):
        if self._h and self.ctx._h:
            self.ctx._lib.irgl_pipe_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- convenience drivers (the IrGL programs of the north star, in host form) ------------------
def bfs(ctx: Context, graph: Graph, src: int, *, pipe: Pipe | None = None, outline=-1,
        direction=0):
    """Listing 2: LEVEL=0; Iterate BFS(graph, LEVEL) Initial [src] { LEVEL++ }.
    direction=1: direction-optimising variant (same levels)."""
    p = pipe or ctx.pipe(graph.n)
    p.init_scalars([src])
    st = ctx.iterate(BFS, graph, p, outline=outline, round_start=1, direction=direction)
    return ctx.read_result(BFS, graph), st


def sssp(ctx: Context, graph: Graph, src: int, *, pipe: Pipe | None = None, outline=-1,
         delta=-1, defer=-1):
    """Data-driven SSSP (IrGL form of Listing 2 with dist[n]+weight(e) and atomicMin).
    delta > 0: near-far piles; defer > 0: degree-scaled deferral budget; -1: runtime defaults.
    Same distances in every mode."""
    p = pipe or ctx.pipe(graph.n)
    p.init_scalars([src])
    st = ctx.iterate(SSSP, graph, p, outline=outline, delta=delta, defer=defer)
    return ctx.read_result(SSSP, graph), st


def cc(ctx: Context, graph: Graph):
    """Iterate While Any CC(graph): hook + compress until no hook happens."""
    st = ctx.iterate(CC, graph, None, cond=COND_WHILE, reduction=RED_ANY)
    return ctx.read_result(CC, graph), st


def cc_lp(ctx: Context, graph: Graph, *, outline=-1):
    p = ctx.pipe(graph.n)
    p.init_range(0, graph.n)  # Initial FromArray(all vertices)
    st = ctx.iterate(CC_LP, graph, p, outline=outline)
    return ctx.read_result(CC_LP, graph), st


def pagerank(ctx: Context, graph: Graph, d=0.85, tol=1e-6, max_iter=100, outline=-1):
    """Iterate While Any PR(graph) [Or rounds >= max_iter]."""
    st = ctx.iterate(PR, graph, None, cond=COND_WHILE, reduction=RED_ANY, max_rounds=max_iter,
                     extra_comb=COMB_OR, outline=outline, pr_damping=d, pr_tol=tol)
    return ctx.read_result(PR, graph), st


def mst(ctx: Context, graph: Graph):
    """Boruvka (Listing 1) under Iterate While Any: returns ((forest weight, edges), Stats)."""
    st = ctx.iterate(MST, graph, None, cond=COND_WHILE, reduction=RED_ANY)
    return ctx.read_result(MST, graph), st


def triangle_count(ctx: Context, graph: Graph):
    _, st = ctx.invoke(TC, graph)
    return ctx.read_result(TC, graph), st


# ---- IrGL source front end ----------------------------------------------------
class Module:
    """An IrGL program parsed by the runtime's front end (frontend.h): parse_source
    plus the recognition of each plain kernel as one of the runtime's operators."""

    def __init__(self, text: str, filename: str = "<input>"):
        L = load_library()
        self._lib = L
        h = C.c_void_p()
        diag = C.create_string_buffer(8192)
        st = L.irgl_module_parse(text.encode(), filename.encode(), C.byref(h), diag, len(diag))
        if st != OK:
            raise IrglError(st, diag.value.decode())
        self._h = h

    @classmethod
    def from_file(cls, path):
        with open(path) as f:
            return cls(f.read(), os.path.basename(path))

    def kernels(self):
        """[(name, op or -1, written field, is_host)]"""
        out = []
        for i in range(self._lib.irgl_module_kernel_count(self._h)):
            name, field = C.create_string_buffer(256), C.create_string_buffer(256)
            op, host = C.c_int32(), C.c_int32()
            _check(self._lib.irgl_module_kernel_info(self._h, i, name, 256, C.byref(op), field, 256,
                                                     C.byref(host)))
            out.append((name.value.decode(), op.value, field.value.decode(), bool(host.value)))
        return out

    def pretty(self) -> str:
        need = C.c_size_t(0)
        self._lib.irgl_module_print(self._h, None, 0, C.byref(need))
        buf = C.create_string_buffer(need.value)
        _check(self._lib.irgl_module_print(self._h, buf, need.value, None))
        return buf.value.decode()

    def run_host(self, ctx: "Context", graph: "Graph", entry: str | None = None, **bindings):
        """run_host: execute the host code; returns the RunInfo as a dict."""
        names = (C.c_char_p * max(len(bindings), 1))(*[k.encode() for k in bindings])
        vals = (C.c_double * max(len(bindings), 1))(*[float(v) for v in bindings.values()])
        info = RunInfo()
        diag = C.create_string_buffer(8192)
        st = self._lib.irgl_run_host(ctx.handle, self._h, entry.encode() if entry else None,
                                     graph.handle if graph else None, names, vals, len(bindings),
                                     C.byref(info), diag, len(diag))
        if st != OK:
            raise IrglError(st, diag.value.decode() or _err(ctx.handle))
        return {"last_op": info.last_op, "last_reduced": info.last_reduced,
                "invocations": info.invocations, "orchestrations": info.orchestrations}

    def scalar(self, name: str) -> float:
        v = C.c_double()
        _check(self._lib.irgl_module_scalar(self._h, name.encode(), C.byref(v)))
        return v.value

    def close(self):
        if getattr(self, "_h", None):
            self._lib.irgl_module_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
