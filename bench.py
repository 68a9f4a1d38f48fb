#!/usr/bin/env python3
"""bench.py — GTEPS of the IrGL worklist hot path on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl irgl|reference] [--op sssp|bfs]
                  [--scale S]

Workload (config[1] of BASELINE.json at N=1): data-driven SSSP (integer weights in [1,255]) on a
device-generated Philox RMAT graph (Graph500 A/B/C/D .57/.19/.19/.05, edge factor 16, scrambled
ids, seed 1; weights seed 11), scale 22 at N=1 and 22+log2(N) at N GPUs (weak scaling: per-GPU
edges fixed; N=8 -> RMAT-25).  One step = one full traversal from the next of 16 sources
(non-isolated, Philox seed 7), operator-state reset included.  GTEPS (Graph500) = undirected
edges of the traversed component / time.  The CSR (col+weight, 1 GB at s22) is larger than L2,
so no flush is needed between steps.

N>1: one process per GPU (torchrun); the graph is 1D vertex-partitioned, ranks exchange
frontier updates with NCCL inside irgl_iterate; rank 0 prints one JSON line.  Device time is the
max over ranks.  --impl reference: the CPU reference arm (the oracle's OpenMP bulk-synchronous
IrGL executor on the host cores; the reference itself ships no executable code).
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GTEPS (BFS/SSSP, RMAT) at 1/2/4/8 B200; % of HBM roofline; speedup vs host CPU"
INF = 2147483647


# ---- Philox-4x32-10 (source selection; same stream as the oracle's orc_pick_sources) -------------
def _philox(c, k):
    c0, c1, c2, c3 = c
    k0, k1 = k
    M = 0xFFFFFFFF
    for _ in range(10):
        p0 = 0xD2511F53 * c0
        p1 = 0xCD9E8D57 * c2
        c0, c1, c2, c3 = ((p1 >> 32) ^ c1 ^ k0) & M, p1 & M, ((p0 >> 32) ^ c3 ^ k1) & M, p0 & M
        k0 = (k0 + 0x9E3779B9) & M
        k1 = (k1 + 0xBB67AE85) & M
    return c0, c1, c2, c3


def pick_sources(n, degree_of, count=16, seed=7):
    out = []
    for i in range(count):
        for att in range(1_000_000):
            r = _philox((i, att, 0, 0x53524353), (seed & 0xFFFFFFFF, seed >> 32))
            x = ((r[1] << 32) | r[0]) % n
            if degree_of(x) > 0:
                out.append(x)
                break
    return out


# ---- clocks sampler ---------------------------------------------------------------------------------
class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML polled every 2 ms from
    a thread (nvidia-smi's 100 ms loop misses a region of a few tens of ms); nvidia-smi fallback."""
    NAMES = ("sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")

    def __init__(self, gpu_index):
        self.rows = []  # (sm_mhz, max_mhz, reasons bitmask-decoded tuple)
        self.stop_ev = threading.Event()
        self.proc = None
        self.t = None
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(int(gpu_index))
            bits = (N.nvmlClocksEventReasonSwPowerCap, N.nvmlClocksEventReasonHwSlowdown,
                    N.nvmlClocksEventReasonHwThermalSlowdown, N.nvmlClocksEventReasonSwThermalSlowdown)
            mx = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))

            def poll():
                while not self.stop_ev.is_set():
                    try:
                        sm = float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
                        r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append((sm, mx, tuple(n for n, b in zip(self.NAMES, bits) if r & b)))
                    except Exception:
                        pass
                    time.sleep(0.002)
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            self.kind = "nvml"
            return
        except Exception:
            pass
        try:
            fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,"
                      "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                      "clocks_event_reasons.sw_thermal_slowdown")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={fields}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)

            def read():
                for line in self.proc.stdout:
                    parts = [x.strip() for x in line.split(",")]
                    if len(parts) == 6 and parts[0].replace(".", "").isdigit():
                        self.rows.append((float(parts[0]), float(parts[1]),
                                          tuple(n for n, v in zip(self.NAMES, parts[2:]) if v == "Active")))
            self.t = threading.Thread(target=read, daemon=True)
            self.t.start()
            self.kind = "nvidia-smi"
        except Exception:
            self.proc = None

    def stop(self):
        self.stop_ev.set()
        if self.proc:
            time.sleep(0.05)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        if not self.rows:
            return None
        sm = [r[0] for r in self.rows]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": sorted({n for r in self.rows for n in r[2]}),
                "samples": len(self.rows), "source": self.kind}


# ---- distributed plumbing (gloo for host-side barrier / reductions / NCCL id broadcast) ---------
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group("gloo", rank=self.rank, world_size=self.world)
            self.dist = dist

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def reduce(self, x, op):
        if self.world == 1:
            return x
        import torch
        t = torch.tensor([float(x)], dtype=torch.float64)
        self.dist.all_reduce(t, op={"max": self.dist.ReduceOp.MAX,
                                    "sum": self.dist.ReduceOp.SUM}[op])
        return t.item()

    def reduce_vec(self, v, op):
        if self.world == 1:
            return v
        import torch
        t = torch.tensor(np.asarray(v, dtype=np.float64))
        self.dist.all_reduce(t, op={"max": self.dist.ReduceOp.MAX,
                                    "sum": self.dist.ReduceOp.SUM}[op])
        return t.numpy()

    def bcast_bytes(self, b):
        if self.world == 1:
            return b
        obj = [b]
        self.dist.broadcast_object_list(obj, src=0)
        return obj[0]


def algorithmic_bytes(op, vr, er):
    """BFS 20 V_r + 8 E_r;  SSSP 24 V_r + 12 E_r  (bytes of CSR + labels touched)."""
    return (20 * vr + 8 * er) if op == "bfs" else (24 * vr + 12 * er)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(op, scale):
    p = os.path.join(ROOT, "profiles", f"ncu_{op}_rmat{scale}.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d
    except Exception:
        return None, None


# ---- CPU arms --------------------------------------------------------------------------------------
def cpu_run(op, scale, steps, warmup, budget_s=None):
    """Oracle OpenMP BSP executor on host cores; returns (GTEPS, cores, sample, host graph)."""
    from oracle import oracle as O  # checker / CPU baseline only
    O.build()
    og = O.rmat(scale)
    srcs = [int(s) for s in og.sources(16)]
    fn = O.sssp_bsp_omp if op == "sssp" else O.bfs_bsp_omp
    deg = og.degrees()
    for i in range(warmup):
        fn(og, srcs[i % 16])
    tot_e, tot_t, done = 0, 0.0, 0
    for i in range(steps):
        s = srcs[(warmup + i) % 16]
        t0 = time.perf_counter()
        res, _, _ = fn(og, s)
        tot_t += time.perf_counter() - t0
        tot_e += int(deg[res < INF].sum())
        done += 1
        if budget_s is not None and tot_t > budget_s:
            break
    gteps = tot_e / 2 / tot_t / 1e9
    return gteps, O.max_threads(), done, tot_t, og, srcs


def run_reference(args, d):
    if d.rank != 0:
        return 0
    scale = args.scale
    gteps, cores, done, tt, _, _ = cpu_run(args.op, scale, args.steps, args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gteps, 4), "unit": "GTEPS",
        "n_gpus": args.gpus, "steps": done, "warmup": args.warmup,
        "ms_per_step": round(tt / max(done, 1) * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic Philox RMAT (host-generated, identical to the device graph)",
        "config": workload_config(args, None),
        "cpu_baseline": {"value": round(gteps, 4), "unit": "GTEPS", "cores": cores, "kind": "port",
                         "sample": f"{done} single-source {args.op.upper()} traversals of "
                                   f"RMAT-{scale} on the OpenMP bulk-synchronous IrGL executor"},
        "e2e": {"value": round(gteps, 4), "unit": "GTEPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(args, g):
    cfg = {"workload": f"{args.op.upper()}{'-DO' if args.direction and args.op == 'bfs' else ''} "
                       f"on RMAT-{args.scale} (edge factor 16, weights [1,255]), "
                       f"one traversal per step over 16 sources",
           "op": args.op, "graph": "rmat", "scale": args.scale, "edge_factor": 16,
           "sources": 16, "partitions": args.gpus, "outline": args.outline,
           "l2": "inputs larger than L2 (CSR col+weight >> 126 MB); no flush",
           "layout": ("degree-ordered vertex relabelling (untimed preprocessing; API ids unchanged)"
                      if args.relabel and args.gpus == 1 else "generator ids")}
    if g is not None:
        cfg["n"] = int(g.n)
        cfg["m_directed"] = int(g.m)
    return cfg


# ---- GPU arm -----------------------------------------------------------------------------------------
def run_irgl(args, d):
    import paper_1607_05707_b200 as irgl
    op_id = irgl.SSSP if args.op == "sssp" else irgl.BFS
    if d.world > 1:
        uid = d.bcast_bytes(irgl.nccl_unique_id() if d.rank == 0 else None)
        ctx = irgl.Context(nccl=(d.local_rank, d.rank, d.world, uid), outline=args.outline)
    else:
        ctx = irgl.Context(devices=[d.local_rank], outline=args.outline)
    t0 = time.time()
    g = ctx.generate_rmat(args.scale)
    gen_s = time.time() - t0
    relabel_s = None
    if args.relabel and d.world == 1:
        # data layout: degree-ordered vertex ids (preprocessing, like the CSR build: untimed);
        # every id crossing the API stays the generator's
        t0 = time.time()
        g.relabel()
        relabel_s = time.time() - t0
    info = g.info
    # local degrees -> sources (Philox stream of the oracle), agreed across ranks
    rp = _local_row_ptr(ctx, g)
    lo, hi = info.lo, info.hi
    if relabel_s is not None:  # degrees in the caller's ids for the source pick
        dg = np.diff(rp)[g.perm()]
        rp = np.zeros(g.n + 1, dtype=np.int64)
        rp[1:] = np.cumsum(dg)

    def local_deg(x):
        return int(rp[x - lo + 1] - rp[x - lo]) if lo <= x < hi else 0

    cand = pick_sources(g.n, lambda x: d.reduce(local_deg(x), "sum"))
    p = ctx.pipe(max(info.local_n, 1) if d.world > 1 else g.n)

    # E_r / V_r per source from one BFS each (BFS expands every reached vertex exactly once)
    er, vr = [], []
    for s in cand:
        p.init_scalars([s])
        st = ctx.iterate(irgl.BFS, g, p)
        er.append(d.reduce(st.edges, "sum"))
        vr.append(d.reduce(st.popped, "sum"))

    kw = {"direction": 1} if (args.op == "bfs" and args.direction) else {}

    def step(i):
        s = cand[i % 16]
        p.init_scalars([s])
        return ctx.iterate(op_id, g, p, **kw)

    for i in range(args.warmup):
        step(i)
    # ---- device-timed region: inputs resident in HBM
    d.barrier()
    ctx.sync()
    sampler = ClockSampler(d.local_rank) if d.rank == 0 else None
    l0 = irgl.launch_count()
    ctx.event_record(0)
    kms, tot_e, tot_b = 0.0, 0.0, 0.0
    if args.batch:  # the K steps as one irgl_traverse_batch call (no per-step Python overhead)
        stats = ctx.traverse_batch(op_id, g, p, [cand[(args.warmup + i) % 16] for i in range(args.steps)],
                                   **kw)
    else:
        stats = [step(args.warmup + i) for i in range(args.steps)]
    ctx.event_record(1)
    ctx.sync()
    for i, st in enumerate(stats):
        k = (args.warmup + i) % 16
        kms += st.kernel_ms
        tot_e += er[k]
        # direction-optimising BFS examines fewer edges than E_r: bytes from the actual counter
        # (SURVEY §8f F1); otherwise the fixed work-efficient formula of §8d
        e_bytes = d.reduce(st.edges, "sum") if kw else er[k]
        tot_b += algorithmic_bytes(args.op, vr[k], e_bytes)
    dev_ms = ctx.event_elapsed(0, 1)
    launches = irgl.launch_count() - l0
    d.barrier()
    clocks = sampler.stop() if sampler else None
    dev_ms = d.reduce(dev_ms, "max")
    kms = d.reduce(kms, "max")
    gteps = tot_e / 2 / (dev_ms * 1e-3) / 1e9

    # ---- end to end through the public API: host source in, host distances out (pinned).  Queries
    # are pipelined the way a serving loop would issue them: each step's result copy is queued
    # (irgl_read_result_async) and overlaps the next traversal, which writes the graph's second
    # label buffer; every copy has landed before the timed region closes (irgl_results_wait).
    try:
        import torch
        host_out = [torch.empty(g.n, dtype=torch.int32, pin_memory=True).numpy() for _ in range(2)]
    except Exception:
        host_out = [np.empty(g.n, dtype=np.int32) for _ in range(2)]
    # untimed warm-up of the serving loop: the first asynchronous read allocates the graph's second
    # label buffer and the copy events (a cudaMalloc inside the timed loop cost 1-100+ ms)
    for i in range(max(2, args.warmup)):
        step(i)
        ctx.read_result_async(op_id, g, host_out[i % 2])
    ctx.results_wait()
    d.barrier()
    t0 = time.perf_counter()
    if args.batch:
        ctx.traverse_batch(op_id, g, p, [cand[(args.warmup + i) % 16] for i in range(args.steps)],
                           host_out, **kw)
    else:
        for i in range(args.steps):
            step(args.warmup + i)
            ctx.read_result_async(op_id, g, host_out[i % 2])
        ctx.results_wait()
    wall = d.reduce(time.perf_counter() - t0, "max")
    e2e = tot_e / 2 / wall / 1e9
    # the host link's speed on this box right now: one result copy alone (the e2e copies are
    # PCIe-bound; the same build measured 14-44 GTEPS e2e on different boxes at equal device time)
    ctx.sync()
    t1 = time.perf_counter()
    for _ in range(4):
        ctx.read_result_async(op_id, g, host_out[0])
        ctx.results_wait()
    d2h_gbps = 4 * 4 * int(g.n) / (time.perf_counter() - t1) / 1e9

    peak, peak_kind = load_peaks()
    achieved = tot_b / (kms * 1e-3) / 1e9 if kms > 0 else None
    traffic, ncu = ncu_traffic(args.op, args.scale)
    line = {
        "metric": METRIC, "value": round(gteps, 4), "unit": "GTEPS", "n_gpus": d.world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dev_ms / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic: device Philox RMAT (Graph500 .57/.19/.19/.05, ef 16, scrambled ids, "
                "seed 1), int32 weights in [1,255] (seed 11)",
        "config": workload_config(args, g),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1) if achieved else None,
                     "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4) if achieved else None,
                     "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": (f"persistent_kernel<{args.op.upper()}> (outlined Iterate)"
                                if not kw else "persistent_bfs_do_kernel (outlined, direction-optimising)")
                     if args.outline != 0 else "expand_kernel + chunk_kernel",
                     "algorithmic_bytes_per_step": round(tot_b / args.steps),
                     "kernel_ms_per_step": round(kms / args.steps, 4)},
        "e2e": {"value": round(e2e, 4), "unit": "GTEPS", "h2d_bytes_per_step": 8,
                "d2h_bytes_per_step": 4 * int(g.n), "d2h_GBps_alone": round(d2h_gbps, 1)},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "detail": {"gen_s": round(gen_s, 3), "relabel_s": round(relabel_s, 3) if relabel_s else None, "rounds_per_step": float(np.mean([s.rounds for s in stats])),
                   "edges_scanned_per_step": float(np.mean([s.edges for s in stats])),
                   "E_r_mean": float(np.mean(er)), "V_r_mean": float(np.mean(vr)),
                   "outlined": int(stats[-1].outlined) if stats else None,
                   "directed_edges_per_s": round(tot_e / (dev_ms * 1e-3), 1)},
    }
    # ---- CPU baseline (rank 0, N=1 only): oracle OpenMP executor on the host cores
    if d.world == 1 and not args.no_cpu_baseline:
        cg, cores, done, tt, og, osrc = cpu_run(args.op, args.scale, 16, 1, budget_s=12.0)
        line["cpu_baseline"] = {"value": round(cg, 4), "unit": "GTEPS", "cores": cores,
                                "kind": "port",
                                "sample": f"{done} single-source {args.op.upper()} traversals of "
                                          f"RMAT-{args.scale} (OpenMP bulk-synchronous IrGL "
                                          f"executor, {tt:.1f} s)"}
        # parity of the measured workload: GPU result == oracle for source 0
        from oracle import oracle as O
        assert osrc == cand, "source selection differs from the oracle"
        p.init_scalars([cand[0]])
        ctx.iterate(op_id, g, p)
        gpu = ctx.read_result(op_id, g)
        ref = O.sssp(og, cand[0]) if args.op == "sssp" else O.bfs(og, cand[0])[0]
        line["parity"] = "bit-exact" if np.array_equal(gpu, ref) else "MISMATCH"
    if d.rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    return 0


def _local_row_ptr(ctx, g):
    import ctypes as C
    rp = np.zeros(g.info.local_n + 1, dtype=np.int64)
    st = ctx._lib.irgl_graph_download(g.handle, rp.ctypes.data_as(C.POINTER(C.c_int64)), None, None)
    if st != 0:
        raise RuntimeError("irgl_graph_download failed")
    return rp


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="irgl", choices=["irgl", "reference"])
    ap.add_argument("--op", default="sssp", choices=["sssp", "bfs"])
    ap.add_argument("--scale", type=int, default=0)
    ap.add_argument("--outline", type=int, default=-1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--batch", type=int, default=1,
                    help="1: the K steps as one irgl_traverse_batch call; 0: one Python-level "
                         "init/iterate/read per step")
    ap.add_argument("--relabel", type=int, default=1,
                    help="1 = degree-ordered vertex relabelling before timing (one GPU only)")
    ap.add_argument("--direction", type=int, default=0,
                    help="BFS: 1 = direction-optimising (SURVEY §8f F1), 0 = Listing-2 top-down")
    args = ap.parse_args()
    d = Dist()
    if d.world > 1:
        args.gpus = d.world
    if args.scale <= 0:
        args.scale = 22 + int(round(math.log2(max(args.gpus, 1))))
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args, d)
    return run_irgl(args, d)


if __name__ == "__main__":
    sys.exit(main())
