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

    def __init__(self, gpu_index, start=True):
        self.rows = []  # (sm_mhz, max_mhz, reasons bitmask-decoded tuple)
        self.stop_ev = threading.Event()
        self.proc = None
        self.t = None
        self.gpu_index = gpu_index
        if start:
            self.start()

    def start(self):
        gpu_index = self.gpu_index
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
    def __init__(self, single=False):
        self.world = 1 if single else int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = 0 if single else int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        # the rank's GPU: LOCAL_RANK, wrapped when ranks outnumber the box's GPUs (--transport gloo)
        self.device = self.local_rank
        if os.environ.get("IRGL_BENCH_WRAP_DEVICES") == "1":
            try:
                import torch
                self.device = self.local_rank % max(torch.cuda.device_count(), 1)
            except Exception:
                pass
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


def kernel_source_hash():
    """sha256 (16 hex) over the library's kernel sources and build flags: the stamp a committed
    ncu capture carries, so a capture of an older kernel is never reported as this one's traffic."""
    import glob
    import hashlib
    h = hashlib.sha256()
    pkg = os.path.join(ROOT, "paper_1607_05707_b200")
    files = sorted(glob.glob(os.path.join(pkg, "csrc", "*.cu")) + glob.glob(os.path.join(pkg, "csrc", "*.cuh"))
                   + glob.glob(os.path.join(pkg, "csrc", "kernels.h")) + [os.path.join(pkg, "Makefile")])
    for f in files:
        with open(f, "rb") as fh:
            h.update(os.path.basename(f).encode() + b"\0" + fh.read())
    return h.hexdigest()[:16]


def ncu_traffic(op, scale, world=1, relabel=1):
    """DRAM bytes per launch of the dominant kernel from the committed `ncu --set full` capture of
    this workload (profiles/ncu_<op>_rmat<scale>.json, written by tools/ncu_json.py); null when
    the capture's kernel-source stamp differs from the current sources (stale) or is absent."""
    if world > 1 or not relabel:
        return None, "no capture for this configuration"
    p = os.path.join(ROOT, "profiles", f"ncu_{op}_rmat{scale}.json")
    try:
        with open(p) as f:
            d = json.load(f)
    except Exception:
        return None, "no capture"
    if d.get("source_hash") != kernel_source_hash():
        return None, f"stale capture ({os.path.basename(p)}: source_hash {d.get('source_hash')} != {kernel_source_hash()})"
    return d.get("dram_bytes_per_launch"), f"profiles/{os.path.basename(p)} (source_hash {d['source_hash']})"


# ---- CPU arms --------------------------------------------------------------------------------------
def cpu_run(op, scale, steps, warmup, budget_s=None):
    """Oracle OpenMP BSP executor on host cores; returns (GTEPS, cores, sample, host graph)."""
    from oracle import oracle as O  # checker / CPU baseline only
    O.build()
    # every host core: torchrun exports OMP_NUM_THREADS=1 per rank (only rank 0 runs this arm)
    O.set_threads(len(os.sched_getaffinity(0)))
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


CPU_ALGO = {"sssp": "data-driven Bellman-Ford: every round relaxes all edges of the frontier, "
                    "the IrGL SSSP program's semantics; no priority ordering",
            "bfs": "Listing-2 top-down BFS, one level per round"}


def cpu_serial(op, og, srcs, budget_s=10.0):
    """CPU(i) of SURVEY §8d: the serial textbook algorithm on one core (queue BFS / binary-heap
    Dijkstra), a bounded sample of the same sources."""
    from oracle import oracle as O
    deg = og.degrees()
    tot_e, tot_t, done = 0, 0.0, 0
    for s in srcs:
        t0 = time.perf_counter()
        res = O.sssp(og, s) if op == "sssp" else O.bfs(og, s)[0]
        tot_t += time.perf_counter() - t0
        tot_e += int(deg[res < INF].sum())
        done += 1
        if tot_t > budget_s:
            break
    return {"value": round(tot_e / 2 / tot_t / 1e9, 4), "unit": "GTEPS", "cores": 1,
            "algorithm": "binary-heap Dijkstra" if op == "sssp" else "queue BFS",
            "sample": f"{done} single-source traversals, {tot_t:.1f} s"}


def cpu_work_efficient(og, srcs, budget_s=8.0):
    """The OpenMP executor with the GPU's degree-scaled deferral (K = 1024): a work-efficient CPU
    SSSP beside the IrGL-semantics baseline, so the speed-up is also shown against a CPU code that
    does not re-scan edges ~3x (bounded sample of the same sources, every host core)."""
    from oracle import oracle as O
    deg = og.degrees()
    tot_e, tot_t, done = 0, 0.0, 0
    for s in srcs:
        t0 = time.perf_counter()
        res, _, _ = O.sssp_defer_omp(og, s)
        tot_t += time.perf_counter() - t0
        tot_e += int(deg[res < INF].sum())
        done += 1
        if tot_t > budget_s:
            break
    return {"value": round(tot_e / 2 / tot_t / 1e9, 4), "unit": "GTEPS", "cores": O.max_threads(),
            "algorithm": "bulk-synchronous data-driven SSSP with degree-scaled deferral (K = 1024)",
            "sample": f"{done} single-source traversals, {tot_t:.1f} s"}


def scaling_of(args):
    # N=1: configs[1] on one GPU; N>1: configs[4], one RMAT-27 graph split over the N GPUs
    return "strong" if args.gpus > 1 else "weak"


def run_reference(args, d):
    if d.rank != 0:
        return 0
    scale = args.scale
    gteps, cores, done, tt, og, srcs = cpu_run(args.op, scale, args.steps, args.warmup,
                                               budget_s=60.0 if scale > 24 else None)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gteps, 4), "unit": "GTEPS",
        "n_gpus": args.gpus, "steps": done, "warmup": args.warmup,
        "ms_per_step": round(tt / max(done, 1) * 1e3, 3), "higher_is_better": True,
        "vs_baseline": None, "dtype": "int32",
        "data": "synthetic Philox RMAT (host-generated, identical to the device graph)",
        "scaling": scaling_of(args),
        "config": workload_config(args, None, layout="generator (Philox-scrambled) ids, one host "
                                                     "CSR (the CPU arm does not relabel)"),
        "cpu_baseline": {"value": round(gteps, 4), "unit": "GTEPS", "cores": cores, "kind": "port",
                         "sample": f"{done} single-source {args.op.upper()} traversals of "
                                   f"RMAT-{scale} on the OpenMP bulk-synchronous IrGL executor "
                                   f"({CPU_ALGO[args.op]})",
                         "serial": cpu_serial(args.op, og, srcs)},
        "e2e": {"value": round(gteps, 4), "unit": "GTEPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(args, g, layout=None):
    cfg = {"workload": f"{args.op.upper()}{'-DO' if args.direction and args.op == 'bfs' else ''} "
                       f"on RMAT-{args.scale} (edge factor 16, weights [1,255]), "
                       f"one traversal per step over 16 sources",
           "op": args.op, "graph": "rmat", "scale": args.scale, "edge_factor": 16,
           "sources": 16, "partitions": args.gpus, "outline": args.outline,
           "l2": "inputs larger than L2 (CSR col+weight >> 126 MB); no flush",
           "layout": layout or ("degree-ordered vertex relabelling (untimed preprocessing; API ids "
                                "unchanged)" if args.relabel and args.gpus == 1 else
                                "1D vertex partition, block-diagonal degree order (each rank "
                                "renumbers its own range; untimed; API ids unchanged)"
                                if args.relabel else
                                "generator (Philox-scrambled) ids, 1D vertex partition"
                                if args.gpus > 1 else "generator (Philox-scrambled) ids")}
    if args.gpus > 1:
        cfg["partition"] = ("1D vertex ranges of ceil(N/P) (multiples of 32), one per GPU, exchange per "
                            "round over " + ("NCCL" if getattr(args, "transport", "nccl") == "nccl" else
                                             "the host transport plugin (gloo; ranks may share a GPU)"))
    if g is not None:
        cfg["n"] = int(g.n)
        cfg["m_directed"] = int(g.m)
    return cfg


# ---- GPU arm -----------------------------------------------------------------------------------------
def _sources_and_work(ctx, g, p, d, relabelled):
    """16 sources (the oracle's Philox stream over degrees in the caller's ids) and E_r / V_r per
    source from one BFS each (BFS expands every reached vertex exactly once)."""
    import paper_1607_05707_b200 as irgl
    info = g.info
    rp = _local_row_ptr(ctx, g)
    lo, hi = info.lo, info.hi
    perm = g.perm() if relabelled else None  # caller id -> new id (same owner range)

    def local_deg(x):  # degree of caller id x if this rank owns it
        if not (lo <= x < hi):
            return 0
        y = int(perm[x]) if perm is not None else x
        return int(rp[y - lo + 1] - rp[y - lo])

    cand = pick_sources(g.n, lambda x: d.reduce(local_deg(x), "sum"))
    er, vr = [], []
    for s in cand:
        p.init_scalars([s])
        st = ctx.iterate(irgl.BFS, g, p)
        er.append(d.reduce(st.edges, "sum"))
        vr.append(d.reduce(st.popped, "sum"))
    return cand, er, vr


def _timed_traversals(args, d, ctx, g, p, op_id, cand, er, vr, kw, sampler=None):
    """W untimed traversals, then K timed ones issued as one irgl_traverse_batch (or per-step
    calls), CUDA events on the runtime's stream; returns the device numbers, max over ranks."""
    import paper_1607_05707_b200 as irgl

    def step(i):
        p.init_scalars([cand[i % 16]])
        return ctx.iterate(op_id, g, p, **kw)

    for i in range(args.warmup):
        step(i)
    d.barrier()
    ctx.sync()
    if sampler is not None:
        sampler.start()
    l0 = irgl.launch_count()
    ctx.event_record(0)
    if args.batch:  # the K steps as one irgl_traverse_batch call (no per-step Python overhead)
        stats = ctx.traverse_batch(op_id, g, p, [cand[(args.warmup + i) % 16] for i in range(args.steps)],
                                   **kw)
    else:
        stats = [step(args.warmup + i) for i in range(args.steps)]
    ctx.event_record(1)
    ctx.sync()
    launches = irgl.launch_count() - l0
    dev_ms = ctx.event_elapsed(0, 1)
    d.barrier()
    clocks = sampler.stop() if sampler is not None else None
    kms, tot_e, tot_b = 0.0, 0.0, 0.0
    for i, st in enumerate(stats):
        k = (args.warmup + i) % 16
        kms += st.kernel_ms
        tot_e += er[k]
        # direction-optimising BFS examines fewer edges than E_r: bytes from the actual counter
        # (SURVEY §8f F1); otherwise the fixed work-efficient formula of §8d
        e_bytes = d.reduce(st.edges, "sum") if kw else er[k]
        tot_b += algorithmic_bytes(args.op, vr[k], e_bytes)
    return dict(dev_ms=d.reduce(dev_ms, "max"), kms=d.reduce(kms, "max"), tot_e=tot_e, tot_b=tot_b,
                stats=stats, launches=int(d.reduce(launches, "sum")), clocks=clocks, step=step)


def one_gpu_reference_point(args, op_id, kw, relabel):
    """configs[4]'s one-GPU reference point (run by rank 0 before the partitioned run, on its own
    GPU alone): the same RMAT-27 graph, sources and K steps in one partition."""
    import paper_1607_05707_b200 as irgl
    solo = Dist(single=True)
    with irgl.Context(devices=[int(os.environ.get("LOCAL_RANK", "0"))], outline=args.outline) as c1:
        g1 = c1.generate_rmat(args.scale)
        if relabel:
            g1.relabel()
        p1 = c1.pipe(g1.n)
        cand, er, vr = _sources_and_work(c1, g1, p1, solo, relabel)
        r = _timed_traversals(args, solo, c1, g1, p1, op_id, cand, er, vr, kw)
        gteps = r["tot_e"] / 2 / (r["dev_ms"] * 1e-3) / 1e9
        out = {"value": round(gteps, 4), "unit": "GTEPS", "ms_per_step": round(r["dev_ms"] / args.steps, 4),
               "layout": "degree-ordered ids" if relabel else "generator ids (the partitioned layout)"}
        g1.close()
        p1.close()
    return out


def secondary_entries(args, scales_ops):
    """Secondary driver-timed workloads of the same metric (BASELINE configs: BFS on RMAT-22, the
    north-star RMAT-24 BFS / SSSP), each on its own context in the bench's layout (degree-ordered
    ids), K traversals over the 16 sources through irgl_traverse_batch, with the roofline of
    SURVEY §8d and bit-exact parity of source 0 against the oracle."""
    import argparse as _ap
    import paper_1607_05707_b200 as irgl
    from oracle import oracle as O  # checker only
    solo = Dist(single=True)
    peak, _ = load_peaks()
    out = []
    og_cache = {}
    for entry in scales_ops:
        scale, op = entry[0], entry[1]
        kw = entry[2] if len(entry) > 2 else {}
        a = _ap.Namespace(**vars(args))
        a.scale, a.op = scale, op
        op_id = irgl.SSSP if op == "sssp" else irgl.BFS
        with irgl.Context(devices=[int(os.environ.get("LOCAL_RANK", "0"))], outline=args.outline) as c:
            g = c.generate_rmat(scale)
            g.relabel()
            p = c.pipe(g.n)
            cand, er, vr = _sources_and_work(c, g, p, solo, True)
            r = _timed_traversals(a, solo, c, g, p, op_id, cand, er, vr, kw)
            gteps = r["tot_e"] / 2 / (r["dev_ms"] * 1e-3) / 1e9
            ach = r["tot_b"] / (r["kms"] * 1e-3) / 1e9 if r["kms"] > 0 else None
            p.init_scalars([cand[0]])
            c.iterate(op_id, g, p, **kw)
            gpu = c.read_result(op_id, g)
            p.close()
            g.close()
        if scale not in og_cache:
            og_cache.clear()
            og_cache[scale] = O.rmat(scale)
        og = og_cache[scale]
        ref = O.sssp(og, cand[0]) if op == "sssp" else O.bfs(og, cand[0])[0]
        traffic, note = ncu_traffic(op, scale, 1, 1) if not kw else (None, "no capture of the DO kernel")
        name = "BFS (direction-optimising; roofline on the edges it examined)" if kw else op.upper()
        out.append({"workload": f"{name} on RMAT-{scale} (degree-ordered ids), {args.steps} "
                                f"traversals over 16 sources", "value": round(gteps, 3),
                    "unit": "GTEPS", "ms_per_step": round(r["dev_ms"] / args.steps, 4),
                    "roofline": {"achieved": round(ach, 1) if ach else None, "peak": peak,
                                 "frac": round(ach / peak, 4) if ach else None,
                                 "kernel_ms_per_step": round(r["kms"] / args.steps, 4),
                                 "algorithmic_bytes_per_step": round(r["tot_b"] / args.steps),
                                 "traffic": traffic, "traffic_source": note},
                    "gpu_launches": r["launches"],
                    "parity": "bit-exact" if np.array_equal(gpu, ref) else "MISMATCH",
                    "parity_check": f"source {cand[0]} against the serial oracle "
                                    f"({'Dijkstra' if op == 'sssp' else 'queue BFS'})"})
    return out


def partitioned_entry(args, scale=24, parts=(2, 4)):
    """The multi-partition code path measured on the one GPU: RMAT-`scale` split into
    P logical partitions (block-diagonal degree order), each Iterate the distributed persistent
    kernel (one cooperative kernel per partition meeting at a device-side rendezvous); ms per
    traversal from the runtime's CUDA events over 8 sources, parity of one source against the
    oracle.  The partitions share this GPU's SMs and L2: a functional stand-in for P GPUs, not a
    scaling number (the one-partition numbers are the secondary entries)."""
    import paper_1607_05707_b200 as irgl
    from oracle import oracle as O  # checker only
    og = O.rmat(scale)
    deg = np.diff(og.row_ptr)
    srcs = pick_sources(og.n, lambda x: int(deg[x]), count=8)
    refs = {"bfs": O.bfs(og, srcs[0])[0], "sssp": O.sssp(og, srcs[0])}
    dev = int(os.environ.get("LOCAL_RANK", "0"))
    out = []
    for P in parts:
        ent = {"workload": f"RMAT-{scale} in {P} logical partitions on one GPU (distributed persistent "
                           f"kernel, block-diagonal degree order), 8 sources", "P": P}
        ok, outl = True, True
        with irgl.Context(devices=[dev], logical_partitions=P, outline=args.outline) as c:
            g = c.generate_rmat(scale)
            g.relabel()
            p = c.pipe(g.n)
            for name, op_id, kw in (("bfs", irgl.BFS, {}), ("bfs_do", irgl.BFS, {"direction": 1}),
                                    ("sssp", irgl.SSSP, {})):
                ms, edges, xb = [], [], []
                for i, s in enumerate([srcs[0]] + list(srcs)):  # first: warm-up
                    p.init_scalars([s])
                    st = c.iterate(op_id, g, p, **kw)
                    outl = outl and st.outlined == 1
                    if i:
                        ms.append(st.device_ms)
                        edges.append(st.edges)
                        xb.append(st.exchange_bytes)
                p.init_scalars([srcs[0]])
                c.iterate(op_id, g, p, **kw)
                ok = ok and np.array_equal(c.read_result(op_id, g), refs["sssp" if op_id == irgl.SSSP else "bfs"])
                ent[f"{name}_ms_per_traversal"] = round(float(np.mean(ms)), 4)
                ent[f"{name}_edges_scanned"] = int(np.mean(edges))
                ent[f"{name}_exchange_bytes"] = int(np.mean(xb))  # ids + values stored into peers' inboxes
            p.close()
            g.close()
        ent["outlined"] = outl
        ent["parity"] = "bit-exact" if ok else "MISMATCH"
        ent["parity_check"] = f"source {srcs[0]}: BFS, DO-BFS levels and SSSP distances against the serial oracle"
        out.append(ent)
    return out


def run_irgl(args, d):
    import paper_1607_05707_b200 as irgl
    op_id = irgl.SSSP if args.op == "sssp" else irgl.BFS
    kw = {"direction": 1} if (args.op == "bfs" and args.direction) else {}
    one_gpu = None
    if d.world > 1:
        # the scaling denominator of configs[4]: rank 0 alone on its GPU first (others wait)
        if d.rank == 0 and not args.no_one_gpu_point:
            one_gpu = {"generator_ids": one_gpu_reference_point(args, op_id, kw, relabel=False)}
            if args.relabel:
                one_gpu["degree_ordered"] = one_gpu_reference_point(args, op_id, kw, relabel=True)
        d.barrier()
        if args.transport == "gloo":
            # the rank transport over the bench's own gloo group (irgl_ctx_create_transport):
            # the multi-process path on a box with fewer GPUs than ranks (ranks share devices;
            # NCCL refuses two ranks on one device) — a plumbing check, not a scaling number
            from paper_1607_05707_b200.dist import TorchTransport
            ctx = irgl.Context(transport=TorchTransport(device=d.device), outline=args.outline)
        else:
            uid = d.bcast_bytes(irgl.nccl_unique_id() if d.rank == 0 else None)
            ctx = irgl.Context(nccl=(d.device, d.rank, d.world, uid), outline=args.outline)
    else:
        ctx = irgl.Context(devices=[d.device], outline=args.outline)
    t0 = time.time()
    g = ctx.generate_rmat(args.scale)
    gen_s = time.time() - t0
    relabel_s = None
    if args.relabel:
        # data layout: degree-ordered vertex ids (preprocessing, like the CSR build: untimed); at
        # N > 1 block-diagonal (each rank orders its own range); every id crossing the API stays
        # the generator's
        t0 = time.time()
        g.relabel()
        relabel_s = time.time() - t0
    info = g.info
    p = ctx.pipe(max(info.local_n, 1) if d.world > 1 else g.n)
    cand, er, vr = _sources_and_work(ctx, g, p, d, relabel_s is not None)

    # ---- device-timed region: inputs resident in HBM
    sampler = ClockSampler(d.device, start=False) if d.rank == 0 else None
    r = _timed_traversals(args, d, ctx, g, p, op_id, cand, er, vr, kw, sampler)
    dev_ms, kms, tot_e, tot_b, stats = r["dev_ms"], r["kms"], r["tot_e"], r["tot_b"], r["stats"]
    step = r["step"]
    gteps = tot_e / 2 / (dev_ms * 1e-3) / 1e9

    # ---- end to end through the public API: host source in, host distances out (pinned).  Queries
    # are pipelined the way a serving loop would issue them: each step's result copy is queued
    # (irgl_read_result_async) and overlaps the next traversal, which writes the graph's second
    # label buffer; every copy has landed before the timed region closes (irgl_results_wait).
    # At N>1 each rank copies its own vertex range (the result is distributed like the graph).
    nres = int(info.local_n) if d.world > 1 else int(g.n)
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
    d2h_gbps = 4 * 4 * nres / (time.perf_counter() - t1) / 1e9

    peak, peak_kind = load_peaks()
    achieved = tot_b / (kms * 1e-3) / 1e9 if kms > 0 else None
    traffic, traffic_note = ncu_traffic(args.op, args.scale, d.world, args.relabel)
    assert d.world == args.gpus, (d.world, args.gpus)
    line = {
        "metric": METRIC, "value": round(gteps, 4), "unit": "GTEPS", "n_gpus": d.world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dev_ms / args.steps, 4), "higher_is_better": True,
        "scaling": scaling_of(args), "vs_baseline": None, "dtype": "int32",
        "data": "synthetic: device Philox RMAT (Graph500 .57/.19/.19/.05, ef 16, scrambled ids, "
                "seed 1), int32 weights in [1,255] (seed 11)",
        "config": workload_config(args, g),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1) if achieved else None,
                     "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4) if achieved else None,
                     "traffic": traffic, "traffic_source": traffic_note, "peak_kind": peak_kind,
                     "kernel": (f"persistent_kernel<{args.op.upper()}> (outlined Iterate)"
                                if not kw else "persistent_bfs_do_kernel (outlined, direction-optimising)")
                     if args.outline != 0 and d.world == 1 else "expand_kernel + chunk_kernel",
                     "algorithmic_bytes_per_step": round(tot_b / args.steps),
                     "kernel_ms_per_step": round(kms / args.steps, 4)},
        "e2e": {"value": round(e2e, 4), "unit": "GTEPS", "h2d_bytes_per_step": 8 * d.world,
                "d2h_bytes_per_step": 4 * int(g.n), "d2h_GBps_alone": round(d2h_gbps, 1)},
        "gpu_launches": r["launches"],
        "clocks": r["clocks"],
        "detail": {"gen_s": round(gen_s, 3), "relabel_s": round(relabel_s, 3) if relabel_s else None, "rounds_per_step": float(np.mean([s.rounds for s in stats])),
                   "edges_scanned_per_step": float(np.mean([s.edges for s in stats])),
                   "E_r_mean": float(np.mean(er)), "V_r_mean": float(np.mean(vr)),
                   "outlined": int(stats[-1].outlined) if stats else None,
                   "directed_edges_per_s": round(tot_e / (dev_ms * 1e-3), 1)},
    }
    if d.world > 1:
        line["detail"]["exchange_bytes_per_step"] = float(np.mean([s.exchange_bytes for s in stats]))
        if one_gpu:
            line["detail"]["one_gpu"] = one_gpu  # scaling denominator: same graph on one GPU
    # ---- CPU baseline (rank 0, N=1 only): oracle OpenMP executor on the host cores
    if d.world == 1 and not args.no_cpu_baseline:
        cg, cores, done, tt, og, osrc = cpu_run(args.op, args.scale, 16, 1, budget_s=12.0)
        line["cpu_baseline"] = {"value": round(cg, 4), "unit": "GTEPS", "cores": cores,
                                "kind": "port",
                                "sample": f"{done} single-source {args.op.upper()} traversals of "
                                          f"RMAT-{args.scale} (OpenMP bulk-synchronous IrGL "
                                          f"executor, {CPU_ALGO[args.op]}; {tt:.1f} s)",
                                "serial": cpu_serial(args.op, og, osrc[:4], budget_s=8.0)}
        if args.op == "sssp":
            line["cpu_baseline"]["work_efficient"] = cpu_work_efficient(og, osrc, budget_s=8.0)
        # parity of the measured workload: GPU result == oracle for source 0
        from oracle import oracle as O
        assert osrc == cand, "source selection differs from the oracle"
        p.init_scalars([cand[0]])
        ctx.iterate(op_id, g, p)
        gpu = ctx.read_result(op_id, g)
        ref = O.sssp(og, cand[0]) if args.op == "sssp" else O.bfs(og, cand[0])[0]
        line["parity"] = "bit-exact" if np.array_equal(gpu, ref) else "MISMATCH"
    ctx.close()
    # ---- secondary entries (N=1): BFS at the headline scale, the north-star RMAT-24 BFS / SSSP
    if d.world == 1 and args.secondary and args.scale == 22 and args.op == "sssp" and not args.direction:
        line["detail"]["secondary"] = secondary_entries(
            args, [(22, "bfs"), (24, "bfs"), (24, "sssp"), (24, "bfs", {"direction": 1})])
        line["detail"]["partitioned_one_gpu"] = partitioned_entry(args)
    if d.rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def _local_row_ptr(ctx, g):
    import ctypes as C
    rp = np.zeros(g.info.local_n + 1, dtype=np.int64)
    st = ctx._lib.irgl_graph_download(g.handle, rp.ctypes.data_as(C.POINTER(C.c_int64)), None, None)
    if st != 0:
        raise RuntimeError("irgl_graph_download failed")
    return rp


def _free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def self_launch(n):
    """`python bench.py --gpus N` without a launcher: start the N ranks ourselves (one process per
    GPU, the same torchrun command the driver uses) and pass rank 0's JSON line through."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, IRGL_BENCH_SELF_LAUNCHED="1")
    return subprocess.call(cmd, env=env)


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
    ap.add_argument("--transport", default="nccl", choices=["nccl", "gloo"],
                    help="N>1 rank transport: NCCL (default) or the host plugin over gloo (ranks may "
                         "share a GPU: a plumbing check on boxes with fewer GPUs than ranks)")
    ap.add_argument("--secondary", type=int, default=1,
                    help="N=1 default workload: also time BFS RMAT-22 and BFS / SSSP RMAT-24 "
                         "(detail.secondary, with parity)")
    ap.add_argument("--no-one-gpu-point", action="store_true",
                    help="N>1: skip the one-GPU RMAT-27 reference point in detail.one_gpu")
    ap.add_argument("--batch", type=int, default=1,
                    help="1: the K steps as one irgl_traverse_batch call; 0: one Python-level "
                         "init/iterate/read per step")
    ap.add_argument("--relabel", type=int, default=1,
                    help="1 = degree-ordered vertex relabelling before timing (one GPU only)")
    ap.add_argument("--direction", type=int, default=0,
                    help="BFS: 1 = direction-optimising (SURVEY §8f F1), 0 = Listing-2 top-down")
    args = ap.parse_args()
    if args.transport == "gloo":
        os.environ["IRGL_BENCH_WRAP_DEVICES"] = "1"
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args.gpus)
    d = Dist()
    if d.world > 1 and args.gpus != d.world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={d.world}")
    args.gpus = d.world
    if args.scale <= 0:
        # N=1: configs[1] (SSSP RMAT-22); N>1: configs[4] (RMAT-27 vertex-partitioned over the N
        # GPUs, total work fixed -> strong scaling)
        args.scale = 22 if args.gpus == 1 else 27
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args, d)
    return run_irgl(args, d)


if __name__ == "__main__":
    sys.exit(main())
