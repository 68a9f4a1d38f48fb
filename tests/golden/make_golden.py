"""Generates tests/golden/spec_examples.json — the reference's own pins for this path.

The reference (arXiv 1607.05707 re-spec, /root/reference/SPEC.md) ships no fixtures, test files or
executable code for the hot path.  Its only known-answer examples are the
[OP] examples and acceptance items quoted below; this script writes them down verbatim as data,
and derives the random-graph BFS cases of acceptance item 1 with an independent
pure-Python sequential BFS (not the oracle), so the oracle can be checked against them.

Run: python tests/golden/make_golden.py   (deterministic; committed output)
"""
import json
import os
import random
from collections import deque

HERE = os.path.dirname(os.path.abspath(__file__))


def seq_bfs(n, adj, src):
    INF = 2147483647
    lv = [INF] * n
    lv[src] = 0
    q = deque([src])
    while q:
        u = q.popleft()
        for v in adj[u]:
            if lv[v] == INF:
                lv[v] = lv[u] + 1
                q.append(v)
    return lv


def random_connected(rng, n):
    edges = set()
    for i in range(1, n):  # random spanning tree
        edges.add((rng.randrange(0, i), i))
    for _ in range(rng.randrange(0, 2 * n)):
        a, b = rng.randrange(n), rng.randrange(n)
        if a != b:
            edges.add((min(a, b), max(a, b)))
    return sorted(edges)


def main():
    g = {"source": "/root/reference/SPEC.md (examples quoted per case)", "cases": {}}
    c = g["cases"]
    c["bfs_path5"] = {
        "ref": "SPEC.md:438 'Listing 2 with a 5-node path graph, src=0 -> level array [0,1,2,3,4]'"
               " and SPEC.md:523 `irglc run bfs.irgl --graph path5.txt --bind src=0` -> "
               "`level = [0, 1, 2, 3, 4]`; invocations = ecc(src)+1 = 5 (SPEC.md:549, App. B1)",
        "n": 5, "edges": [[0, 1], [1, 2], [2, 3], [3, 4]], "src": 0,
        "level": [0, 1, 2, 3, 4], "invocations": 5}
    c["iterate_nonpushing"] = {"ref": "SPEC.md:439 'Iterate over a kernel that never pushes -> "
                                      "exactly 1 round'", "rounds": 1}
    c["countdown_guard3"] = {"ref": "SPEC.md:465 'kernel pushing each popped item once more with a "
                                    "countdown guard of 3 -> exactly 3 invocations'",
                             "init": [0], "guard": 3, "invocations": 3}
    c["retry_odd_once"] = {"ref": "SPEC.md:466 'kernel retrying every odd item once -> 2 runs of the "
                                  "kernel per invocation, out contains all processed items'",
                           "init": list(range(8)), "guard": 1, "launches": 2,
                           "out_sorted": list(range(8))}
    c["retry_trace_3round"] = {
        "ref": "SPEC.md:554 'golden trace comparison on a 3-round hand-computed scenario' "
               "(odd items retried twice; rows = [launch, |in|, |out| after, |retry| after])",
        "init": list(range(8)), "guard": 2,
        "trace": [[1, 8, 4, 4], [2, 4, 4, 4], [3, 4, 8, 0]]}
    c["reduce_identities"] = {"ref": "SPEC.md:448 (Any over all-false -> false), SPEC.md:557 "
                                     "(zero-iteration launches return false (Any) / true (All))",
                              "any_all_false": False, "any_empty": False, "all_empty": True}
    c["forall_consecutive_100_8"] = {
        "ref": "SPEC.md:449 'ForAll of 100 iterations, 8 threads, consecutive mapping -> thread t "
               "executes iterations {t, t+8, ...}'",
        "n": 100, "threads": 8, "thread_of": [i % 8 for i in range(100)]}
    c["forall_blocked_100_10"] = {
        "ref": "SPEC.md:321 'blocked over N=100, threads=10 -> thread t covers [10t, 10t+10)'",
        "n": 100, "threads": 10, "thread_of": [i // 10 for i in range(100)]}
    c["t_control"] = {
        "ref": "SPEC.md:254-256, :379 (kinds: 0 Elastic, 1 Shrinkable(max), 2 Fixed(n))",
        "cases": [[[[0, 0], [0, 0]], 1024], [[[0, 0], [1, 512], [2, 128]], 128],
                  [[[2, 128], [2, 256]], None], [[[0, 0], [1, 256]], 256]]}
    rng = random.Random(549)
    rg = []
    for t in range(20):  # 20 random connected graphs (<= 64 nodes)
        n = rng.randrange(2, 65)
        edges = random_connected(rng, n)
        adj = [[] for _ in range(n)]
        for a, b in edges:
            adj[a].append(b)
            adj[b].append(a)
        for a in adj:
            a.sort()
        src = rng.randrange(n)
        lv = seq_bfs(n, adj, src)
        rg.append({"n": n, "edges": [list(e) for e in edges], "src": src, "level": lv,
                   "invocations": max(lv) + 1})
    c["bfs_random_connected"] = {"ref": "SPEC.md:549 acceptance item 1 (levels = sequential BFS, "
                                        "rounds = ecc(src)+1)", "graphs": rg}
    with open(os.path.join(HERE, "spec_examples.json"), "w") as f:
        json.dump(g, f, indent=1, sort_keys=True)
        f.write("\n")


if __name__ == "__main__":
    main()
