// bfs_listing2.cpp — Listing 2 of the paper written against the C++ operator
// API, both as the runtime's Iterate and as a host loop of Invoke with between_rounds {LEVEL++}.
//
//   Kernel BFS(graph, LEVEL) { ForAll(wlidx In wl) { n = wl.pop(wlidx)
//     ForAll(e In graph.edges(n)) { if (e.dst.level == INF) { e.dst.level = LEVEL; wl.push(e.dst.id) } } } }
//   LEVEL = 0; Iterate BFS(graph, LEVEL) Initial [src] { LEVEL++; }
//
// Usage: bfs_listing2 [scale]   (prints levels of the 5-node path, then an RMAT summary)
#include <cstdio>
#include <cstdlib>

#include "irgl/irgl.hpp"

int main(int argc, char** argv) {
  try {
    irgl::Context ctx;
    // 5-node path, src = 0 -> [0, 1, 2, 3, 4]
    std::vector<int64_t> rp = {0, 1, 3, 5, 7, 8};
    std::vector<int32_t> col = {1, 0, 2, 1, 3, 2, 4, 3};
    irgl::Graph path = ctx.csr(5, rp, col);
    irgl::Pipe wl = ctx.pipe(5);
    wl.initial({0});
    int64_t LEVEL = 1;  // level[src] = 0 is preset by the operator reset (App. B2)
    const int64_t rounds = ctx.iterate_host(IRGL_OP_BFS, path, wl, LEVEL, [&] { ++LEVEL; });
    std::vector<int32_t> level = ctx.result<int32_t>(IRGL_OP_BFS, path);
    std::printf("level = [%d, %d, %d, %d, %d]  invocations = %lld\n", level[0], level[1], level[2],
                level[3], level[4], (long long)rounds);
    if (level != std::vector<int32_t>{0, 1, 2, 3, 4} || rounds != 5) return 1;

    const int scale = argc > 1 ? std::atoi(argv[1]) : 16;
    irgl::Graph g = ctx.rmat(scale);
    irgl::Pipe p = ctx.pipe(g.info().n);
    p.initial({1});
    irgl_iter_stats st = ctx.iterate(IRGL_OP_BFS, &g, &p);
    std::printf("RMAT-%d BFS: rounds=%lld edges=%lld outlined=%d %.3f ms\n", scale,
                (long long)st.rounds, (long long)st.edges, st.outlined, st.device_ms);
    return 0;
  } catch (const irgl::Error& e) {
    std::fprintf(stderr, "irgl error: %s\n", e.what());
    return 2;
  }
}
