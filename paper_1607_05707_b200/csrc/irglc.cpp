// irglc — GPU-backed command line over the IrGL front end (the reference's CLI
// is specified at SPEC.md:507-545 and not shipped).  Subcommands:
//
//   irglc check FILE.irgl                       parse + recognise; prints each kernel's role
//   irglc run FILE.irgl --graph G.txt [--bind name=value ...] [--entry K] [--out PATH]
//         runs the host code on GPU 0 over the text edge list G.txt ("N M" then "u v [w]",
//         SPEC.md:497, symmetrised) and writes the last operator's node result as "v value"
//         lines (stdout by default)
//
// Exit codes: 0 success, 1 program / runtime diagnostics, 2 usage error.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "irgl/frontend.h"
#include "irgl/rt.h"

static int usage() {
  fprintf(stderr,
          "usage: irglc check FILE.irgl\n"
          "       irglc run FILE.irgl --graph EDGELIST [--bind NAME=VALUE]... [--entry KERNEL] [--out PATH]\n");
  return 2;
}

static const char* op_name(int op) {
  switch (op) {
    case IRGL_OP_BFS: return "BFS";
    case IRGL_OP_SSSP: return "SSSP";
    case IRGL_OP_CC_LP: return "CC_LP";
    case IRGL_OP_PR: return "PR";
    default: return "-";
  }
}

int main(int argc, char** argv) {
  if (argc < 3) return usage();
  const std::string cmd = argv[1], file = argv[2];
  std::ifstream in(file);
  if (!in) {
    fprintf(stderr, "irglc: cannot read %s\n", file.c_str());
    return 2;
  }
  std::stringstream ss;
  ss << in.rdbuf();
  std::vector<char> diag(1 << 16);
  irgl_module* m = nullptr;
  if (irgl_module_parse(ss.str().c_str(), file.c_str(), &m, diag.data(), diag.size()) != IRGL_OK) {
    fputs(diag.data(), stderr);
    return 1;
  }
  if (cmd == "check") {
    for (int i = 0; i < irgl_module_kernel_count(m); ++i) {
      char name[256], field[256];
      int32_t op = -1, host = 0;
      irgl_module_kernel_info(m, i, name, sizeof name, &op, field, sizeof field, &host);
      printf("%s: %s\n", name, host ? "host" : op >= 0 ? op_name(op) : "plain (not recognised)");
    }
    irgl_module_destroy(m);
    return 0;
  }
  if (cmd != "run") return usage();
  std::string graph, entry, out;
  std::vector<std::string> names;
  std::vector<double> vals;
  for (int i = 3; i < argc; ++i) {
    const std::string a = argv[i];
    if (i + 1 >= argc) return usage();
    if (a == "--graph") graph = argv[++i];
    else if (a == "--entry") entry = argv[++i];
    else if (a == "--out") out = argv[++i];
    else if (a == "--bind") {
      const std::string b = argv[++i];
      const size_t eq = b.find('=');
      if (eq == std::string::npos) return usage();
      names.push_back(b.substr(0, eq));
      vals.push_back(atof(b.c_str() + eq + 1));
    } else {
      return usage();
    }
  }
  if (graph.empty()) return usage();
  int dev = 0;
  irgl_ctx* ctx = nullptr;
  irgl_config cfg;
  memset(&cfg, 0, sizeof cfg);
  cfg.outline = -1;
  if (irgl_ctx_create(&dev, 1, &cfg, &ctx) != IRGL_OK) {
    fprintf(stderr, "irglc: %s\n", irgl_last_error(nullptr));
    return 1;
  }
  irgl_graph* g = nullptr;
  if (irgl_graph_read_edgelist(ctx, graph.c_str(), 1, &g) != IRGL_OK) {
    fprintf(stderr, "irglc: %s\n", irgl_last_error(ctx));
    return 1;
  }
  std::vector<const char*> np;
  for (const std::string& s : names) np.push_back(s.c_str());
  irgl_run_info info;
  if (irgl_run_host(ctx, m, entry.empty() ? nullptr : entry.c_str(), g, np.data(), vals.data(), (int)np.size(),
                    &info, diag.data(), diag.size()) != IRGL_OK) {
    fputs(diag.data(), stderr);
    return 1;
  }
  int rc = 0;
  if (info.last_op >= 0) {
    irgl_graph_info gi;
    irgl_graph_info_get(g, &gi);
    FILE* f = out.empty() ? stdout : fopen(out.c_str(), "w");
    if (!f) {
      fprintf(stderr, "irglc: cannot write %s\n", out.c_str());
      return 2;
    }
    if (info.last_op == IRGL_OP_PR) {
      std::vector<double> r(gi.n);
      if (irgl_read_result(ctx, g, IRGL_OP_PR, r.data(), r.size() * sizeof(double)) != IRGL_OK) rc = 1;
      for (int64_t v = 0; v < gi.n && !rc; ++v) fprintf(f, "%lld %.17g\n", (long long)v, r[v]);
    } else {
      std::vector<int32_t> r(gi.n);
      if (irgl_read_result(ctx, g, (irgl_op)info.last_op, r.data(), r.size() * 4) != IRGL_OK) rc = 1;
      for (int64_t v = 0; v < gi.n && !rc; ++v) {
        if (r[v] == 2147483647) fprintf(f, "%lld INF\n", (long long)v);
        else fprintf(f, "%lld %d\n", (long long)v, r[v]);
      }
    }
    if (f != stdout) fclose(f);
    if (rc) fprintf(stderr, "irglc: %s\n", irgl_last_error(ctx));
  }
  irgl_graph_destroy(g);
  irgl_ctx_destroy(ctx);
  irgl_module_destroy(m);
  return rc;
}
