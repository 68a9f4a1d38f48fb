/* frontend.h — IrGL source front end over the B200 runtime.
 *
 * Parses the concrete IrGL notation of the paper's listings (Kernel / ForAll / Iterate / Invoke /
 * Pipe / ReduceAndReturn / wl.pop / wl.push ..., Table 1 :63-103, Listing 2 :288-304)
 * into an AST, recognises the plain kernels this runtime implements (BFS, SSSP, CC label
 * propagation, PageRank) by structural match against their IrGL form, and executes the host
 * code: the orchestration statements drive irgl_iterate / irgl_invoke on the GPU.
 *
 * Replaces (reference, specified but not shipped): frontend::parse_source and
 * interp::run_host for programs whose plain kernels are recognised; the
 * statement-level CBlock interpreter is out of scope, so an unrecognised plain
 * kernel is an IRGL_E_UNSUPPORTED diagnostic, never a silent skip.  Errors are values with stable
 * rule ids ("file:line:col: error[RULE]: message", diag.hpp:20-29 convention).
 */
#ifndef IRGL_FRONTEND_H
#define IRGL_FRONTEND_H

#include "irgl/rt.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct irgl_module irgl_module;

/* parse_source: text -> Module.  On failure returns IRGL_E_INVALID and writes the
 * diagnostics into diag (NUL-terminated, truncated to diag_len). */
irgl_status_t irgl_module_parse(const char* text, const char* filename, irgl_module** out,
                                char* diag, size_t diag_len);
irgl_status_t irgl_module_destroy(irgl_module* m);

/* Number of kernels, and the runtime operator a kernel was recognised as (-1: not recognised, or
 * a host kernel).  `field` receives the node property the kernel writes (e.g. "level"). */
int irgl_module_kernel_count(const irgl_module* m);
irgl_status_t irgl_module_kernel_info(const irgl_module* m, int index, char* name, size_t name_len,
                                      int32_t* op, char* field, size_t field_len, int32_t* host);

/* Canonical pretty print: parse(print(m)) is structurally equal to m. */
irgl_status_t irgl_module_print(const irgl_module* m, char* out, size_t out_len, size_t* needed);

typedef struct irgl_run_info {
  int32_t last_op;        /* operator of the last orchestration statement run (-1: none)      */
  int32_t last_reduced;   /* last Any/All value (-1: none)                                       */
  int64_t invocations;    /* kernel invocations (Iterate rounds + Invokes)                       */
  int64_t orchestrations; /* Iterate / Invoke statements executed                                 */
  int64_t reserved[4];
} irgl_run_info;

/* run_host: executes the host code of `entry` (NULL: the module's top-level
 * statements) sequentially.  `g` is bound to every graph-typed name; names[i] = values[i] bind the
 * host scalars (e.g. src = 0).  Orchestration statements run on the GPU through irgl_iterate /
 * irgl_invoke; node results are then read with irgl_read_result(ctx, g, info.last_op, ...). */
irgl_status_t irgl_run_host(irgl_ctx* ctx, irgl_module* m, const char* entry, irgl_graph* g,
                            const char* const* names, const double* values, int nbind,
                            irgl_run_info* info, char* diag, size_t diag_len);

/* Final value of a host scalar after irgl_run_host (e.g. LEVEL). */
irgl_status_t irgl_module_scalar(const irgl_module* m, const char* name, double* out);

#ifdef __cplusplus
}
#endif
#endif /* IRGL_FRONTEND_H */
