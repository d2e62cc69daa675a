/*
 * flashrnn_csp.h -- C ABI of the tiling solver's integer CSP engine (part of
 * libflashrnn.so; see paper_2412_07752_b200/csrc/csp.h).
 *
 * Replaces, for FFI callers, the reference's ConstrINT core:
 *   rnnkit::csp::solve             (/root/reference/proj/core/include/rnnkit/csp/solver.hpp:20-22)
 *   rnnkit::csp::brute_force_solve (solver.hpp:24-29)
 * Problems travel in a line-oriented text form (csp.h `parse`):
 *   v <id> <C|R|I> r <lo> <hi> | s <lo> <hi> <step> | e <v1> <v2> ...   variables (index = order)
 *   n v <var> | n + <node> <node> | n * <node> <node>                    expression nodes
 *   c = <node> <node> | c < <node> <node> | c | <node> <node>            ==, <=, divides
 *   h <var> <S|L>                                                        heuristic order
 * Results are written as "id=value" lines (resolution variables).
 */
#ifndef FLASHRNN_CSP_H_
#define FLASHRNN_CSP_H_
#include <stddef.h>
#include <stdint.h>

#include "flashrnn.h"
#ifdef __cplusplus
extern "C" {
#endif
/* First solution in heuristic order.  FRNN_OK (written to out), FRNN_EINFEASIBLE
 * (no solution), FRNN_EINVAL_ARG (malformed problem / out too small).
 * stats (nullable): [0] search nodes, [1] backtracks, [2] solve time in ns. */
FRNN_API int frnn_csp_solve(const char* problem, char* out, size_t out_bytes, int64_t* stats);
/* Every solution (exhaustive; the search space must be <= cap).  Solutions are
 * separated by a line "--".  *count receives the number of solutions. */
FRNN_API int frnn_csp_brute_force(const char* problem, int64_t cap, char* out, size_t out_bytes, int64_t* count);
#ifdef __cplusplus
}
#endif
#endif
