/*
 * flashrnn.h -- C ABI of the B200-native FlashRNN engine (libflashrnn.so).
 *
 * Drop-in boundary for the reference's C++ operator API
 *   rnnkit::rnn::forward   (/root/reference/proj/core/include/rnnkit/rnn/engine.hpp:143-203)
 *   rnnkit::rnn::backward  (engine.hpp:221-339)
 * The C++ shim <flashrnn/engine.hpp> restores those exact signatures on top of
 * this ABI; INTEGRATION.md shows the binding a maintainer adds.
 *
 * Conventions
 *   - All tensor pointers are DEVICE pointers owned by the caller; nothing is
 *     allocated on the hot path.  Scratch comes from the caller's workspace
 *     (size from frnn_workspace_size).
 *   - Layouts are exactly rnnkit's (D = num_heads * head_dim):
 *       R       [NH][NG][DH][DH]   row = gate output, col = input state (engine.hpp:20, :24-27)
 *       bias    [NG][D]            (engine.hpp:21)
 *       x       [T][B][NG][D]      gate pre-inputs, W already applied (engine.hpp:50)
 *       s0      [NS][B][D]         (engine.hpp:51)
 *       states  [T+1][NS][B][D]    index 0 = s0 (engine.hpp:81)
 *       gates   [T][NG][B][D]      raw pre-activations (engine.hpp:82, :188)
 *       dx [T][B][NG][D], dbias [NG][D], dR [NH][NG][DH][DH], ds0 [NS][B][D] (engine.hpp:94-97)
 *       d_hidden [T][B][D]         StepGradients::hidden, nullable (engine.hpp:208-211)
 *   - dtype selects the element type of every tensor argument: FRNN_F32
 *     (float) or FRNN_BF16 (bfloat16 bits).  Arithmetic accumulates in fp32.
 *   - Launches are ordered on `stream` (a cudaStream_t, NULL = legacy default).
 *     Functions are reentrant across streams; the plan cache is mutex-guarded.
 *   - Errors are status codes; frnn_last_error() gives a thread-local message.
 *     There is NO CPU fallback: a missing/unsupported GPU returns FRNN_ECUDA or
 *     FRNN_EUNSUPPORTED.
 */
#ifndef FLASHRNN_H_
#define FLASHRNN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FRNN_ABI_VERSION 1

#if defined(__GNUC__)
#define FRNN_API __attribute__((visibility("default")))
#else
#define FRNN_API
#endif

/* Status codes.  EINVAL_* mirror the std::invalid_argument throws of the
 * reference: shape/count mismatch (engine.hpp:119-128), non-finite inputs
 * (:131-135, :146-147), trace/gradient size (:231-236), clip magnitude (:107). */
typedef enum {
  FRNN_OK = 0,
  FRNN_EINVAL_SHAPE = 1,   /* cell/params/batch counts or sizes disagree, degenerate shape */
  FRNN_ENONFINITE = 2,     /* non-finite input or initial state (forward only) */
  FRNN_EUNSUPPORTED = 3,   /* valid but not implemented on this device (e.g. dtype) */
  FRNN_EINFEASIBLE = 4,    /* the tiling solver found no plan */
  FRNN_ECUDA = 5,          /* CUDA runtime/driver error, or no sm_100 device */
  FRNN_EINVAL_ARG = 6      /* NULL pointer, workspace too small, bad clip magnitude */
} frnn_status;

typedef enum { FRNN_F32 = 0, FRNN_BF16 = 1 } frnn_dtype;

/* cell.hpp:11 Variant */
typedef enum { FRNN_ELMAN = 0, FRNN_LSTM = 1, FRNN_GRU = 2, FRNN_SLSTM = 3 } frnn_variant;

/* cell.hpp:16-23 CellSpec (the name string is implied by the variant). */
typedef struct {
  int32_t variant;             /* frnn_variant: selects the pointwise map */
  int32_t num_states;          /* N_s */
  int32_t num_gates;           /* N_g (<= 4) */
  uint8_t uses_recurrent[4];   /* gate_uses_recurrent */
  uint8_t uses_input[4];       /* gate_uses_input */
} frnn_cell;

typedef struct {
  int32_t seq_len;    /* T  (>= 0) */
  int32_t batch;      /* B  (>= 1) */
  int32_t num_heads;  /* NH (>= 1) */
  int32_t head_dim;   /* DH (>= 1) */
} frnn_shape;

/* engine.hpp:100-111 ClipPolicy */
typedef enum { FRNN_CLIP_OFF = 0, FRNN_CLIP_VALUE = 1, FRNN_CLIP_ZERO = 2 } frnn_clip_mode;
typedef struct {
  int32_t mode;       /* frnn_clip_mode */
  double magnitude;   /* > 0 for FRNN_CLIP_VALUE */
} frnn_clip;

typedef enum { FRNN_PASS_FORWARD = 0, FRNN_PASS_BACKWARD = 1 } frnn_pass;

/* Kernel family chosen by the planner (or forced through frnn_options). */
typedef enum {
  FRNN_ALGO_AUTO = 0,
  FRNN_ALGO_FUSED = 1,        /* persistent kernel, R resident on-chip (tcgen05, bf16) */
  FRNN_ALGO_ALTERNATING = 2,  /* one fused GEMM+pointwise launch per step, R streamed */
  FRNN_ALGO_SIMT = 3          /* persistent fp32 FFMA kernel, R in shared memory */
} frnn_algo;

/* Flags for frnn_options.flags */
#define FRNN_FLAG_CHECK_FINITE 0x1u  /* forward: scan x/s0, return FRNN_ENONFINITE (syncs) */

typedef struct {
  uint32_t flags;     /* FRNN_FLAG_* */
  int32_t algo;       /* frnn_algo; FRNN_ALGO_AUTO lets the solver choose */
} frnn_options;

/* Solved tiling (the ConstrINT-style solver's output). */
typedef struct {
  int32_t algo;              /* frnn_algo actually used */
  int32_t rows_per_cta;      /* gate rows (M) per CTA: tcgen05 M tile */
  int32_t batch_tile;        /* batch columns (N) per CTA */
  int32_t ctas_per_group;    /* CTAs that synchronise per step (one head x batch tile) */
  int32_t groups;            /* independent groups = heads x batch tiles */
  int32_t grid;              /* total CTAs */
  int32_t threads;           /* threads per CTA */
  int32_t smem_bytes;        /* dynamic shared memory per CTA */
  int32_t tmem_cols;         /* TMEM columns allocated per CTA */
  int32_t k_split;           /* accumulating-axis split (alternating path) */
  int64_t workspace_bytes;   /* scratch the pass needs */
  double solve_us;           /* solver wall time */
  int32_t cluster;           /* >0: thread-block cluster size of the cluster-resident fused kernels */
} frnn_plan_info;

/* -- metadata ----------------------------------------------------------- */
FRNN_API const char* frnn_version(void);
FRNN_API const char* frnn_last_error(void);           /* thread-local; "" when none */
FRNN_API int frnn_cell_spec(int32_t variant, frnn_cell* out);          /* cell.hpp:25-53 */

/* -- planning ----------------------------------------------------------- */
FRNN_API int frnn_plan(const frnn_cell* cell, frnn_shape shape, int32_t dtype, int32_t pass,
              const frnn_options* opts, frnn_plan_info* out);
FRNN_API int frnn_workspace_size(const frnn_cell* cell, frnn_shape shape, int32_t dtype, int32_t pass,
                        const frnn_options* opts, size_t* bytes);
/* The plan as JSON (schema_version 1, the counterpart of rnnkit::plan::plan_to_json,
 * planner.cpp:428-453): shape, kernel family, tiling, footprint, solve time. */
FRNN_API int frnn_plan_json(const frnn_cell* cell, frnn_shape shape, int32_t dtype, int32_t pass,
                            const frnn_options* opts, char* out, size_t out_bytes);
/* Re-check of the solved plan against every constraint of its kernel family
 * (the counterpart of rnnkit::plan::plan_residuals, planner.cpp:349-402): writes
 * a JSON array of violations ("[]" when every residual is zero) and returns
 * FRNN_OK, or FRNN_EINFEASIBLE when there is any.  frnn_plan_json also reports
 * the plan's per-step traffic (hbm_traffic_per_step, planner.cpp:233-243). */
FRNN_API int frnn_plan_check(const frnn_cell* cell, frnn_shape shape, int32_t dtype, int32_t pass,
                             const frnn_options* opts, char* out, size_t out_bytes);
/* Persistent plan cache (the paper's cached solver solutions):
 * JSON lines, one solved plan per line (schema_version 1), tagged with the
 * library version and device limits; load skips lines from another build or
 * device.  Setting FRNN_PLAN_CACHE=<file> loads it before the first plan and
 * appends every new solve. */
FRNN_API int frnn_plan_cache_save(const char* path);
FRNN_API int frnn_plan_cache_load(const char* path, int32_t* loaded);
FRNN_API int frnn_plan_cache_clear(void);

/* -- the hot path --------------------------------------------------------- */
/* engine.hpp:143-203.  Writes states (incl. states[0] = s0) and gates. */
FRNN_API int frnn_forward(const frnn_cell* cell, frnn_shape shape, int32_t dtype,
                 const void* R, const void* bias, const void* x, const void* s0,
                 void* states, void* gates,
                 void* workspace, size_t workspace_bytes,
                 const frnn_options* opts, void* stream);

/* engine.hpp:221-339.  d_hidden may be NULL.  dx/dbias/dR/ds0 are fully
 * overwritten (dx is zero for gates with uses_input == 0, dR zero for gates
 * with uses_recurrent == 0). */
FRNN_API int frnn_backward(const frnn_cell* cell, frnn_shape shape, int32_t dtype,
                  const void* R, const void* bias, const void* states, const void* gates,
                  const void* d_states_final, const void* d_hidden, frnn_clip clip,
                  void* dx, void* dbias, void* dR, void* ds0,
                  void* workspace, size_t workspace_bytes,
                  const frnn_options* opts, void* stream);

/* -- the step before the path: input projection ---------------------------- */
/* x = u . W^T, the gate pre-inputs rnnkit's engine takes already projected
 * (SPEC.md:376):
 *   u [tokens][in_features]            tokens = T*B, row-major (u[t][b][k])
 *   W [out_features][in_features]      out_features = NG*D, row j*D + e
 *   x [tokens][out_features]           = rnnkit's x[T][B][NG][D]
 * bf16 in, fp32 accumulate (tcgen05), bf16 out; in_features % 8 == 0. */
FRNN_API int frnn_input_projection(const void* W, const void* u, void* x, int64_t tokens, int32_t out_features,
                                   int32_t in_features, int32_t dtype, void* stream);

/* -- multi-GPU partitioner (batch x head sharding) --------------- */
typedef struct {
  int32_t batch_begin, batch_end;   /* [begin, end) rows of B owned by this rank */
  int32_t head_begin, head_end;     /* [begin, end) heads owned by this rank */
  int32_t reduce_params;            /* 1: dR/db must be sum-reduced across batch shards */
} frnn_shard;
FRNN_API int frnn_partition(frnn_shape shape, int32_t world_size, int32_t rank, frnn_shard* out);

#ifdef __cplusplus
}
#endif
#endif /* FLASHRNN_H_ */
