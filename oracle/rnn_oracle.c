/*
 * oracle/rnn_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference rnnkit engine (the FlashRNN reference
 * implementation) used as the parity CHECKER for the B200 kernels.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library.  The product path (paper_2412_07752_b200/) never links or
 * calls it; there is no CPU fallback.
 *
 * Parity of this restatement is PINNED against the unmodified reference
 * compiled from /root/reference (oracle/_ref/libref.so, built by
 * oracle/Makefile) and against the golden vectors in tests/golden/ that the
 * reference produced (tests/golden/make_golden.py).
 *
 * Every function cites the reference file:line it restates.  Paths are
 * relative to /root/reference/proj/core/include/rnnkit/rnn/.
 *
 * Build: gcc -O3 -fopenmp -ffp-contract=off -fPIC -shared (oracle/Makefile).  No
 * FMA contraction, so float results are bit-identical to the reference
 * engine<float> compiled with the same flags.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- cells -- */
/* cell.hpp:11 enum class Variant { Elman, Lstm, Gru, Slstm } */
enum { ORC_ELMAN = 0, ORC_LSTM = 1, ORC_GRU = 2, ORC_SLSTM = 3 };

typedef struct {
  int variant;
  int num_states;
  int num_gates;
  int uses_rec[4];
  int uses_in[4];
} orc_cell;

/* cell.hpp:25-53 cell_spec */
orc_cell orc_cell_spec(int v) {
  orc_cell c;
  c.variant = v;
  for (int j = 0; j < 4; ++j) { c.uses_rec[j] = 1; c.uses_in[j] = 1; }
  switch (v) {
    case ORC_ELMAN: c.num_states = 1; c.num_gates = 1; break;
    case ORC_LSTM: c.num_states = 2; c.num_gates = 4; break;
    case ORC_GRU:
      c.num_states = 1; c.num_gates = 4;
      c.uses_rec[2] = 0; /* n skips the R term, cell.hpp:43 */
      c.uses_in[3] = 0;  /* g skips the input,  cell.hpp:44 */
      break;
    default: c.num_states = 4; c.num_gates = 4; break; /* sLSTM h,c,n,m */
  }
  return c;
}

/* --------------------------------------------------------------- numerics */
/* scalar.hpp:50-76.  Instantiated for double (suffix d) and float (f). */
#define DEF_NUM(S, SUF, TANH, EXP, LOG1P)                                          \
  static inline S sig_##SUF(S x) { return (S)1 / ((S)1 + EXP(-x)); } /* :58-62 */ \
  static inline S logsig_##SUF(S x) { /* :64-70 */                                 \
    return x >= 0 ? -LOG1P(EXP(-x)) : x - LOG1P(EXP(x));                           \
  }                                                                                \
  static inline S max_##SUF(S a, S b) { return a > b ? a : b; } /* :73-76 */

DEF_NUM(double, d, tanh, exp, log1p)
DEF_NUM(float, f, tanhf, expf, log1pf)

/* cell.hpp:65-99 pointwise_forward ; cell.hpp:108-201 pointwise_jacobians */
#define DEF_CELL(S, SUF, TANH, EXP)                                                     \
  static void pw_fwd_##SUF(const orc_cell* cell, const S* prev, const S* g, S* next) { \
    switch (cell->variant) {                                                           \
      case ORC_ELMAN: next[0] = TANH(g[0]); break; /* :69-72 */                        \
      case ORC_LSTM: { /* :73-78 */                                                    \
        S c = sig_##SUF(g[1]) * prev[1] + sig_##SUF(g[2]) * TANH(g[0]);                \
        next[0] = sig_##SUF(g[3]) * TANH(c);                                           \
        next[1] = c;                                                                   \
        break;                                                                         \
      }                                                                                \
      case ORC_GRU: { /* :79-84 */                                                     \
        S sz = sig_##SUF(g[0]);                                                        \
        S inner = g[2] + sig_##SUF(g[1]) * TANH(g[3]);                                 \
        next[0] = sz * prev[0] + ((S)1 - sz) * TANH(inner);                            \
        break;                                                                         \
      }                                                                                \
      default: { /* :85-97 */                                                          \
        S a = logsig_##SUF(g[1]) + prev[3];                                            \
        S m = max_##SUF(a, g[2]);                                                      \
        S fexp = EXP(a - m);                                                           \
        S iexp = EXP(g[2] - m);                                                        \
        S c = fexp * prev[1] + iexp * TANH(g[0]);                                      \
        S n = fexp * prev[2] + iexp;                                                   \
        next[0] = sig_##SUF(g[3]) * (c / n);                                           \
        next[1] = c;                                                                   \
        next[2] = n;                                                                   \
        next[3] = m;                                                                   \
        break;                                                                         \
      }                                                                                \
    }                                                                                  \
  }                                                                                    \
  static void pw_jac_##SUF(const orc_cell* cell, const S* prev, const S* g, S dg[4][4], \
                           S dp[4][4]) {                                               \
    memset(dg, 0, sizeof(S) * 16);                                                     \
    memset(dp, 0, sizeof(S) * 16);                                                     \
    switch (cell->variant) {                                                           \
      case ORC_ELMAN: { S t = TANH(g[0]); dg[0][0] = (S)1 - t * t; break; }            \
      case ORC_LSTM: { /* :119-135 */                                                  \
        S sf = sig_##SUF(g[1]), si = sig_##SUF(g[2]), so = sig_##SUF(g[3]);            \
        S tz = TANH(g[0]);                                                             \
        S c = sf * prev[1] + si * tz;                                                  \
        S tc = TANH(c);                                                                \
        S dtc = (S)1 - tc * tc;                                                        \
        dg[1][0] = si * ((S)1 - tz * tz);                                              \
        dg[1][1] = sf * ((S)1 - sf) * prev[1];                                         \
        dg[1][2] = si * ((S)1 - si) * tz;                                              \
        dp[1][1] = sf;                                                                 \
        for (int j = 0; j < 3; ++j) dg[0][j] = so * dtc * dg[1][j];                    \
        dg[0][3] = so * ((S)1 - so) * tc;                                              \
        dp[0][1] = so * dtc * sf;                                                      \
        break;                                                                         \
      }                                                                                \
      case ORC_GRU: { /* :136-149 */                                                   \
        S sz = sig_##SUF(g[0]), sr = sig_##SUF(g[1]);                                  \
        S tg = TANH(g[3]);                                                             \
        S u = g[2] + sr * tg;                                                          \
        S tu = TANH(u);                                                                \
        S dtu = (S)1 - tu * tu;                                                        \
        S omz = (S)1 - sz;                                                             \
        dg[0][0] = sz * ((S)1 - sz) * (prev[0] - tu);                                  \
        dg[0][1] = omz * dtu * sr * ((S)1 - sr) * tg;                                  \
        dg[0][2] = omz * dtu;                                                          \
        dg[0][3] = omz * dtu * sr * ((S)1 - tg * tg);                                  \
        dp[0][0] = sz;                                                                 \
        break;                                                                         \
      }                                                                                \
      default: { /* :150-198 */                                                        \
        S sf = sig_##SUF(g[1]), so = sig_##SUF(g[3]);                                  \
        S a = logsig_##SUF(g[1]) + prev[3];                                            \
        int use_a = !(a < g[2]); /* ties -> forget branch, :153 */                    \
        S m = use_a ? a : g[2];                                                        \
        S fexp = EXP(a - m);                                                           \
        S iexp = EXP(g[2] - m);                                                        \
        S tz = TANH(g[0]);                                                             \
        S c = fexp * prev[1] + iexp * tz;                                              \
        S n = fexp * prev[2] + iexp;                                                   \
        S da_df = (S)1 - sf;                                                           \
        S dm_df = use_a ? da_df : (S)0;                                                \
        S dm_di = use_a ? (S)0 : (S)1;                                                 \
        S dm_dmp = use_a ? (S)1 : (S)0;                                                \
        S dfexp_df = fexp * (da_df - dm_df);                                           \
        S diexp_df = -iexp * dm_df;                                                    \
        S dfexp_di = -fexp * dm_di;                                                    \
        S diexp_di = iexp * ((S)1 - dm_di);                                            \
        S dfexp_dmp = fexp * ((S)1 - dm_dmp);                                          \
        S diexp_dmp = -iexp * dm_dmp;                                                  \
        dg[1][0] = iexp * ((S)1 - tz * tz);                                            \
        dg[1][1] = dfexp_df * prev[1] + diexp_df * tz;                                 \
        dg[1][2] = dfexp_di * prev[1] + diexp_di * tz;                                 \
        dp[1][1] = fexp;                                                               \
        dp[1][3] = dfexp_dmp * prev[1] + diexp_dmp * tz;                               \
        dg[2][1] = dfexp_df * prev[2] + diexp_df;                                      \
        dg[2][2] = dfexp_di * prev[2] + diexp_di;                                      \
        dp[2][2] = fexp;                                                               \
        dp[2][3] = dfexp_dmp * prev[2] + diexp_dmp;                                    \
        dg[3][1] = dm_df;                                                              \
        dg[3][2] = dm_di;                                                              \
        dp[3][3] = dm_dmp;                                                             \
        S inv_n = (S)1 / n;                                                            \
        S h_over = c * inv_n;                                                          \
        for (int j = 0; j < 4; ++j) dg[0][j] = so * (dg[1][j] - h_over * dg[2][j]) * inv_n; \
        dg[0][3] = dg[0][3] + so * ((S)1 - so) * h_over;                               \
        for (int k = 0; k < 4; ++k) dp[0][k] = so * (dp[1][k] - h_over * dp[2][k]) * inv_n; \
        break;                                                                         \
      }                                                                                \
    }                                                                                  \
  }

DEF_CELL(double, d, tanh, exp)
DEF_CELL(float, f, tanhf, expf)

/* ------------------------------------------------------------- engine --- */
/* Layouts (engine.hpp:20-21, :50-51, :81-82, :94-97):
 *   R[NH][NG][DH][DH], bias[NG][D], x[T][B][NG][D], s0[NS][B][D],
 *   states[T+1][NS][B][D], gates[T][NG][B][D], D = NH*DH.               */
#define RIDX(hd, j, r, c) ((((size_t)(hd) * NG + (j)) * DH + (r)) * DH + (c))
#define XIDX(t, b, j, e) ((((size_t)(t) * B + (b)) * NG + (j)) * D + (e))
#define SIDX(t, i, b, e) ((((size_t)(t) * NS + (i)) * B + (b)) * D + (e))
#define GIDX(t, j, b, e) ((((size_t)(t) * NG + (j)) * B + (b)) * D + (e))
#define DSIDX(i, b, e) (((size_t)(i) * B + (b)) * D + (e))

/* Loop orders.  Every output element below is produced by EXACTLY the
 * sequence of floating-point operations the reference performs for it
 * (same operands, same order, same rounding; -ffp-contract=off), so the
 * results are bit-identical to the reference engine -- pinned by
 * tests/test_oracle.py.  What differs is only which element is computed when:
 *   - R.h (engine.hpp:178-182) keeps each gate's ascending-c sum but runs the
 *     B sums of one R row side by side (h transposed to [D][B]), so R is read
 *     once per step and the inner loop vectorises across b;
 *   - R^T.dg (:291-305) keeps each column's (j ascending, r ascending) sum but
 *     walks R row-major with the column accumulators in a [B][chunk] array;
 *   - dR (:321-334) keeps each element's ascending-b sum in an accumulator
 *     row before the single += into dR.
 * Independent elements are spread over OpenMP threads (OMP_NUM_THREADS);
 * nothing is reduced across threads, so the thread count
 * never changes a bit.  This is what lets the checker run the headline
 * shape (T=1024, B=16, H=768) in seconds.                                  */
#define ORC_BT 16   /* batch rows per R.h register block   */
#define ORC_CC 32   /* R^T.dg columns per task              */

/* engine.hpp:143-203 forward (finiteness/shape checks are the caller's). */
#define DEF_FWD(S, SUF, CS)                                                               \
  void orc_forward_##SUF(const orc_cell* cell, int T, int B, int NH, int DH,        \
                         const S* R, const S* bias, const S* x, const S* s0,       \
                         S* states, S* gates) {                                    \
    const int NS = cell->num_states, NG = cell->num_gates, D = NH * DH;             \
    memcpy(states, s0, sizeof(S) * (size_t)NS * B * D); /* :161-164 */             \
    S* hT = (S*)malloc(sizeof(S) * (size_t)D * (B > 0 ? B : 1));                   \
    for (int t = 0; t < T; ++t) {                                                  \
      const S* sp0 = &states[SIDX(t, 0, 0, 0)];                                    \
      _Pragma("omp parallel for schedule(static)")                                 \
      for (int e = 0; e < D; ++e)                                                  \
        for (int b = 0; b < B; ++b) hT[(size_t)e * B + b] = sp0[(size_t)b * D + e]; \
      _Pragma("omp parallel for collapse(2) schedule(dynamic, 8)")                 \
      for (int j = 0; j < NG; ++j)                                                 \
        for (int e = 0; e < D; ++e) {                                              \
          const int hd = e / DH, r = e % DH;                                       \
          for (int b0 = 0; b0 < B; b0 += ORC_BT) {                                 \
            const int nb = B - b0 < ORC_BT ? B - b0 : ORC_BT;                       \
            S y[ORC_BT];                                                           \
            for (int k = 0; k < ORC_BT; ++k) y[k] = 0;                             \
            if (cell->uses_rec[j]) { /* :178-182 ascending c */                   \
              const S* row = &R[RIDX(hd, j, r, 0)];                                \
              const S* hc = hT + (size_t)hd * DH * B + b0;                         \
              if (nb == ORC_BT) {                                                  \
                for (int c = 0; c < DH; ++c)                                       \
                  for (int k = 0; k < ORC_BT; ++k) y[k] += row[c] * hc[(size_t)c * B + k]; \
              } else {                                                             \
                for (int c = 0; c < DH; ++c)                                       \
                  for (int k = 0; k < nb; ++k) y[k] += row[c] * hc[(size_t)c * B + k]; \
              }                                                                    \
            }                                                                      \
            for (int k = 0; k < nb; ++k) {                                         \
              const int b = b0 + k;                                                \
              S acc = cell->uses_in[j] ? x[XIDX(t, b, j, e)] : (S)0; /* :183-187 */ \
              acc += bias[(size_t)j * D + e];                                      \
              acc += y[k];                                                         \
              gates[GIDX(t, j, b, e)] = acc;                                       \
            }                                                                      \
          }                                                                        \
        }                                                                          \
      _Pragma("omp parallel for collapse(2) schedule(static)") /* :193-200 */     \
      for (int b = 0; b < B; ++b)                                                  \
        for (int e = 0; e < D; ++e) {                                              \
          S prev[4], g[4], next[4];                                                \
          for (int i = 0; i < NS; ++i) prev[i] = states[SIDX(t, i, b, e)];          \
          for (int j = 0; j < NG; ++j) g[j] = gates[GIDX(t, j, b, e)];              \
          pw_fwd_##CS(cell, prev, g, next);                                       \
          for (int i = 0; i < NS; ++i) states[SIDX(t + 1, i, b, e)] = next[i];      \
        }                                                                          \
    }                                                                              \
    free(hT);                                                                      \
  }

DEF_FWD(double, f64, d)
DEF_FWD(float, f32, f)

/* engine.hpp:100-111 ClipPolicy modes */
enum { ORC_CLIP_OFF = 0, ORC_CLIP_VALUE = 1, ORC_CLIP_ZERO = 2 };

/* engine.hpp:221-339 backward.  d_hidden (StepGradients::hidden, [T][B][D])
 * may be NULL.  Outputs are fully overwritten.                            */
#define DEF_BWD(S, SUF, CS)                                                               \
  void orc_backward_##SUF(const orc_cell* cell, int T, int B, int NH, int DH,       \
                          const S* R, const S* states, const S* gates,             \
                          const S* d_states_final, int clip_mode, double clip_mag, \
                          const S* d_hidden, S* dx, S* dbias, S* dR, S* ds0) {     \
    const int NS = cell->num_states, NG = cell->num_gates, D = NH * DH;             \
    const size_t nst = (size_t)NS * B * D;                                         \
    memset(dx, 0, sizeof(S) * (size_t)T * B * NG * D);                             \
    memset(dbias, 0, sizeof(S) * (size_t)NG * D);                                  \
    memset(dR, 0, sizeof(S) * (size_t)NH * NG * DH * DH);                          \
    S* ds_cur = (S*)malloc(sizeof(S) * (nst ? nst : 1));                           \
    S* ds_prev = (S*)malloc(sizeof(S) * (nst ? nst : 1));                          \
    S* dg = (S*)malloc(sizeof(S) * ((size_t)NG * B * D + 1));                      \
    memcpy(ds_cur, d_states_final, sizeof(S) * nst); /* :248 */                    \
    const S mag = (S)clip_mag; /* :255 */                                          \
    const int ncc = (DH + ORC_CC - 1) / ORC_CC;                                    \
    for (int t = T - 1; t >= 0; --t) {                                             \
      if (d_hidden) /* :258-263 */                                                 \
        for (int b = 0; b < B; ++b)                                                \
          for (int e = 0; e < D; ++e)                                              \
            ds_cur[DSIDX(0, b, e)] += d_hidden[((size_t)t * B + b) * D + e];        \
      _Pragma("omp parallel for collapse(2) schedule(static)") /* :267-286 */     \
      for (int b = 0; b < B; ++b)                                                  \
        for (int e = 0; e < D; ++e) {                                              \
          S prev[4], g[4], dsl[4], Jg[4][4], Jp[4][4];                             \
          for (int i = 0; i < NS; ++i) {                                           \
            prev[i] = states[SIDX(t, i, b, e)];                                    \
            dsl[i] = ds_cur[DSIDX(i, b, e)];                                       \
          }                                                                        \
          for (int j = 0; j < NG; ++j) g[j] = gates[GIDX(t, j, b, e)];              \
          pw_jac_##CS(cell, prev, g, Jg, Jp);                                     \
          for (int j = 0; j < NG; ++j) {                                           \
            S acc = 0;                                                             \
            for (int i = 0; i < NS; ++i) acc += Jg[i][j] * dsl[i];                 \
            dg[((size_t)j * B + b) * D + e] = acc;                                 \
          }                                                                        \
          for (int k = 0; k < NS; ++k) {                                           \
            S acc = 0;                                                             \
            for (int i = 0; i < NS; ++i) acc += Jp[i][k] * dsl[i];                 \
            ds_prev[DSIDX(k, b, e)] = acc;                                         \
          }                                                                        \
        }                                                                          \
      if (clip_mode != ORC_CLIP_ZERO) { /* :289-308 */                             \
        _Pragma("omp parallel for collapse(2) schedule(dynamic, 1)")               \
        for (int hd = 0; hd < NH; ++hd)                                            \
          for (int cc = 0; cc < ncc; ++cc) {                                       \
            const int c0 = cc * ORC_CC;                                            \
            const int nc = DH - c0 < ORC_CC ? DH - c0 : ORC_CC;                     \
            S* term = (S*)calloc((size_t)B * ORC_CC, sizeof(S));                   \
            for (int j = 0; j < NG; ++j) {                                         \
              if (!cell->uses_rec[j]) continue;                                    \
              for (int r = 0; r < DH; ++r) {                                       \
                const S* Rr = &R[RIDX(hd, j, r, c0)];                              \
                for (int b = 0; b < B; ++b) {                                      \
                  const S d = dg[((size_t)j * B + b) * D + hd * DH + r];           \
                  S* tb = term + (size_t)b * ORC_CC;                               \
                  for (int c = 0; c < nc; ++c) tb[c] += Rr[c] * d;                 \
                }                                                                  \
              }                                                                    \
            }                                                                      \
            for (int b = 0; b < B; ++b)                                            \
              for (int c = 0; c < nc; ++c) {                                       \
                S v = term[(size_t)b * ORC_CC + c];                                \
                if (clip_mode == ORC_CLIP_VALUE) {                                 \
                  if (v > mag) v = mag;                                            \
                  if (v < -mag) v = -mag;                                          \
                }                                                                  \
                ds_prev[DSIDX(0, b, hd * DH + c0 + c)] += v;                       \
              }                                                                    \
            free(term);                                                            \
          }                                                                        \
      }                                                                            \
      _Pragma("omp parallel for collapse(2) schedule(static)") /* :311-320 */     \
      for (int j = 0; j < NG; ++j)                                                 \
        for (int e = 0; e < D; ++e)                                                \
          for (int b = 0; b < B; ++b) {                                            \
            S v = dg[((size_t)j * B + b) * D + e];                                 \
            if (cell->uses_in[j]) dx[XIDX(t, b, j, e)] = v;                        \
            dbias[(size_t)j * D + e] += v;                                         \
          }                                                                        \
      _Pragma("omp parallel for collapse(3) schedule(dynamic, 4)") /* :321-334 */ \
      for (int hd = 0; hd < NH; ++hd)                                              \
        for (int j = 0; j < NG; ++j)                                               \
          for (int r = 0; r < DH; ++r) {                                           \
            if (!cell->uses_rec[j]) continue;                                      \
            S* acc = (S*)calloc((size_t)DH, sizeof(S));                            \
            for (int b = 0; b < B; ++b) {                                          \
              const S d = dg[((size_t)j * B + b) * D + hd * DH + r];               \
              const S* h = &states[SIDX(t, 0, b, hd * DH)];                        \
              for (int c = 0; c < DH; ++c) acc[c] += d * h[c];                     \
            }                                                                      \
            S* out = &dR[RIDX(hd, j, r, 0)];                                       \
            for (int c = 0; c < DH; ++c) out[c] += acc[c];                         \
            free(acc);                                                             \
          }                                                                        \
      S* tmp = ds_cur; ds_cur = ds_prev; ds_prev = tmp; /* :335 */                 \
    }                                                                              \
    memcpy(ds0, ds_cur, sizeof(S) * nst); /* :337 */                               \
    free(ds_cur); free(ds_prev); free(dg);                                         \
  }

DEF_BWD(double, f64, d)
DEF_BWD(float, f32, f)

/* Pointwise maps exposed for per-element parity tests (cell.hpp:65, :108). */
void orc_pointwise_forward_f64(const orc_cell* c, const double* p, const double* g, double* n) {
  pw_fwd_d(c, p, g, n);
}
void orc_pointwise_jacobians_f64(const orc_cell* c, const double* p, const double* g,
                                 double* dgate16, double* dprev16) {
  double a[4][4], b[4][4];
  pw_jac_d(c, p, g, a, b);
  memcpy(dgate16, a, sizeof a);
  memcpy(dprev16, b, sizeof b);
}

/* ---------------------------------------------------------------- rng ---- */
/* rng.hpp:12-50: std::mt19937_64 + explicit Box-Muller (bit-reproducible). */
typedef struct {
  uint64_t mt[312];
  int mti;
  int have_spare;
  double spare;
} orc_rng;

orc_rng* orc_rng_new(uint64_t seed) {
  orc_rng* r = (orc_rng*)calloc(1, sizeof(orc_rng));
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->mti = 312;
  return r;
}
void orc_rng_free(orc_rng* r) { free(r); }

uint64_t orc_rng_u64(orc_rng* r) { /* std::mt19937_64 operator() */
  static const uint64_t MAG[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (r->mti >= 312) {
    int i;
    for (i = 0; i < 312 - 156; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + 156] ^ (x >> 1) ^ MAG[x & 1ULL];
    }
    for (; i < 311; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + (156 - 312)] ^ (x >> 1) ^ MAG[x & 1ULL];
    }
    uint64_t x = (r->mt[311] & UM) | (r->mt[0] & LM);
    r->mt[311] = r->mt[155] ^ (x >> 1) ^ MAG[x & 1ULL];
    r->mti = 0;
  }
  uint64_t x = r->mt[r->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

double orc_rng_uniform(orc_rng* r) { /* rng.hpp:20-22 */
  return ldexp((double)(orc_rng_u64(r) >> 11), -53);
}

double orc_rng_normal(orc_rng* r) { /* rng.hpp:26-38 */
  if (r->have_spare) { r->have_spare = 0; return r->spare; }
  double u1 = orc_rng_uniform(r);
  while (u1 <= 0.0) u1 = orc_rng_uniform(r);
  double u2 = orc_rng_uniform(r);
  double rr = sqrt(-2.0 * log(u1));
  double theta = 2.0 * M_PI * u2;
  r->spare = rr * sin(theta);
  r->have_spare = 1;
  return rr * cos(theta);
}

void orc_rng_fill_normal(orc_rng* r, double scale, size_t n, double* out) {
  for (size_t i = 0; i < n; ++i) out[i] = scale * orc_rng_normal(r);
}

/* random_init.hpp:10-18 random_params */
void orc_random_params(orc_rng* rng, const orc_cell* cell, int NH, int DH, double r_scale,
                       double bias_scale, double* R, double* bias) {
  size_t nr = (size_t)NH * cell->num_gates * DH * DH, nb = (size_t)cell->num_gates * NH * DH;
  double rs = r_scale / sqrt((double)DH);
  for (size_t i = 0; i < nr; ++i) R[i] = rs * orc_rng_normal(rng);
  for (size_t i = 0; i < nb; ++i) bias[i] = bias_scale * orc_rng_normal(rng);
}

/* random_init.hpp:22-40 random_batch */
void orc_random_batch(orc_rng* rng, const orc_cell* cell, int T, int B, int NH, int DH,
                      double input_scale, double state_scale, double* x, double* s0) {
  const int D = NH * DH, NS = cell->num_states;
  size_t nx = (size_t)T * B * cell->num_gates * D;
  for (size_t i = 0; i < nx; ++i) x[i] = input_scale * orc_rng_normal(rng);
  for (int i = 0; i < NS; ++i)
    for (int b = 0; b < B; ++b)
      for (int e = 0; e < D; ++e) {
        double v = state_scale * orc_rng_normal(rng);
        if (cell->variant == ORC_SLSTM && i == 2) v = 1.0 + 0.1 * fabs(v);
        if (cell->variant == ORC_SLSTM && i == 3) v = 0.0;
        s0[((size_t)i * B + b) * D + e] = v;
      }
}

/* bf16 round-to-nearest-even, scalar.hpp:20-27 (used to build bf16-mode
 * oracle inputs: round R, b, x, s0 then run the f64 engine).   */
void orc_round_bf16(size_t n, const double* in, double* out) {
  for (size_t i = 0; i < n; ++i) {
    float f = (float)in[i];
    if (!isfinite(f)) { out[i] = f; continue; }
    uint32_t bits;
    memcpy(&bits, &f, 4);
    uint32_t lsb = (bits >> 16) & 1u;
    bits += 0x7FFFu + lsb;
    bits &= 0xFFFF0000u;
    memcpy(&f, &bits, 4);
    out[i] = f;
  }
}
