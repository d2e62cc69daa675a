// abi.cpp -- the C ABI (include/flashrnn.h): argument validation mirroring the
// reference's std::invalid_argument checks, the mutex-guarded plan cache, and
// dispatch to the CUDA kernels.  No CPU fallback: every compute call runs on
// an sm_100 device or returns an error.
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <initializer_list>
#include <utility>

#include "../../include/flashrnn.h"
#include "../../include/flashrnn_debug.h"
#include "kernels.h"
#include "planner.h"

namespace frnn {
extern long long* g_prof_buf;
extern int g_prof_steps;
extern int g_skeleton;
}  // namespace frnn

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(FRNN_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// cell.hpp:25-53
frnn_cell spec_of(int v) {
  frnn_cell c{};
  c.variant = v;
  for (int j = 0; j < 4; ++j) c.uses_recurrent[j] = c.uses_input[j] = 1;
  switch (v) {
    case FRNN_ELMAN: c.num_states = 1; c.num_gates = 1; break;
    case FRNN_LSTM: c.num_states = 2; c.num_gates = 4; break;
    case FRNN_GRU:
      c.num_states = 1; c.num_gates = 4;
      c.uses_recurrent[2] = 0;
      c.uses_input[3] = 0;
      break;
    default: c.num_states = 4; c.num_gates = 4; break;
  }
  return c;
}

// Shape checks of engine.hpp:116-129 (counts, dims, degenerate shape).  The
// storage-size check is implicit: the ABI takes raw pointers sized by shape.
int validate(const frnn_cell* cell, const frnn_shape& s, int dtype) {
  if (!cell) return fail(FRNN_EINVAL_ARG, "null cell");
  if (cell->variant < FRNN_ELMAN || cell->variant > FRNN_SLSTM)
    return fail(FRNN_EINVAL_SHAPE, "unknown cell variant");
  frnn_cell ref = spec_of(cell->variant);
  if (cell->num_states != ref.num_states || cell->num_gates != ref.num_gates)
    return fail(FRNN_EINVAL_SHAPE, "cell/params/batch gate or state counts disagree");
  if (s.head_dim < 1 || s.seq_len < 0 || s.batch < 1 || s.num_heads < 1)
    return fail(FRNN_EINVAL_SHAPE, "degenerate shape");
  if (dtype != FRNN_F32 && dtype != FRNN_BF16) return fail(FRNN_EUNSUPPORTED, "unsupported dtype");
  return FRNN_OK;
}

int validate_pass(int32_t pass) {
  if (pass != FRNN_PASS_FORWARD && pass != FRNN_PASS_BACKWARD)
    return fail(FRNN_EINVAL_ARG, "pass must be FRNN_PASS_FORWARD (0) or FRNN_PASS_BACKWARD (1)");
  return FRNN_OK;
}

// The kernels move R/s0/state rows with 16-byte vector loads and TMA (16-byte
// aligned global addresses), so every tensor base must be 16-byte aligned; a
// sliced tensor that is not would fault inside a kernel and poison the context.
int check_aligned(std::initializer_list<std::pair<const void*, const char*>> ptrs) {
  for (const auto& pr : ptrs)
    if (pr.first && (reinterpret_cast<uintptr_t>(pr.first) & 15u))
      return fail(FRNN_EINVAL_ARG, std::string(pr.second) + " is not 16-byte aligned");
  return FRNN_OK;
}

int check_device() {
  static std::once_flag once;
  static int status = FRNN_OK;
  static std::string msg;
  std::call_once(once, [] {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    cudaDeviceProp prop{};
    if (e == cudaSuccess) e = cudaGetDeviceProperties(&prop, dev);
    if (e != cudaSuccess) {
      status = FRNN_ECUDA;
      msg = std::string("no CUDA device: ") + cudaGetErrorString(e);
    } else if (prop.major != 10 || prop.minor != 0) {  // the fatbin carries sm_100a SASS only
      status = FRNN_ECUDA;
      msg = "libflashrnn is built for sm_100a (B200); found sm_" + std::to_string(prop.major * 10 + prop.minor);
    }
  });
  if (status != FRNN_OK) return fail(status, msg);
  return FRNN_OK;
}

frnn::Problem make_problem(const frnn_cell* c, const frnn_shape& s, int dtype) {
  frnn::Problem p{};
  p.variant = c->variant;
  p.NS = c->num_states;
  p.NG = c->num_gates;
  for (int j = 0; j < 4; ++j) {
    p.rec[j] = j < p.NG && c->uses_recurrent[j];
    p.inp[j] = j < p.NG && c->uses_input[j];
  }
  p.T = s.seq_len;
  p.B = s.batch;
  p.NH = s.num_heads;
  p.DH = s.head_dim;
  p.D = s.num_heads * s.head_dim;
  p.bf16 = dtype == FRNN_BF16;
  return p;
}

// ---------------------------------------------------------- plan cache ----
using Key = std::tuple<int, int, int, int, int, int, int, int, int, int, int, int>;
std::mutex g_mu;
std::map<Key, frnn::Plan> g_cache;

// ---------------------------------------------- persistent plan cache ----
// The counterpart of the paper's cached solver solutions: solved
// plans as JSON lines (schema_version 1, like frnn_plan_json), one per line,
// keyed by the problem and the requested algorithm, tagged with the library
// version and the device limits they were solved against.  Lines that do not
// match this build and device are skipped on load.  FRNN_PLAN_CACHE=<file>
// loads the file before the first plan and appends every new solve to it.
int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    dev = 0;
  }
  return dev;
}

std::string plan_line(const Key& k, const frnn::Plan& pl) {
  const auto& lim = frnn::device_limits();
  char buf[1024];
  std::snprintf(
      buf, sizeof buf,
      "{\"schema_version\": 1, \"version\": \"%s\", \"sm_count\": %d, \"smem_optin\": %d, "
      "\"tmem_cols\": %d, \"cluster_max\": %d, \"variant\": %d, \"rec_mask\": %d, \"inp_mask\": %d, "
      "\"seq_len\": %d, \"batch\": %d, \"num_heads\": %d, \"head_dim\": %d, \"bf16\": %d, \"pass\": %d, "
      "\"req_algo\": %d, \"algo\": %d, \"rows_per_cta\": %d, \"batch_tile\": %d, \"units_per_cta\": %d, "
      "\"ctas_per_group\": %d, \"groups\": %d, \"grid\": %d, \"threads\": %d, \"smem_bytes\": %d, "
      "\"plan_tmem_cols\": %d, \"k_split\": %d, \"cluster\": %d, \"ka\": %d, \"stages\": %d, "
      "\"ffma\": %d, \"ws_bytes\": %lld, \"solve_us\": %.3f}",
      frnn_version(), lim.sm_count, lim.smem_optin, lim.tmem_cols, lim.cluster_max, std::get<0>(k), std::get<1>(k),
      std::get<2>(k), std::get<3>(k), std::get<4>(k), std::get<5>(k), std::get<6>(k), std::get<7>(k),
      std::get<8>(k), std::get<9>(k), pl.algo, pl.rows_per_cta, pl.batch_tile, pl.units_per_cta, pl.ctas_per_group,
      pl.groups, pl.grid, pl.threads, pl.smem_bytes, pl.tmem_cols, pl.k_split, pl.cluster, pl.ka, pl.stages, pl.ffma,
      (long long)pl.ws_bytes, pl.solve_us);
  return buf;
}

bool field(const std::string& line, const char* name, double* v) {
  const std::string pat = std::string("\"") + name + "\": ";
  const size_t pos = line.find(pat);
  if (pos == std::string::npos) return false;
  char* end = nullptr;
  *v = std::strtod(line.c_str() + pos + pat.size(), &end);
  return end != line.c_str() + pos + pat.size();
}

// Parses one cache line; false when malformed or solved for another build/device.
bool parse_plan_line(const std::string& line, int dev, Key* k, frnn::Plan* pl) {
  const auto& lim = frnn::device_limits();
  if (line.find(std::string("\"version\": \"") + frnn_version() + "\"") == std::string::npos) return false;
  static const char* names[] = {"schema_version", "sm_count", "smem_optin", "tmem_cols", "cluster_max",
                                "variant", "rec_mask", "inp_mask", "seq_len", "batch", "num_heads", "head_dim",
                                "bf16", "pass", "req_algo", "algo", "rows_per_cta", "batch_tile",
                                "units_per_cta", "ctas_per_group", "groups", "grid", "threads", "smem_bytes",
                                "plan_tmem_cols", "k_split", "cluster", "ka", "stages", "ffma", "ws_bytes",
                                "solve_us"};
  double v[32];
  for (int i = 0; i < 32; ++i)
    if (!field(line, names[i], &v[i])) return false;
  if (v[0] != 1 || v[1] != lim.sm_count || v[2] != lim.smem_optin || v[3] != lim.tmem_cols ||
      v[4] != lim.cluster_max)
    return false;
  *k = Key{(int)v[5], (int)v[6], (int)v[7], (int)v[8], (int)v[9], (int)v[10], (int)v[11], (int)v[12],
           (int)v[13], (int)v[14], dev, 0};
  *pl = frnn::Plan{};
  pl->algo = (int)v[15];
  pl->rows_per_cta = (int)v[16];
  pl->batch_tile = (int)v[17];
  pl->units_per_cta = (int)v[18];
  pl->ctas_per_group = (int)v[19];
  pl->groups = (int)v[20];
  pl->grid = (int)v[21];
  pl->threads = (int)v[22];
  pl->smem_bytes = (int)v[23];
  pl->tmem_cols = (int)v[24];
  pl->k_split = (int)v[25];
  pl->cluster = (int)v[26];
  pl->ka = (int)v[27];
  pl->stages = (int)v[28];
  pl->ffma = (int)v[29];
  pl->solve_us = v[31];
  // never trust the persisted size: the kernels' workspace layout may have
  // changed since the line was written (recomputed from the plan's fields)
  const int var = (int)v[5];
  if (var < FRNN_ELMAN || var > FRNN_SLSTM || (int)v[13] < 0 || (int)v[13] > 1) return false;
  frnn_cell cell = spec_of(var);
  for (int j = 0; j < 4; ++j) {
    cell.uses_recurrent[j] = ((int)v[6] >> j) & 1;
    cell.uses_input[j] = ((int)v[7] >> j) & 1;
  }
  const frnn_shape sh{(int)v[8], (int)v[9], (int)v[10], (int)v[11]};
  if (sh.seq_len < 0 || sh.batch < 1 || sh.num_heads < 1 || sh.head_dim < 1) return false;
  pl->ws_bytes = frnn::plan_workspace(make_problem(&cell, sh, (int)v[12] ? FRNN_BF16 : FRNN_F32), (int)v[13], *pl);
  return true;
}

int load_plans(const char* path, int* loaded) {  // caller holds g_mu
  std::FILE* f = std::fopen(path, "r");
  if (!f) return fail(FRNN_EINVAL_ARG, std::string("cannot open plan cache ") + path);
  const int dev = current_device();
  int n = 0;
  std::string line;
  char chunk[512];
  while (std::fgets(chunk, sizeof chunk, f)) {
    line += chunk;
    if (line.empty() || line.back() != '\n') continue;
    Key k;
    frnn::Plan pl;
    if (parse_plan_line(line, dev, &k, &pl)) {
      g_cache[k] = pl;
      ++n;
    }
    line.clear();
  }
  Key k;
  frnn::Plan pl;
  if (!line.empty() && parse_plan_line(line, dev, &k, &pl)) {
    g_cache[k] = pl;
    ++n;
  }
  std::fclose(f);
  if (loaded) *loaded = n;
  return FRNN_OK;
}

const char* env_cache() {
  const char* e = std::getenv("FRNN_PLAN_CACHE");
  return e && *e ? e : nullptr;
}

int get_plan(const frnn::Problem& p, int pass, const frnn_options* o, frnn::Plan* out) {
  static std::once_flag env_once;
  std::call_once(env_once, [] {
    if (const char* path = env_cache()) {
      std::lock_guard<std::mutex> lk(g_mu);
      if (std::FILE* f = std::fopen(path, "r")) {  // a missing file is created on the first solve
        std::fclose(f);
        load_plans(path, nullptr);
        g_err.clear();
      }
    }
  });
  const int dev = current_device();
  int recm = 0, inm = 0;
  for (int j = 0; j < 4; ++j) {
    recm |= p.rec[j] << j;
    inm |= p.inp[j] << j;
  }
  const int algo = o ? o->algo : FRNN_ALGO_AUTO;
  Key k{p.variant, recm, inm, p.T, p.B, p.NH, p.DH, (int)p.bf16, pass, algo, dev, 0};
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_cache.find(k);
    if (it != g_cache.end()) {
      *out = it->second;
      return FRNN_OK;
    }
  }
  std::string why;
  auto t0 = std::chrono::steady_clock::now();
  int rc = frnn::solve_plan(p, pass, algo, frnn::device_limits(), out, &why);
  out->solve_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  if (rc != FRNN_OK) return fail(rc, why);
  std::lock_guard<std::mutex> lk(g_mu);
  g_cache[k] = *out;
  if (const char* path = env_cache()) {  // persist the new solve
    if (std::FILE* f = std::fopen(path, "a")) {
      std::fprintf(f, "%s\n", plan_line(k, *out).c_str());
      std::fclose(f);
    }
  }
  return FRNN_OK;
}

size_t elem(const frnn::Problem& p) { return p.bf16 ? 2 : 4; }

}  // namespace

namespace frnn {  // the thread-local error string, for the other C-ABI translation units (dist.cu)
int set_error(int code, const std::string& msg) { return fail(code, msg); }
void clear_error() { g_err.clear(); }
}  // namespace frnn

extern "C" {

const char* frnn_version(void) { return "flashrnn-b200 0.1.0 (sm_100a, abi 1)"; }

const char* frnn_last_error(void) { return g_err.c_str(); }

int frnn_cell_spec(int32_t variant, frnn_cell* out) {
  if (!out) return fail(FRNN_EINVAL_ARG, "null output");
  if (variant < FRNN_ELMAN || variant > FRNN_SLSTM) return fail(FRNN_EINVAL_SHAPE, "unknown cell variant");
  *out = spec_of(variant);
  return FRNN_OK;
}

int frnn_plan(const frnn_cell* cell, frnn_shape shape, int32_t dtype, int32_t pass, const frnn_options* opts,
              frnn_plan_info* out) {
  g_err.clear();
  int rc = validate(cell, shape, dtype);
  if (rc) return rc;
  if ((rc = validate_pass(pass))) return rc;
  if (!out) return fail(FRNN_EINVAL_ARG, "null output");
  frnn::Problem p = make_problem(cell, shape, dtype);
  frnn::Plan pl{};
  if ((rc = get_plan(p, pass, opts, &pl))) return rc;
  out->algo = pl.algo;
  out->rows_per_cta = pl.rows_per_cta;
  out->batch_tile = pl.batch_tile;
  out->ctas_per_group = pl.ctas_per_group;
  out->groups = pl.groups;
  out->grid = pl.grid;
  out->threads = pl.threads;
  out->smem_bytes = pl.smem_bytes;
  out->tmem_cols = pl.tmem_cols;
  out->k_split = pl.k_split;
  out->cluster = pl.cluster;
  out->workspace_bytes = (int64_t)pl.ws_bytes;
  out->solve_us = pl.solve_us;
  return FRNN_OK;
}

int frnn_plan_cache_save(const char* path) {
  g_err.clear();
  if (!path) return fail(FRNN_EINVAL_ARG, "null path");
  std::lock_guard<std::mutex> lk(g_mu);
  std::FILE* f = std::fopen(path, "w");
  if (!f) return fail(FRNN_EINVAL_ARG, std::string("cannot write plan cache ") + path);
  for (const auto& kv : g_cache) std::fprintf(f, "%s\n", plan_line(kv.first, kv.second).c_str());
  std::fclose(f);
  return FRNN_OK;
}

int frnn_plan_cache_load(const char* path, int32_t* loaded) {
  g_err.clear();
  if (!path) return fail(FRNN_EINVAL_ARG, "null path");
  std::lock_guard<std::mutex> lk(g_mu);
  int n = 0;
  const int rc = load_plans(path, &n);
  if (loaded) *loaded = n;
  return rc;
}

int frnn_plan_cache_clear(void) {
  g_err.clear();
  std::lock_guard<std::mutex> lk(g_mu);
  g_cache.clear();
  return FRNN_OK;
}

// planner.cpp:428-453 plan_to_json, for the B200 plan (schema_version 1).
int frnn_plan_json(const frnn_cell* cell, frnn_shape shape, int32_t dtype, int32_t pass, const frnn_options* opts,
                   char* out, size_t out_bytes) {
  g_err.clear();
  int rc = validate(cell, shape, dtype);
  if (rc) return rc;
  if ((rc = validate_pass(pass))) return rc;
  frnn::Problem p = make_problem(cell, shape, dtype);
  frnn::Plan pl{};
  if ((rc = get_plan(p, pass, opts, &pl))) return rc;
  static const char* algos[] = {"auto", "fused", "alternating", "simt"};
  const auto& lim = frnn::device_limits();
  const frnn::PlanTraffic tr = frnn::plan_traffic(p, pass, pl);
  const std::vector<std::string> res = frnn::plan_residuals(p, pass, pl, lim);
  char buf[2560];
  const int n = std::snprintf(
      buf, sizeof buf,
      "{\n  \"schema_version\": 1,\n  \"gpu\": \"B200\",\n  \"sm_count\": %d,\n  \"pass\": \"%s\",\n"
      "  \"shape\": {\"num_states\": %d, \"num_gates\": %d, \"head_dim\": %d, \"num_heads\": %d, "
      "\"batch\": %d, \"seq_len\": %d, \"dtype\": \"%s\"},\n"
      "  \"algo\": \"%s\",\n"
      "  \"tiling\": {\"cluster\": %d, \"units_per_cta\": %d, \"rows_per_cta\": %d, \"batch_tile\": %d, "
      "\"ctas_per_group\": %d, \"groups\": %d, \"k_split\": %d, \"k_atoms_per_stage\": %d, \"stages\": %d, "
      "\"step_kernels\": \"%s\"},\n"
      "  \"grid_blocks\": %d,\n  \"threads_per_block\": %d,\n"
      "  \"footprint\": {\"smem_bytes\": %d, \"tmem_columns\": %d, \"workspace_bytes\": %lld, "
      "\"r_matrix_bytes_per_head\": %lld},\n"
      "  \"traffic_per_step_bytes\": {\"io\": %.0f, \"exchange_onchip\": %.0f, \"exchange_l2\": %.0f, "
      "\"r_stream\": %.0f},\n  \"residuals\": %d,\n  \"solve_us\": %.1f\n}\n",
      lim.sm_count, pass == FRNN_PASS_FORWARD ? "forward" : "backward", p.NS, p.NG, p.DH, p.NH, p.B, p.T,
      p.bf16 ? "bf16" : "fp32", algos[pl.algo & 3], pl.cluster, pl.units_per_cta, pl.rows_per_cta, pl.batch_tile,
      pl.ctas_per_group, pl.groups, pl.k_split, pl.ka, pl.stages,
      pl.algo == FRNN_ALGO_SIMT ? "simt" : (pl.ffma || !p.bf16) ? "ffma" : "tcgen05", pl.grid, pl.threads, pl.smem_bytes, pl.tmem_cols,
      (long long)pl.ws_bytes, (long long)p.NG * p.DH * p.DH * (p.bf16 ? 2 : 4), tr.io, tr.exchange_onchip,
      tr.exchange_l2, tr.r_stream, (int)res.size(), pl.solve_us);
  if (!out || n < 0 || (size_t)n + 1 > out_bytes) return fail(FRNN_EINVAL_ARG, "output buffer too small");
  std::memcpy(out, buf, (size_t)n + 1);
  return FRNN_OK;
}

namespace {
std::string json_escape(const std::string& m) {
  std::string o;
  for (char c : m) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  return o;
}
int write_residuals(const std::vector<std::string>& res, char* out, size_t out_bytes) {
  std::string j = "[";
  for (size_t i = 0; i < res.size(); ++i) j += (i ? ", \"" : "\"") + json_escape(res[i]) + "\"";
  j += "]";
  if (!out || j.size() + 1 > out_bytes) return fail(FRNN_EINVAL_ARG, "output buffer too small");
  std::memcpy(out, j.c_str(), j.size() + 1);
  return res.empty() ? FRNN_OK : fail(FRNN_EINFEASIBLE, "plan residuals: " + res[0]);
}
frnn::Plan plan_from_fields(const int64_t* f) {
  frnn::Plan pl{};
  pl.algo = (int)f[0];
  pl.rows_per_cta = (int)f[1];
  pl.batch_tile = (int)f[2];
  pl.units_per_cta = (int)f[3];
  pl.ctas_per_group = (int)f[4];
  pl.groups = (int)f[5];
  pl.grid = (int)f[6];
  pl.threads = (int)f[7];
  pl.smem_bytes = (int)f[8];
  pl.tmem_cols = (int)f[9];
  pl.k_split = (int)f[10];
  pl.cluster = (int)f[11];
  pl.ka = (int)f[12];
  pl.stages = (int)f[13];
  pl.ffma = (int)f[14];
  pl.ws_bytes = (size_t)f[15];
  return pl;
}
}  // namespace

int frnn_plan_check(const frnn_cell* cell, frnn_shape shape, int32_t dtype, int32_t pass, const frnn_options* opts,
                    char* out, size_t out_bytes) {
  g_err.clear();
  int rc = validate(cell, shape, dtype);
  if (rc) return rc;
  if ((rc = validate_pass(pass))) return rc;
  frnn::Problem p = make_problem(cell, shape, dtype);
  frnn::Plan pl{};
  if ((rc = get_plan(p, pass, opts, &pl))) return rc;
  return write_residuals(frnn::plan_residuals(p, pass, pl, frnn::device_limits()), out, out_bytes);
}

int frnn_debug_plan_fields(const frnn_cell* cell, frnn_shape shape, int32_t dtype, int32_t pass,
                           const frnn_options* opts, int64_t* fields16) {
  g_err.clear();
  int rc = validate(cell, shape, dtype);
  if (rc) return rc;
  if ((rc = validate_pass(pass))) return rc;
  if (!fields16) return fail(FRNN_EINVAL_ARG, "null output");
  frnn::Problem p = make_problem(cell, shape, dtype);
  frnn::Plan pl{};
  if ((rc = get_plan(p, pass, opts, &pl))) return rc;
  const int64_t f[16] = {pl.algo, pl.rows_per_cta, pl.batch_tile, pl.units_per_cta, pl.ctas_per_group, pl.groups,
                         pl.grid, pl.threads, pl.smem_bytes, pl.tmem_cols, pl.k_split, pl.cluster, pl.ka, pl.stages,
                         pl.ffma, (int64_t)pl.ws_bytes};
  std::memcpy(fields16, f, sizeof f);
  return FRNN_OK;
}

int frnn_debug_plan_residuals(const frnn_cell* cell, frnn_shape shape, int32_t dtype, int32_t pass,
                              const int64_t* fields16, char* out, size_t out_bytes) {
  g_err.clear();
  int rc = validate(cell, shape, dtype);
  if (rc) return rc;
  if ((rc = validate_pass(pass))) return rc;
  if (!fields16) return fail(FRNN_EINVAL_ARG, "null plan");
  frnn::Problem p = make_problem(cell, shape, dtype);
  return write_residuals(frnn::plan_residuals(p, pass, plan_from_fields(fields16), frnn::device_limits()), out,
                         out_bytes);
}

int frnn_workspace_size(const frnn_cell* cell, frnn_shape shape, int32_t dtype, int32_t pass,
                        const frnn_options* opts, size_t* bytes) {
  g_err.clear();
  int rc = validate(cell, shape, dtype);
  if (rc) return rc;
  if ((rc = validate_pass(pass))) return rc;
  if (!bytes) return fail(FRNN_EINVAL_ARG, "null output");
  frnn::Problem p = make_problem(cell, shape, dtype);
  frnn::Plan pl{};
  if ((rc = get_plan(p, pass, opts, &pl))) return rc;
  *bytes = pl.ws_bytes + 256;  // + the non-finite flag
  return FRNN_OK;
}

int frnn_forward(const frnn_cell* cell, frnn_shape shape, int32_t dtype, const void* R, const void* bias,
                 const void* x, const void* s0, void* states, void* gates, void* workspace, size_t ws_bytes,
                 const frnn_options* opts, void* stream) {
  g_err.clear();
  int rc = validate(cell, shape, dtype);
  if (rc) return rc;
  if (!R || !bias || !s0 || !states || (shape.seq_len > 0 && (!x || !gates)))
    return fail(FRNN_EINVAL_ARG, "null tensor pointer");
  if ((rc = check_aligned({{R, "R"}, {bias, "bias"}, {x, "x"}, {s0, "s0"}, {states, "states"}, {gates, "gates"},
                           {workspace, "workspace"}})))
    return rc;
  if ((rc = check_device())) return rc;
  frnn::Problem p = make_problem(cell, shape, dtype);
  p.R = R; p.bias = bias; p.x = x; p.s0 = s0; p.states = states; p.gates = gates;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t nstate = (size_t)p.NS * p.B * p.D;
  frnn::Plan pl{};
  if (p.T > 0 && (rc = get_plan(p, FRNN_PASS_FORWARD, opts, &pl))) return rc;
  const size_t need = (p.T > 0 ? pl.ws_bytes : 0) + 256;
  if (!workspace || ws_bytes < need)
    return fail(FRNN_EINVAL_ARG, "workspace too small: need " + std::to_string(need) + " bytes");
  cudaError_t e;
  if (opts && (opts->flags & FRNN_FLAG_CHECK_FINITE)) {  // engine.hpp:146-147
    int* flag = reinterpret_cast<int*>(static_cast<char*>(workspace) + need - 256);
    int h = 0;
    if ((e = cudaMemsetAsync(flag, 0, sizeof(int), s)) != cudaSuccess) return cuda_fail(e, "memset");
    if ((e = frnn::check_finite(x, (size_t)p.T * p.B * p.NG * p.D, p.bf16, flag, s))) return cuda_fail(e, "finite");
    if ((e = cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s))) return cuda_fail(e, "finite");
    if ((e = cudaStreamSynchronize(s))) return cuda_fail(e, "finite");
    if (h) return fail(FRNN_ENONFINITE, "non-finite input");
    if ((e = frnn::check_finite(s0, nstate, p.bf16, flag, s))) return cuda_fail(e, "finite");
    if ((e = cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s))) return cuda_fail(e, "finite");
    if ((e = cudaStreamSynchronize(s))) return cuda_fail(e, "finite");
    if (h) return fail(FRNN_ENONFINITE, "non-finite initial state");
  }
  if (p.T == 0) {  // states = [s0]
    if ((e = cudaMemcpyAsync(states, s0, nstate * elem(p), cudaMemcpyDeviceToDevice, s)))
      return cuda_fail(e, "copy s0");
    return FRNN_OK;
  }
  switch (pl.algo) {
    case FRNN_ALGO_SIMT: e = frnn::simt_forward(p, pl, workspace, s); break;
    case FRNN_ALGO_FUSED:
      e = pl.cluster ? frnn::cluster_forward(p, pl, workspace, s) : frnn::fused_forward(p, pl, workspace, s);
      break;
    default: e = frnn::alt_forward(p, pl, workspace, s); break;
  }
  if (e == cudaErrorNotSupported) return fail(FRNN_EUNSUPPORTED, "algorithm not implemented for this shape");
  if (e != cudaSuccess) return cuda_fail(e, "forward launch");
  return FRNN_OK;
}

int frnn_backward(const frnn_cell* cell, frnn_shape shape, int32_t dtype, const void* R, const void* bias,
                  const void* states, const void* gates, const void* d_states_final, const void* d_hidden,
                  frnn_clip clip, void* dx, void* dbias, void* dR, void* ds0, void* workspace, size_t ws_bytes,
                  const frnn_options* opts, void* stream) {
  g_err.clear();
  int rc = validate(cell, shape, dtype);
  if (rc) return rc;
  if (clip.mode == FRNN_CLIP_VALUE && !(clip.magnitude > 0))  // engine.hpp:107
    return fail(FRNN_EINVAL_ARG, "clip magnitude must be positive");
  if (clip.mode < FRNN_CLIP_OFF || clip.mode > FRNN_CLIP_ZERO) return fail(FRNN_EINVAL_ARG, "bad clip mode");
  if (!R || !states || !d_states_final || !dbias || !dR || !ds0 || (shape.seq_len > 0 && (!gates || !dx)))
    return fail(FRNN_EINVAL_ARG, "null tensor pointer");
  if ((rc = check_aligned({{R, "R"}, {bias, "bias"}, {states, "states"}, {gates, "gates"},
                           {d_states_final, "d_states_final"}, {d_hidden, "d_hidden"}, {dx, "dx"},
                           {dbias, "dbias"}, {dR, "dR"}, {ds0, "ds0"}, {workspace, "workspace"}})))
    return rc;
  if ((rc = check_device())) return rc;
  frnn::Problem p = make_problem(cell, shape, dtype);
  p.R = R; p.bias = bias; p.cstates = states; p.cgates = gates; p.dsf = d_states_final; p.dh = d_hidden;
  p.clip_mode = clip.mode;
  p.clip_mag = (float)clip.magnitude;
  p.dx = dx; p.dbias = dbias; p.dR = dR; p.ds0 = ds0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (p.T == 0) {  // no steps: ds0 = d_states_final, zero parameter grads
    const size_t nstate = (size_t)p.NS * p.B * p.D;
    if ((e = cudaMemcpyAsync(ds0, d_states_final, nstate * elem(p), cudaMemcpyDeviceToDevice, s)) ||
        (e = cudaMemsetAsync(dbias, 0, (size_t)p.NG * p.D * elem(p), s)) ||
        (e = cudaMemsetAsync(dR, 0, (size_t)p.NH * p.NG * p.DH * p.DH * elem(p), s)))
      return cuda_fail(e, "T=0 backward");
    return FRNN_OK;
  }
  frnn::Plan pl{};
  if ((rc = get_plan(p, FRNN_PASS_BACKWARD, opts, &pl))) return rc;
  const size_t need = pl.ws_bytes + 256;
  if (!workspace || ws_bytes < need)
    return fail(FRNN_EINVAL_ARG, "workspace too small: need " + std::to_string(need) + " bytes");
  switch (pl.algo) {
    case FRNN_ALGO_SIMT: e = frnn::simt_backward(p, pl, workspace, s); break;
    case FRNN_ALGO_FUSED:
      e = pl.cluster ? frnn::cluster_backward(p, pl, workspace, s) : frnn::fused_backward(p, pl, workspace, s);
      break;
    default: e = frnn::alt_backward(p, pl, workspace, s); break;
  }
  if (e == cudaErrorNotSupported) return fail(FRNN_EUNSUPPORTED, "algorithm not implemented for this shape");
  if (e != cudaSuccess) return cuda_fail(e, "backward launch");
  return FRNN_OK;
}

int frnn_input_projection(const void* W, const void* u, void* x, int64_t tokens, int32_t out_features,
                          int32_t in_features, int32_t dtype, void* stream) {
  g_err.clear();
  if (!W || !u || !x) return fail(FRNN_EINVAL_ARG, "null tensor pointer");
  if (tokens < 1 || out_features < 1 || in_features < 1) return fail(FRNN_EINVAL_SHAPE, "degenerate shape");
  if (dtype != FRNN_BF16) return fail(FRNN_EUNSUPPORTED, "input projection: bf16 only");
  if (in_features % 8) return fail(FRNN_EINVAL_SHAPE, "in_features must be a multiple of 8 (16-byte TMA rows)");
  int rc = check_aligned({{W, "W"}, {u, "u"}, {x, "x"}});
  if (rc) return rc;
  rc = check_device();
  if (rc) return rc;
  cudaError_t e = frnn::wx_gemm(W, u, x, tokens, out_features, in_features, static_cast<cudaStream_t>(stream));
  if (e == cudaErrorNotSupported) return fail(FRNN_EUNSUPPORTED, "TMA tensor maps unavailable");
  if (e != cudaSuccess) return cuda_fail(e, "input projection");
  return FRNN_OK;
}

// Batch x head sharding over world_size ranks: heads split by the
// largest factor of world_size dividing NH; the rest of world_size splits B.
int frnn_partition(frnn_shape shape, int32_t world_size, int32_t rank, frnn_shard* out) {
  g_err.clear();
  if (!out) return fail(FRNN_EINVAL_ARG, "null output");
  if (world_size < 1 || rank < 0 || rank >= world_size) return fail(FRNN_EINVAL_ARG, "bad rank/world size");
  if (shape.batch < 1 || shape.num_heads < 1) return fail(FRNN_EINVAL_SHAPE, "degenerate shape");
  int hs = 1;
  for (int f = 1; f <= world_size; ++f)
    if (world_size % f == 0 && shape.num_heads % f == 0) hs = f;
  int bs = world_size / hs;
  if (bs > shape.batch) return fail(FRNN_EINVAL_SHAPE, "more batch shards than batch rows");
  const int hp = rank / bs, bp = rank % bs;
  const int hper = shape.num_heads / hs;
  out->head_begin = hp * hper;
  out->head_end = (hp + 1) * hper;
  out->batch_begin = (int)((long long)shape.batch * bp / bs);
  out->batch_end = (int)((long long)shape.batch * (bp + 1) / bs);
  out->reduce_params = bs > 1;
  return FRNN_OK;
}

int frnn_debug_cluster_shape(const frnn_cell* cell, frnn_shape shape, int32_t dtype, int32_t pass, int32_t* out10) {
  g_err.clear();
  int rc = validate(cell, shape, dtype);
  if (rc) return rc;
  if ((rc = validate_pass(pass))) return rc;
  if (!out10) return fail(FRNN_EINVAL_ARG, "null output");
  frnn::Problem p = make_problem(cell, shape, dtype);
  frnn::Plan pl{};
  if ((rc = get_plan(p, pass, nullptr, &pl))) return rc;
  for (int i = 0; i < 10; ++i) out10[i] = 0;
  out10[0] = pl.algo;
  out10[1] = pl.cluster;
  if (pl.algo != FRNN_ALGO_FUSED || pl.cluster <= 0) return FRNN_OK;
  const frnn::ClusterShape cs = frnn::cluster_shape(p, pl.units_per_cta, pl.batch_tile, pass == FRNN_PASS_BACKWARD);
  const int32_t v[8] = {cs.UPC, cs.CL, cs.MBT, cs.MS, cs.SSM, cs.KBP, cs.R1, cs.R2};
  for (int i = 0; i < 8; ++i) out10[2 + i] = v[i];
  return FRNN_OK;
}

int frnn_debug_plan_csp(const frnn_cell* cell, frnn_shape shape, int32_t dtype, int32_t pass, int32_t algo,
                        char* out, size_t out_bytes) {
  g_err.clear();
  int rc = validate(cell, shape, dtype);
  if (rc) return rc;
  try {
    const std::string t = frnn::plan_csp_text(make_problem(cell, shape, dtype), pass, algo, frnn::device_limits());
    if (!out || t.size() + 1 > out_bytes) return fail(FRNN_EINVAL_ARG, "output buffer too small");
    std::memcpy(out, t.c_str(), t.size() + 1);
    return FRNN_OK;
  } catch (const std::exception& e) {
    return fail(FRNN_EINVAL_ARG, e.what());
  }
}

int frnn_debug_skeleton(int32_t enable) {
  frnn::g_skeleton = enable != 0;
  return FRNN_OK;
}

int frnn_debug_profile(void* device_buffer, int32_t steps) {
  frnn::g_prof_buf = static_cast<long long*>(device_buffer);
  frnn::g_prof_steps = device_buffer ? steps : 0;
  return FRNN_OK;
}

}  // extern "C"
