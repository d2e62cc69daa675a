// csp_abi.cpp -- C ABI of the CSP engine (include/flashrnn_csp.h).
#include <chrono>
#include <cstring>
#include <stdexcept>
#include <string>

#include "../../include/flashrnn_csp.h"
#include "csp.h"

namespace {
int put(const std::string& s, char* out, size_t cap) {
  if (!out || s.size() + 1 > cap) return FRNN_EINVAL_ARG;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return FRNN_OK;
}
}  // namespace

extern "C" {

int frnn_csp_solve(const char* problem, char* out, size_t out_bytes, int64_t* stats) {
  if (!problem) return FRNN_EINVAL_ARG;
  try {
    const frnn::csp::Problem p = frnn::csp::parse(problem);
    const auto t0 = std::chrono::steady_clock::now();
    const auto sol = frnn::csp::solve(p);
    const auto ns = std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
    if (stats) {
      stats[0] = sol ? sol->nodes : 0;
      stats[1] = sol ? sol->backtracks : 0;
      stats[2] = (int64_t)ns;
    }
    if (!sol) return FRNN_EINFEASIBLE;
    std::string s;
    for (const auto& [id, v] : sol->values) s += id + "=" + std::to_string(v) + "\n";
    return put(s, out, out_bytes);
  } catch (const std::exception&) {
    return FRNN_EINVAL_ARG;
  }
}

int frnn_csp_brute_force(const char* problem, int64_t cap, char* out, size_t out_bytes, int64_t* count) {
  if (!problem) return FRNN_EINVAL_ARG;
  try {
    const auto all = frnn::csp::brute_force(frnn::csp::parse(problem), cap);
    if (count) *count = (int64_t)all.size();
    std::string s;
    for (const auto& m : all) {
      for (const auto& [id, v] : m) s += id + "=" + std::to_string(v) + "\n";
      s += "--\n";
    }
    return put(s, out, out_bytes);
  } catch (const std::exception&) {
    return FRNN_EINVAL_ARG;
  }
}

}  // extern "C"
