// ktimer.cpp -- optional per-kernel-class CUDA-event timing (developer hook
// behind flashrnn_debug.h; bench.py uses it to time the dominant kernel on its
// launch stream).  Disabled by default: kt_begin/kt_end are then no-ops.
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <vector>

#include "../../include/flashrnn_debug.h"
#include "kernels.h"

namespace frnn {
namespace {

struct Span {
  int cls;
  cudaEvent_t b, e;
};
std::mutex g_mu;
bool g_on = false;
std::vector<Span> g_spans;
std::vector<cudaEvent_t> g_pool;
cudaEvent_t g_open[KT_N] = {};

cudaEvent_t take() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

std::atomic<long long> g_launches{0};

}  // namespace

void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void kt_begin(int cls, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_on) return;
  g_open[cls] = take();
  cudaEventRecord(g_open[cls], s);
}

void kt_end(int cls, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_on || !g_open[cls]) return;
  cudaEvent_t e = take();
  cudaEventRecord(e, s);
  g_spans.push_back({cls, g_open[cls], e});
  g_open[cls] = nullptr;
}

}  // namespace frnn

extern "C" {

int frnn_debug_timing(int32_t enable) {
  std::lock_guard<std::mutex> lk(frnn::g_mu);
  frnn::g_on = enable != 0;
  return FRNN_OK;
}

// Sums the recorded spans per kernel class (fwd loop, bwd loop, dR/db) in ms,
// waiting for their events; clears the record.
int frnn_debug_kernel_ms(double* ms3, int64_t* count3) {
  std::lock_guard<std::mutex> lk(frnn::g_mu);
  for (int i = 0; i < frnn::KT_N; ++i) {
    if (ms3) ms3[i] = 0;
    if (count3) count3[i] = 0;
  }
  for (auto& sp : frnn::g_spans) {
    cudaEventSynchronize(sp.e);
    float ms = 0;
    cudaEventElapsedTime(&ms, sp.b, sp.e);
    if (ms3) ms3[sp.cls] += ms;
    if (count3) count3[sp.cls] += 1;
    frnn::g_pool.push_back(sp.b);
    frnn::g_pool.push_back(sp.e);
  }
  frnn::g_spans.clear();
  return FRNN_OK;
}

// Total kernels launched by the library since load (bench.py gpu_launches).
int frnn_debug_launches(int64_t* count) {
  if (count) *count = frnn::g_launches.load();
  return FRNN_OK;
}

}  // extern "C"
