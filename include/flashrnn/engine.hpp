// flashrnn/engine.hpp -- C++ drop-in for rnnkit's operator API, backed by the
// B200 kernels through the C ABI (flashrnn.h).  Header-only; link with
// -lflashrnn -lcudart -lpthread.
//
// Same types, members, layouts and signatures as the reference
//   rnnkit::rnn::forward   (/root/reference/proj/core/include/rnnkit/rnn/engine.hpp:143-144)
//   rnnkit::rnn::backward  (engine.hpp:221-225)
// in namespace flashrnn::rnn, so a caller switches engines by changing the
// namespace.  Value semantics: host std::vectors in, host
// std::vectors out.  Errors: the reference's std::invalid_argument cases
// (engine.hpp:107, :119-134, :231-236) throw std::invalid_argument;
// device/runtime failures throw std::runtime_error.  Element types: float
// (fp32 mode, FFMA kernels) and BFloat16 (bf16 mode, tcgen05 kernels); double
// is rejected (there is no CPU fallback).
//
// Host path (what a value-semantics call costs beyond the kernels):
//  * per calling thread, one CUDA stream and grow-only PINNED staging buffers;
//    device tensors come from the stream-ordered pool allocator (cudaMallocAsync
//    with the pool's release threshold raised), so steady-state calls allocate
//    nothing from the driver;
//  * host<->pinned conversion (BFloat16's float storage <-> bf16 bits, or a
//    plain copy for float) runs on a worker pool, chunk by chunk, and each
//    chunk's async copy overlaps the conversion of the next; the reference's
//    finiteness check of x/s0 (engine.hpp:131-135) happens in that same pass;
//  * forward() keeps the device copy of the trace (states, gates) attached to
//    the returned ForwardTrace; backward() uses it instead of re-uploading
//    while the trace's vectors still own the storage forward() returned
//    (a copied trace re-uploads).  Code that edits a trace in place calls
//    tr.drop_device() first; FRNN_SHIM_REUSE_TRACE=0 disables the reuse.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <future>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "../flashrnn.h"

#if defined(__linux__)
#include <sys/mman.h>
#endif

namespace flashrnn::rnn {

// ---- cell.hpp:11-53 ----
enum class Variant { Elman, Lstm, Gru, Slstm };

struct CellSpec {
  Variant variant = Variant::Elman;
  std::string name;
  int num_states = 1;
  int num_gates = 1;
  std::array<bool, 4> gate_uses_recurrent{true, true, true, true};
  std::array<bool, 4> gate_uses_input{true, true, true, true};
};

inline CellSpec cell_spec(Variant v) {
  frnn_cell c{};
  frnn_cell_spec(static_cast<int32_t>(v), &c);
  CellSpec s;
  s.variant = v;
  static const char* names[] = {"elman", "lstm", "gru", "slstm"};
  s.name = names[static_cast<int>(v)];
  s.num_states = c.num_states;
  s.num_gates = c.num_gates;
  for (int j = 0; j < 4; ++j) {
    s.gate_uses_recurrent[j] = c.uses_recurrent[j] != 0;
    s.gate_uses_input[j] = c.uses_input[j] != 0;
  }
  return s;
}

inline std::optional<Variant> variant_from_name(const std::string& n) {
  if (n == "elman") return Variant::Elman;
  if (n == "lstm") return Variant::Lstm;
  if (n == "gru") return Variant::Gru;
  if (n == "slstm") return Variant::Slstm;
  return std::nullopt;
}

// ---- scalar.hpp:12-43: bf16 value type (float storage, RNE rounding) ----
struct BFloat16 {
  float v = 0.0f;
  BFloat16() = default;
  explicit BFloat16(double x) : v(round(static_cast<float>(x))) {}
  explicit BFloat16(float x) : v(round(x)) {}
  explicit BFloat16(int x) : v(round(static_cast<float>(x))) {}
  static float round(float x) {
    if (!std::isfinite(x)) return x;
    uint32_t bits;
    std::memcpy(&bits, &x, 4);
    bits += 0x7FFFu + ((bits >> 16) & 1u);
    bits &= 0xFFFF0000u;
    std::memcpy(&x, &bits, 4);
    return x;
  }
  explicit operator double() const { return v; }
  explicit operator float() const { return v; }
  uint16_t bits() const {
    uint32_t b;
    std::memcpy(&b, &v, 4);
    return static_cast<uint16_t>(b >> 16);
  }
  static BFloat16 from_bits(uint16_t h) {
    BFloat16 r;
    uint32_t b = static_cast<uint32_t>(h) << 16;
    std::memcpy(&r.v, &b, 4);
    return r;
  }
};

// ---- engine.hpp:15-111 ----
template <class S>
struct Params {
  int num_heads = 1;
  int head_dim = 0;
  int num_gates = 1;
  std::vector<S> recurrent;  // [head][gate][row][col]
  std::vector<S> bias;       // [gate][dim]
  int dim() const { return num_heads * head_dim; }
  std::size_t r_index(int head, int gate, int row, int col) const {
    return ((static_cast<std::size_t>(head) * num_gates + gate) * head_dim + row) * head_dim + col;
  }
  std::size_t b_index(int gate, int e) const { return static_cast<std::size_t>(gate) * dim() + e; }
  static Params zeros(int num_heads, int head_dim, int num_gates) {
    Params p;
    p.num_heads = num_heads;
    p.head_dim = head_dim;
    p.num_gates = num_gates;
    p.recurrent.assign(static_cast<std::size_t>(num_heads) * num_gates * head_dim * head_dim, S(0));
    p.bias.assign(static_cast<std::size_t>(num_gates) * num_heads * head_dim, S(0));
    return p;
  }
};

template <class S>
struct SequenceBatch {
  int seq_len = 0, batch = 0, num_gates = 1, num_states = 1, dim = 0;
  std::vector<S> inputs;       // [T][batch][gate][dim]
  std::vector<S> init_states;  // [state][batch][dim]
  std::size_t x_index(int t, int b, int gate, int e) const {
    return ((static_cast<std::size_t>(t) * batch + b) * num_gates + gate) * dim + e;
  }
  std::size_t s_index(int state, int b, int e) const {
    return (static_cast<std::size_t>(state) * batch + b) * dim + e;
  }
  static SequenceBatch zeros(int seq_len, int batch, int num_gates, int num_states, int dim) {
    SequenceBatch sb;
    sb.seq_len = seq_len;
    sb.batch = batch;
    sb.num_gates = num_gates;
    sb.num_states = num_states;
    sb.dim = dim;
    sb.inputs.assign(static_cast<std::size_t>(seq_len) * batch * num_gates * dim, S(0));
    sb.init_states.assign(static_cast<std::size_t>(num_states) * batch * dim, S(0));
    return sb;
  }
};

namespace detail {
struct DeviceTrace;
}

template <class S>
struct ForwardTrace {
  int seq_len = 0, batch = 0, num_states = 1, num_gates = 1, dim = 0;
  std::vector<S> states;  // [T+1][state][batch][dim]
  std::vector<S> gates;   // [T][gate][batch][dim]
  // Not in rnnkit's struct: the device copy forward() produced, reused by
  // backward() while `states`/`gates` still own forward()'s storage.
  std::shared_ptr<detail::DeviceTrace> device;
  void drop_device() { device.reset(); }
  std::size_t s_index(int t, int state, int b, int e) const {
    return ((static_cast<std::size_t>(t) * num_states + state) * batch + b) * dim + e;
  }
  std::size_t g_index(int t, int gate, int b, int e) const {
    return ((static_cast<std::size_t>(t) * num_gates + gate) * batch + b) * dim + e;
  }
};

template <class S>
struct Gradients {
  std::vector<S> d_inputs, d_bias, d_recurrent, d_init_states;
};

struct ClipPolicy {
  enum class Mode { Off, ClipValue, Zero };
  Mode mode = Mode::Off;
  double magnitude = 0.0;
  static ClipPolicy off() { return {Mode::Off, 0.0}; }
  static ClipPolicy value(double m) {
    if (m <= 0) throw std::invalid_argument("clip magnitude must be positive");  // engine.hpp:107
    return {Mode::ClipValue, m};
  }
  static ClipPolicy zero() { return {Mode::Zero, 0.0}; }
};

template <class S>
struct StepGradients {
  std::vector<S> hidden;  // [T][batch][dim]; empty means none
};

namespace detail {

template <class S>
constexpr int32_t dtype_of() {
  static_assert(std::is_same_v<S, float> || std::is_same_v<S, BFloat16>,
                "flashrnn GPU engine supports float and BFloat16 (no fp64, no CPU fallback)");
  return std::is_same_v<S, float> ? FRNN_F32 : FRNN_BF16;
}
template <class S>
constexpr std::size_t dev_size() {
  return std::is_same_v<S, float> ? 4 : 2;
}

[[noreturn]] inline void raise(int rc) {
  const std::string msg = frnn_last_error();
  if (rc == FRNN_EINVAL_SHAPE || rc == FRNN_ENONFINITE || rc == FRNN_EINVAL_ARG) throw std::invalid_argument(msg);
  throw std::runtime_error("flashrnn: " + msg);
}
inline void check(int rc) {
  if (rc != FRNN_OK) raise(rc);
}
inline void cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("flashrnn: ") + what + ": " + cudaGetErrorString(e));
}

// Fixed worker pool for the host-side conversions: run(n, f) calls f(begin, end)
// over [0, n) in chunks of `grain`, on the workers and the calling thread.
class Pool {
 public:
  static Pool& get() {
    static Pool p;
    return p;
  }
  void run(std::size_t n, std::size_t grain, const std::function<void(std::size_t, std::size_t)>& f) {
    if (n == 0) return;
    const std::size_t chunks = (n + grain - 1) / grain;
    if (workers_.empty() || chunks == 1) {
      f(0, n);
      return;
    }
    std::unique_lock<std::mutex> job_lock(job_mutex_);  // one job at a time
    {
      std::lock_guard<std::mutex> g(m_);
      fn_ = &f;
      n_ = n;
      grain_ = grain;
      chunks_ = chunks;
      next_.store(0);
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    const std::size_t mine = drain();
    std::unique_lock<std::mutex> l(m_);
    done_ += mine;
    done_cv_.wait(l, [&] { return done_ == chunks_; });
    fn_ = nullptr;
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }

 private:
  Pool() {
    const char* e = std::getenv("FRNN_SHIM_THREADS");
    unsigned n = e ? static_cast<unsigned>(std::atoi(e)) : std::min(16u, std::thread::hardware_concurrency());
    for (unsigned i = 1; i < n; ++i) workers_.emplace_back([this] { loop(); });
  }
  std::size_t drain() {
    std::size_t did = 0;
    for (;;) {
      const std::size_t c = next_.fetch_add(1);
      if (c >= chunks_) return did;
      const std::size_t b = c * grain_;
      (*fn_)(b, std::min(n_, b + grain_));
      ++did;
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> l(m_);
        cv_.wait(l, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        if (!fn_) continue;
      }
      const std::size_t did = drain();
      std::lock_guard<std::mutex> g(m_);
      done_ += did;
      if (done_ == chunks_) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex m_, job_mutex_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(std::size_t, std::size_t)>* fn_ = nullptr;
  std::size_t n_ = 0, grain_ = 1, chunks_ = 0, done_ = 0;
  std::atomic<std::size_t> next_{0};
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// Per-thread stream, pinned staging and events (grow-only; reused by every call).
struct Staging {
  cudaStream_t stream = nullptr;
  void* pin = nullptr;
  std::size_t pin_bytes = 0;
  std::vector<cudaEvent_t> events;
  int device = -1;
  Staging() {
    cuda(cudaGetDevice(&device), "cudaGetDevice");
    cuda(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
    cudaMemPool_t pool;  // keep freed blocks in the stream-ordered pool (no driver frees between calls)
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  // The stream is deliberately never destroyed: a ForwardTrace may outlive the
  // thread that produced it, and its device copy is freed stream-ordered on
  // this stream (DevMem).  One stream per calling thread for the process lifetime.
  ~Staging() {
    if (stream) cudaStreamSynchronize(stream);
    for (auto e : events) cudaEventDestroy(e);
    if (pin) cudaFreeHost(pin);
  }
  uint8_t* pinned(std::size_t bytes) {
    if (bytes > pin_bytes) {
      if (pin) {
        cuda(cudaStreamSynchronize(stream), "stream sync");
        cudaFreeHost(pin);
        pin = nullptr;
      }
      const std::size_t nb = std::max(bytes, pin_bytes + pin_bytes / 2);
      cuda(cudaHostAlloc(&pin, nb, cudaHostAllocDefault), "cudaHostAlloc");
      pin_bytes = nb;
    }
    return static_cast<uint8_t*>(pin);
  }
  cudaEvent_t event(std::size_t i) {
    while (events.size() <= i) {
      cudaEvent_t e;
      cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
      events.push_back(e);
    }
    return events[i];
  }
  static Staging& get() {
    thread_local Staging s;
    return s;
  }
};

// Stream-ordered device allocation (pooled), freed on the stream it was used on.
struct DevMem {
  void* ptr = nullptr;
  cudaStream_t stream = nullptr;
  DevMem() = default;
  DevMem(std::size_t bytes, cudaStream_t s) : stream(s) {
    if (bytes) cuda(cudaMallocAsync(&ptr, bytes, s), "cudaMallocAsync");
  }
  DevMem(const DevMem&) = delete;
  DevMem& operator=(const DevMem&) = delete;
  DevMem(DevMem&& o) noexcept : ptr(o.ptr), stream(o.stream) { o.ptr = nullptr; }
  DevMem& operator=(DevMem&& o) noexcept {
    if (this != &o) {
      if (ptr) cudaFreeAsync(ptr, stream);
      ptr = o.ptr;
      stream = o.stream;
      o.ptr = nullptr;
    }
    return *this;
  }
  ~DevMem() {
    if (ptr) cudaFreeAsync(ptr, stream);
  }
};

struct DeviceTrace {
  DevMem states, gates;
  const void* host_states = nullptr;  // storage identity of the trace forward() returned
  const void* host_gates = nullptr;
  std::size_t n_states = 0, n_gates = 0;
  int32_t dtype = 0, device = -1;
};

constexpr std::size_t kChunk = std::size_t(1) << 21;  // elements per pipelined chunk
constexpr std::size_t kGrain = std::size_t(1) << 16;  // elements per worker task

// One host tensor bound for the device: element count, its device destination
// and the byte offset of its image in the pinned staging buffer.
template <class S>
struct Up {
  const std::vector<S>* v;
  void* dst;
  std::size_t off;
  bool check_finite;
};

// host vectors -> pinned (parallel convert, optional finiteness scan) -> device,
// chunk by chunk so each chunk's H2D overlaps the next chunk's conversion.
// Throws invalid_argument (before any launch) on a non-finite checked tensor.
template <class S>
void upload(std::vector<Up<S>> ups, Staging& st) {
  std::size_t total = 0;
  for (auto& u : ups) {
    u.off = total;
    total += (u.v->size() * dev_size<S>() + 255) & ~std::size_t(255);
  }
  uint8_t* pin = st.pinned(total);
  for (auto& u : ups) {
    const std::size_t n = u.v->size();
    const S* src = u.v->data();
    for (std::size_t c0 = 0; c0 < n; c0 += kChunk) {
      const std::size_t c1 = std::min(n, c0 + kChunk);
      std::atomic<bool> bad{false};
      Pool::get().run(c1 - c0, kGrain, [&](std::size_t b, std::size_t e) {
        bool nonfinite = false;
        if constexpr (std::is_same_v<S, float>) {
          float* out = reinterpret_cast<float*>(pin + u.off) + c0;
          std::memcpy(out + b, src + c0 + b, (e - b) * 4);
          if (u.check_finite)
            for (std::size_t i = b; i < e; ++i) nonfinite |= !std::isfinite(out[i]);
        } else {
          uint16_t* out = reinterpret_cast<uint16_t*>(pin + u.off) + c0;
          for (std::size_t i = b; i < e; ++i) {
            uint32_t w;
            std::memcpy(&w, &src[c0 + i].v, 4);
            out[i] = static_cast<uint16_t>(w >> 16);  // values are bf16-exact (BFloat16 rounds on construction)
            nonfinite |= u.check_finite && (w & 0x7F800000u) == 0x7F800000u;
          }
        }
        if (nonfinite) bad = true;
      });
      if (bad) throw std::invalid_argument("non-finite input or initial state");  // engine.hpp:131-135
      cuda(cudaMemcpyAsync(static_cast<uint8_t*>(u.dst) + c0 * dev_size<S>(), pin + u.off + c0 * dev_size<S>(),
                           (c1 - c0) * dev_size<S>(), cudaMemcpyHostToDevice, st.stream),
           "H2D");
    }
  }
}

// device -> pinned -> host vectors: every chunk's D2H is queued first (with an
// event), then each chunk is converted as soon as it lands.
template <class S>
void download(const std::vector<std::pair<const void*, std::vector<S>*>>& downs, Staging& st) {
  std::size_t total = 0;
  std::vector<std::size_t> offs;
  for (auto& d : downs) {
    offs.push_back(total);
    total += (d.second->size() * dev_size<S>() + 255) & ~std::size_t(255);
  }
  uint8_t* pin = st.pinned(total);
  std::size_t ev = 0;
  for (std::size_t k = 0; k < downs.size(); ++k) {
    const std::size_t n = downs[k].second->size();
    for (std::size_t c0 = 0; c0 < n; c0 += kChunk) {
      const std::size_t c1 = std::min(n, c0 + kChunk);
      cuda(cudaMemcpyAsync(pin + offs[k] + c0 * dev_size<S>(),
                           static_cast<const uint8_t*>(downs[k].first) + c0 * dev_size<S>(),
                           (c1 - c0) * dev_size<S>(), cudaMemcpyDeviceToHost, st.stream),
           "D2H");
      cuda(cudaEventRecord(st.event(ev++), st.stream), "cudaEventRecord");
    }
  }
  ev = 0;
  for (std::size_t k = 0; k < downs.size(); ++k) {
    std::vector<S>& out = *downs[k].second;
    const std::size_t n = out.size();
    for (std::size_t c0 = 0; c0 < n; c0 += kChunk) {
      const std::size_t c1 = std::min(n, c0 + kChunk);
      cuda(cudaEventSynchronize(st.event(ev++)), "D2H");
      Pool::get().run(c1 - c0, kGrain, [&](std::size_t b, std::size_t e) {
        if constexpr (std::is_same_v<S, float>) {
          std::memcpy(out.data() + c0 + b, reinterpret_cast<const float*>(pin + offs[k]) + c0 + b, (e - b) * 4);
        } else {
          const uint16_t* in = reinterpret_cast<const uint16_t*>(pin + offs[k]) + c0;
          for (std::size_t i = b; i < e; ++i) {
            const uint32_t w = static_cast<uint32_t>(in[i]) << 16;
            std::memcpy(&out[c0 + i].v, &w, 4);
          }
        }
      });
    }
  }
}

// A value-semantics output vector of n elements.  Fresh multi-hundred-MB
// buffers are page-fault bound (every call allocates new result vectors, as
// rnnkit's API returns by value): ask for transparent huge pages before the
// elements are constructed, and build the outputs of one call concurrently
// (alloc_outputs) while the uploads and kernels run.
template <class S>
void alloc_out(std::vector<S>& v, std::size_t n) {
  v.reserve(n);
#if defined(__linux__) && defined(MADV_HUGEPAGE)
  const std::uintptr_t lo = (reinterpret_cast<std::uintptr_t>(v.data()) + (2u << 20) - 1) & ~std::uintptr_t((2u << 20) - 1);
  const std::uintptr_t hi = (reinterpret_cast<std::uintptr_t>(v.data() + n)) & ~std::uintptr_t((2u << 20) - 1);
  if (hi > lo) madvise(reinterpret_cast<void*>(lo), hi - lo, MADV_HUGEPAGE);
#endif
  v.resize(n);
}
// Ready-made large output vectors: a call takes one (a move, no page faults,
// no zero fill on its critical path) and a background thread builds the
// replacement for the next call of the same shape while the caller does
// whatever it does between calls.  At most 2 spares per size; only sizes of
// >= 1 Mi elements; FRNN_SHIM_PREBUILD=0 turns it off.
template <class S>
class OutputCache {
 public:
  static OutputCache& get() {
    static OutputCache c;
    return c;
  }
  // Called on the worker of an alloc_outputs future.
  std::vector<S> take(std::size_t n) {
    std::vector<S> v;
    bool hit = false;
    {
      std::lock_guard<std::mutex> g(m_);
      auto it = ready_.find(n);
      if (it != ready_.end() && !it->second.empty()) {
        v = std::move(it->second.back());
        it->second.pop_back();
        hit = true;
      }
    }
    if (!hit) alloc_out(v, n);
    refill(n);
    return v;
  }
  static bool enabled(std::size_t n) {
    static const bool on = [] {
      const char* e = std::getenv("FRNN_SHIM_PREBUILD");
      return !e || std::atoi(e) != 0;
    }();
    return on && n >= (std::size_t(1) << 20);
  }
  ~OutputCache() {
    std::vector<std::future<void>> fs;
    {
      std::lock_guard<std::mutex> g(m_);
      fs.swap(builders_);
    }
    for (auto& f : fs) f.wait();
  }

 private:
  void refill(std::size_t n) {
    std::lock_guard<std::mutex> g(m_);
    builders_.erase(std::remove_if(builders_.begin(), builders_.end(),
                                   [](std::future<void>& f) {
                                     return f.wait_for(std::chrono::seconds(0)) == std::future_status::ready;
                                   }),
                    builders_.end());
    if (ready_[n].size() + pending_[n] >= 2) return;
    ++pending_[n];
    builders_.push_back(std::async(std::launch::async, [this, n] {
      std::vector<S> v;
      alloc_out(v, n);
      std::lock_guard<std::mutex> l(m_);
      ready_[n].push_back(std::move(v));
      --pending_[n];
    }));
  }
  std::mutex m_;
  std::map<std::size_t, std::vector<std::vector<S>>> ready_;
  std::map<std::size_t, int> pending_;
  std::vector<std::future<void>> builders_;
};

// Build a call's large outputs concurrently with its uploads and kernels.
template <class S>
std::vector<std::future<void>> alloc_outputs(const std::vector<std::pair<std::vector<S>*, std::size_t>>& outs) {
  std::vector<std::future<void>> f;
  for (auto& o : outs)
    f.push_back(std::async(std::launch::async, [o] {
      if (OutputCache<S>::enabled(o.second)) *o.first = OutputCache<S>::get().take(o.second);
      else alloc_out(*o.first, o.second);
    }));
  return f;
}

// FRNN_SHIM_PROFILE=1: per-call phase times on stderr.
struct PhaseClock {
  bool on;
  const char* name;
  std::chrono::steady_clock::time_point t0, last;
  std::string out;
  explicit PhaseClock(const char* n) : on(std::getenv("FRNN_SHIM_PROFILE") != nullptr), name(n) {
    t0 = last = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    const auto t = std::chrono::steady_clock::now();
    char buf[96];
    std::snprintf(buf, sizeof buf, " %s %.2f", what, std::chrono::duration<double, std::milli>(t - last).count());
    out += buf;
    last = t;
  }
  ~PhaseClock() {
    if (on)
      std::fprintf(stderr, "[flashrnn shim] %s:%s | total %.2f ms\n", name, out.c_str(),
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
};

inline frnn_cell to_c(const CellSpec& c) {
  frnn_cell r{};
  r.variant = static_cast<int32_t>(c.variant);
  r.num_states = c.num_states;
  r.num_gates = c.num_gates;
  for (int j = 0; j < 4; ++j) {
    r.uses_recurrent[j] = c.gate_uses_recurrent[j];
    r.uses_input[j] = c.gate_uses_input[j];
  }
  return r;
}

// engine.hpp:116-128 (check_shapes): counts, dims and every storage size.
template <class S>
void check_shapes(const CellSpec& cell, const Params<S>& p, const SequenceBatch<S>& sb) {
  if (p.num_gates != cell.num_gates || sb.num_gates != cell.num_gates || sb.num_states != cell.num_states)
    throw std::invalid_argument("cell/params/batch gate or state counts disagree");
  if (sb.dim != p.dim()) throw std::invalid_argument("batch dim != params dim");
  if (p.num_heads < 1 || p.head_dim < 1 || sb.batch < 1 || sb.seq_len < 0)
    throw std::invalid_argument("degenerate shape");
  const std::size_t NG = cell.num_gates, NS = cell.num_states, D = sb.dim, T = sb.seq_len, B = sb.batch;
  if (p.recurrent.size() != (std::size_t)p.num_heads * NG * p.head_dim * p.head_dim ||
      p.bias.size() != NG * D || sb.inputs.size() != T * B * NG * D || sb.init_states.size() != NS * B * D)
    throw std::invalid_argument("tensor storage size mismatch");
}

inline bool reuse_trace() {
  const char* e = std::getenv("FRNN_SHIM_REUSE_TRACE");
  return !e || std::atoi(e) != 0;
}

}  // namespace detail

/// engine.hpp:143-203 on the GPU.
template <class S>
ForwardTrace<S> forward(const CellSpec& cell, const Params<S>& p, const SequenceBatch<S>& sb) {
  detail::check_shapes(cell, p, sb);
  const frnn_cell c = detail::to_c(cell);
  const frnn_shape sh{sb.seq_len, sb.batch, p.num_heads, p.head_dim};
  const int32_t dt = detail::dtype_of<S>();
  const std::size_t NS = cell.num_states, NG = cell.num_gates, D = sb.dim, T = sb.seq_len, B = sb.batch;
  const frnn_options opt{0u, FRNN_ALGO_AUTO};  // finiteness is checked on the host during staging
  std::size_t wsb = 0;
  detail::check(frnn_workspace_size(&c, sh, dt, FRNN_PASS_FORWARD, &opt, &wsb));
  detail::Staging& stg = detail::Staging::get();
  const cudaStream_t s = stg.stream;
  constexpr std::size_t E = detail::dev_size<S>();
  detail::DevMem R(p.recurrent.size() * E, s), bias(p.bias.size() * E, s), x(sb.inputs.size() * E, s),
      s0(sb.init_states.size() * E, s), ws(wsb, s);
  detail::PhaseClock pc("forward");
  auto dtr = std::make_shared<detail::DeviceTrace>();
  dtr->states = detail::DevMem((T + 1) * NS * B * D * E, s);
  dtr->gates = detail::DevMem(T * NG * B * D * E, s);
  ForwardTrace<S> tr;
  tr.seq_len = sb.seq_len;
  tr.batch = sb.batch;
  tr.num_states = cell.num_states;
  tr.num_gates = cell.num_gates;
  tr.dim = sb.dim;
  auto allocs = detail::alloc_outputs<S>({{&tr.states, (T + 1) * NS * B * D}, {&tr.gates, T * NG * B * D}});
  detail::upload<S>({{&p.recurrent, R.ptr, 0, false}, {&p.bias, bias.ptr, 0, false},
                     {&sb.init_states, s0.ptr, 0, true}, {&sb.inputs, x.ptr, 0, true}},
                    stg);
  pc.mark("upload");
  detail::check(frnn_forward(&c, sh, dt, R.ptr, bias.ptr, x.ptr, s0.ptr, dtr->states.ptr, dtr->gates.ptr, ws.ptr,
                             wsb, &opt, s));
  for (auto& f : allocs) f.get();
  pc.mark("alloc-wait");
  detail::download<S>({{dtr->states.ptr, &tr.states}, {dtr->gates.ptr, &tr.gates}}, stg);
  detail::cuda(cudaStreamSynchronize(s), "forward");
  pc.mark("kernel+download");
  dtr->host_states = tr.states.data();
  dtr->host_gates = tr.gates.data();
  dtr->n_states = tr.states.size();
  dtr->n_gates = tr.gates.size();
  dtr->dtype = dt;
  dtr->device = stg.device;
  if (detail::reuse_trace()) tr.device = std::move(dtr);
  return tr;
}

/// engine.hpp:221-339 on the GPU.
template <class S>
Gradients<S> backward(const CellSpec& cell, const Params<S>& p, const SequenceBatch<S>& sb,
                      const ForwardTrace<S>& tr, const std::vector<S>& d_states_final,
                      const ClipPolicy& clip = ClipPolicy::off(), const StepGradients<S>* extra = nullptr) {
  detail::check_shapes(cell, p, sb);
  const std::size_t NS = cell.num_states, NG = cell.num_gates, D = sb.dim, T = sb.seq_len, B = sb.batch;
  if (tr.seq_len != sb.seq_len || tr.batch != sb.batch || tr.dim != sb.dim || tr.num_states != cell.num_states ||
      tr.num_gates != cell.num_gates || tr.states.size() != (T + 1) * NS * B * D ||
      tr.gates.size() != T * NG * B * D)
    throw std::invalid_argument("trace does not match batch");  // engine.hpp:229-231
  if (d_states_final.size() != NS * B * D) throw std::invalid_argument("terminal state gradient has wrong size");
  const bool has_dh = extra && !extra->hidden.empty();
  if (has_dh && extra->hidden.size() != T * B * D)
    throw std::invalid_argument("per-step hidden gradients have wrong size");
  const frnn_cell c = detail::to_c(cell);
  const frnn_shape sh{sb.seq_len, sb.batch, p.num_heads, p.head_dim};
  const int32_t dt = detail::dtype_of<S>();
  std::size_t wsb = 0;
  detail::check(frnn_workspace_size(&c, sh, dt, FRNN_PASS_BACKWARD, nullptr, &wsb));
  detail::Staging& stg = detail::Staging::get();
  const cudaStream_t s = stg.stream;
  constexpr std::size_t E = detail::dev_size<S>();
  detail::DevMem R(p.recurrent.size() * E, s), bias(p.bias.size() * E, s), dsf(d_states_final.size() * E, s),
      dh(has_dh ? extra->hidden.size() * E : 0, s), dx(sb.inputs.size() * E, s), db(p.bias.size() * E, s),
      dR(p.recurrent.size() * E, s), ds0(d_states_final.size() * E, s), ws(wsb, s), st_up, ga_up;
  std::vector<detail::Up<S>> ups{{&p.recurrent, R.ptr, 0, false}, {&p.bias, bias.ptr, 0, false},
                                 {&d_states_final, dsf.ptr, 0, false}};
  if (has_dh) ups.push_back({&extra->hidden, dh.ptr, 0, false});
  const void* st = nullptr;
  const void* ga = nullptr;
  const detail::DeviceTrace* dev = tr.device.get();
  if (dev && detail::reuse_trace() && dev->host_states == tr.states.data() && dev->host_gates == tr.gates.data() &&
      dev->n_states == tr.states.size() && dev->n_gates == tr.gates.size() && dev->dtype == dt &&
      dev->device == stg.device) {
    st = dev->states.ptr;  // forward()'s device trace, still the one these vectors hold
    ga = dev->gates.ptr;
  } else {
    st_up = detail::DevMem(tr.states.size() * E, s);
    ga_up = detail::DevMem(tr.gates.size() * E, s);
    ups.push_back({&tr.states, st_up.ptr, 0, false});
    ups.push_back({&tr.gates, ga_up.ptr, 0, false});
    st = st_up.ptr;
    ga = ga_up.ptr;
  }
  detail::PhaseClock pc("backward");
  Gradients<S> g;
  auto allocs = detail::alloc_outputs<S>({{&g.d_inputs, sb.inputs.size()}});
  g.d_bias.resize(p.bias.size());
  g.d_recurrent.resize(p.recurrent.size());
  g.d_init_states.resize(d_states_final.size());
  detail::upload<S>(std::move(ups), stg);
  pc.mark(st_up.ptr ? "upload(+trace)" : "upload");
  const frnn_clip cl{static_cast<int32_t>(clip.mode), clip.magnitude};
  detail::check(frnn_backward(&c, sh, dt, R.ptr, bias.ptr, st, ga, dsf.ptr, has_dh ? dh.ptr : nullptr, cl, dx.ptr,
                              db.ptr, dR.ptr, ds0.ptr, ws.ptr, wsb, nullptr, s));
  for (auto& f : allocs) f.get();
  pc.mark("alloc-wait");
  detail::download<S>({{db.ptr, &g.d_bias}, {dR.ptr, &g.d_recurrent}, {ds0.ptr, &g.d_init_states},
                       {dx.ptr, &g.d_inputs}},
                      stg);
  detail::cuda(cudaStreamSynchronize(s), "backward");
  pc.mark("kernel+download");
  return g;
}

}  // namespace flashrnn::rnn
