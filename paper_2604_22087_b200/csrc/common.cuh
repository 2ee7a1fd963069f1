// Common infrastructure for libafem_b200: error types (1:1 with the reference's exception types,
// reference errors.hpp:10-38), RAII device arrays, the context (device + stream + scratch), and a
// counted kernel-launch helper.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace afem {

struct LeaseError : std::logic_error { using std::logic_error::logic_error; };
struct StaleEpochError : std::logic_error { using std::logic_error::logic_error; };
struct CapabilityError : std::logic_error { using std::logic_error::logic_error; };
struct FactorizationError : std::runtime_error { using std::runtime_error::runtime_error; };
struct InvertedElementError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };
struct NomemError : std::runtime_error { using std::runtime_error::runtime_error; };

[[noreturn]] inline void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
  char buf[512];
  std::snprintf(buf, sizeof buf, "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e), cudaGetErrorString(e),
                file, line, what);
  if (e == cudaErrorMemoryAllocation) throw NomemError(buf);
  throw CudaError(buf);
}

#define AFEM_CK(x)                                                           \
  do {                                                                       \
    cudaError_t e_ = (x);                                                    \
    if (e_ != cudaSuccess) ::afem::throw_cuda(e_, #x, __FILE__, __LINE__);   \
  } while (0)

// Device array owned by the library (move-only).
template <class T>
struct DevArray {
  T* p = nullptr;
  size_t n = 0;
  DevArray() = default;
  explicit DevArray(size_t count) { alloc(count); }
  DevArray(const DevArray&) = delete;
  DevArray& operator=(const DevArray&) = delete;
  DevArray(DevArray&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DevArray& operator=(DevArray&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DevArray() { release(); }
  void alloc(size_t count) {
    release();
    if (count == 0) return;
    AFEM_CK(cudaMalloc(reinterpret_cast<void**>(&p), count * sizeof(T)));
    n = count;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  size_t bytes() const { return n * sizeof(T); }
  T* get() const { return p; }
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;
  int64_t launches = 0;
  // scratch for deterministic two-stage reductions
  DevArray<double> red_partials;  // kMaxBlocks * 4
  DevArray<double> red_out;       // 64 scalars
  DevArray<unsigned int> red_counter;
  // Grow-only staging buffers for host-pointer arguments at the ABI (slot k of the current call).
  std::vector<DevArray<uint8_t>> staging;
  int staging_next = 0;
  // copy streams + events of the pipelined host-buffer operator apply (created on first use)
  cudaStream_t s_in = nullptr, s_out = nullptr;
  std::vector<cudaEvent_t> events;
  void copy_streams(size_t n_events) {
    if (!s_in) {
      AFEM_CK(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking));
      AFEM_CK(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking));
    }
    while (events.size() < n_events) {
      cudaEvent_t e;
      AFEM_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      events.push_back(e);
    }
  }
  void release_copy_streams() {
    for (cudaEvent_t e : events) cudaEventDestroy(e);
    events.clear();
    if (s_in) cudaStreamDestroy(s_in);
    if (s_out) cudaStreamDestroy(s_out);
    s_in = s_out = nullptr;
  }
  // Per-context resources of the graph paths (created lazily on this context's device, so two
  // contexts on different devices driven from one host thread never share them):
  //   cap        private capture stream (the context stream may be the legacy default stream)
  //   snap/snap_ev  pinned host slots + events for the CG loop's status snapshots
  //   pcg_parts  block partials of the persistent cooperative CG
  cudaStream_t cap = nullptr;
  void* snap = nullptr;
  size_t snap_bytes = 0;
  cudaEvent_t snap_ev[2] = {nullptr, nullptr};
  DevArray<double> pcg_parts;
  cudaStream_t capture_stream() {
    if (!cap) AFEM_CK(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    return cap;
  }
  void* pinned_snap(size_t bytes) {
    if (snap_bytes < bytes) {
      if (snap) cudaFreeHost(snap);
      snap = nullptr;
      snap_bytes = 0;
      AFEM_CK(cudaMallocHost(&snap, bytes));
      snap_bytes = bytes;
    }
    for (cudaEvent_t& e : snap_ev)
      if (!e) AFEM_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return snap;
  }
  void release_graph_resources() {
    for (cudaEvent_t& e : snap_ev)
      if (e) cudaEventDestroy(e), e = nullptr;
    if (snap) cudaFreeHost(snap);
    snap = nullptr;
    snap_bytes = 0;
    if (cap) cudaStreamDestroy(cap);
    cap = nullptr;
    pcg_parts.release();
  }
  void* stage(size_t bytes) {
    if (staging_next >= (int)staging.size()) staging.emplace_back();
    DevArray<uint8_t>& b = staging[staging_next++];
    if (b.n < bytes) b.alloc(bytes);
    return b.p;
  }
};

// Stream capture of library launches into a graph, exception-safe: the context's stream is
// redirected to its private capture stream for the guard's lifetime. end() returns the captured
// graph; if the guard dies without end() (a launch threw), the capture is ended and discarded and
// the context's stream and launch counter are restored, so the context stays usable.
struct CaptureGuard {
  Ctx& c;
  cudaStream_t home;
  int64_t l0;
  bool open = true;
  explicit CaptureGuard(Ctx& ctx) : c(ctx), home(ctx.stream), l0(ctx.launches) {
    cudaStream_t s = c.capture_stream();
    AFEM_CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    c.stream = s;
  }
  // ends the capture; returns the graph (caller owns it) and the number of launches captured
  cudaGraph_t end(int64_t* captured = nullptr) {
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(c.stream, &g);
    open = false;
    if (captured) *captured = c.launches - l0;
    c.stream = home;
    c.launches = l0;
    AFEM_CK(e);
    return g;
  }
  ~CaptureGuard() {
    if (!open) return;
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(c.stream, &g);
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();  // clear the capture-invalidation error
    c.stream = home;
    c.launches = l0;
  }
  CaptureGuard(const CaptureGuard&) = delete;
  CaptureGuard& operator=(const CaptureGuard&) = delete;
};

// Runs a callable on scope exit (cleanup on every path, exceptions included).
template <class F>
struct ScopeExit {
  F f;
  bool armed = true;
  explicit ScopeExit(F fn) : f(std::move(fn)) {}
  ~ScopeExit() {
    if (armed) f();
  }
  ScopeExit(const ScopeExit&) = delete;
  ScopeExit& operator=(const ScopeExit&) = delete;
};

constexpr int kRedBlocks = 1184;  // 8 x 148 SMs: partial-sum slots for the deterministic reductions
constexpr int kRedThreads = 256;

// Counted launch on the context stream. Every kernel the library issues goes through here so
// bench.py can report how many of OUR kernels ran in a timed region.
template <class... KArgs, class... Args>
inline void launch(Ctx& c, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, Args&&... args) {
  if (grid.x == 0 || grid.y == 0 || grid.z == 0) return;
  k<<<grid, block, smem, c.stream>>>(std::forward<Args>(args)...);
  ++c.launches;
  AFEM_CK(cudaGetLastError());
}

inline unsigned grid_for(int64_t n, int threads, int64_t cap = 1 << 30) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g);
}

}  // namespace afem
