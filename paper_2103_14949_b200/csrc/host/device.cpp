// device.cpp — per-process device context: device selection, the engine
// stream, stream-ordered memory pool, engine mode.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <map>
#include <cstdlib>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "quantc/device.hpp"

namespace quantc::device {

namespace {

struct Context {
  int dev = -1;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // host->device uploads overlapping engine work
  std::atomic<int> mode{static_cast<int>(EngineMode::kAuto)};
};

Context& ctx() {
  static Context c;
  static std::once_flag once;
  std::call_once(once, [] {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
      throw DeviceError(std::string("quantc-b200 needs a CUDA device (sm_100a): ") +
                        (e != cudaSuccess ? cudaGetErrorString(e) : "no device visible"));
    }
    int dev = 0;
    if (const char* v = std::getenv("QUANTC_DEVICE")) {
      dev = std::atoi(v);
    } else if (const char* r = std::getenv("LOCAL_RANK")) {
      dev = std::atoi(r) % n;
    }
    if (cudaSetDevice(dev) != cudaSuccess) throw DeviceError("cudaSetDevice failed");
    cudaDeviceProp prop{};
    cudaGetDeviceProperties(&prop, dev);
    if (prop.major != 10) {
      throw DeviceError("quantc-b200 kernels are built for sm_100a; device " +
                        std::string(prop.name) + " is sm_" + std::to_string(prop.major) +
                        std::to_string(prop.minor));
    }
    // keep freed blocks in the pool: per-batch activations are re-allocated
    // every step
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thresh = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh);
    }
    cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking);
    c.dev = dev;
    if (const char* m = std::getenv("QUANTC_ENGINE")) {
      std::string s(m);
      if (s == "exact") c.mode = static_cast<int>(EngineMode::kExact);
      if (s == "fast") c.mode = static_cast<int>(EngineMode::kFast);
      if (s == "auto") c.mode = static_cast<int>(EngineMode::kAuto);
    }
  });
  // the engine may be driven from several host threads; bind the device
  cudaSetDevice(c.dev);
  return c;
}

}  // namespace

void set_engine_mode(EngineMode m) { ctx().mode = static_cast<int>(m); }
EngineMode engine_mode() { return static_cast<EngineMode>(ctx().mode.load()); }
int current_device() { return ctx().dev; }
namespace {
struct PinRegistry {
  std::mutex mu;
  std::map<uintptr_t, size_t> ranges;  // start -> bytes
  size_t total = 0;
};
PinRegistry& pins() {
  static PinRegistry* r = new PinRegistry;  // outlives static destructors
  return *r;
}
}  // namespace

bool pin_host(const void* p, size_t bytes) {
  if (!p || bytes == 0) return false;
  static const size_t cap = [] {
    const char* e = std::getenv("QUANTC_PIN_MAX_MB");
    return (e ? static_cast<size_t>(std::max(0, std::atoi(e))) : size_t{16384}) << 20;
  }();
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return false;
  }
  PinRegistry& r = pins();
  std::lock_guard<std::mutex> lk(r.mu);
  const auto key = reinterpret_cast<uintptr_t>(p);
  if (r.ranges.count(key)) return true;
  if (r.total + bytes > cap) return false;
  ctx();
  if (cudaHostRegister(const_cast<void*>(p), bytes, cudaHostRegisterDefault) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  r.ranges[key] = bytes;
  r.total += bytes;
  return true;
}

void unpin_host(const void* p) {
  PinRegistry& r = pins();
  std::lock_guard<std::mutex> lk(r.mu);
  auto it = r.ranges.find(reinterpret_cast<uintptr_t>(p));
  if (it == r.ranges.end()) return;
  cudaHostUnregister(const_cast<void*>(p));
  r.total -= it->second;
  r.ranges.erase(it);
}

bool host_pinned(const void* p, size_t bytes) {
  PinRegistry& r = pins();
  std::lock_guard<std::mutex> lk(r.mu);
  if (r.ranges.empty()) return false;
  const auto a = reinterpret_cast<uintptr_t>(p);
  auto it = r.ranges.upper_bound(a);
  if (it == r.ranges.begin()) return false;
  --it;
  return a + bytes <= it->first + it->second;
}

namespace {
struct Mirror {
  const void* pinned;
  size_t bytes_per;
  int64_t n;
};
std::mutex& mirror_mu() {
  static std::mutex* m = new std::mutex;
  return *m;
}
std::map<const void*, Mirror>& mirrors() {
  static auto* m = new std::map<const void*, Mirror>;
  return *m;
}
}  // namespace

void* alloc_pinned(size_t bytes) {
  static const size_t cap = [] {
    const char* e = std::getenv("QUANTC_PIN_MAX_MB");
    return (e ? static_cast<size_t>(std::max(0, std::atoi(e))) : size_t{16384}) << 20;
  }();
  if (bytes == 0 || bytes > cap) return nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return nullptr;
  }
  ctx();
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void free_pinned(void* p) {
  if (p) cudaFreeHost(p);
}

void set_dataset_mirror(const void* dataset, const void* pinned, size_t bytes_per, int64_t n) {
  std::lock_guard<std::mutex> lk(mirror_mu());
  mirrors()[dataset] = Mirror{pinned, bytes_per, n};
}

void clear_dataset_mirror(const void* dataset) {
  std::lock_guard<std::mutex> lk(mirror_mu());
  mirrors().erase(dataset);
}

bool dataset_mirror(const void* dataset, const void** pinned, size_t* bytes_per, int64_t* n) {
  std::lock_guard<std::mutex> lk(mirror_mu());
  auto it = mirrors().find(dataset);
  if (it == mirrors().end()) return false;
  *pinned = it->second.pinned;
  *bytes_per = it->second.bytes_per;
  *n = it->second.n;
  return true;
}

void* stream() { return ctx().stream; }
void* copy_stream() { return ctx().copy_stream; }

void* aux_stream(int i) {
  static std::mutex mu;
  static std::vector<cudaStream_t>* streams = new std::vector<cudaStream_t>;  // never destroyed
  ctx();
  std::lock_guard<std::mutex> lk(mu);
  while (static_cast<int>(streams->size()) <= i) {
    cudaStream_t s = nullptr;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    streams->push_back(s);
  }
  return (*streams)[static_cast<size_t>(i)];
}

void synchronize() {
  cudaError_t e = cudaStreamSynchronize(ctx().stream);
  if (e != cudaSuccess) throw DeviceError(std::string("CUDA error: ") + cudaGetErrorString(e));
}

void pool_reserve(size_t bytes) {
  static size_t reserved = 0;
  if (bytes <= reserved) return;
  cudaStream_t s = static_cast<cudaStream_t>(stream());
  void* p = nullptr;
  if (cudaMallocAsync(&p, bytes, s) == cudaSuccess) {
    cudaFreeAsync(p, s);
    reserved = bytes;
  } else {
    cudaGetLastError();
  }
}

size_t memory_budget_bytes() {
  if (const char* v = std::getenv("QUANTC_BATCH_BYTES")) return std::strtoull(v, nullptr, 10);
  size_t free_b = 0, total = 0;
  cudaMemGetInfo(&free_b, &total);
  size_t budget = free_b / 4;
  const size_t cap = size_t{24} << 30;
  return budget > cap ? cap : budget;
}

Counters& counters() {
  static Counters c;
  return c;
}

namespace {
struct Profile {
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events;
  std::vector<double> ops;
  std::vector<double> bytes;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t take() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};
Profile& prof() {
  static Profile p;
  return p;
}
}  // namespace

void profile_enable(bool on) { prof().on = on; }
bool profile_enabled() { return prof().on; }

void profile_gemm_begin() {
  Profile& p = prof();
  cudaEvent_t a = p.take(), b = p.take();
  cudaEventRecord(a, ctx().stream);
  p.events.push_back({a, b});
}

void profile_gemm_end(double ops, double bytes) {
  Profile& p = prof();
  cudaEventRecord(p.events.back().second, ctx().stream);
  p.ops.push_back(ops);
  p.bytes.push_back(bytes);
}

void profile_read(double* gemm_ms, int64_t* gemm_launches, double* gemm_ops,
                  double* gemm_bytes) {
  Profile& p = prof();
  synchronize();
  double ms = 0.0, ops = 0.0, bytes = 0.0;
  for (size_t i = 0; i < p.events.size(); ++i) {
    float t = 0.0f;
    cudaEventElapsedTime(&t, p.events[i].first, p.events[i].second);
    ms += t;
    ops += p.ops[i];
    bytes += p.bytes[i];
    p.pool.push_back(p.events[i].first);
    p.pool.push_back(p.events[i].second);
  }
  if (gemm_ms) *gemm_ms = ms;
  if (gemm_launches) *gemm_launches = static_cast<int64_t>(p.events.size());
  if (gemm_ops) *gemm_ops = ops;
  if (gemm_bytes) *gemm_bytes = bytes;
  p.events.clear();
  p.ops.clear();
  p.bytes.clear();
}

}  // namespace quantc::device
