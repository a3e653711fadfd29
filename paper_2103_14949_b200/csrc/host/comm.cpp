// comm.cpp — communicators for the distributed hot path (quantc/comm.hpp).
//
// NCCL is bound at run time (dlopen of libnccl.so.2: the copy torch ships in
// site-packages/nvidia/nccl, or whatever the process already loaded) so the
// library has no link-time NCCL dependency and a single-GPU user never loads
// it.  Collectives run on the engine stream over device staging buffers; the
// payloads of this path are small (8 bytes per candidate, 16 bytes per edge,
// 16 KB of int64 counts per edge), so one staging round trip per call is
// noise next to the forwards they merge.
#include "quantc/comm.hpp"

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "engine.hpp"
#include "quantc/device.hpp"

namespace quantc {

std::pair<int64_t, int64_t> shard_range(int64_t n, int rank, int world) {
  if (world < 1 || rank < 0 || rank >= world) throw CommError("bad rank / world size");
  const int64_t base = n / world, extra = n % world;
  const int64_t first = rank * base + std::min<int64_t>(rank, extra);
  return {first, first + base + (rank < extra ? 1 : 0)};
}

namespace {

class LocalComm final : public Communicator {
 public:
  int rank() const override { return 0; }
  int size() const override { return 1; }
  void allreduce_sum(int64_t*, size_t) override {}
  void allreduce_min(double*, size_t) override {}
  void allreduce_max(double*, size_t) override {}
  void allgather(const double* send, size_t n, double* recv) override {
    if (n) std::memcpy(recv, send, n * sizeof(double));
  }
};

class HookComm final : public Communicator {
 public:
  explicit HookComm(const CommHooks& h) : h_(h) {
    if (h_.size < 1 || h_.rank < 0 || h_.rank >= h_.size) throw CommError("bad rank / world size");
    if (!h_.allreduce_sum_i64 || !h_.allreduce_f64 || !h_.allgather_f64) {
      throw CommError("communicator callbacks missing");
    }
  }
  int rank() const override { return h_.rank; }
  int size() const override { return h_.size; }
  void allreduce_sum(int64_t* d, size_t n) override {
    check(h_.allreduce_sum_i64(d, n, h_.user), "allreduce(sum)");
  }
  void allreduce_min(double* d, size_t n) override {
    check(h_.allreduce_f64(d, n, 0, h_.user), "allreduce(min)");
  }
  void allreduce_max(double* d, size_t n) override {
    check(h_.allreduce_f64(d, n, 1, h_.user), "allreduce(max)");
  }
  void allgather(const double* s, size_t n, double* r) override {
    check(h_.allgather_f64(s, n, r, h_.user), "allgather");
  }

 private:
  static void check(int rc, const char* what) {
    if (rc != 0) throw CommError(std::string("communicator callback failed: ") + what);
  }
  CommHooks h_;
};

// ---- NCCL through dlopen ---------------------------------------------------------
// The ABI subset of nccl.h this file uses (stable since NCCL 2.0).
using ncclComm_t = void*;
using ncclResult_t = int;
enum { kNcclInt64 = 4, kNcclFloat64 = 8 };
enum { kNcclSum = 0, kNcclMax = 2, kNcclMin = 3 };

struct NcclApi {
  void* so = nullptr;
  ncclResult_t (*get_unique_id)(NcclId*) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t*, int, NcclId, int) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string why;
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    std::vector<std::string> names;
    if (const char* e = std::getenv("QUANTC_NCCL_LIB")) names.push_back(e);
    names.push_back("libnccl.so.2");
#ifdef QUANTC_NCCL_PATH
    names.push_back(QUANTC_NCCL_PATH);
#endif
    for (const std::string& n : names) {
      a.so = dlopen(n.c_str(), RTLD_NOW | RTLD_GLOBAL);
      if (a.so) break;
    }
    if (!a.so) {
      a.why = "libnccl.so.2 not found (set QUANTC_NCCL_LIB)";
      return a;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(a.so, name));
      if (!fn && a.why.empty()) a.why = std::string("NCCL symbol missing: ") + name;
    };
    sym(a.get_unique_id, "ncclGetUniqueId");
    sym(a.init_rank, "ncclCommInitRank");
    sym(a.destroy, "ncclCommDestroy");
    sym(a.all_reduce, "ncclAllReduce");
    sym(a.all_gather, "ncclAllGather");
    sym(a.error_string, "ncclGetErrorString");
    return a;
  }();
  return api;
}

NcclApi& nccl_or_throw() {
  NcclApi& a = nccl();
  if (!a.why.empty()) throw CommError(a.why);
  return a;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != 0) {
    throw CommError(std::string(what) + ": " + nccl().error_string(r));
  }
}

class NcclComm final : public Communicator {
 public:
  NcclComm(int rank, int world, const NcclId& id) : rank_(rank), world_(world) {
    if (world < 1 || rank < 0 || rank >= world) throw CommError("bad rank / world size");
    NcclApi& a = nccl_or_throw();
    device::current_device();  // binds the engine device before NCCL picks it up
    nccl_check(a.init_rank(&comm_, world, id, rank), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm_) nccl().destroy(comm_);
  }
  int rank() const override { return rank_; }
  int size() const override { return world_; }
  void allreduce_sum(int64_t* d, size_t n) override { reduce(d, n, 8, kNcclInt64, kNcclSum); }
  void allreduce_min(double* d, size_t n) override { reduce(d, n, 8, kNcclFloat64, kNcclMin); }
  void allreduce_max(double* d, size_t n) override { reduce(d, n, 8, kNcclFloat64, kNcclMax); }
  void allgather(const double* s, size_t n, double* r) override {
    if (n == 0) return;
    std::lock_guard<std::mutex> lk(mu_);
    const size_t bytes = n * 8;
    auto buf = engine::device_alloc(bytes * static_cast<size_t>(world_ + 1));
    char* send = static_cast<char*>(buf.get());
    char* recv = send + bytes;
    cudaStream_t st = static_cast<cudaStream_t>(device::stream());
    cudaMemcpyAsync(send, s, bytes, cudaMemcpyHostToDevice, st);
    nccl_check(nccl().all_gather(send, recv, n, kNcclFloat64, comm_, st), "ncclAllGather");
    cudaMemcpyAsync(r, recv, bytes * static_cast<size_t>(world_), cudaMemcpyDeviceToHost, st);
    device::synchronize();
  }

 private:
  void reduce(void* d, size_t n, size_t esize, int dtype, int op) {
    if (n == 0) return;
    std::lock_guard<std::mutex> lk(mu_);
    const size_t bytes = n * esize;
    auto buf = engine::device_alloc(bytes);
    cudaStream_t st = static_cast<cudaStream_t>(device::stream());
    cudaMemcpyAsync(buf.get(), d, bytes, cudaMemcpyHostToDevice, st);
    nccl_check(nccl().all_reduce(buf.get(), buf.get(), n, dtype, op, comm_, st), "ncclAllReduce");
    cudaMemcpyAsync(d, buf.get(), bytes, cudaMemcpyDeviceToHost, st);
    device::synchronize();
  }

  int rank_, world_;
  ncclComm_t comm_ = nullptr;
  std::mutex mu_;
};

}  // namespace

std::unique_ptr<Communicator> make_local_communicator() { return std::make_unique<LocalComm>(); }

std::unique_ptr<Communicator> make_callback_communicator(const CommHooks& hooks) {
  return std::make_unique<HookComm>(hooks);
}

bool nccl_available() { return nccl().why.empty(); }

NcclId nccl_unique_id() {
  NcclId id{};
  nccl_check(nccl_or_throw().get_unique_id(&id), "ncclGetUniqueId");
  return id;
}

std::unique_ptr<Communicator> make_nccl_communicator(int rank, int world, const NcclId& id) {
  return std::make_unique<NcclComm>(rank, world, id);
}

}  // namespace quantc
