// quantc/comm.hpp — the communicator the distributed calibrate-and-search
// path runs over (B200 extension; the reference is single-process, its only
// parallelism a std::thread pool over samples, parallel.cpp:25-56).
//
// One process per GPU.  Every rank calls the same collectives in the same
// order.  All collectives used by the hot path are EXACT (min / max of
// doubles, sums of int64, gathers), so results are independent of the rank
// count and identical to one process and to the reference:
//   * calibration: MIN / MAX of per-edge extrema between the passes, SUM of
//     int64 histograms after pass 2 (reference calibration.cpp:81-91, :108-113)
//   * search, samples sharded: SUM of int64 agreement counts per candidate
//   * search, candidates sharded: ALLGATHER of per-candidate losses
//
// Backends: NCCL (dlopen'ed libnccl.so.2 over NVLink / NVSwitch; one
// communicator per GPU, collectives issued on the engine stream) and host
// callbacks (any transport the caller owns, e.g. torch.distributed / gloo in
// the multi-process CPU tests).
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>

namespace quantc {

class CommError : public std::runtime_error {
 public:
  explicit CommError(const std::string& what) : std::runtime_error(what) {}
};

class Communicator {
 public:
  virtual ~Communicator() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  // In place on host buffers; every rank passes the same n.
  virtual void allreduce_sum(int64_t* data, size_t n) = 0;
  virtual void allreduce_min(double* data, size_t n) = 0;
  virtual void allreduce_max(double* data, size_t n) = 0;
  // recv holds size() * n values, rank r's at [r*n, (r+1)*n).
  virtual void allgather(const double* send, size_t n, double* recv) = 0;
};

// Contiguous balanced partition of n units over `world` ranks: [first, last).
// The first n % world ranks own one extra unit.
std::pair<int64_t, int64_t> shard_range(int64_t n, int rank, int world);

// A single-process communicator (world 1): every collective is the identity.
std::unique_ptr<Communicator> make_local_communicator();

// NCCL.  The unique id is created by one rank (nccl_unique_id) and shared out
// of band (e.g. over torch.distributed); the communicator binds the current
// device (quantc::device) and runs its collectives on the engine stream.
using NcclId = std::array<char, 128>;
NcclId nccl_unique_id();
std::unique_ptr<Communicator> make_nccl_communicator(int rank, int world, const NcclId& id);
bool nccl_available();

// Host callbacks (status 0 = success).  op: 0 = min, 1 = max.
struct CommHooks {
  int rank = 0;
  int size = 1;
  void* user = nullptr;
  int (*allreduce_sum_i64)(int64_t* data, size_t n, void* user) = nullptr;
  int (*allreduce_f64)(double* data, size_t n, int op, void* user) = nullptr;
  int (*allgather_f64)(const double* send, size_t n, double* recv, void* user) = nullptr;
};
std::unique_ptr<Communicator> make_callback_communicator(const CommHooks& hooks);

}  // namespace quantc
