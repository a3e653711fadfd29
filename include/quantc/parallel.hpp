// quantc/parallel.hpp — host worker resolution (B200 build).
//
// Drop-in for /root/reference/proj/include/quantc/parallel.hpp.  On the B200
// path the per-sample parallelism of the reference's thread pool
// (calibration.cpp:68,95; interpreter.cpp:546) is the GPU batch dimension, and
// process-level sharding is one rank per GPU (parallel.py + NCCL).  The host
// utility is kept for API compatibility and host-side loops.
#pragma once

#include <cstddef>
#include <functional>

namespace quantc {

int resolve_workers(int requested);
void parallel_for(size_t n, int workers, const std::function<void(size_t)>& fn);

}  // namespace quantc
