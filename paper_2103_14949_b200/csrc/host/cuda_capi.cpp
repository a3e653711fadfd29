// cuda_capi.cpp — include/quantc_cuda.h: the C-ABI over the sm_100a kernels.
#include <algorithm>
#include "quantc_cuda.h"

#include <cuda_runtime.h>

#include <atomic>
#include <cstring>
#include <stdexcept>
#include <string>

#include "../kernels/kernels.h"
#include "engine.hpp"
#include "quantc/device.hpp"
#include "quantc/parallel.hpp"

using namespace quantc;

// shared with capi.cpp's error slot
namespace {
thread_local std::string g_err;

cudaStream_t st(void* s) {
  return s ? static_cast<cudaStream_t>(s) : static_cast<cudaStream_t>(device::stream());
}

template <typename F>
int wrap(F&& f) {
  try {
    (void)device::stream();  // device context first (fails loudly without a GPU)
    f();
    return QC_OK;
  } catch (const DeviceError& e) {
    g_err = e.what();
    return QC_ERR_CUDA;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return QC_ERR_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_err = e.what();
    return QC_ERR_CUDA;
  }
}

QParams from_pod(const qc_qparams& p) {
  QParams q;
  q.threshold = p.threshold;
  q.bit = p.bit;
  q.sign = p.sign;
  q.in_dtype = DType(static_cast<DTypeKind>(p.in_dtype));
  q.out_dtype = DType(static_cast<DTypeKind>(p.out_dtype));
  q.zero_point = p.zero_point;
  q.passthrough = p.passthrough != 0;
  if (p.acc_dtype != QC_NONE) q.acc_dtype = DType(static_cast<DTypeKind>(p.acc_dtype));
  q.acc_scale = p.acc_scale;
  return q;
}

kern::ConvShape shape(int N, int C, int H, int W, int O, int KH, int KW, int sh, int sw, int ph,
                      int pw) {
  kern::ConvShape cs{N, C, H, W, O, KH, KW, (H + 2 * ph - KH) / sh + 1, (W + 2 * pw - KW) / sw + 1,
                     sh, sw, ph, pw};
  return cs;
}
}  // namespace

extern "C" {

const char* qcu_last_error(void) { return g_err.c_str(); }

int qcu_sim_quant(const float* x, float* y, int64_t n, const qc_qparams* p, void* stream) {
  return wrap([&] { kern::sim_quant(x, y, n, engine::resolve_sq(from_pod(*p)), st(stream)); });
}

int qcu_minmax(const float* x, int64_t n, double* out_minmax, void* stream) {
  return wrap([&] {
    auto keys = engine::device_alloc(16);
    auto* k = static_cast<unsigned long long*>(keys.get());
    kern::minmax_init(k, 1, st(stream));
    kern::minmax_accumulate(x, n, k, st(stream));
    kern::minmax_decode(k, out_minmax, 1, st(stream));
    cudaStreamSynchronize(st(stream));
  });
}

int qcu_histogram(const float* x, int64_t n, double absmax, int bins, uint64_t* counts,
                  void* stream) {
  return wrap([&] {
    kern::histogram_accumulate(x, n, absmax, bins, reinterpret_cast<unsigned long long*>(counts),
                               1ull, st(stream));
  });
}

int qcu_kl_sweep(const int64_t* counts, int n_edges, int bins, int target_bit, int* best_i,
                 double* best_kl, void* stream) {
  return wrap([&] {
    if (target_bit < 1 || target_bit > 16 || bins < (1 << target_bit)) {
      throw std::invalid_argument("kl_sweep: bins must be >= 2^target_bit, target_bit in [1,16]");
    }
    kern::kl_sweep(counts, n_edges, bins, target_bit, best_i, best_kl, st(stream));
  });
}

int qcu_conv2d_f64acc(const float* x, const float* w, const float* bias, float* y, int N, int C,
                      int H, int W, int O, int KH, int KW, int sh, int sw, int ph, int pw,
                      void* stream) {
  return wrap([&] {
    kern::conv2d_f64acc(x, w, bias, y, shape(N, C, H, W, O, KH, KW, sh, sw, ph, pw), st(stream));
  });
}

int qcu_conv2d_grouped_f64acc(const float* x, const float* w, const float* bias, float* y, int N,
                              int C, int H, int W, int O, int KH, int KW, int sh, int sw, int ph,
                              int pw, int groups, void* stream) {
  return wrap([&] {
    if (groups < 1 || C % groups != 0 || O % groups != 0) {
      throw std::invalid_argument("qcu_conv2d_grouped_f64acc: groups must divide C and O");
    }
    kern::ConvShape cs = shape(N, C, H, W, O, KH, KW, sh, sw, ph, pw);
    cs.G = groups;
    kern::conv2d_f64acc(x, w, bias, y, cs, st(stream));
  });
}

int qcu_avg_pool2d_f32(const float* x, float* y, int N, int C, int H, int W, int KH, int KW,
                       int sh, int sw, int ph, int pw, void* stream) {
  return wrap([&] {
    const int OH = (H + 2 * ph - KH) / sh + 1, OW = (W + 2 * pw - KW) / sw + 1;
    kern::avgpool_f32(x, y, N, C, H, W, OH, OW, KH, KW, sh, sw, ph, pw, st(stream));
  });
}

int qcu_conv2d_int(const int32_t* x, const int32_t* w, const int32_t* bias, int32_t* y, int N,
                   int C, int H, int W, int O, int KH, int KW, int sh, int sw, int ph, int pw,
                   int64_t zp0, int64_t zp1, int acc_dtype, int trap, int64_t* overflow_flat,
                   void* stream) {
  return wrap([&] {
    DType acc(static_cast<DTypeKind>(acc_dtype));
    std::shared_ptr<void> flag;
    unsigned long long* f = nullptr;
    if (trap) {
      flag = engine::device_alloc(8);
      f = static_cast<unsigned long long*>(flag.get());
      unsigned long long init = ~0ull;
      cudaMemcpyAsync(f, &init, 8, cudaMemcpyHostToDevice, st(stream));
    }
    kern::conv2d_int(x, w, bias, y, shape(N, C, H, W, O, KH, KW, sh, sw, ph, pw), zp0, zp1,
                     acc.min_value(), acc.max_value(), f, st(stream));
    if (trap) {
      unsigned long long h = ~0ull;
      cudaMemcpyAsync(&h, f, 8, cudaMemcpyDeviceToHost, st(stream));
      cudaStreamSynchronize(st(stream));
      *overflow_flat = h == ~0ull ? -1 : static_cast<int64_t>(h);
    }
  });
}

int qcu_requantize(const int32_t* x, int32_t* y, int64_t n, int64_t multiplier, int shift,
                   int64_t in_zp, int64_t out_zp, int64_t qmin, int64_t qmax, void* stream) {
  return wrap([&] {
    kern::requantize_int(x, y, n, multiplier, shift, in_zp, out_zp, qmin, qmax, st(stream));
  });
}

int qcu_argmax_rows(const float* x, int rows, int64_t cols, int grouped, int64_t* out,
                    void* stream) {
  return wrap([&] {
    if (grouped) {
      // the grouped-candidate kernel: rows split into up to 4 equal groups
      const int g = std::min(grouped, 4);
      if (rows % g) throw std::invalid_argument("rows not divisible by the group count");
      const int per = rows / g;
      const float* xs[4];
      int64_t* outs[4];
      for (int i = 0; i < g; ++i) {
        xs[i] = x + static_cast<int64_t>(i) * per * cols;
        outs[i] = out + static_cast<int64_t>(i) * per;
      }
      kern::argmax_rows_multi(xs, outs, g, per, cols, st(stream));
    } else {
      kern::argmax_rows(x, rows, cols, out, st(stream));
    }
  });
}

int qcu_gemm_s8(const int8_t* A, const int8_t* B, int M, int N, int K, double scale,
                const float* bias, float* y, int OHW, void* stream) {
  return wrap([&] {
    if (!kern::gemm_s8_tcgen05_available()) throw DeviceError("tcgen05 path unavailable");
    kern::GemmEpilogue ep{y, bias, scale, OHW};
    kern::gemm_s8_tcgen05(A, B, M, N, K, ep, st(stream));
  });
}

int qcu_synchronize(void* stream) {
  return wrap([&] {
    cudaError_t e = cudaStreamSynchronize(st(stream));
    if (e != cudaSuccess) throw DeviceError(cudaGetErrorString(e));
  });
}

int qcu_tcgen05_available(void) {
  try {
    (void)device::stream();
    return kern::gemm_s8_tcgen05_available() ? 1 : 0;
  } catch (...) {
    return 0;
  }
}

int qcu_set_engine_mode(int mode) {
  return wrap([&] {
    if (mode < 0 || mode > 2) throw std::invalid_argument("engine mode must be 0, 1 or 2");
    device::set_engine_mode(static_cast<device::EngineMode>(mode));
  });
}

void* qcu_engine_stream(void) {
  try {
    return device::stream();
  } catch (...) {
    return nullptr;
  }
}

int qcu_profile_enable(int on) {
  return wrap([&] { device::profile_enable(on != 0); });
}

int qcu_parallel_selftest(size_t n, int workers, int64_t throw_at, int64_t* sum) {
  // host-only: no device context
  try {
    std::atomic<int64_t> acc{0};
    parallel_for(n, workers, [&](size_t i) {
      if (throw_at >= 0 && static_cast<int64_t>(i) >= throw_at) {
        throw std::runtime_error("selftest index " + std::to_string(i));
      }
      acc.fetch_add(static_cast<int64_t>(i));
    });
    *sum = acc.load();
    return QC_OK;
  } catch (const std::exception& e) {
    g_err = e.what();
    return QC_ERR_INTERNAL;
  }
}

int qcu_profile_read(double* gemm_ms, int64_t* gemm_launches, double* gemm_ops,
                     double* gemm_bytes) {
  return wrap([&] { device::profile_read(gemm_ms, gemm_launches, gemm_ops, gemm_bytes); });
}

int qcu_counters(int64_t* steps, int64_t* tcgen05_gemms, int64_t* f64_convs,
                 int64_t* fused_batches) {
  if (fused_batches) *fused_batches = device::counters().fused_batches;
  const auto& c = device::counters();
  if (steps) *steps = c.kernel_launches;
  if (tcgen05_gemms) *tcgen05_gemms = c.tcgen05_gemms;
  if (f64_convs) *f64_convs = c.f64_convs;
  return QC_OK;
}

int qcu_simt_int_convs(int64_t* n) {
  if (n) *n = device::counters().simt_int_convs;
  return QC_OK;
}

}  // extern "C"
