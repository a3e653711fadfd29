// core.cpp — DType, Tensor, BigUInt and the host worker helper.
//
// Semantics follow reference dtype.cpp:10-79, tensor.cpp:14-124 and
// parallel.cpp:15-56 (ranges, error messages' meaning, first-by-index
// exception rethrow).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <mutex>
#include <numeric>
#include <condition_variable>
#include <stdexcept>
#include <thread>
#include <vector>

#include "quantc/bigint.hpp"
#include "quantc/dtype.hpp"
#include "quantc/parallel.hpp"
#include "quantc/tensor.hpp"

namespace quantc {

// ---- DType ------------------------------------------------------------------

namespace {
struct KindRow {
  DTypeKind kind;
  const char* name;
  int width;  // 0 for float
  size_t bytes;
};
constexpr KindRow kKinds[] = {
    {DTypeKind::kFloat32, "float32", 0, 4}, {DTypeKind::kInt8, "int8", 8, 1},
    {DTypeKind::kUInt8, "uint8", 8, 1},     {DTypeKind::kInt16, "int16", 16, 2},
    {DTypeKind::kInt32, "int32", 32, 4},
};
const KindRow& row_of(DTypeKind k) {
  for (const KindRow& r : kKinds) {
    if (r.kind == k) return r;
  }
  throw std::invalid_argument("bad dtype kind");
}
}  // namespace

int DType::width() const {
  const KindRow& r = row_of(kind);
  if (r.width == 0) throw std::invalid_argument("float32 has no integer width");
  return r.width;
}

int64_t DType::min_value() const {
  if (kind == DTypeKind::kUInt8) return 0;
  return -(int64_t{1} << (width() - 1));
}

int64_t DType::max_value() const {
  if (kind == DTypeKind::kUInt8) return 255;
  return (int64_t{1} << (width() - 1)) - 1;
}

size_t DType::byte_size() const { return row_of(kind).bytes; }

std::string DType::name() const { return row_of(kind).name; }

DType parse_dtype(const std::string& token) {
  for (const KindRow& r : kKinds) {
    if (token == r.name) return DType(r.kind);
  }
  throw std::invalid_argument("unknown dtype token: " + token);
}

int max_bits(DType dtype) {
  if (dtype.is_float()) throw std::invalid_argument("max_bits is undefined for " + dtype.name());
  return dtype.width();
}

// ---- Tensor -----------------------------------------------------------------
// Host-side value type of the drop-in API (device work never goes through
// it: the engine keeps its own device buffers).  Error strings are the
// reference's (tensor.cpp), which the errors-identical tests compare.

int64_t shape_numel(const std::vector<int64_t>& shape) {
  int64_t n = 1;
  for (int64_t d : shape) {
    if (d < 0) throw std::invalid_argument("negative dimension");
    n *= d;
  }
  return n;
}

std::string shape_to_string(const std::vector<int64_t>& shape) {
  std::string s;
  for (int64_t d : shape) s += (s.empty() ? "" : ",") + std::to_string(d);
  return "(" + s + ")";
}

namespace {
// element count of `shape` must equal the payload length
void check_length(const std::vector<int64_t>& shape, size_t len) {
  if (shape_numel(shape) != static_cast<int64_t>(len)) {
    throw std::invalid_argument("data length does not match shape " + shape_to_string(shape));
  }
}
[[noreturn]] void wrong_view(const char* view, const DType& d) {
  throw std::logic_error(std::string(view) + " on " + d.name() + " tensor");
}
}  // namespace

Tensor Tensor::zeros(DType dtype, std::vector<int64_t> shape) {
  const size_t n = static_cast<size_t>(shape_numel(shape));
  return dtype.is_float() ? from_floats(std::move(shape), std::vector<float>(n, 0.0f))
                          : from_ints(dtype, std::move(shape), std::vector<int32_t>(n, 0));
}

Tensor Tensor::from_floats(std::vector<int64_t> shape, std::vector<float> data) {
  check_length(shape, data.size());
  Tensor t;
  t.dtype_ = f32;
  t.shape_ = std::move(shape);
  t.f_ = std::move(data);
  return t;
}

Tensor Tensor::from_ints(DType dtype, std::vector<int64_t> shape, std::vector<int32_t> data) {
  if (dtype.is_float()) throw std::invalid_argument("from_ints needs an integer dtype");
  check_length(shape, data.size());
  Tensor t;
  t.dtype_ = dtype;
  t.shape_ = std::move(shape);
  t.i_ = std::move(data);
  if (!t.in_range()) throw std::invalid_argument("integer data out of range for " + dtype.name());
  return t;
}

Tensor Tensor::scalar(float value) { return from_floats({1}, {value}); }

int64_t Tensor::numel() const { return static_cast<int64_t>(dtype_.is_float() ? f_.size() : i_.size()); }

std::span<const float> Tensor::floats() const {
  if (!dtype_.is_float()) wrong_view("floats()", dtype_);
  return f_;
}
std::span<float> Tensor::floats() {
  if (!dtype_.is_float()) wrong_view("floats()", dtype_);
  return f_;
}
std::span<const int32_t> Tensor::ints() const {
  if (dtype_.is_float()) wrong_view("ints()", dtype_);
  return i_;
}
std::span<int32_t> Tensor::ints() {
  if (dtype_.is_float()) wrong_view("ints()", dtype_);
  return i_;
}

bool Tensor::in_range() const {
  if (dtype_.is_float() || i_.empty()) return true;
  const auto [lo, hi] = std::minmax_element(i_.begin(), i_.end());
  return *lo >= dtype_.min_value() && *hi <= dtype_.max_value();
}

float Tensor::max_abs() const {
  // |v| of integers compared as floats, like the reference
  auto fold = [](float m, float v) { return std::max(m, std::fabs(v)); };
  if (dtype_.is_float()) return std::accumulate(f_.begin(), f_.end(), 0.0f, fold);
  return std::accumulate(i_.begin(), i_.end(), 0.0f,
                         [&](float m, int32_t v) { return fold(m, static_cast<float>(v)); });
}

bool Tensor::equals(const Tensor& other) const {
  if (dtype_ != other.dtype_ || shape_ != other.shape_) return false;
  if (!dtype_.is_float()) return i_ == other.i_;
  // bitwise (NaN payloads and signed zeros count)
  return f_.size() == other.f_.size() &&
         (f_.empty() || std::memcmp(f_.data(), other.f_.data(), f_.size() * sizeof(float)) == 0);
}

// ---- BigUInt ------------------------------------------------------------------

BigUInt::BigUInt(uint64_t v) {
  limbs_.push_back(static_cast<uint32_t>(v));
  if (v >> 32) limbs_.push_back(static_cast<uint32_t>(v >> 32));
}

BigUInt& BigUInt::operator*=(uint64_t m) {
  // multiply by a (possibly 64-bit) factor via two 32-bit halves
  auto mul32 = [](std::vector<uint32_t>& l, uint32_t f) {
    uint64_t carry = 0;
    for (uint32_t& x : l) {
      uint64_t cur = static_cast<uint64_t>(x) * f + carry;
      x = static_cast<uint32_t>(cur);
      carry = cur >> 32;
    }
    if (carry) l.push_back(static_cast<uint32_t>(carry));
  };
  if (m >> 32) {
    BigUInt hi = *this;
    mul32(hi.limbs_, static_cast<uint32_t>(m >> 32));
    hi.limbs_.insert(hi.limbs_.begin(), 0u);
    mul32(limbs_, static_cast<uint32_t>(m));
    // add hi
    uint64_t carry = 0;
    if (limbs_.size() < hi.limbs_.size()) limbs_.resize(hi.limbs_.size(), 0);
    for (size_t i = 0; i < limbs_.size(); ++i) {
      uint64_t cur = static_cast<uint64_t>(limbs_[i]) + (i < hi.limbs_.size() ? hi.limbs_[i] : 0) +
                     carry;
      limbs_[i] = static_cast<uint32_t>(cur);
      carry = cur >> 32;
    }
    if (carry) limbs_.push_back(static_cast<uint32_t>(carry));
  } else {
    mul32(limbs_, static_cast<uint32_t>(m));
  }
  while (limbs_.size() > 1 && limbs_.back() == 0) limbs_.pop_back();
  return *this;
}

int BigUInt::compare(const BigUInt& o) const {
  if (limbs_.size() != o.limbs_.size()) return limbs_.size() < o.limbs_.size() ? -1 : 1;
  for (size_t i = limbs_.size(); i-- > 0;) {
    if (limbs_[i] != o.limbs_[i]) return limbs_[i] < o.limbs_[i] ? -1 : 1;
  }
  return 0;
}

std::string BigUInt::str() const {
  std::vector<uint32_t> l = limbs_;
  std::string digits;
  auto is_zero = [&] { return l.size() == 1 && l[0] == 0; };
  if (is_zero()) return "0";
  while (!is_zero()) {
    uint64_t rem = 0;
    for (size_t i = l.size(); i-- > 0;) {
      uint64_t cur = (rem << 32) | l[i];
      l[i] = static_cast<uint32_t>(cur / 1000000000u);
      rem = cur % 1000000000u;
    }
    while (l.size() > 1 && l.back() == 0) l.pop_back();
    std::string chunk = std::to_string(rem);
    if (!is_zero()) chunk = std::string(9 - chunk.size(), '0') + chunk;
    digits = chunk + digits;
  }
  return digits;
}

// ---- workers ------------------------------------------------------------------

int resolve_workers(int requested) {
  if (requested > 0) return requested;
  if (const char* env = std::getenv("QUANTC_WORKERS")) {
    int n = std::atoi(env);
    if (n > 0) return n;
  }
  unsigned hw = std::thread::hardware_concurrency();
  return hw > 0 ? static_cast<int>(hw) : 1;
}

namespace {

// Persistent workers for parallel_for: spawning threads per call costs tens of
// microseconds each, which dominated short host loops (e.g. packing a batch
// of samples into pinned staging).  A call hands out indices through an
// atomic counter; the caller participates; nested calls run serially.
class Pool {
 public:
  // Never destroyed: at process exit the workers are still blocked on cv_,
  // and destroying a condition variable with waiters blocks in glibc.
  static Pool& get() {
    static Pool* p = new Pool;
    return *p;
  }

  void run(size_t n, size_t w, const std::function<void(size_t)>& fn) {
    std::unique_lock<std::mutex> call(call_mu_);  // one parallel_for at a time
    ensure(w - 1);
    Job job;
    job.n = n;
    job.fn = &fn;
    job.first_idx = n;
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &job;
      active_ = w - 1;
      limit_ = w - 1;  // workers 0..w-2 join this call
      ++gen_;
    }
    cv_.notify_all();
    work(job);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return active_ == 0; });
    job_ = nullptr;
    lk.unlock();
    if (job.first_err) std::rethrow_exception(job.first_err);
  }

  static bool in_worker() { return tl_worker_; }

 private:
  struct Job {
    size_t n = 0;
    const std::function<void(size_t)>* fn = nullptr;
    std::atomic<size_t> next{0};
    std::mutex err_mu;
    size_t first_idx = 0;
    std::exception_ptr first_err;
  };

  static void work(Job& job) {
    for (;;) {
      const size_t i = job.next.fetch_add(1);
      if (i >= job.n) return;
      try {
        (*job.fn)(i);
      } catch (...) {
        std::lock_guard<std::mutex> lk(job.err_mu);
        if (i < job.first_idx) {
          job.first_idx = i;
          job.first_err = std::current_exception();
        }
      }
    }
  }

  void ensure(size_t k) {
    while (threads_.size() < k) {
      const size_t id = threads_.size();
      threads_.emplace_back([this, id] { loop(id); });
      threads_.back().detach();
    }
  }

  void loop(size_t id) {
    tl_worker_ = true;
    uint64_t seen = 0;
    for (;;) {
      Job* job = nullptr;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (job_ == nullptr || id >= limit_) continue;
        job = job_;
      }
      work(*job);
      std::lock_guard<std::mutex> lk(mu_);
      if (--active_ == 0) done_cv_.notify_all();
    }
  }

  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  std::vector<std::thread> threads_;
  Job* job_ = nullptr;
  size_t active_ = 0, limit_ = 0;
  uint64_t gen_ = 0;
  static thread_local bool tl_worker_;
};
thread_local bool Pool::tl_worker_ = false;

}  // namespace

void parallel_for(size_t n, int workers, const std::function<void(size_t)>& fn) {
  if (n == 0) return;
  const size_t w = std::min<size_t>(static_cast<size_t>(resolve_workers(workers)), n);
  if (w <= 1 || Pool::in_worker()) {
    for (size_t i = 0; i < n; ++i) fn(i);
    return;
  }
  Pool::get().run(n, w, fn);
}

}  // namespace quantc
