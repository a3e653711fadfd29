// fastplan.cpp — compiler + executor of the fused int8 dataflow (engine v2).
#include "fastplan.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <numeric>
#include <set>

#include "quantc/device.hpp"
#include "quantc/simulate.hpp"

namespace quantc::fast {

using kern::FSq;
using kern::ProgArgs;
using kern::ProgBuf;
using kern::ProgInstr;

namespace {
cudaStream_t S() { return static_cast<cudaStream_t>(device::stream()); }
// inside FastPlan members: the instance's stream
#define ST() static_cast<cudaStream_t>(stream_ ? stream_ : device::stream())
void ok_cuda(cudaError_t e) {
  if (e != cudaSuccess) throw DeviceError(std::string("fastplan: ") + cudaGetErrorString(e));
}
int r16(int c) { return (c + 15) / 16 * 16; }

struct Attr2 {
  int a, b;
};
Attr2 pair_of(const Node& n, const char* key, Attr2 d) {
  if (!n.has_attr(key)) return d;
  auto v = n.attr<std::vector<int64_t>>(key);
  return {static_cast<int>(v[0]), static_cast<int>(v[1])};
}

bool is_pow2(double t) {
  if (!(t > 0.0) || !std::isfinite(t)) return false;
  int e = 0;
  return std::frexp(t, &e) == 0.5;
}
}  // namespace

struct FastPlan::Val {
  int step = -1;        // node whose value is stored
  int sq_step = -1;     // sq that produced the codes (kind 0)
  int kind = 0;         // 0 int8 codes, 1 fp32
  int64_t rows_ps = 0;  // rows per sample in the (m, n) space
  int C = 0;
  int hw = 1, cs = 0;
  int64_t ld = 0;
  bool zero_fill = false;
  // a column slice of another fp32 value (a concat input writing into the
  // concat's buffer): no storage of its own, columns [col_off, col_off + C)
  int alias_root = -1;
  int64_t col_off = 0;
  // space-to-depth layout of a tiny-channel graph input feeding a stride-2
  // conv: pixel (h, w, c) of an [H, W, C] image lives at s2d pixel
  // (h/2, w/2), channel ((h%2)*2 + w%2)*C + c, 16-byte rows
  bool s2d = false;
  int s2d_C = 0, s2d_H = 0, s2d_W = 0;
  int64_t bytes_ps() const {
    return (rows_ps / hw) * ld * (kind == 0 ? 1 : 4);
  }
};

struct FastPlan::Stage {
  enum Kind { kInput, kGemm, kMaxpool, kGap, kDw, kAvg, kCat } kind = kInput;
  int step = -1;
  int code_off = 0, code_len = 0;
  int in_val = -1;
  // input
  int input_k = 0, n0 = 1, C = 0, HW = 1;
  // gemm
  bool dense = false, gather = false, packed = false;
  int w_sq = -1, w_const = -1, bias_const = -1;
  int O = 0, KH = 1, KW = 1, sh = 1, sw = 1, ph = 0, pw = 0, H = 1, W = 1, OH = 1, OW = 1;
  int taps = 1, ldk = 0, Ktrue = 0, Kpad = 0;
  int64_t rows_out_ps = 0;
  // pool
  int pkh = 1, pkw = 1;
  // program with stage-local indices (see kern::StageTables)
  std::vector<ProgInstr> code;
  std::vector<int> sq_slots;  // local sq index -> global FSq slot
  std::vector<int> buf_vals;  // local buf index -> Val id
  std::vector<int> clips;     // local clip index -> global clip id
  int depth = 0;
  // GEMM epilogue smem slots (kern::ProgBuf::slot) per local buffer
  std::vector<int> buf_slot;
  int n_out = 0;
  int out_vals[2] = {-1, -1};
  int res_val = -1;
  double bias_absmax = 0.0;
  double bias_absmin = std::numeric_limits<double>::infinity();  // smallest nonzero |bias|
  // space-to-depth stem conv (see Val::s2d): original channels / kernel and
  // the tap alignment shift
  bool s2d = false;
  int s2d_C = 0, s2d_KH = 0, s2d_KW = 0, s2d_dh = 0, s2d_dw = 0;
};

namespace {

double code_absmax(const FSq& f) {
  return std::max(std::fabs(static_cast<double>(f.qmin) - f.zp),
                  std::fabs(static_cast<double>(f.qmax) - f.zp));
}

// a CUDA-core stage whose program is [passthrough accumulator sq,] sq_store8
// into plain code rows runs it inline (kern::DwFast) instead of through the
// table interpreter (whose registers cut the kernel's occupancy ~3x)
kern::DwFast inline_store_program(const kern::StageTables& t) {
  static const bool off = std::getenv("QUANTC_NO_DW_FAST") != nullptr;
  kern::DwFast fast{};
  const int k = t.n_code - 1;
  if (off || (t.n_code != 1 && t.n_code != 2) || t.code[k].op != kern::kPSqStore8 ||
      t.buf[t.code[k].b].kind != 0 || t.buf[t.code[k].b].hw != 1) {
    return fast;
  }
  if (t.n_code == 2) {
    if (t.code[0].op != kern::kPSq || !t.sq[t.code[0].a].passthrough) return fast;
    fast.fa = t.sq[t.code[0].a];
  }
  fast.n = t.n_code;
  fast.fs = t.sq[t.code[k].a];
  fast.buf = t.buf[t.code[k].b];
  return fast;
}

bool no_acc_shape() {
  static const bool off = std::getenv("QUANTC_NO_ACC_SHAPE") != nullptr;
  return off;
}

bool no_clip_fold() {
  static const bool off = std::getenv("QUANTC_NO_CLIP_FOLD") != nullptr;
  return off;
}

// Per-run table optimisation of one stage (observable results unchanged):
//  * interval analysis of |v| along the program; an accumulator clamp that
//    the bound proves can never fire is dropped (has_acc = 0);
//  * sq -> relu folds into the code clamp: relu((q-zp)*s) == (max(q,zp)-zp)*s.
// `v0` bounds the stage's produced value before the program.
void optimise_tables(kern::StageTables& t, double v0) {
  std::vector<double> stack;
  double b = v0;
  std::vector<kern::ProgInstr> out;
  for (int pc = 0; pc < t.n_code; ++pc) {
    kern::ProgInstr ins = t.code[pc];
    switch (ins.op) {
      case kern::kPSq:
      case kern::kPSqStore8: {
        FSq& f = t.sq[ins.a];
        if (f.has_acc && std::isfinite(b) && -b * 1.001 > static_cast<double>(f.lo_up) &&
            b * 1.001 < static_cast<double>(f.hi_dn)) {
          f.has_acc = 0;
        }
        if (f.has_acc) {
          b = std::min(b, std::max(std::fabs(static_cast<double>(f.lo_rn)),
                                   std::fabs(static_cast<double>(f.hi_rn))) * 1.001);
        }
        if (!f.passthrough) b = code_absmax(f) * static_cast<double>(f.s);
        // a passthrough sq without a live accumulator clamp is the identity
        if (ins.op == kern::kPSq && f.passthrough && !f.has_acc) continue;
        // a passthrough accumulator clamp followed by a clip whose bounds lie
        // inside the saturation range is absorbed by the clip (v < lo_up <= a
        // gives clip(lo_rn) = a = clip(v); symmetric above): e.g. MobileNetV2's
        // int16 accumulator sq before relu6
        if (ins.op == kern::kPSq && f.passthrough && f.has_acc && !no_clip_fold() && pc + 1 < t.n_code &&
            t.code[pc + 1].op == kern::kPClip) {
          const float2 c = t.clip[t.code[pc + 1].a];
          if (f.lo_up <= c.x && f.lo_rn <= c.x && f.hi_dn >= c.y && f.hi_rn >= c.y) continue;
        }
        const bool relu_next = pc + 1 < t.n_code && t.code[pc + 1].op == kern::kPRelu;
        if (ins.op == kern::kPSq && relu_next && !f.passthrough) {
          f.qmin = std::max(f.qmin, f.zp);
          f.q_lo = std::max(f.q_lo, f.zp);
          f.q_hi = std::max(f.q_hi, f.zp);
          out.push_back(ins);
          ++pc;  // relu folded
          continue;
        }
        // sq -> clip(lo, hi) (e.g. relu6) folds into the code clamp when both
        // bounds sit on the sq's grid: clip((q-zp)*s, lo, hi) ==
        // (clamp(q, zp + lo/s, zp + hi/s) - zp)*s for integral lo/s, hi/s
        const bool clip_next = pc + 1 < t.n_code && t.code[pc + 1].op == kern::kPClip;
        if (ins.op == kern::kPSq && clip_next && !f.passthrough && !no_clip_fold()) {
          const float2 c = t.clip[t.code[pc + 1].a];
          const double ql = static_cast<double>(c.x) / f.s, qh = static_cast<double>(c.y) / f.s;
          if (std::isfinite(ql) && std::isfinite(qh) && ql == std::floor(ql) && qh == std::floor(qh) &&
              ql <= qh && std::fabs(ql) < 1e6 && std::fabs(qh) < 1e6) {
            const float lo = static_cast<float>(f.zp + ql), hi = static_cast<float>(f.zp + qh);
            f.qmin = std::min(std::max(f.qmin, lo), hi);
            f.qmax = std::max(std::min(f.qmax, hi), lo);
            f.q_lo = std::min(std::max(f.q_lo, lo), hi);
            f.q_hi = std::min(std::max(f.q_hi, lo), hi);
            b = std::min(b, std::max(std::fabs(static_cast<double>(c.x)), std::fabs(static_cast<double>(c.y))));
            out.push_back(ins);
            ++pc;  // clip folded
            continue;
          }
        }
        break;
      }
      case kern::kPClip: {
        const float2 c = t.clip[ins.a];
        b = std::min(b, std::max(std::fabs(static_cast<double>(c.x)), std::fabs(static_cast<double>(c.y))));
        // clip(a, b) -> sq folds into the sq's code clamp when a/s and b/s
        // are integers: round is monotonic and both bounds are grid points
        if (pc + 1 < t.n_code && !no_clip_fold() &&
            (t.code[pc + 1].op == kern::kPSq || t.code[pc + 1].op == kern::kPSqStore8)) {
          FSq& f = t.sq[t.code[pc + 1].a];
          const double ql = static_cast<double>(c.x) / f.s, qh = static_cast<double>(c.y) / f.s;
          if (!f.passthrough && !f.has_acc && std::isfinite(ql) && std::isfinite(qh) &&
              ql == std::floor(ql) && qh == std::floor(qh) && ql <= qh && std::fabs(ql) < 1e6 &&
              std::fabs(qh) < 1e6) {
            const float lo = static_cast<float>(f.zp + ql), hi = static_cast<float>(f.zp + qh);
            f.qmin = std::min(std::max(f.qmin, lo), hi);
            f.qmax = std::max(std::min(f.qmax, hi), lo);
            continue;  // clip folded into the next sq
          }
        }
        break;
      }
      case kern::kPAdd: {
        const kern::ProgBuf& pb = t.buf[ins.b];
        b = pb.kind == 0 ? b + 128.0 * static_cast<double>(pb.scale)
                         : std::numeric_limits<double>::infinity();
        break;
      }
      case kern::kPPush:
        stack.push_back(b);
        break;
      case kern::kPPop:
        b = stack.back();
        stack.pop_back();
        break;
      default:
        break;
    }
    out.push_back(ins);
  }
  t.n_code = static_cast<int32_t>(out.size());
  std::copy(out.begin(), out.end(), t.code);
}

}  // namespace

namespace {

// per-element program builder
struct Builder {
  const engine::Plan& plan;
  std::vector<ProgInstr>& code;
  std::map<int, int>& sq_index;
  std::vector<int>& sq_steps;
  std::vector<float>& clip_lo;
  std::vector<float>& clip_hi;
  std::vector<std::unique_ptr<FastPlan::Val>>& vals;
  std::map<int, int>& val_of;  // materialised step -> val index
  std::set<int>& absorbed;
  std::function<void(const std::string&)> fail;
  // current register value space
  int64_t rows_ps = 0;
  int C = 0;
  int flat_hw = 1, flat_cs = 0;
  int depth = 0;
  int max_depth = 0;
  int* out_val = nullptr;
  int64_t* out_per_sample = nullptr;
  // set by compile() for a graph-input stage: its step and image geometry
  int input_step = -1;
  int input_H = 0, input_W = 0;

  const Graph& g() const { return plan.graph(); }
  const Node& node(int step) const { return *plan.steps()[static_cast<size_t>(step)].node; }

  std::vector<std::pair<int, int>> consumers(int step) const {
    std::vector<std::pair<int, int>> out;
    for (const Edge* e : g().out_edges(node(step).id)) {
      out.push_back({plan.step_of(e->dst.node), e->dst.port});
    }
    return out;
  }
  // conv2d step with groups == C_in == O and weights [O, 1, KH, KW]
  bool depthwise(int step) const {
    const Node& n = node(step);
    if (n.op != OpKind::kConv2d) return false;
    const auto& st = plan.steps()[static_cast<size_t>(step)];
    if (st.in.size() < 2 || st.in[0] < 0 || st.in[1] < 0) return false;
    const auto& ds = plan.shape(st.in[0]);
    const auto& ws = plan.shape(st.in[1]);
    const int64_t groups = n.attr_or<int64_t>("groups", 1);
    return ds.size() == 4 && ws.size() == 4 && groups > 1 && groups == ds[1] && ws[0] == groups &&
           ws[1] == 1 && ws[2] * ws[3] <= 1024;
  }
  // concat step x feeding another concat (its sole consumer, not an output):
  // that concat's step and the port x occupies, else -1
  std::pair<int, int> concat_outer(int x) const {
    const auto cs = consumers(x);
    if (cs.size() == 1 && !is_output(x) && node(cs[0].first).op == OpKind::kConcat) return cs[0];
    return {-1, -1};
  }
  // channel offset of input `port` of concat step x, within x
  int64_t concat_port_off(int x, int port) const {
    const auto& in = plan.steps()[static_cast<size_t>(x)].in;
    int64_t off = 0;
    for (int p = 0; p < port; ++p) off += plan.shape(in[static_cast<size_t>(p)])[1];
    return off;
  }
  // the outermost concat's buffer (fp32, created when its first input lands)
  // and the column slice of input `port` of concat x inside it
  std::map<int, int>* concat_root_val = nullptr;
  int concat_slice(int x, int port) {
    int64_t off = concat_port_off(x, port);
    int root = x;
    for (auto o = concat_outer(root); o.first >= 0; o = concat_outer(root)) {
      off += concat_port_off(o.first, o.second);
      root = o.first;
    }
    const auto& rshape = plan.shape(root);
    if (rshape.size() != 4) {
      fail("concat of non-4-D values");
      return -1;
    }
    const int C_total = static_cast<int>(rshape[1]);
    auto it = concat_root_val->find(root);
    if (it == concat_root_val->end()) {
      const int keepC = C;
      C = C_total;
      const int v = make_val(root, -1, 1, C_total, 1, 0, false);
      C = keepC;
      it = concat_root_val->emplace(root, v).first;
    }
    const int rv = it->second;
    if (vals[static_cast<size_t>(rv)]->rows_ps != rows_ps) {
      fail("concat inputs with different row spaces");
      return -1;
    }
    // (not registered in val_of: step x's own value is the concat, not a slice)
    auto v = std::make_unique<FastPlan::Val>();
    v->step = x;
    v->kind = 1;
    v->rows_ps = rows_ps;
    v->C = C;
    v->ld = C_total;
    v->alias_root = rv;
    v->col_off = off;
    vals.push_back(std::move(v));
    return static_cast<int>(vals.size()) - 1;
  }
  bool is_output(int step) const {
    for (const PortRef& o : g().outputs()) {
      if (o.node == node(step).id) return true;
    }
    return false;
  }
  int sq_slot(int step) {
    auto it = sq_index.find(step);
    if (it != sq_index.end()) return it->second;
    const int s = static_cast<int>(sq_steps.size());
    sq_index[step] = s;
    sq_steps.push_back(step);
    return s;
  }
  void op(uint8_t k, int a = 0, int b = 0) {
    code.push_back(ProgInstr{k, 0, static_cast<uint16_t>(a), static_cast<uint32_t>(b)});
  }
  int make_val(int step, int sq_step, int kind, int64_t ld, int hw, int cs, bool zero) {
    auto v = std::make_unique<FastPlan::Val>();
    v->step = step;
    v->sq_step = sq_step;
    v->kind = kind;
    v->rows_ps = rows_ps;
    v->C = C;
    v->hw = hw;
    v->cs = cs;
    v->ld = ld;
    v->zero_fill = zero;
    vals.push_back(std::move(v));
    const int id = static_cast<int>(vals.size()) - 1;
    val_of[step] = id;
    return id;
  }

  // layout for the codes of sq `x` consumed by step `y` at `port`
  bool codes_for(int x, int y, int port) {
    const Node& ny = node(y);
    int64_t ld = r16(C);
    int hw = 1, cs = 0;
    bool zero = false;
    switch (ny.op) {
      case OpKind::kConv2d: {
        if (ny.attr_or<int64_t>("groups", 1) != 1) {
          // depthwise (groups == C == O): CUDA-core stage over NHWC codes
          if (!depthwise(y) || port != 0 || flat_hw != 1) {
            fail("grouped conv2d (other than depthwise) runs on the exact engine");
            return false;
          }
          ld = r16(C);
          zero = ld != C;
          break;
        }
        if (port != 0) {
          fail("conv2d weight is not a constant");
          return false;
        }
        if (flat_hw != 1) {
          fail("conv2d after flatten");
          return false;
        }
        const auto& ws = plan.shape(plan.steps()[static_cast<size_t>(y)].in[1]);
        Attr2 st = pair_of(ny, "strides", {1, 1}), pd = pair_of(ny, "padding", {0, 0});
        const bool direct = ws[2] == 1 && ws[3] == 1 && st.a == 1 && st.b == 1 && pd.a == 0 &&
                            pd.b == 0 && C % 16 == 0;
        ld = direct ? C : r16(C);
        zero = ld != C;
        // the RGB stem: a graph input quantized straight into a stride-2 KxK
        // conv with <= 4 channels is stored space-to-depth, making the conv a
        // stride-1 conv over 16-byte pixels (one gather chunk per tap)
        if (input_step >= 0 && C <= 4 && st.a == 2 && st.b == 2 && ws[2] > 1 && ws[3] > 1 &&
            consumers(input_step).size() == 1 && consumers(x).size() == 1 && rows_ps > 0 &&
            !std::getenv("QUANTC_NO_S2D")) {
          const int H2 = (input_H + 1) / 2, W2 = (input_W + 1) / 2;
          const int64_t n0 = rows_ps / (static_cast<int64_t>(input_H) * input_W);
          const int64_t keep_rows = rows_ps;
          rows_ps = n0 * H2 * W2;
          const int v = make_val(x, x, 0, 16, 1, 0, true);
          rows_ps = keep_rows;
          FastPlan::Val& val = *vals[static_cast<size_t>(v)];
          val.s2d = true;
          val.s2d_C = C;
          val.s2d_H = input_H;
          val.s2d_W = input_W;
          op(kern::kPSqStore8, sq_slot(x), v);
          return true;
        }
        break;
      }
      case OpKind::kDense:
        if (port != 0) {
          fail("dense weight is not a constant");
          return false;
        }
        if (flat_hw > 1) {
          hw = flat_hw;
          cs = flat_cs;
          ld = static_cast<int64_t>(flat_hw) * flat_cs;
        } else {
          ld = C;
        }
        if (ld % 16 != 0) {
          fail("dense reduction not a multiple of 16 bytes");
          return false;
        }
        break;
      case OpKind::kMaxPool2d:
      case OpKind::kAdd:
        if (flat_hw != 1) {
          fail("pool/add after flatten");
          return false;
        }
        break;
      default:
        fail("unsupported consumer of a quantized edge: " + op_name(ny.op));
        return false;
    }
    op(kern::kPSqStore8, sq_slot(x), make_val(x, x, 0, ld, hw, cs, zero));
    return true;
  }

  void store_f32(int step, bool output) {
    if (flat_hw != 1 && !output) {
      fail("fp32 materialisation after flatten");
      return;
    }
    const int v = make_val(step, -1, 1, C, 1, 0, false);
    op(kern::kPStoreF32, 0, v);
    if (output) {
      // argmax runs over the per-sample tensor in reference (NCHW) order:
      // identical to NHWC only when there is one pixel per row
      const auto& shp = plan.shape(step);
      int64_t pix = 1;
      for (size_t i = 2; i < shp.size(); ++i) pix *= shp[i];
      if (pix != 1 && C != 1) fail("4-D graph output with H*W > 1");
      *out_val = v;
      *out_per_sample = rows_ps * C;
    }
  }

  // u's value is in the register
  void emit(int u) {
    auto cons = consumers(u);
    const bool out = is_output(u);
    const size_t n = cons.size() + (out ? 1 : 0);
    for (size_t i = 0; i < n; ++i) {
      const bool branch = i + 1 < n;
      if (branch) {
        if (++depth > 3) {
          fail("fan-out deeper than the program stack");
          return;
        }
        max_depth = std::max(max_depth, depth);
        op(kern::kPPush);
      }
      if (i < cons.size()) {
        handle(u, cons[i].first, cons[i].second);
      } else {
        store_f32(u, true);
      }
      if (branch) {
        op(kern::kPPop);
        --depth;
      }
    }
  }

  // consumer x of the register value u
  void handle(int u, int x, int port) {
    const Node& nx = node(x);
    switch (nx.op) {
      case OpKind::kSimulatedQuantize: {
        absorbed.insert(x);
        auto cy = consumers(x);
        if (cy.empty()) {
          op(kern::kPSq, sq_slot(x));
          if (is_output(x)) store_f32(x, true);
          return;
        }
        if (cy.size() > 1 || is_output(x)) {
          fail("simulated_quantize with several consumers");
          return;
        }
        const int y = cy[0].first;
        const Node& ny = node(y);
        switch (ny.op) {
          case OpKind::kRelu:
          case OpKind::kClip:
          case OpKind::kFlatten:
            op(kern::kPSq, sq_slot(x));
            handle(x, y, cy[0].second);
            return;
          case OpKind::kAdd: {
            if (nx.attr_or<bool>("boundary", false)) {
              // a boundary sq is always a passthrough (fp32 out): fp32 add
              op(kern::kPSq, sq_slot(x));
              handle(x, y, cy[0].second);
              return;
            }
            const auto& yin = plan.steps()[static_cast<size_t>(y)].in;
            const int other = yin[static_cast<size_t>(1 - cy[0].second)];
            auto it = val_of.find(other);
            if (it != val_of.end()) {
              op(kern::kPSq, sq_slot(x));
              op(kern::kPAdd, 0, it->second);
              absorbed.insert(y);
              emit(y);
            } else {
              codes_for(x, y, cy[0].second);
            }
            return;
          }
          case OpKind::kGlobalAvgPool2d:
            op(kern::kPSq, sq_slot(x));
            store_f32(x, false);
            return;
          case OpKind::kConcat:
            op(kern::kPSq, sq_slot(x));
            handle(x, y, cy[0].second);
            return;
          case OpKind::kAvgPool2d:
            // float-only op (its input edge is a passthrough in every
            // binding Algorithm 1 allows): the sq's fp32 value, pooled by
            // an avg stage with the exact engine's double arithmetic
            op(kern::kPSq, sq_slot(x));
            store_f32(x, false);
            return;
          default:
            codes_for(x, y, cy[0].second);
            return;
        }
      }
      case OpKind::kRelu:
        absorbed.insert(x);
        op(kern::kPRelu);
        emit(x);
        return;
      case OpKind::kClip: {
        absorbed.insert(x);
        if (!nx.has_attr("a_min")) {
          fail("integer clip in the fp32 graph");
          return;
        }
        clip_lo.push_back(static_cast<float>(nx.attr<double>("a_min")));
        clip_hi.push_back(static_cast<float>(nx.attr<double>("a_max")));
        op(kern::kPClip, static_cast<int>(clip_lo.size()) - 1);
        emit(x);
        return;
      }
      case OpKind::kFlatten: {
        absorbed.insert(x);
        if (flat_hw != 1) {
          fail("double flatten");
          return;
        }
        const auto& in_shape = plan.shape(plan.steps()[static_cast<size_t>(x)].in[0]);
        int64_t hw = 1;
        for (size_t i = 2; i < in_shape.size(); ++i) hw *= in_shape[i];
        flat_hw = static_cast<int>(hw);
        flat_cs = C;
        emit(x);
        flat_hw = 1;
        flat_cs = 0;
        return;
      }
      case OpKind::kGlobalAvgPool2d:
        // an fp32 value pooled by a GAP stage (which reads it from rows)
        store_f32(u, false);
        return;
      case OpKind::kAvgPool2d: {
        // an fp32 value pooled by an avg stage; a concat's value already is
        // fp32 rows (the concat buffer the register was loaded from)
        if (flat_hw != 1) {
          fail("avg_pool2d after flatten");
          return;
        }
        auto it = val_of.find(u);
        if (it == val_of.end() || vals[static_cast<size_t>(it->second)]->kind != 1 ||
            vals[static_cast<size_t>(it->second)]->C != C) {
          store_f32(u, false);
        }
        return;
      }
      case OpKind::kConcat: {
        // channel placement: the value lands as fp32 in its column slice of
        // the (outermost) concat buffer; the concat's stage runs its
        // consumers over the whole buffer once every input has landed
        if (flat_hw != 1) {
          fail("concat after flatten");
          return;
        }
        const int sv = concat_slice(x, port);
        if (sv >= 0) op(kern::kPStoreF32, 0, sv);
        return;
      }
      case OpKind::kAdd: {
        // fp32 add (an add the spec does not quantize, e.g. arm_vmlal_like's
        // residuals): float + float like the reference (interpreter.cpp
        // add).  The first operand to arrive is materialised as fp32 rows;
        // the program of the second reads it and carries on with the sum.
        if (flat_hw != 1) {
          fail("add after flatten");
          return;
        }
        const auto& xin = plan.steps()[static_cast<size_t>(x)].in;
        const int other = xin[static_cast<size_t>(1 - port)];
        auto it = val_of.find(other);
        if (it != val_of.end()) {
          op(kern::kPAdd, 0, it->second);
          absorbed.insert(x);
          emit(x);
        } else {
          store_f32(u, false);
        }
        return;
      }
      default:
        fail("operator " + op_name(nx.op) + " consumes an unquantized value (port " +
             std::to_string(port) + ")");
        return;
    }
  }
};

FSq make_fsq(const QParams& p) {
  FSq f{};
  f.passthrough = p.passthrough ? 1 : 0;
  f.has_acc = p.acc_dtype.has_value() && p.acc_scale > 0.0;
  double s = 1.0, qmin = 0, qmax = 0, zp = 0;
  if (!p.passthrough) {
    s = compute_scale(p.threshold, p.bit, p.sign);
    QuantBounds b = quant_bounds(p.bit, p.sign);
    qmin = static_cast<double>(b.qmin);
    qmax = static_cast<double>(b.qmax);
    zp = static_cast<double>(p.zero_point);
  }
  f.s = static_cast<float>(s);
  f.inv_s = static_cast<float>(1.0 / s);
  f.qmin = static_cast<float>(qmin);
  f.qmax = static_cast<float>(qmax);
  f.zp = static_cast<float>(zp);
  if (f.has_acc) {
    const double lo = static_cast<double>(p.acc_dtype->min_value()) * p.acc_scale;
    const double hi = static_cast<double>(p.acc_dtype->max_value()) * p.acc_scale;
    float lu = static_cast<float>(lo);
    if (static_cast<double>(lu) < lo) lu = std::nextafter(lu, std::numeric_limits<float>::infinity());
    float hd = static_cast<float>(hi);
    if (static_cast<double>(hd) > hi) hd = std::nextafter(hd, -std::numeric_limits<float>::infinity());
    f.lo_up = lu;
    f.hi_dn = hd;
    f.lo_rn = static_cast<float>(lo);
    f.hi_rn = static_cast<float>(hi);
    if (!p.passthrough) {
      auto code = [&](double v) {
        double q = std::round(v / s) + zp;
        return static_cast<float>(std::clamp(q, qmin, qmax));
      };
      f.q_lo = code(lo);
      f.q_hi = code(hi);
    }
  }
  return f;
}

// straight-line epilogue shape of a GEMM stage program (fused.cuh kShape*)
// The shape kernels keep 4 sq parameters in registers and address all code
// I/O through tile slots, so they require: symmetric grids (zp = 0), no live
// accumulator clamp, no passthrough, slot-resident stores / add operand, and
// O % 16 == 0 (whole 16-column chunks).  Anything else runs the interpreter.
int classify_shape(const kern::StageTables& t, int O) {
  std::vector<uint8_t> ops;
  bool acc0 = false;  // the conv output's sq carries a live accumulator clamp
  bool pt0 = false;   // ... as a passthrough (a float edge's accumulator simulation)
  for (int i = 0; i < t.n_code; ++i) {
    const kern::ProgInstr& in = t.code[i];
    ops.push_back(in.op);
    if (in.op == kern::kPSq || in.op == kern::kPSqStore8) {
      const kern::FSq& f = t.sq[in.a];
      if (f.zp != 0.0f) return 0;
      if (f.passthrough) {
        if (i != 0 || in.op != kern::kPSq || !f.has_acc || no_acc_shape()) return 0;
        pt0 = acc0 = true;
        continue;
      }
      if (f.has_acc) {
        if (i != 0 || no_acc_shape()) return 0;
        acc0 = true;
      }
    }
    if ((in.op == kern::kPSqStore8 || in.op == kern::kPAdd) &&
        (t.buf[in.b].slot < 0 || t.buf[in.b].kind != 0)) {
      return 0;
    }
    if (in.op == kern::kPStoreF32 && (t.buf[in.b].kind != 1 || t.buf[in.b].hw != 1)) return 0;
  }
  using V = std::vector<uint8_t>;
  // fp32 scores (masked tail chunk): any O
  if ((ops == V{kern::kPSq, kern::kPStoreF32} || ops == V{kern::kPStoreF32}) && O % 4 == 0) {
    return kern::kShapeSqF32;
  }
  if (O % 16 != 0) return 0;
  if (acc0) {
    // [passthrough acc sq, sq_store8]: the clamp overrides the store's code
    if (pt0) return ops == V{kern::kPSq, kern::kPSqStore8} ? kern::kShapeStoreAcc : 0;
    if (ops == V{kern::kPSq, kern::kPSqStore8}) return kern::kShapeSqStoreAcc;
    if (ops == V{kern::kPSqStore8}) return kern::kShapeStoreAcc;
    return 0;
  }
  if (ops == V{kern::kPSqStore8}) return 1;
  if (ops == V{kern::kPSq, kern::kPSqStore8}) return 2;
  if (ops == V{kern::kPSq, kern::kPAdd, kern::kPSq, kern::kPPush, kern::kPSqStore8, kern::kPPop,
               kern::kPSqStore8}) {
    return 3;
  }
  if (ops == V{kern::kPSq, kern::kPAdd, kern::kPSq, kern::kPSqStore8}) return 4;
  if (ops == V{kern::kPSq, kern::kPAdd, kern::kPSq, kern::kPStoreF32}) return 5;
  return 0;
}

// v as an exactly representable normal float
bool exact_float(double v, float& out) {
  out = static_cast<float>(v);
  return static_cast<double>(out) == v && (v == 0.0 || std::fpclassify(out) == FP_NORMAL);
}

// rounding bounds of sq f: x clamped to the nearest floats inside
// [qmin - 1/2, qmax + 1/2] rounds (half away) into [qmin, qmax]
bool round_bounds(const kern::FSq& f, kern::EpiSq& q) {
  q.lo = std::nextafter(f.qmin - 0.5f, std::numeric_limits<float>::infinity());
  q.hi = std::nextafter(f.qmax + 0.5f, -std::numeric_limits<float>::infinity());
  return std::fabs(f.qmin) < 65536.0f && std::fabs(f.qmax) < 65536.0f;
}

// sq f applied to a previous integer code R on grid prev_s (T-domain when
// prev_T): x = fma(R, s_prev/s, off); k >= 1 needs no rounding (kEpiExact)
bool epi_from_code(double prev_s, bool prev_T, const kern::FSq& f, kern::EpiSq& q,
                   double in_lo, double in_hi) {
  const double M = kern::kMagic;
  const double k = prev_s / f.s;
  if (!exact_float(k, q.k)) return false;
  const bool nonneg = f.qmin >= 0.0f || prev_T;
  q.flags = nonneg ? kern::kEpiNonneg : 0;
  double off = 0.0;
  if (k >= 1.0) {
    // r * 2^d is already an integer: clamp in the output domain only
    q.flags |= kern::kEpiExact;
    if (nonneg) {
      off = prev_T ? M - M * k : M;
      q.lo = static_cast<float>(M + f.qmin);
      q.hi = static_cast<float>(M + f.qmax);
    } else {
      q.lo = f.qmin;
      q.hi = f.qmax;
    }
    // the input codes span [in_lo, in_hi]: scaled, they may already fit
    if (k * in_lo >= f.qmin && k * in_hi <= f.qmax) q.flags |= kern::kEpiNoClamp;
  } else {
    off = prev_T ? -M * k : 0.0;
    if (!round_bounds(f, q)) return false;
  }
  return exact_float(off, q.off);
}

// Saturating form of shapes 6/7 (fused.cuh run_shape_epi): sq i's input is
// pre-scaled by 1/P_i (P_i a power of two, code range [-P_i, P_i - 1] for a
// signed sq0 of shape 7, [0, P_i - 1] otherwise), so that add.rz.sat clamps
// the low side and one min caps the high side.  Scaling by a power of two
// commutes with RN / RZ rounding for normal floats, so every folded constant
// must stay an exact normal float, and so must the smallest nonzero bias
// term bias / s0 / P0.  Returns false when the shape must fall back.
bool fold_saturating(int shape, double bias_absmin, kern::EpiConsts& e) {
  auto code_range = [](const kern::EpiSq& q, double& lo, double& hi) {
    lo = std::nearbyint(static_cast<double>(q.lo) + 0.5);
    hi = std::nearbyint(static_cast<double>(q.hi) - 0.5);
  };
  auto pow2 = [](double v) { return v >= 1.0 && std::exp2(std::round(std::log2(v))) == v; };
  auto scaled = [](float& v, double p) {
    float out;
    if (!exact_float(static_cast<double>(v) / p, out)) return false;
    v = out;
    return true;
  };
  const double M = kern::kMagic;
  kern::EpiConsts f = e;
  double lo0, hi0;
  code_range(f.q[0], lo0, hi0);
  const bool signed0 = shape == kern::kShapeAddForkId;
  const double P0 = signed0 ? -lo0 : hi0 + 1.0;
  if (!pow2(P0) || hi0 != P0 - 1.0 || lo0 != (signed0 ? -P0 : 0.0)) return false;
  if (!scaled(f.q[0].k, P0) || !scaled(f.inv0, P0)) return false;
  // the bias table entries bias * inv0 / P0 must stay normal floats
  if (std::isfinite(bias_absmin) && bias_absmin * static_cast<double>(f.inv0) < 0x1p-125) {
    return false;
  }
  f.sat_half[0] = static_cast<float>(0.5 / P0);
  f.sat_p[0] = static_cast<float>(P0);
  f.sat_top[0] = static_cast<float>(signed0 ? P0 - 1.0 : M + hi0);
  if (signed0) {
    double lo1, hi1;
    code_range(f.q[1], lo1, hi1);
    const double P1 = hi1 + 1.0;
    if (lo1 != 0.0 || !pow2(P1)) return false;
    if (!scaled(f.q[1].k, P1) || !scaled(f.ka, P1) || !scaled(f.ka_off, P1)) return false;
    f.sat_half[1] = static_cast<float>(0.5 / P1);
    f.sat_p[1] = static_cast<float>(P1);
    f.sat_top[1] = static_cast<float>(M + hi1);
  }
  e = f;
  return true;
}

// Fold the shape's sq chain into EpiConsts (fused.h).  Every factor is a
// power of two, so each folded product / offset must be an exact float;
// returns false (interpreter fallback) when one is not.
bool make_epi(const kern::StageTables& t, int shape, double sxw, kern::EpiConsts& e) {
  using kern::kEpiExact;
  using kern::kEpiNonneg;
  std::memset(&e, 0, sizeof(e));
  const kern::ProgInstr* c = t.code;
  std::vector<int> qs;  // local sq indices in program order
  int res = -1, out0 = -1, out1 = -1;
  switch (shape) {
    case 1: qs = {c[0].a}; out0 = static_cast<int>(c[0].b); break;
    case kern::kShapeStoreAcc: {
      const int k = t.n_code == 2 ? 1 : 0;  // [pt acc sq, sq_store8] or [sq_store8 with acc]
      qs = {c[k].a};
      out0 = static_cast<int>(c[k].b);
      break;
    }
    case 2:
    case kern::kShapeSqStoreAcc: qs = {c[0].a, c[1].a}; out0 = static_cast<int>(c[1].b); break;
    case 3:
      qs = {c[0].a, c[2].a, c[4].a, c[6].a};
      res = static_cast<int>(c[1].b);
      out0 = static_cast<int>(c[4].b);
      out1 = static_cast<int>(c[6].b);
      break;
    case 4:
      qs = {c[0].a, c[2].a, c[3].a};
      res = static_cast<int>(c[1].b);
      out0 = static_cast<int>(c[3].b);
      break;
    case 5:
      qs = {c[0].a, c[2].a};
      res = static_cast<int>(c[1].b);
      out0 = static_cast<int>(c[3].b);
      break;
    case kern::kShapeSqF32:
      if (t.n_code == 1) {
        // bare fp32 store of the conv output: x0 = fma(a, s_x*s_w, bias), one
        // rounding (the reference's float conv value), no sq
        if (!exact_float(sxw, e.q[0].k)) return false;
        e.q[0].flags = kern::kEpiNoClamp;
        e.inv0 = 1.0f;
        e.f32_s = 1.0f;
        e.f32_off = 0.0f;
        const kern::ProgBuf& fb = t.buf[c[0].b];
        if (fb.kind != 1 || fb.hw != 1 || (reinterpret_cast<uintptr_t>(fb.ptr) & 15) != 0 || fb.ld % 4 != 0) {
          return false;  // (concat column slices: the interpreter's scalar stores)
        }
        e.f32_ptr = static_cast<float*>(fb.ptr);
        e.f32_ld = fb.ld;
        e.slot_out[0] = e.slot_out[1] = -1;
        return true;
      }
      qs = {c[0].a};
      out0 = static_cast<int>(c[1].b);
      break;
    default: return false;
  }
  // sq0 on the conv output: x0 = fma(a, s_x*s_w / s0, bias / s0)
  const kern::FSq& f0 = t.sq[qs[0]];
  kern::EpiSq& q0 = e.q[0];
  if (!exact_float(sxw / f0.s, q0.k) || !exact_float(f0.inv_s, e.inv0) || !round_bounds(f0, q0)) {
    return false;
  }
  // bias / s0 must stay exact: scaling by 2^j >= 1 never leaves the normal range downwards
  if (!(f0.inv_s >= 1.0f)) return false;
  q0.flags = f0.qmin >= 0.0f ? kEpiNonneg : 0;
  bool prev_nonneg = (q0.flags & kEpiNonneg) != 0;
  double prev_s = f0.s;
  size_t next = 1;
  if (res >= 0) {
    // x1 = fma(r0, s0/s1, c * s_res/s1); rounding (the sum is not integral in general)
    const kern::FSq& f1 = t.sq[qs[1]];
    kern::EpiSq& q1 = e.q[1];
    const double sres = t.buf[res].scale;
    if (!exact_float(prev_s / f1.s, q1.k) || !exact_float(sres / f1.s, e.ka) ||
        !exact_float(-(8388608.0 + 128.0) * (sres / f1.s), e.ka_off) || !round_bounds(f1, q1)) {
      return false;
    }
    q1.flags = f1.qmin >= 0.0f ? kEpiNonneg : 0;
    prev_nonneg = (q1.flags & kEpiNonneg) != 0;
    prev_s = f1.s;
    e.slot_res = t.buf[res].slot;
    next = 2;
  }
  // the remaining sqs read the previous rounded code (a fork, shape 3, reads
  // the same R1 twice)
  for (size_t i = next; i < qs.size(); ++i) {
    const kern::FSq& fp = t.sq[qs[next - 1]];  // the code R all of them read
    if (!epi_from_code(prev_s, prev_nonneg, t.sq[qs[i]], e.q[i], fp.qmin, fp.qmax)) {
      return false;
    }
  }
  if (shape == 5 || shape == kern::kShapeSqF32) {
    // fp32 output value v = r * s of the last sq (T-domain: fma(R, s, -M*s))
    const double s_last = prev_s;
    if (!exact_float(s_last, e.f32_s) ||
        !exact_float(prev_nonneg ? -kern::kMagic * s_last : 0.0, e.f32_off)) {
      return false;
    }
    const kern::ProgBuf& fb = t.buf[out0];
    if (fb.kind != 1 || fb.hw != 1 || (reinterpret_cast<uintptr_t>(fb.ptr) & 15) != 0 || fb.ld % 4 != 0) {
      return false;  // (concat column slices: the interpreter's scalar stores)
    }
    e.f32_ptr = static_cast<float*>(fb.ptr);
    e.f32_ld = fb.ld;
  }
  e.slot_out[0] = out0 >= 0 && shape != 5 && shape != kern::kShapeSqF32 ? t.buf[out0].slot : -1;
  e.slot_out[1] = out1 >= 0 ? t.buf[out1].slot : -1;
  if (shape == kern::kShapeSqStoreAcc || shape == kern::kShapeStoreAcc) {
    // sq0's accumulator clamp on x0 = v / s0 (power-of-two scaling: exact),
    // saturation codes in the domain epi_round leaves x0 in (T: M + code)
    const kern::FSq& f0 = t.sq[qs[0]];  // the grid sq x0 is in
    const bool pt = shape == kern::kShapeStoreAcc && t.n_code == 2;
    const kern::FSq& fa = pt ? t.sq[c[0].a] : f0;  // the accumulator clamp
    float alo = 0.0f, ahi = 0.0f;
    if (!exact_float(static_cast<double>(fa.lo_up) / f0.s, alo) ||
        !exact_float(static_cast<double>(fa.hi_dn) / f0.s, ahi)) {
      return false;
    }
    double clo = f0.q_lo, chi = f0.q_hi;
    if (pt) {
      // the store sq's code of the saturated value (round half away, clamp)
      clo = std::clamp(std::round(static_cast<double>(fa.lo_rn) / f0.s) + f0.zp, static_cast<double>(f0.qmin),
                       static_cast<double>(f0.qmax));
      chi = std::clamp(std::round(static_cast<double>(fa.hi_rn) / f0.s) + f0.zp, static_cast<double>(f0.qmin),
                       static_cast<double>(f0.qmax));
    }
    const double base = (e.q[0].flags & kEpiNonneg) ? kern::kMagic : 0.0;
    e.q[3].lo = alo;
    e.q[3].hi = ahi;
    if (!exact_float(base + clo, e.q[3].k) || !exact_float(base + chi, e.q[3].off)) return false;
  }
  return true;
}

// A max-pool whose program only stores codes of the pooled value ([sq_store8]
// or the fork [push, sq_store8, pop, sq_store8]) into plain NHWC rows runs the
// stores-only kernel; every store folds to code -> code constants.
bool pool_stores(const kern::StageTables& t, double s_in, kern::PoolStores& ps) {
  std::memset(&ps, 0, sizeof(ps));
  std::vector<int> stores;
  if (t.n_code == 1 && t.code[0].op == kern::kPSqStore8) {
    stores = {0};
  } else if (t.n_code == 4 && t.code[0].op == kern::kPPush && t.code[1].op == kern::kPSqStore8 &&
             t.code[2].op == kern::kPPop && t.code[3].op == kern::kPSqStore8) {
    stores = {1, 3};
  } else {
    return false;
  }
  for (size_t i = 0; i < stores.size(); ++i) {
    const kern::ProgInstr& in = t.code[stores[i]];
    const kern::FSq& f = t.sq[in.a];
    const kern::ProgBuf& b = t.buf[in.b];
    if (f.zp != 0.0f || f.has_acc || f.passthrough || b.kind != 0 || b.hw != 1 || b.ld % 16 != 0) {
      return false;
    }
    // pooled codes span the input grid's int8 range at most
    if (!epi_from_code(s_in, false, f, ps.q[i], -128.0, 127.0)) return false;
    ps.out[i] = static_cast<int8_t*>(b.ptr);
    ps.ld[i] = b.ld;
  }
  ps.n_out = static_cast<int>(stores.size());
  return true;
}

}  // namespace

FastPlan::~FastPlan() = default;

void FastPlan::fail(const std::string& why) {
  if (ok_ || why_.empty()) why_ = why;
  ok_ = false;
}

FastPlan::FastPlan(const engine::Plan& plan) : plan_(plan) {
  ok_ = true;
  try {
    compile();
  } catch (const std::exception& e) {
    fail(std::string("compile: ") + e.what());
  }
}

void FastPlan::compile() {
  const auto& steps = plan_.steps();
  std::vector<ProgInstr> code;
  std::map<int, int> val_of;
  std::set<int> absorbed;
  Builder b{plan_, code, sq_index_, sq_steps_, clip_lo_, clip_hi_, vals_, val_of, absorbed,
            [this](const std::string& w) { fail(w); }};
  b.out_val = &out_val_;
  b.out_per_sample = &out_per_sample_;
  std::map<int, int> concat_root_val;
  b.concat_root_val = &concat_root_val;
  const Graph& g = plan_.graph();

  for (size_t i = 0; i < steps.size() && ok_; ++i) {
    const int step = static_cast<int>(i);
    const Node& n = *steps[i].node;
    if (absorbed.count(step)) continue;
    auto st = std::make_unique<Stage>();
    st->step = step;
    st->code_off = static_cast<int>(code.size());
    const auto& shp = plan_.shape(step);
    switch (n.op) {
      case OpKind::kConstant:
        continue;  // weights / biases, consumed by GEMM stages
      case OpKind::kSimulatedQuantize: {
        // weight sq (constant input) belongs to its GEMM; anything else here
        // was not reached by a program
        const int src = steps[i].in[0];
        if (src >= 0 && steps[static_cast<size_t>(src)].node->op == OpKind::kConstant) continue;
        fail("simulated_quantize not reachable from a producing stage");
        continue;
      }
      case OpKind::kInput: {
        auto it = std::find(g.inputs().begin(), g.inputs().end(), n.id);
        st->kind = Stage::kInput;
        st->input_k = static_cast<int>(it - g.inputs().begin());
        if (shp.size() == 4) {
          st->n0 = static_cast<int>(shp[0]);
          st->C = static_cast<int>(shp[1]);
          st->HW = static_cast<int>(shp[2] * shp[3]);
        } else if (shp.size() == 2) {
          st->n0 = static_cast<int>(shp[0]);
          st->C = static_cast<int>(shp[1]);
          st->HW = 1;
        } else {
          fail("input rank");
          continue;
        }
        b.rows_ps = static_cast<int64_t>(st->n0) * st->HW;
        b.C = st->C;
        if (shp.size() == 4) {
          b.input_step = step;
          b.input_H = static_cast<int>(shp[2]);
          b.input_W = static_cast<int>(shp[3]);
        }
        break;
      }
      case OpKind::kConv2d:
      case OpKind::kDense: {
        if (n.attr_or<int64_t>("groups", 1) != 1) {
          if (!b.depthwise(step)) {
            fail("grouped conv2d (other than depthwise) runs on the exact engine");
            continue;
          }
          // depthwise: CUDA-core stage (kern::stage_dw_conv), the consumers'
          // program like any producing stage
          st->kind = Stage::kDw;
          const auto& in = steps[i].in;
          const Node& wsq = *steps[static_cast<size_t>(in[1])].node;
          auto vit = val_of.find(in[0]);
          if (steps[static_cast<size_t>(in[0])].node->op != OpKind::kSimulatedQuantize || vit == val_of.end() ||
              vals_[static_cast<size_t>(vit->second)]->kind != 0) {
            fail("depthwise data input is not an int8 simulated_quantize");
            continue;
          }
          if (wsq.op != OpKind::kSimulatedQuantize ||
              steps[static_cast<size_t>(steps[static_cast<size_t>(in[1])].in[0])].node->op != OpKind::kConstant) {
            fail("depthwise weight is not a simulated-quantized constant");
            continue;
          }
          st->in_val = vit->second;
          st->w_sq = in[1];
          st->w_const = steps[static_cast<size_t>(in[1])].in[0];
          if (in.size() > 2 && in[2] >= 0) {
            if (steps[static_cast<size_t>(in[2])].node->op != OpKind::kConstant ||
                !steps[static_cast<size_t>(in[2])].node->payload->dtype().is_float()) {
              fail("bias is not a float constant");
              continue;
            }
            st->bias_const = in[2];
            for (float bv : steps[static_cast<size_t>(in[2])].node->payload->floats()) {
              st->bias_absmax = std::max(st->bias_absmax, std::fabs(static_cast<double>(bv)));
            }
          }
          const auto& ds = plan_.shape(in[0]);
          const auto& ws = plan_.shape(st->w_const);
          Attr2 strd = pair_of(n, "strides", {1, 1}), pad = pair_of(n, "padding", {0, 0});
          st->n0 = static_cast<int>(ds[0]);
          st->C = static_cast<int>(ds[1]);
          st->H = static_cast<int>(ds[2]);
          st->W = static_cast<int>(ds[3]);
          st->O = static_cast<int>(ws[0]);
          st->KH = static_cast<int>(ws[2]);
          st->KW = static_cast<int>(ws[3]);
          st->sh = strd.a;
          st->sw = strd.b;
          st->ph = pad.a;
          st->pw = pad.b;
          st->OH = static_cast<int>(shp[2]);
          st->OW = static_cast<int>(shp[3]);
          st->taps = st->KH * st->KW;
          st->ldk = (st->C + 15) / 16 * 16;  // weight codes [tap][ldk]
          st->Ktrue = st->taps * st->ldk;
          st->Kpad = st->Ktrue;
          st->rows_out_ps = static_cast<int64_t>(st->n0) * st->OH * st->OW;
          b.rows_ps = st->rows_out_ps;
          b.C = st->O;
          absorbed.insert(in[1]);
          break;
        }
        st->kind = Stage::kGemm;
        st->dense = n.op == OpKind::kDense;
        const auto& in = steps[i].in;
        if (in.size() < 2 || in[0] < 0 || in[1] < 0) {
          fail("gemm inputs");
          continue;
        }
        const Node& dsq = *steps[static_cast<size_t>(in[0])].node;
        const Node& wsq = *steps[static_cast<size_t>(in[1])].node;
        auto vit = val_of.find(in[0]);
        if (dsq.op != OpKind::kSimulatedQuantize || vit == val_of.end() ||
            vals_[static_cast<size_t>(vit->second)]->kind != 0) {
          fail("conv/dense data input is not an int8 simulated_quantize");
          continue;
        }
        if (wsq.op != OpKind::kSimulatedQuantize ||
            steps[static_cast<size_t>(steps[static_cast<size_t>(in[1])].in[0])].node->op != OpKind::kConstant) {
          fail("conv/dense weight is not a simulated-quantized constant");
          continue;
        }
        st->in_val = vit->second;
        st->w_sq = in[1];
        st->w_const = steps[static_cast<size_t>(in[1])].in[0];
        if (in.size() > 2 && in[2] >= 0) {
          if (steps[static_cast<size_t>(in[2])].node->op != OpKind::kConstant ||
              !steps[static_cast<size_t>(in[2])].node->payload->dtype().is_float()) {
            fail("bias is not a float constant");
            continue;
          }
          st->bias_const = in[2];
          for (float bv : steps[static_cast<size_t>(in[2])].node->payload->floats()) {
            st->bias_absmax = std::max(st->bias_absmax, std::fabs(static_cast<double>(bv)));
            if (bv != 0.0f) st->bias_absmin = std::min(st->bias_absmin, std::fabs(static_cast<double>(bv)));
          }
        }
        const Val& dv = *vals_[static_cast<size_t>(st->in_val)];
        const auto& ws = plan_.shape(st->w_const);
        st->O = static_cast<int>(ws[0]);
        if (st->dense) {
          st->Ktrue = static_cast<int>((dv.rows_ps / dv.hw) > 0 ? dv.ld : dv.ld);
          st->Ktrue = static_cast<int>(dv.hw > 1 ? static_cast<int64_t>(dv.hw) * dv.cs : dv.C);
          st->taps = dv.hw;
          st->ldk = dv.hw > 1 ? dv.cs : dv.C;
          st->gather = false;
          st->rows_out_ps = dv.rows_ps / dv.hw;
          b.rows_ps = st->rows_out_ps;
        } else {
          const auto& ds = plan_.shape(in[0]);
          Attr2 strd = pair_of(n, "strides", {1, 1}), pad = pair_of(n, "padding", {0, 0});
          st->H = static_cast<int>(ds[2]);
          st->W = static_cast<int>(ds[3]);
          st->KH = static_cast<int>(ws[2]);
          st->KW = static_cast<int>(ws[3]);
          st->sh = strd.a;
          st->sw = strd.b;
          st->ph = pad.a;
          st->pw = pad.b;
          st->OH = static_cast<int>(shp[2]);
          st->OW = static_cast<int>(shp[3]);
          st->n0 = static_cast<int>(ds[0]);
          st->C = static_cast<int>(ds[1]);
          st->taps = st->KH * st->KW;
          st->gather = !(st->taps == 1 && st->sh == 1 && st->sw == 1 && st->ph == 0 &&
                         st->pw == 0 && dv.ld == st->C);
          st->ldk = st->gather ? static_cast<int>(dv.ld) : st->C;
          // 64-channel stride-1 KxK convs: weight taps at a 128-byte stride
          // (zero channels 64..127) so the conv runs on the 2-D band producer
          // (conv_tc.cu TcArgs::b2_*), which reads 128-byte channel chunks
          static const bool no_band2 = std::getenv("QUANTC_BAND2") == nullptr;  // opt-in, conv_tc.cu
          if (!no_band2 && st->gather && dv.ld == 64 && st->C == 64 && st->taps > 1 && st->sh == 1 &&
              st->sw == 1 && st->ph < st->KH && st->pw < st->KW && st->OW + st->KW - 1 <= 128 && !dv.s2d) {
            st->ldk = 128;
          }
          st->Ktrue = st->gather ? st->taps * st->ldk : st->C;
          // tiny-channel convs (e.g. the RGB stem, C=3 in 16-byte rows): pack
          // dense im2col rows k = tap*C + c first, then run the GEMM direct
          if (st->gather && st->C <= 8 && st->taps > 1) {
            st->packed = true;
            st->gather = false;
            st->ldk = st->C;
            st->Ktrue = st->taps * st->C;
          }
          if (dv.s2d) {
            // stride-2 KxK conv over the space-to-depth input: a stride-1
            // ceil((K+d)/2)^2 conv, pad ceil(p/2), where d = 2*ceil(p/2) - p
            // aligns original tap k = 2*ka + dy - d (fastplan weight_codes_s2d)
            st->s2d = true;
            st->s2d_C = dv.s2d_C;
            st->s2d_KH = st->KH;
            st->s2d_KW = st->KW;
            const int ph2 = (st->ph + 1) / 2, pw2 = (st->pw + 1) / 2;
            st->s2d_dh = 2 * ph2 - st->ph;
            st->s2d_dw = 2 * pw2 - st->pw;
            st->KH = (st->s2d_KH + st->s2d_dh + 1) / 2;
            st->KW = (st->s2d_KW + st->s2d_dw + 1) / 2;
            st->ph = ph2;
            st->pw = pw2;
            st->sh = st->sw = 1;
            st->H = (dv.s2d_H + 1) / 2;
            st->W = (dv.s2d_W + 1) / 2;
            st->C = 4 * dv.s2d_C;
            st->taps = st->KH * st->KW;
            st->gather = true;
            st->packed = false;
            st->ldk = 16;
            st->Ktrue = st->taps * 16;
          }
          // the gather producer tracks tap validity in a 64-bit mask
          if (st->gather && st->taps > 63) fail("conv kernel with more than 63 taps");
          st->rows_out_ps = static_cast<int64_t>(st->n0) * st->OH * st->OW;
          b.rows_ps = st->rows_out_ps;
        }
        st->Kpad = (st->Ktrue + 127) / 128 * 128;
        b.C = st->O;
        absorbed.insert(in[1]);
        break;
      }
      case OpKind::kMaxPool2d: {
        st->kind = Stage::kMaxpool;
        const int src = steps[i].in[0];
        auto vit = val_of.find(src);
        if (vit == val_of.end() || vals_[static_cast<size_t>(vit->second)]->kind != 0) {
          fail("max_pool2d input is not int8 codes");
          continue;
        }
        st->in_val = vit->second;
        const auto& ds = plan_.shape(src);
        auto k = n.attr<std::vector<int64_t>>("pool_size");
        Attr2 strd = pair_of(n, "strides", {static_cast<int>(k[0]), static_cast<int>(k[1])});
        Attr2 pad = pair_of(n, "padding", {0, 0});
        st->n0 = static_cast<int>(ds[0]);
        st->C = static_cast<int>(ds[1]);
        st->H = static_cast<int>(ds[2]);
        st->W = static_cast<int>(ds[3]);
        st->OH = static_cast<int>(shp[2]);
        st->OW = static_cast<int>(shp[3]);
        st->pkh = static_cast<int>(k[0]);
        st->pkw = static_cast<int>(k[1]);
        st->sh = strd.a;
        st->sw = strd.b;
        st->ph = pad.a;
        st->pw = pad.b;
        b.rows_ps = static_cast<int64_t>(st->n0) * st->OH * st->OW;
        b.C = st->C;
        break;
      }
      case OpKind::kAvgPool2d: {
        // average of materialised fp32 rows (zero padding counted: the op's
        // semantics are the constant depthwise conv it rewrites to)
        st->kind = Stage::kAvg;
        const int src = steps[i].in[0];
        auto vit = val_of.find(src);
        if (vit == val_of.end() || vals_[static_cast<size_t>(vit->second)]->kind != 1) {
          fail("avg_pool2d input is not materialised fp32");
          continue;
        }
        st->in_val = vit->second;
        const auto& ds = plan_.shape(src);
        auto k = n.attr<std::vector<int64_t>>("pool_size");
        Attr2 strd = pair_of(n, "strides", {static_cast<int>(k[0]), static_cast<int>(k[1])});
        Attr2 pad = pair_of(n, "padding", {0, 0});
        st->n0 = static_cast<int>(ds[0]);
        st->C = static_cast<int>(ds[1]);
        st->H = static_cast<int>(ds[2]);
        st->W = static_cast<int>(ds[3]);
        st->OH = static_cast<int>(shp[2]);
        st->OW = static_cast<int>(shp[3]);
        st->pkh = static_cast<int>(k[0]);
        st->pkw = static_cast<int>(k[1]);
        st->sh = strd.a;
        st->sw = strd.b;
        st->ph = pad.a;
        st->pw = pad.b;
        b.rows_ps = static_cast<int64_t>(st->n0) * st->OH * st->OW;
        b.C = st->C;
        break;
      }
      case OpKind::kConcat: {
        // a concat inside another concat has no stage: its inputs wrote
        // straight into the outer buffer
        if (b.concat_outer(step).first >= 0) continue;
        auto cit = concat_root_val.find(step);
        if (cit == concat_root_val.end()) {
          fail("concat not reached by its inputs");
          continue;
        }
        if (n.attr_or<int64_t>("axis", 1) != 1) {
          fail("concat along an axis other than channels");
          continue;
        }
        st->kind = Stage::kCat;
        st->in_val = cit->second;
        const Val& cv = *vals_[static_cast<size_t>(cit->second)];
        st->C = cv.C;
        b.rows_ps = cv.rows_ps;
        b.C = cv.C;
        break;
      }
      case OpKind::kGlobalAvgPool2d: {
        st->kind = Stage::kGap;
        const int src = steps[i].in[0];
        auto vit = val_of.find(src);
        if (vit == val_of.end() || vals_[static_cast<size_t>(vit->second)]->kind != 1) {
          fail("global_avg_pool2d input is not materialised fp32");
          continue;
        }
        st->in_val = vit->second;
        const auto& ds = plan_.shape(src);
        st->n0 = static_cast<int>(ds[0]);
        st->C = static_cast<int>(ds[1]);
        st->HW = static_cast<int>(ds[2] * ds[3]);
        b.rows_ps = st->n0;
        b.C = st->C;
        break;
      }
      default:
        fail("operator " + op_name(n.op) + " (node " + std::to_string(n.id) +
             ") outside the fused dataflow");
        continue;
    }
    if (st->kind != Stage::kInput) b.input_step = -1;
    b.flat_hw = 1;
    b.flat_cs = 0;
    b.depth = 0;
    b.max_depth = 0;
    b.emit(step);
    st->code_len = static_cast<int>(code.size()) - st->code_off;
    st->depth = b.max_depth;
    // re-index the stage's program against its own compact tables
    std::map<int, int> lsq, lbuf, lclip;
    for (int pc = st->code_off; pc < st->code_off + st->code_len; ++pc) {
      ProgInstr ins = code[static_cast<size_t>(pc)];
      auto local = [](std::map<int, int>& m, std::vector<int>& v, int g) {
        auto it = m.find(g);
        if (it != m.end()) return it->second;
        const int l = static_cast<int>(v.size());
        m[g] = l;
        v.push_back(g);
        return l;
      };
      switch (ins.op) {
        case kern::kPSq:
          ins.a = static_cast<uint16_t>(local(lsq, st->sq_slots, ins.a));
          break;
        case kern::kPSqStore8:
          ins.a = static_cast<uint16_t>(local(lsq, st->sq_slots, ins.a));
          ins.b = static_cast<uint32_t>(local(lbuf, st->buf_vals, static_cast<int>(ins.b)));
          break;
        case kern::kPAdd:
        case kern::kPStoreF32:
          ins.b = static_cast<uint32_t>(local(lbuf, st->buf_vals, static_cast<int>(ins.b)));
          break;
        case kern::kPClip:
          ins.a = static_cast<uint16_t>(local(lclip, st->clips, ins.a));
          break;
        default:
          break;
      }
      st->code.push_back(ins);
    }
    // GEMM stages: route plain-row int8 code outputs (<= 2) and one residual
    // operand through shared-memory tile slots (TMA store / TMA prefetch)
    st->buf_slot.assign(st->buf_vals.size(), -1);
    if (st->kind == Stage::kGemm) {
      auto slot_ok = [&](int vid) {
        const Val& v = *vals_[static_cast<size_t>(vid)];
        return v.kind == 0 && v.hw == 1 && v.ld % 16 == 0 && v.rows_ps == st->rows_out_ps &&
               v.C == st->O;
      };
      std::vector<int> produced;
      for (const ProgInstr& ins : st->code) {
        if (ins.op != kern::kPSqStore8) continue;
        const int lb = static_cast<int>(ins.b);
        produced.push_back(lb);
        if (st->buf_slot[static_cast<size_t>(lb)] < 0 && st->n_out < 2 &&
            slot_ok(st->buf_vals[static_cast<size_t>(lb)])) {
          st->buf_slot[static_cast<size_t>(lb)] = st->n_out;
          st->out_vals[st->n_out++] = st->buf_vals[static_cast<size_t>(lb)];
        }
      }
      for (const ProgInstr& ins : st->code) {
        if (ins.op != kern::kPAdd) continue;
        const int lb = static_cast<int>(ins.b);
        const bool mine = std::find(produced.begin(), produced.end(), lb) != produced.end();
        if (!mine && st->res_val < 0 && slot_ok(st->buf_vals[static_cast<size_t>(lb)])) {
          st->res_val = st->buf_vals[static_cast<size_t>(lb)];
          st->buf_slot[static_cast<size_t>(lb)] = 2;  // fixed below to n_out
        }
      }
      for (size_t k = 0; k < st->buf_slot.size(); ++k) {
        if (st->buf_slot[k] == 2 && st->buf_vals[k] == st->res_val) st->buf_slot[k] = st->n_out;
      }
    }
    if (st->code.size() > static_cast<size_t>(kern::kMaxCode) ||
        st->sq_slots.size() > static_cast<size_t>(kern::kMaxSq) ||
        st->buf_vals.size() > static_cast<size_t>(kern::kMaxBuf) ||
        st->clips.size() > static_cast<size_t>(kern::kMaxClip)) {
      fail("stage program exceeds the StageTables limits");
    }
    stages_.push_back(std::move(st));
  }
  if (ok_ && out_val_ < 0) fail("graph output not reached");
  if (std::getenv("QUANTC_DUMP_PLAN")) {
    static const char* kind[] = {"input", "gemm", "maxpool", "gap", "dw", "avg", "cat"};
    static const char* opn[] = {"end", "sq", "sq_store8", "relu", "clip", "add", "store_f32",
                                "push", "pop"};
    for (const auto& st : stages_) {
      std::fprintf(stderr, "stage %-7s step %4d C %4d O %4d K %4dx%-2d s%d gather %d s2d %d n_out %d res %d:",
                   kind[st->kind], st->step, st->C, st->O, st->KH, st->KW, st->sh,
                   st->gather ? 1 : 0, st->s2d ? 1 : 0, st->n_out, st->res_val >= 0 ? 1 : 0);
      for (const ProgInstr& in : st->code) std::fprintf(stderr, " %s", opn[in.op]);
      std::fprintf(stderr, "\n");
    }
  }
  if (ok_ && sq_steps_.size() > 65535) fail("too many simulated_quantize nodes");
}

bool FastPlan::eligible(const SimBinding* binding, bool exact, std::string* why) const {
  if (!ok_) {
    if (why) *why = why_;
    return false;
  }
  std::set<int> coded;
  for (const auto& v : vals_) {
    if (v->kind == 0) coded.insert(v->sq_step);
  }
  for (const auto& st : stages_) {
    if (st->kind == Stage::kGemm || st->kind == Stage::kDw) coded.insert(st->w_sq);
  }
  auto check = [&](int step) -> bool {
    const QParams p = engine::qparams_of(*plan_.steps()[static_cast<size_t>(step)].node, binding);
    try {
      engine::resolve_sq(p);
    } catch (...) {
      if (why) *why = "invalid QParams";
      return false;
    }
    if (!p.passthrough) {
      const double s = compute_scale(p.threshold, p.bit, p.sign);
      if (exact && !is_pow2(s)) {
        if (why) *why = "non power-of-two scale";
        return false;
      }
      const float sf = static_cast<float>(s);
      if (!(std::isfinite(sf) && sf > 0 && std::isfinite(1.0f / sf) && std::fpclassify(sf) == FP_NORMAL)) {
        if (why) *why = "scale outside fp32 range";
        return false;
      }
    }
    if (p.acc_dtype.has_value() && p.acc_scale > 0.0) {
      const double lo = static_cast<double>(p.acc_dtype->min_value()) * p.acc_scale;
      if (!std::isfinite(static_cast<float>(lo))) {
        if (why) *why = "accumulator bound outside fp32 range";
        return false;
      }
    }
    if (coded.count(step)) {
      if (p.passthrough || p.sign != 1 || p.zero_point != 0 || p.bit > 8) {
        if (why) *why = "materialised code is not int8";
        return false;
      }
    }
    return true;
  };
  for (int step : sq_steps_) {
    if (!check(step)) return false;
  }
  for (const auto& st : stages_) {
    if ((st->kind == Stage::kGemm || st->kind == Stage::kDw) && !check(st->w_sq)) return false;
  }
  return true;
}

void FastPlan::ensure_arena(int batch, int group) {
  // buffers are batch-major rows: a smaller batch runs on a prefix
  Arena& ar = arenas_[static_cast<size_t>(group)];
  if (ar.batch >= batch) return;
  ar.bufs.clear();
  for (const auto& v : vals_) {
    if (v->alias_root >= 0) {
      ar.bufs.push_back(nullptr);  // a column slice of its root's buffer
      continue;
    }
    const size_t bytes = static_cast<size_t>(v->bytes_ps()) * batch;
    auto buf = engine::device_alloc_on(ST(), bytes + 64);
    if (v->zero_fill) ok_cuda(cudaMemsetAsync(buf.get(), 0, bytes + 64, ST()));
    ar.bufs.push_back(buf);
  }
  ar.tables = engine::device_alloc_on(ST(), std::max<size_t>(1, stages_.size()) * sizeof(kern::StageTables));
  ar.batch = batch;
}

// Per-binding state of one forward: the host-built tables, epilogue shapes /
// constants, fork aliases, and the arena (group) it runs in.
struct FastPlan::Run {
  int group = 0;
  int batch = 0;
  std::vector<const float*> inputs;
  const SimBinding* binding = nullptr;
  int64_t* d_preds = nullptr;
  float* d_scores = nullptr;
  std::vector<FSq> fsq, wfsq;
  std::map<int, float> scale_by_step;
  std::vector<double> acc_bound;
  std::vector<kern::StageTables> tabs;
  std::vector<int> shape0, shape_of;
  std::vector<kern::EpiConsts> epi_of;
  std::vector<double> sxw_of;
  std::vector<char> drop2;
  std::vector<char> pool_drop2;  // max-pool stage stores once (aliased outputs)
  std::vector<int> alias;
  const kern::StageTables* d_tabs = nullptr;
  std::vector<std::shared_ptr<void>> keep;  // per-run temporaries (stream-ordered frees)
};

void FastPlan::prepare(Run& r) {
  ensure_arena(r.batch, r.group);
  const SimBinding* binding = r.binding;
  auto& fsq = r.fsq;
  auto& scale_by_step = r.scale_by_step;
  auto& wfsq = r.wfsq;
  auto& acc_bound = r.acc_bound;
  auto& tabs = r.tabs;
  // ---- per-run tables: FSq per sq node, clip bounds, buffer descriptors
  fsq.assign(sq_steps_.size(), FSq{});
  for (size_t k = 0; k < sq_steps_.size(); ++k) {
    const QParams p = engine::qparams_of(*plan_.steps()[static_cast<size_t>(sq_steps_[k])].node, binding);
    fsq[k] = make_fsq(p);
    scale_by_step[sq_steps_[k]] = fsq[k].s;
  }
  // weight-edge sq parameters and |accumulator| bounds of the GEMM stages
  wfsq.assign(stages_.size(), FSq{});
  acc_bound.assign(stages_.size(), 0.0);
  for (size_t si = 0; si < stages_.size(); ++si) {
    const Stage& st = *stages_[si];
    if (st.kind != Stage::kGemm && st.kind != Stage::kDw) continue;
    wfsq[si] = make_fsq(engine::qparams_of(*plan_.steps()[static_cast<size_t>(st.w_sq)].node, binding));
    const Val& dv = *vals_[static_cast<size_t>(st.in_val)];
    const FSq& df = fsq[static_cast<size_t>(sq_index_.at(dv.sq_step))];
    const double kreal = st.kind == Stage::kDw ? static_cast<double>(st.taps)
                         : st.dense            ? st.Ktrue
                                               : static_cast<double>(st.C) * st.KH * st.KW;
    acc_bound[si] = kreal * code_absmax(df) * code_absmax(wfsq[si]);
  }
  // one compact table block per stage (instructions + referenced params)
  tabs.assign(stages_.size(), kern::StageTables{});
  for (size_t si = 0; si < stages_.size(); ++si) {
    const Stage& st = *stages_[si];
    kern::StageTables& t = tabs[si];
    std::memset(&t, 0, sizeof(t));
    t.n_code = static_cast<int32_t>(st.code.size());
    t.n_sq = static_cast<int32_t>(st.sq_slots.size());
    t.n_buf = static_cast<int32_t>(st.buf_vals.size());
    t.n_clip = static_cast<int32_t>(st.clips.size());
    std::copy(st.code.begin(), st.code.end(), t.code);
    for (size_t k = 0; k < st.sq_slots.size(); ++k) t.sq[k] = fsq[static_cast<size_t>(st.sq_slots[k])];
    for (size_t k = 0; k < st.buf_vals.size(); ++k) {
      const int vid = st.buf_vals[k];
      const Val& v = *vals_[static_cast<size_t>(vid)];
      // the value's own buffer (shape 5 folds it into f32_ptr); re-pointed
      // below once fork aliases are known
      t.buf[k] = ProgBuf{arena_ptr(r.group, vid),
                         v.ld, v.hw, v.cs, v.kind,
                         v.kind == 0 ? scale_by_step.at(v.sq_step) : 1.0f,
                         k < st.buf_slot.size() ? st.buf_slot[k] : -1, 0};
    }
    for (size_t k = 0; k < st.clips.size(); ++k) {
      const int c = st.clips[k];
      t.clip[k] = make_float2(clip_lo_[static_cast<size_t>(c)], clip_hi_[static_cast<size_t>(c)]);
    }
    double v0 = std::numeric_limits<double>::infinity();
    if (st.kind == Stage::kGemm || st.kind == Stage::kDw) {
      const Val& dv = *vals_[static_cast<size_t>(st.in_val)];
      const double sxw = static_cast<double>(scale_by_step.at(dv.sq_step)) *
                         static_cast<double>(wfsq[si].s);
      v0 = acc_bound[si] * sxw * 1.0001 + st.bias_absmax;
    } else if (st.kind == Stage::kMaxpool) {
      const Val& v = *vals_[static_cast<size_t>(st.in_val)];
      const FSq& f = fsq[static_cast<size_t>(sq_index_.at(v.sq_step))];
      v0 = code_absmax(f) * static_cast<double>(f.s);
    }
    optimise_tables(t, v0);
  }
  // ---- epilogue shapes and fork aliasing.  A fork whose two stores carry
  // identical constants writes identical bytes: the second value becomes an
  // alias of the first buffer and the kernel stores once (one TMA store
  // stream fewer on the add-fork layers, the largest writers of a step).
  static const bool no_shapes = std::getenv("QUANTC_NO_SHAPES") != nullptr;
  static const bool no_special = std::getenv("QUANTC_NO_SPECIAL") != nullptr;
  static const bool no_alias = std::getenv("QUANTC_NO_FORK_ALIAS") != nullptr;
  static const bool no_res_alias = std::getenv("QUANTC_NO_RES_ALIAS") != nullptr;
  auto& shape0 = r.shape0;
  auto& shape_of = r.shape_of;
  auto& epi_of = r.epi_of;
  auto& sxw_of = r.sxw_of;
  auto& drop2 = r.drop2;
  auto& alias = r.alias;
  shape0.assign(stages_.size(), 0);
  shape_of.assign(stages_.size(), 0);
  epi_of.assign(stages_.size(), kern::EpiConsts{});
  sxw_of.assign(stages_.size(), 0.0);
  drop2.assign(stages_.size(), 0);
  alias.resize(vals_.size());
  std::iota(alias.begin(), alias.end(), 0);
  for (size_t si = 0; si < stages_.size(); ++si) {
    const Stage& st = *stages_[si];
    if (st.kind != Stage::kGemm) continue;
    const Val& dv = *vals_[static_cast<size_t>(st.in_val)];
    sxw_of[si] = static_cast<double>(scale_by_step.count(dv.sq_step) ? scale_by_step.at(dv.sq_step) : 0.0f) *
                 static_cast<double>(wfsq[si].s);
    const int sh0 = no_shapes ? 0 : classify_shape(tabs[si], st.O);
    shape0[si] = sh0;
    kern::EpiConsts& e = epi_of[si];
    int sh = sh0;
    if (sh != 0 && !make_epi(tabs[si], sh, sxw_of[si], e)) sh = 0;
    if (sh == kern::kShapeSqF32) e.f32_cols = st.O;
    // flag-specialised kernels for the common constant profiles (fused.cuh)
    if (!no_special) {
      // a k = 1 store of a T-domain code: exact, at most a clamp
      auto identity = [](const kern::EpiSq& q) {
        return (q.flags & ~kern::kEpiNoClamp) == (kern::kEpiNonneg | kern::kEpiExact) &&
               q.k == 1.0f && q.off == 0.0f;
      };
      auto same = [](const kern::EpiSq& a, const kern::EpiSq& b) {
        return a.flags == b.flags && a.lo == b.lo && a.hi == b.hi;
      };
      // integer shapes first (no float conversion at all), else the
      // saturating float forms
      static const bool no_int = std::getenv("QUANTC_NO_INT_EPI") != nullptr;
      if (sh == kern::kShapeSqStore && e.q[0].flags == kern::kEpiNonneg && identity(e.q[1])) {
        if (!no_int && fold_integer(si, kern::kShapeSqStoreInt, sxw_of[si], r.acc_bound[si], e, r.keep)) {
          sh = kern::kShapeSqStoreInt;
        } else if (fold_saturating(kern::kShapeSqStoreId, st.bias_absmin, e)) {
          sh = kern::kShapeSqStoreId;
        }
      } else if (sh == kern::kShapeAddFork && e.q[0].flags == 0 &&
                 e.q[1].flags == kern::kEpiNonneg && identity(e.q[2]) && identity(e.q[3]) &&
                 same(e.q[2], e.q[3])) {
        if (!no_int && fold_integer(si, kern::kShapeAddForkInt, sxw_of[si], r.acc_bound[si], e, r.keep)) {
          sh = kern::kShapeAddForkInt;
        } else if (fold_saturating(kern::kShapeAddForkId, st.bias_absmin, e)) {
          sh = kern::kShapeAddForkId;
        }
      }
    }
    shape_of[si] = sh;
    if (!no_alias && (sh == kern::kShapeAddFork || sh == kern::kShapeAddForkId || sh == kern::kShapeAddForkInt) &&
        st.n_out == 2 && std::memcmp(&e.q[2], &e.q[3], sizeof(kern::EpiSq)) == 0) {
      const Val& v0 = *vals_[static_cast<size_t>(st.out_vals[0])];
      const Val& v1 = *vals_[static_cast<size_t>(st.out_vals[1])];
      if (v0.kind == v1.kind && v0.C == v1.C && v0.ld == v1.ld && v0.hw == v1.hw &&
          v0.rows_ps == v1.rows_ps && !v0.s2d && !v1.s2d && (v0.zero_fill || !v1.zero_fill)) {
        alias[static_cast<size_t>(st.out_vals[1])] = alias[static_cast<size_t>(st.out_vals[0])];
        drop2[si] = 1;
        // one output slot (0); the residual moves to slot 1 (= n_out)
        e.slot_out[0] = 0;
        e.slot_out[1] = -1;
        // the integer add-fork reads its residual bytes and overwrites them
        // with the output in one slot (TcConvSpec::res_alias): half the slot
        // memory, so 256-wide tiles keep double-buffered sets
        if (e.slot_res >= 0) e.slot_res = (sh == kern::kShapeAddForkInt && !no_res_alias) ? 0 : 1;
      }
    }
  }
  // a max-pool forking into two code stores with identical constants (the
  // pooled value quantized the same way for the first block's conv and its
  // shortcut): one store, the second value aliases the first buffer
  r.pool_drop2.assign(stages_.size(), 0);
  for (size_t si = 0; si < stages_.size() && !no_alias; ++si) {
    const Stage& st = *stages_[si];
    if (st.kind != Stage::kMaxpool) continue;
    const Val& v = *vals_[static_cast<size_t>(st.in_val)];
    kern::PoolStores ps;
    const kern::StageTables& t = tabs[si];
    if (!(st.C % 16 == 0 && v.ld % 16 == 0 && st.ph < st.pkh && st.pw < st.pkw &&
          pool_stores(t, scale_by_step.at(v.sq_step), ps)) ||
        ps.n_out != 2 || std::memcmp(&ps.q[0], &ps.q[1], sizeof(kern::EpiSq)) != 0) {
      continue;
    }
    const int v0 = st.buf_vals[static_cast<size_t>(t.code[1].b)];
    const int v1 = st.buf_vals[static_cast<size_t>(t.code[3].b)];
    const Val& a = *vals_[static_cast<size_t>(v0)];
    const Val& b = *vals_[static_cast<size_t>(v1)];
    if (a.kind == b.kind && a.C == b.C && a.ld == b.ld && a.hw == b.hw && a.rows_ps == b.rows_ps &&
        !a.s2d && !b.s2d && (a.zero_fill || !b.zero_fill)) {
      alias[static_cast<size_t>(v1)] = alias[static_cast<size_t>(v0)];
      r.pool_drop2[si] = 1;
    }
  }
  for (size_t si = 0; si < stages_.size(); ++si) {
    for (size_t k = 0; k < stages_[si]->buf_vals.size(); ++k) {
      tabs[si].buf[k].ptr = buf(r, stages_[si]->buf_vals[k]);
    }
  }
  Arena& ar = arenas_[static_cast<size_t>(r.group)];
  ok_cuda(cudaMemcpyAsync(ar.tables.get(), tabs.data(), tabs.size() * sizeof(kern::StageTables),
                          cudaMemcpyHostToDevice, ST()));
  r.d_tabs = static_cast<const kern::StageTables*>(ar.tables.get());
}

// Integer form of shapes 6/7 (fused.h EpiConsts i_*, fused.cuh run_int_epi).
// Every scale is a power of two.  The code sq0 makes of a conv output is a
// monotone step function of the channel's int32 accumulator a:
//   f(a) = clamp(round(RN24(a*s + b[n]) / s0), lo0, hi0)
// (reference interpreter.cpp:196-236: double sum, + bias, one rounding to
// float; then simulate.cpp:64-78).  The kernel evaluates
//   g(a) = clamp((a*m0 + C[n]) >> r0, lo0, hi0)
// With s/s0 = 2^-r0 (r0 >= 1) g steps at a = k*2^r0 - C[n], C[n] = 2^(r0-1) -
// ceil(-b/s); f steps there too unless the float rounding moves a boundary
// (bias within half an ulp of a step) or a half-way tie is reachable, so both
// sides of every step of every channel are checked with the reference
// arithmetic (a monotone integer step function is pinned by its steps).  With
// s/s0 = 2^L >= 1, g(a) = clamp(a*2^L + C[n]) is checked over its whole
// unclamped range.  Any failing channel leaves the stage on the float shape.
// Shape 7's add and sq1 act on codes: r0*s0 + c*s_res is an exact float when
// the bound below holds, so round((r0*s0 + c*s_res)/s1) is the integer
// half-away rounding of r0*2^a + c*2^b by 2^g (non-negative codes: +2^(g-1),
// then an arithmetic shift; negative sums saturate to 0 in the byte pack).
bool FastPlan::fold_integer(size_t si, int shape, double sxw, double acc_bound, kern::EpiConsts& e,
                            std::vector<std::shared_ptr<void>>& keep) {
  const Stage& st = *stages_[si];
  const double M = kern::kMagic;
  auto code_range = [](const kern::EpiSq& q, double& lo, double& hi) {
    lo = std::nearbyint(static_cast<double>(q.lo) + 0.5);
    hi = std::nearbyint(static_cast<double>(q.hi) - 0.5);
  };
  auto store_clamp = [&](const kern::EpiSq& q, double& lo, double& hi) {
    if (q.flags & kern::kEpiNoClamp) return;
    lo = std::max(lo, static_cast<double>(q.lo) - M);
    hi = std::min(hi, static_cast<double>(q.hi) - M);
  };
  auto log2_exact = [](double v, int& out) {
    int ex = 0;
    if (!(v > 0.0) || std::frexp(v, &ex) != 0.5) return false;
    out = ex - 1;
    return true;
  };
  const bool addfork = shape == kern::kShapeAddForkInt;
  double lo0, hi0;
  code_range(e.q[0], lo0, hi0);
  if (!addfork) {
    store_clamp(e.q[1], lo0, hi0);
    if (lo0 != 0.0 || hi0 < 0.0 || hi0 > 255.0) return false;
  } else if (lo0 < -32768.0 || hi0 > 32767.0 || lo0 > hi0) {
    return false;
  }
  const double inv0 = static_cast<double>(e.inv0);
  int ek = 0;
  if (!log2_exact(static_cast<double>(e.q[0].k), ek) || sxw * inv0 != static_cast<double>(e.q[0].k) ||
      ek > 20 || ek < -30) {
    return false;
  }
  const int m0 = ek >= 0 ? (1 << ek) : 1;
  const int r0 = ek >= 0 ? 0 : -ek;
  // the kernel shifts by multiply-high, which needs a shift >= 2: scale the
  // accumulator side by 2^sc0 (exact) where sq0's shift is shorter
  const int sc0 = r0 < 2 ? 2 - r0 : 0;
  // shape 7: add + sq1 constants
  double lo1 = 0.0, hi1 = 0.0;
  int k0 = 0, kr = 0, h1 = 0, r1 = 0;
  if (addfork) {
    code_range(e.q[1], lo1, hi1);
    store_clamp(e.q[2], lo1, hi1);
    int d0 = 0, dr = 0;
    if (lo1 != 0.0 || hi1 < 0.0 || hi1 > 255.0 || !log2_exact(static_cast<double>(e.q[1].k), d0) ||
        !log2_exact(static_cast<double>(e.ka), dr)) {
      return false;
    }
    const int mm = std::min(d0, dr);
    const double p0 = std::max(std::fabs(lo0), std::fabs(hi0));
    // the reference's float add r0*s0 + c*s_res must be exact (|sum| < 2^24 units)
    if (d0 - mm > 20 || dr - mm > 20 || p0 * std::ldexp(1.0, d0 - mm) + 128.0 * std::ldexp(1.0, dr - mm) >= 0x1p24) {
      return false;
    }
    if (mm >= 0) {
      if (d0 > 20 || dr > 20 || p0 * std::ldexp(1.0, d0) + 128.0 * std::ldexp(1.0, dr) >= 0x1p30) return false;
      k0 = 1 << d0;
      kr = 1 << dr;
    } else {
      if (-mm > 30) return false;
      k0 = 1 << (d0 - mm);
      kr = 1 << (dr - mm);
      r1 = -mm;
      h1 = 1 << (r1 - 1);
    }
  }
  // the folded-bias table, cached per (stage, sq0 grid, code range)
  struct Key {
    int shape, ek;
    double sxw, inv0, lo0, hi0;
  } key{shape, ek, sxw, inv0, lo0, hi0};
  std::string ks(reinterpret_cast<const char*>(&key), sizeof(key));
  auto ck = std::make_pair(static_cast<int>(si), ks);
  auto it = ctab_cache_.find(ck);
  static const bool dbg = std::getenv("QUANTC_DEBUG_INT") != nullptr;
  if (it == ctab_cache_.end()) {
    std::shared_ptr<void> dev;  // null: some channel is irregular
    const int O = st.O;
    const int nmask = (O + 511) / 512;  // one bit per 16-channel chunk
    // device layout: C[O], Tp[O], Tn[O], chunk mask words (kern::IntTable)
    std::vector<int32_t> tab(static_cast<size_t>(3 * O + nmask), 0);
    int32_t* C = tab.data();
    int32_t* Tp = C + O;
    int32_t* Tn = Tp + O;
    uint32_t* mask = reinterpret_cast<uint32_t*>(Tn + O);
    std::span<const float> bias;
    if (st.bias_const >= 0) bias = plan_.steps()[static_cast<size_t>(st.bias_const)].node->payload->floats();
    bool ok = O <= 8192;
    std::string why;
    int64_t cmax = 0;
    const int64_t lo = static_cast<int64_t>(lo0), hi = static_cast<int64_t>(hi0);
    for (int n = 0; n < O && ok; ++n) {
      const float b = bias.empty() ? 0.0f : bias[static_cast<size_t>(n)];
      // the reference's code of accumulator a (double sum + bias, one rounding
      // to float, then round half away on sq0's grid)
      auto f = [&](int64_t a) {
        const float v = static_cast<float>(static_cast<double>(a) * sxw + static_cast<double>(b));
        const double q = std::round(static_cast<double>(v) * inv0);
        return static_cast<int64_t>(std::min(std::max(q, lo0), hi0));
      };
      int64_t c = 0, tp = std::numeric_limits<int32_t>::max(), tn = std::numeric_limits<int32_t>::min();
      if (r0 > 0) {
        const int64_t N = int64_t{1} << r0;
        const double phi = -static_cast<double>(b) / sxw;  // exact (sxw a power of two)
        if (!(std::fabs(phi) < 0x1p40)) {
          ok = false;
          why = "bias/s out of range";
          break;
        }
        c = N / 2 - static_cast<int64_t>(std::ceil(phi));
        // Breakpoint k >= 1 sits at ceil((k - 1/2)N + phi - D) with D = N * 2^(p-24)
        // the fp32 half-spacing below k - 1/2 (binade p) in accumulator units;
        // k <= 0 at floor((k - 1/2)N + phi + D') + 1.  Both equal the regular
        // (k - 1/2)N + ceil(phi) when frac(phi) lies strictly between the
        // largest D and 1 - D' (or phi is an integer and no code is negative):
        // then only the extreme breakpoints are spot-checked.
        const double fr = phi - std::floor(phi);
        auto dmax = [&](double cabs) {
          return cabs < 0.5 ? 0.0 : std::ldexp(1.0, r0 + std::ilogb(cabs) - 24);
        };
        const double dp = hi >= 1 ? dmax(static_cast<double>(hi) - 0.5) : 0.0;
        const double dn = lo < 0 ? dmax(-static_cast<double>(lo) - 0.5) : 0.0;
        const bool regular = dp < 0.25 && dn < 0.25 &&
                             ((fr == 0.0 && lo >= 0) || (fr > 2.0 * dp && 1.0 - fr > 2.0 * dn));
        if (regular) {
          for (int64_t k : {lo + 1, hi}) {
            if (k <= lo || k > hi) continue;
            const int64_t A = k * N - c;
            if (f(A) != k || f(A - 1) != k - 1) {
              ok = false;
              why = "regular breakpoint check failed";
            }
          }
          cmax = std::max(cmax, c < 0 ? -c : c);
          C[n] = static_cast<int32_t>(c * (int64_t{1} << sc0));
          Tp[n] = std::numeric_limits<int32_t>::max();
          Tn[n] = std::numeric_limits<int32_t>::min();
          continue;
        }
        // exact breakpoints A_k (first a with f(a) >= k) next to the regular
        // ones k*N - c: the float rounding of the conv value moves them by at
        // most one, down for the large positive codes (bias just above a grid
        // point) and up for the large negative ones (or all negative codes
        // when half-way ties are reachable)
        int64_t kp = hi + 1, kn = lo;  // shifted ranges [kp, hi] (-1), (lo, kn] (+1)
        int64_t prev_shift = -2;
        for (int64_t k = lo + 1; k <= hi && ok; ++k) {
          int64_t a = k * N - c;
          int guard = 0;
          while (f(a - 1) >= k && guard++ < 4) --a;
          while (f(a) < k && guard++ < 8) ++a;
          const int64_t d = a - (k * N - c);
          if (guard >= 8 || d < -1 || d > 1 || f(a) != k || f(a - 1) != k - 1) {
            ok = false;
            why = "breakpoint moved by more than one";
            break;
          }
          // the shift pattern must be +1... 0... -1 (monotone in k)
          if (d > prev_shift && prev_shift != -2) {
            ok = false;
            why = "non-monotone breakpoint shifts";
            break;
          }
          prev_shift = d;
          if (d == 1) kn = k;
          if (d == -1 && kp > hi) kp = k;
        }
        if (!ok) break;
        if (kp <= hi) tp = kp * N - c - 1;   // a >= Tp: one step earlier
        if (kn > lo) tn = kn * N - c + 1;    // a <  Tn: one step later
        if (kp <= hi || kn > lo) mask[n / 512] |= 1u << ((n / 16) % 32);
        // the folded formula reproduces every breakpoint
        auto g = [&](int64_t a) {
          const int64_t x = a + c + (a >= tp ? 1 : 0) - (a < tn ? 1 : 0);
          return std::min(std::max(x >> r0, lo), hi);
        };
        for (int64_t k = lo + 1; k <= hi && ok; ++k) {
          const int64_t a = k * N - c + (k >= kp ? -1 : 0) + (k <= kn ? 1 : 0);
          ok = g(a) == k && g(a - 1) == k - 1;
        }
        if (!ok) why = "folded formula mismatch";
      } else {
        c = static_cast<int64_t>(std::round(static_cast<double>(b) * inv0));
        const int64_t alo = static_cast<int64_t>(std::floor((lo0 - static_cast<double>(c)) / m0)) - 1;
        const int64_t ahi = static_cast<int64_t>(std::ceil((hi0 - static_cast<double>(c)) / m0)) + 1;
        for (int64_t a = alo; a <= ahi && ok; ++a) {
          ok = f(a) == std::min(std::max(a * m0 + c, lo), hi);
        }
        if (!ok) why = "coarse grid mismatch";
      }
      cmax = std::max(cmax, c < 0 ? -c : c);
      C[n] = static_cast<int32_t>(c * (int64_t{1} << sc0));
      Tp[n] = static_cast<int32_t>(std::min<int64_t>(tp, std::numeric_limits<int32_t>::max()));
      Tn[n] = static_cast<int32_t>(std::max<int64_t>(tn, std::numeric_limits<int32_t>::min()));
    }
    if (ok) {
      dev = engine::device_alloc_on(ST(), tab.size() * sizeof(int32_t));
      // pageable source: staged before the call returns
      ok_cuda(cudaMemcpyAsync(dev.get(), tab.data(), tab.size() * sizeof(int32_t), cudaMemcpyHostToDevice,
                              ST()));
    }
    if (dbg) {
      int corr = 0;
      for (int w = 0; w < nmask; ++w) corr += __builtin_popcount(mask[w]);
      std::fprintf(stderr, "fold_integer stage %zu shape %d r0 %d m0 %d [%g, %g]: %s (%d chunks corrected)\n", si,
                   shape, r0, m0, lo0, hi0, ok ? "ok" : why.c_str(), corr);
    }
    it = ctab_cache_.emplace(ck, std::make_pair(dev, cmax)).first;
  }
  // no int32 overflow of (a*m0 + C) * 2^sc0 for any accumulator this run can reach
  if (!it->second.first ||
      (acc_bound * m0 + static_cast<double>(it->second.second) + 1.0) * std::ldexp(1.0, sc0) >= 0x1p31) {
    return false;
  }
  // shape 7: the second shift likewise made >= 2
  if (addfork && r1 < 2) {
    const int sc1 = 2 - r1;
    k0 <<= sc1;
    kr <<= sc1;
    h1 <<= sc1;
    r1 = 2;
  }
  if (addfork && std::max(std::fabs(lo0), std::fabs(hi0)) * k0 + 128.0 * kr + h1 >= 0x1p31) return false;
  keep.push_back(it->second.first);
  e.ctab = static_cast<const int32_t*>(it->second.first.get());
  e.i_m0 = m0 << sc0;
  e.i_r0 = r0 + sc0;
  e.i_cs = 1 << sc0;
  e.i_mh0 = static_cast<int32_t>(int64_t{1} << (32 - (r0 + sc0)));
  e.i_lo0 = static_cast<int32_t>(lo0);
  e.i_hi0 = static_cast<int32_t>(hi0);
  e.i_k0 = k0;
  e.i_kr = kr;
  e.i_h1 = h1;
  e.i_r1 = r1;
  e.i_mh1 = addfork ? static_cast<int32_t>(int64_t{1} << (32 - r1)) : 0;
  e.i_hi1 = static_cast<int32_t>(hi1);
  return true;
}

void* FastPlan::buf(const Run& r, int vid) const {
  const Val& v = *vals_[static_cast<size_t>(vid)];
  if (v.alias_root >= 0) return static_cast<char*>(buf(r, v.alias_root)) + v.col_off * 4;
  const int root = r.alias.empty() ? vid : r.alias[static_cast<size_t>(vid)];
  return arenas_[static_cast<size_t>(r.group)].bufs[static_cast<size_t>(root)].get();
}

void* FastPlan::arena_ptr(int group, int vid) const {
  const Val& v = *vals_[static_cast<size_t>(vid)];
  if (v.alias_root >= 0) return static_cast<char*>(arena_ptr(group, v.alias_root)) + v.col_off * 4;
  return arenas_[static_cast<size_t>(group)].bufs[static_cast<size_t>(vid)].get();
}

// weight codes of stage si under the run's binding (cached per FSq), and the
// tcgen05 launch spec of the stage for run r
void FastPlan::gemm_spec(Run& r, size_t si, kern::TcConvSpec& sp) {
  const Stage& st = *stages_[si];
  const Val& dv = *vals_[static_cast<size_t>(st.in_val)];
  const FSq wf = r.wfsq[si];
  std::string key(reinterpret_cast<const char*>(&wf), sizeof(FSq));
  auto ck = std::make_pair(static_cast<int>(si), key);
  auto it = wcache_.find(ck);
  if (it == wcache_.end()) {
    // codes [O][Kpad], then one int: max_o sum_k |code| (the accumulator bound)
    const size_t cbytes = static_cast<size_t>(st.O) * st.Kpad;
    auto codes = engine::device_alloc_on(ST(), cbytes + 16);
    if (st.s2d) {
      kern::weight_codes_s2d(plan_.constant(st.w_const).f(), static_cast<int8_t*>(codes.get()),
                             st.O, st.s2d_C, st.s2d_KH, st.s2d_KW, st.KH, st.KW, st.s2d_dh,
                             st.s2d_dw, st.Kpad, wf, ST());
    } else {
      kern::weight_codes_v2(plan_.constant(st.w_const).f(),
                            static_cast<int8_t*>(codes.get()), st.O,
                            st.dense ? (st.taps > 1 ? dv.cs : dv.C) : st.C, st.taps, st.ldk,
                            st.Kpad, wf, ST());
    }
    int* l1 = reinterpret_cast<int*>(static_cast<int8_t*>(codes.get()) + cbytes);
    ok_cuda(cudaMemsetAsync(l1, 0, sizeof(int), ST()));
    kern::weight_l1_max(static_cast<const int8_t*>(codes.get()), st.O, st.Kpad, l1, ST());
    it = wcache_.emplace(ck, codes).first;
    wcache_bytes_ += cbytes + 16;
  }
  r.keep.push_back(it->second);  // a cache clear must not free codes this run uses
  sp = kern::TcConvSpec{};
  sp.x = static_cast<const int8_t*>(buf(r, st.in_val));
  sp.lda = static_cast<int>(dv.ld);
  if (st.packed) {
    auto packed = engine::device_alloc_on(ST(), static_cast<size_t>(st.rows_out_ps * r.batch) * st.Kpad);
    kern::pack_im2col(sp.x, static_cast<int8_t*>(packed.get()), r.batch * st.n0, st.H, st.W,
                      st.C, static_cast<int>(dv.ld), st.KH, st.KW, st.sh, st.sw, st.ph,
                      st.pw, st.OH, st.OW, st.Ktrue, st.Kpad, ST());
    sp.x = static_cast<const int8_t*>(packed.get());
    sp.lda = st.Kpad;
    r.keep.push_back(packed);
  }
  sp.w = static_cast<const int8_t*>(it->second.get());
  sp.w_l1 = reinterpret_cast<const int*>(sp.w + static_cast<size_t>(st.O) * st.Kpad);
  sp.x_absmax = static_cast<int>(code_absmax(r.fsq[static_cast<size_t>(sq_index_.at(dv.sq_step))]));
  sp.M = st.rows_out_ps * r.batch;
  sp.O = st.O;
  sp.Kpad = st.Kpad;
  sp.gather = st.gather ? 1 : 0;
  sp.Ktrue = st.Ktrue;
  sp.Nimg = r.batch * st.n0;
  sp.H = st.H;
  sp.W = st.W;
  sp.C = st.C;
  sp.ld = static_cast<int>(dv.ld);
  sp.ldk = st.ldk;
  sp.KH = st.KH;
  sp.KW = st.KW;
  sp.sh = st.sh;
  sp.sw = st.sw;
  sp.ph = st.ph;
  sp.pw = st.pw;
  sp.OH = st.OH;
  sp.OW = st.OW;
  sp.bias = st.bias_const >= 0 ? plan_.constant(st.bias_const).f() : nullptr;
  sp.scale = r.sxw_of[si];
  sp.prog = ProgArgs{r.d_tabs + si, st.depth, r.shape_of[si]};
  sp.epi = r.epi_of[si];
  if (std::getenv("QUANTC_DUMP_PLAN")) {
    std::fprintf(stderr, "run stage %zu step %d shape %d -> %d flags %d %d %d %d ops", si,
                 st.step, r.shape0[si], sp.prog.shape, sp.epi.q[0].flags, sp.epi.q[1].flags,
                 sp.epi.q[2].flags, sp.epi.q[3].flags);
    for (int pc = 0; pc < r.tabs[si].n_code; ++pc) {
      const kern::ProgInstr& in = r.tabs[si].code[pc];
      std::fprintf(stderr, " %d", in.op);
      if (in.op == kern::kPSq || in.op == kern::kPSqStore8) {
        const FSq& f = r.tabs[si].sq[in.a];
        std::fprintf(stderr, "[zp%g acc%d pt%d q%g..%g s%g]", f.zp, f.has_acc, f.passthrough,
                     f.qmin, f.qmax, f.s);
      }
    }
    std::fprintf(stderr, "\n");
  }
  sp.acc_bound = r.acc_bound[si];
  sp.n_out = r.drop2[si] ? 1 : st.n_out;
  for (int o = 0; o < sp.n_out; ++o) {
    const Val& ov = *vals_[static_cast<size_t>(st.out_vals[o])];
    sp.out_ptr[o] = buf(r, st.out_vals[o]);
    sp.out_cols[o] = ov.C;
    sp.out_ld[o] = ov.ld;
  }
  if (st.res_val >= 0) {
    const Val& rv = *vals_[static_cast<size_t>(st.res_val)];
    sp.res_ptr = buf(r, st.res_val);
    sp.res_cols = rv.C;
    sp.res_ld = rv.ld;
    sp.res_alias = sp.prog.shape == kern::kShapeAddForkInt && sp.n_out == 1 && sp.epi.slot_res == 0 &&
                           sp.epi.slot_out[0] == 0
                       ? 1
                       : 0;
  }
  sp.groups = 1;
}

void FastPlan::launch_gemm(size_t si, const kern::TcConvSpec& sp) {
  const Stage& st = *stages_[si];
  const bool prof = device::profile_enabled();
  if (prof) device::profile_gemm_begin();
  kern::tc_conv(sp, ST());
  if (prof) {
    // algorithmic bytes: input codes once (the NHWC tensor for implicit
    // GEMM), weight codes, bias, code outputs / residual / fp32 outputs
    const double M = static_cast<double>(sp.M) * sp.groups;
    const double a_bytes = st.gather ? static_cast<double>(sp.Nimg) * sp.groups * st.H * st.W * sp.ld
                                     : M * st.Ktrue;
    const double out_bytes = M * st.O * (sp.n_out + (st.res_val >= 0 ? 1 : 0)) +
                             (sp.prog.shape == kern::kShapeAddF32 || sp.prog.shape == kern::kShapeSqF32
                                  ? 4.0 * M * st.O
                                  : 0.0);
    device::profile_gemm_end(
        2.0 * M * st.O *
            (st.dense ? st.Ktrue
                      : (st.s2d ? st.s2d_C * st.s2d_KH * st.s2d_KW : st.C * st.KH * st.KW)),
        a_bytes + static_cast<double>(st.O) * st.Ktrue * sp.groups + 4.0 * st.O + out_bytes);
  }
  device::counters().tcgen05_gemms++;
}

void FastPlan::run_stage(Run& r, size_t si) {
  const Stage& st = *stages_[si];
  ProgArgs pa{r.d_tabs + si, st.depth, r.shape0[si]};
  const int batch = r.batch;
  switch (st.kind) {
    case Stage::kInput: {
      const Val* sv = nullptr;
      for (int vid : st.buf_vals) {
        if (vals_[static_cast<size_t>(vid)]->s2d) sv = vals_[static_cast<size_t>(vid)].get();
      }
      if (sv) {
        // compile guarantees the program is the single store into the s2d value
        if (st.code.size() != 1 || st.code[0].op != kern::kPSqStore8) {
          throw EvalError("fastplan: space-to-depth input stage with a compound program");
        }
        kern::stage_input_s2d(r.inputs.at(static_cast<size_t>(st.input_k)), batch * st.n0,
                              sv->s2d_C, sv->s2d_H, sv->s2d_W, r.tabs[si].sq[st.code[0].a],
                              static_cast<int8_t*>(buf(r, st.buf_vals[0])), ST());
        break;
      }
      kern::stage_input(r.inputs.at(static_cast<size_t>(st.input_k)), batch * st.n0, st.C, st.HW,
                        pa, ST());
      break;
    }
    case Stage::kMaxpool: {
      const Val& v = *vals_[static_cast<size_t>(st.in_val)];
      kern::PoolStores ps;
      if (st.C % 16 == 0 && v.ld % 16 == 0 && st.ph < st.pkh && st.pw < st.pkw &&
          pool_stores(r.tabs[si], r.scale_by_step.at(v.sq_step), ps)) {
        if (!r.pool_drop2.empty() && r.pool_drop2[si]) ps.n_out = 1;
        kern::stage_maxpool_stores(static_cast<const int8_t*>(buf(r, st.in_val)),
                                   static_cast<int>(v.ld), batch * st.n0, st.C, st.H, st.W, st.OH,
                                   st.OW, st.pkh, st.pkw, st.sh, st.sw, st.ph, st.pw, ps, ST());
        break;
      }
      kern::stage_maxpool(static_cast<const int8_t*>(buf(r, st.in_val)),
                          static_cast<int>(v.ld), r.scale_by_step.at(v.sq_step), batch * st.n0,
                          st.C, st.H, st.W, st.OH, st.OW, st.pkh, st.pkw, st.sh, st.sw, st.ph,
                          st.pw, pa, ST());
      break;
    }
    case Stage::kGap: {
      const Val& v = *vals_[static_cast<size_t>(st.in_val)];
      kern::stage_gap(static_cast<const float*>(buf(r, st.in_val)), v.ld, batch * st.n0, st.C,
                      st.HW, pa, ST());
      break;
    }
    case Stage::kAvg: {
      const Val& v = *vals_[static_cast<size_t>(st.in_val)];
      const double wk = static_cast<double>(static_cast<float>(1.0 / (st.pkh * st.pkw)));
      kern::stage_avgpool_f32(static_cast<const float*>(buf(r, st.in_val)), static_cast<int>(v.ld),
                              batch * st.n0, st.C, st.H, st.W, st.OH, st.OW, st.pkh, st.pkw, st.sh,
                              st.sw, st.ph, st.pw, wk, pa, inline_store_program(r.tabs[si]), ST());
      break;
    }
    case Stage::kCat: {
      const Val& v = *vals_[static_cast<size_t>(st.in_val)];
      const kern::ProgBuf src{buf(r, st.in_val), v.ld, 1, 0, 1, 1.0f, -1, 0};
      kern::stage_ew(src, batch * v.rows_ps, v.C, pa, ST());
      break;
    }
    case Stage::kDw: {
      // weight codes [tap][ldk] under this binding's weight sq (cached like
      // the GEMM stages'), then one CUDA-core launch
      const FSq wf = r.wfsq[si];
      std::string key(reinterpret_cast<const char*>(&wf), sizeof(FSq));
      auto ck = std::make_pair(static_cast<int>(si), key);
      auto it = wcache_.find(ck);
      if (it == wcache_.end()) {
        // codes [tap][ldk], then the tap quads [ceil(taps/4)][ldk] words after them
        const size_t cbytes = static_cast<size_t>(st.Kpad);
        const size_t qoff = (cbytes + 15) / 16 * 16;
        const size_t qbytes = static_cast<size_t>((st.taps + 3) / 4) * st.ldk * 4;
        auto codes = engine::device_alloc_on(ST(), qoff + qbytes + 16);
        kern::weight_codes_v2(plan_.constant(st.w_const).f(), static_cast<int8_t*>(codes.get()), 1, st.C,
                              st.taps, st.ldk, st.Kpad, wf, ST());
        kern::dw_weight_quads(static_cast<const int8_t*>(codes.get()), st.taps, st.ldk,
                              reinterpret_cast<int32_t*>(static_cast<int8_t*>(codes.get()) + qoff), ST());
        it = wcache_.emplace(ck, codes).first;
        wcache_bytes_ += qoff + qbytes + 16;
      }
      const size_t qoff = (static_cast<size_t>(st.Kpad) + 15) / 16 * 16;
      const Val& dv = *vals_[static_cast<size_t>(st.in_val)];
      const float sxw = r.scale_by_step.at(dv.sq_step) * wf.s;  // pow2 x pow2: exact
      // [passthrough accumulator sq,] sq_store8 into plain code rows: inline
      const kern::DwFast fast = inline_store_program(r.tabs[si]);
      kern::stage_dw_conv(static_cast<const int8_t*>(buf(r, st.in_val)), static_cast<int>(dv.ld),
                          batch * st.n0, st.C, st.H, st.W, st.KH, st.KW, st.sh, st.sw, st.ph, st.pw,
                          st.OH, st.OW,
                          reinterpret_cast<const int32_t*>(static_cast<const int8_t*>(it->second.get()) + qoff), st.ldk,
                          st.bias_const >= 0 ? plan_.constant(st.bias_const).f() : nullptr, sxw, pa, fast, ST());
      break;
    }
    case Stage::kGemm: {
      kern::TcConvSpec sp;
      gemm_spec(r, si, sp);
      launch_gemm(si, sp);
      break;
    }
  }
}

void FastPlan::finish(Run& r) {
  const float* out = static_cast<const float*>(buf(r, out_val_));
  kern::argmax_rows(out, r.batch, out_per_sample_, r.d_preds, ST());
  if (r.d_scores) {
    ok_cuda(cudaMemcpyAsync(r.d_scores, out, static_cast<size_t>(r.batch) * out_per_sample_ * 4,
                            cudaMemcpyDeviceToDevice, ST()));
  }
  device::counters().fused_batches++;
}

// Weight codes depend only on (stage, weight sq parameters): for a search
// that is (layer, bit-width), a handful of variants per layer.  They are
// kept resident up to QUANTC_WCACHE_MB (default 4096 MB of HBM), so after the
// first visit of each bit-width no candidate re-quantizes its weights
// (ResNet-50: 25.5 MB of codes per variant set).  Over budget the cache is
// dropped (stream-ordered frees: in-flight launches keep their codes).
void FastPlan::trim_weight_cache() {
  static const size_t budget = [] {
    const char* e = std::getenv("QUANTC_WCACHE_MB");
    return static_cast<size_t>(e ? std::max(1, std::atoi(e)) : 4096) << 20;
  }();
  if (wcache_bytes_ > budget) {
    wcache_.clear();
    wcache_bytes_ = 0;
  }
}

void FastPlan::predict(int batch, const std::vector<const float*>& inputs,
                       const SimBinding* binding, int64_t* d_preds, float* d_scores) {
  static const bool hprof = std::getenv("QUANTC_HOST_PROF") != nullptr;
  const auto t_start = std::chrono::steady_clock::now();
  // weight codes are cached per (stage, weight sq parameters); a long search
  // visits many weight bit-widths, so keep roughly the last few bindings
  // (freed stream-ordered: in-flight launches keep their codes)
  trim_weight_cache();
  Run r;
  r.group = 0;
  r.batch = batch;
  r.inputs = inputs;
  r.binding = binding;
  r.d_preds = d_preds;
  r.d_scores = d_scores;
  prepare(r);
  const auto t_prep = std::chrono::steady_clock::now();
  for (size_t si = 0; si < stages_.size(); ++si) run_stage(r, si);
  finish(r);
  if (hprof) {
    auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    std::fprintf(stderr, "predict host us: tables+upload %.1f launches %.1f\\n", us(t_start, t_prep),
                 us(t_prep, std::chrono::steady_clock::now()));
  }
}

// Several bindings (<= kern::kMaxGroups) over the same batch of samples in
// one pass: every GEMM stage whose specs are launch-compatible across the
// bindings runs as ONE grouped tcgen05 launch (G times the tiles: the
// per-layer pipeline fill / drain and launch latency are paid once); other
// stages run per binding.  Each binding has its own arena, tables and
// outputs, so results equal separate predict() calls.
void FastPlan::predict_group(int batch, const std::vector<const float*>& inputs,
                             const std::vector<const SimBinding*>& bindings,
                             const std::vector<int64_t*>& preds,
                             const std::vector<float*>* scores) {
  const int G = static_cast<int>(bindings.size());
  if (G < 1 || G > kern::kMaxGroups) throw std::logic_error("predict_group: 1..kMaxGroups bindings");
  trim_weight_cache();
  std::vector<Run> r(static_cast<size_t>(G));
  for (int g = 0; g < G; ++g) {
    r[g].group = g;
    r[g].batch = batch;
    r[g].inputs = inputs;
    r[g].binding = bindings[g];
    r[g].d_preds = preds[g];
    prepare(r[g]);
  }
  static const bool no_group = std::getenv("QUANTC_NO_GROUPED") != nullptr;
  std::vector<kern::TcConvSpec> sp(static_cast<size_t>(G));
  for (size_t si = 0; si < stages_.size(); ++si) {
    if (stages_[si]->kind == Stage::kInput && G > 1) {
      // space-to-depth input of all bindings in one launch (one read of the images)
      const Stage& st = *stages_[si];
      const Val* sv = nullptr;
      for (int vid : st.buf_vals) {
        if (vals_[static_cast<size_t>(vid)]->s2d) sv = vals_[static_cast<size_t>(vid)].get();
      }
      if (sv && st.code.size() == 1 && st.code[0].op == kern::kPSqStore8 && sv->s2d_C <= 4) {
        std::vector<FSq> ps(static_cast<size_t>(G));
        std::vector<int8_t*> outs(static_cast<size_t>(G));
        for (int g = 0; g < G; ++g) {
          ps[g] = r[g].tabs[si].sq[st.code[0].a];
          outs[g] = static_cast<int8_t*>(buf(r[g], st.buf_vals[0]));
        }
        kern::stage_input_s2d_multi(r[0].inputs.at(static_cast<size_t>(st.input_k)), batch * st.n0,
                                    sv->s2d_C, sv->s2d_H, sv->s2d_W, ps.data(), outs.data(), G, ST());
        continue;
      }
    }
    if (stages_[si]->kind != Stage::kGemm) {
      for (int g = 0; g < G; ++g) run_stage(r[g], si);
      continue;
    }
    for (int g = 0; g < G; ++g) gemm_spec(r[g], si, sp[g]);
    // bindings whose specs are launch-compatible (same epilogue shape, output
    // count, residual and A layout) share one launch
    std::vector<char> launched(static_cast<size_t>(G), 0);
    for (int g0 = 0; g0 < G; ++g0) {
      if (launched[g0]) continue;
      kern::TcConvSpec& head = sp[g0];
      launched[g0] = 1;
      const int sh = head.prog.shape;
      const bool shape_kernel = sh != kern::kShapeGeneric && sh != kern::kShapeInt;
      head.groups = 1;
      for (int g = g0 + 1; g < G && !no_group && shape_kernel; ++g) {
        const kern::TcConvSpec& o = sp[g];
        if (launched[g] || o.prog.shape != sh || o.n_out != head.n_out ||
            (o.res_ptr != nullptr) != (head.res_ptr != nullptr) || o.res_alias != head.res_alias ||
            o.lda != head.lda) {
          continue;
        }
        launched[g] = 1;
        const int k = head.groups - 1;
        head.xg[k] = o.x;
        head.wg[k] = o.w;
        head.w_l1g[k] = o.w_l1;
        head.x_absmaxg[k] = o.x_absmax;
        head.scaleg[k] = o.scale;
        head.out_ptrg[k][0] = o.out_ptr[0];
        head.out_ptrg[k][1] = o.out_ptr[1];
        head.res_ptrg[k] = o.res_ptr;
        head.epig[k] = o.epi;
        head.acc_bound = std::max(head.acc_bound, o.acc_bound);
        ++head.groups;
      }
      launch_gemm(si, head);
    }
  }
  // one argmax launch for the group's outputs (finish() per binding otherwise)
  std::vector<const float*> outs(static_cast<size_t>(G));
  for (int g = 0; g < G; ++g) outs[g] = static_cast<const float*>(buf(r[g], out_val_));
  kern::argmax_rows_multi(outs.data(), preds.data(), G, batch, out_per_sample_, ST());
  if (scores) {
    for (int g = 0; g < G; ++g) {
      if (!(*scores)[g]) continue;
      ok_cuda(cudaMemcpyAsync((*scores)[g], outs[g], static_cast<size_t>(batch) * out_per_sample_ * 4,
                              cudaMemcpyDeviceToDevice, ST()));
    }
  }
  device::counters().fused_batches += G;
}

}  // namespace quantc::fast
