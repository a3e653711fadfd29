/* ORACLE TEST INFRASTRUCTURE — see quantc_oracle.h.  Straight-line scalar C,
 * sequential loops in the reference's order, no vectorisation, no FMA
 * contraction (compiled with -O2 for x86-64 baseline, like the reference). */
#include "quantc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static double clampd(double v, double lo, double hi) {
  return (v < lo) ? lo : ((hi < v) ? hi : v); /* std::clamp */
}

/* simulate.cpp:12-25 + :64-78 */
float orc_sim_quant(float x, double threshold, int bit, int sign, int64_t zero_point,
                    int passthrough, int has_acc, double acc_lo, double acc_hi) {
  double v = (double)x;
  if (has_acc) v = clampd(v, acc_lo, acc_hi);
  if (passthrough) return (float)v;
  double s = threshold / exp2((double)(bit - sign));
  int64_t qmin = sign == 1 ? -((int64_t)1 << (bit - 1)) : 0;
  int64_t qmax = sign == 1 ? ((int64_t)1 << (bit - 1)) - 1 : ((int64_t)1 << bit) - 1;
  double q = round(v / s) + (double)zero_point;
  q = clampd(q, (double)qmin, (double)qmax);
  return (float)((q - (double)zero_point) * s);
}

void orc_sim_quant_array(const float* x, float* y, int64_t n, double threshold, int bit,
                         int sign, int64_t zero_point, int passthrough, int has_acc,
                         double acc_lo, double acc_hi) {
  for (int64_t i = 0; i < n; ++i) {
    y[i] = orc_sim_quant(x[i], threshold, bit, sign, zero_point, passthrough, has_acc, acc_lo,
                         acc_hi);
  }
}

/* calibration.cpp:28-33 */
int orc_bin_index(double a, double absmax, int bins) {
  if (a <= 0.0) return 0;
  double x = a / absmax * (double)bins;
  int idx = (int)ceil(x) - 1;
  return idx < 0 ? 0 : (idx > bins - 1 ? bins - 1 : idx);
}

/* calibration.cpp:97-105 */
void orc_histogram(const float* x, int64_t n, double absmax, int bins, int64_t* counts) {
  for (int64_t i = 0; i < n; ++i) {
    double a = fabs((double)x[i]);
    counts[absmax > 0.0 ? orc_bin_index(a, absmax, bins) : 0]++;
  }
}

/* calibration.cpp:121-134 (absmax > 0, total > 0 assumed) */
double orc_threshold_quantile(const int64_t* counts, int bins, double absmax, double q) {
  int64_t total = 0, cum = 0;
  for (int b = 0; b < bins; ++b) total += counts[b];
  for (int b = 0; b < bins; ++b) {
    cum += counts[b];
    if ((double)cum >= q * (double)total) return absmax * ((double)(b + 1) / (double)bins);
  }
  return absmax;
}

/* calibration.cpp:140-157 */
static double kl_divergence(double* p, double* q, int n) {
  double p_sum = 0.0, q_sum = 0.0, kl = 0.0;
  for (int i = 0; i < n; ++i) {
    if (p[i] == 0.0) p[i] = 1e-9;
    if (q[i] == 0.0) q[i] = 1e-9;
  }
  for (int i = 0; i < n; ++i) p_sum += p[i];
  for (int i = 0; i < n; ++i) q_sum += q[i];
  for (int i = 0; i < n; ++i) {
    double pi = p[i] / p_sum;
    double qi = q[i] / q_sum;
    kl += pi * log(pi / qi);
  }
  return kl;
}

/* calibration.cpp:161-206 */
int orc_kl_best_index(const int64_t* counts, int bins, int target_bit, double* best_kl_out) {
  int levels = 1 << target_bit;
  double best_kl = INFINITY;
  int best_i = levels;
  double* p = (double*)malloc(sizeof(double) * (size_t)bins);
  double* q = (double*)malloc(sizeof(double) * (size_t)bins);
  for (int i = levels; i <= bins; ++i) {
    for (int b = 0; b < i; ++b) p[b] = (double)counts[b];
    for (int b = i; b < bins; ++b) p[i - 1] += (double)counts[b];
    memset(q, 0, sizeof(double) * (size_t)i);
    int merged = i / levels;
    for (int j = 0; j < levels; ++j) {
      int start = j * merged;
      int end = (j == levels - 1) ? i : (j + 1) * merged;
      double sum = 0.0;
      int nonzero = 0;
      for (int b = start; b < end; ++b) {
        sum += p[b];
        if (p[b] != 0.0) ++nonzero;
      }
      if (nonzero == 0) continue;
      double value = sum / (double)nonzero;
      for (int b = start; b < end; ++b) {
        if (p[b] != 0.0) q[b] = value;
      }
    }
    double kl = kl_divergence(p, q, i);
    if (kl < best_kl) {
      best_kl = kl;
      best_i = i;
    }
  }
  free(p);
  free(q);
  if (best_kl_out) *best_kl_out = best_kl;
  return best_i;
}

/* interpreter.cpp:218-234, generalised to groups (op-set extension: output
 * channel o reads the C/G input channels of group o / (O/G); weight
 * [O][C/G][KH][KW]).  groups == 1 is the reference loop verbatim. */
void orc_conv2d_grouped_f64acc(const float* x, const float* w, const float* bias, float* y,
                               int N, int C, int H, int W, int O, int KH, int KW, int sh, int sw,
                               int ph, int pw, int groups) {
  int OH = (H + 2 * ph - KH) / sh + 1, OW = (W + 2 * pw - KW) / sw + 1;
  int Cg = C / groups, Og = O / groups;
  for (int64_t n = 0; n < N; ++n)
    for (int64_t o = 0; o < O; ++o)
      for (int64_t oh = 0; oh < OH; ++oh)
        for (int64_t ow = 0; ow < OW; ++ow) {
          double acc = 0.0;
          int64_t cb = (o / Og) * Cg;
          for (int64_t c = 0; c < Cg; ++c)
            for (int64_t kh = 0; kh < KH; ++kh)
              for (int64_t kw = 0; kw < KW; ++kw) {
                int64_t ih = oh * sh - ph + kh, iw = ow * sw - pw + kw;
                if (ih < 0 || ih >= H || iw < 0 || iw >= W) continue;
                acc += (double)x[((n * C + cb + c) * H + ih) * W + iw] *
                       (double)w[((o * Cg + c) * KH + kh) * KW + kw];
              }
          if (bias) acc += (double)bias[o];
          y[((n * O + o) * OH + oh) * OW + ow] = (float)acc;
        }
}

void orc_conv2d_f64acc(const float* x, const float* w, const float* bias, float* y, int N,
                       int C, int H, int W, int O, int KH, int KW, int sh, int sw, int ph,
                       int pw) {
  orc_conv2d_grouped_f64acc(x, w, bias, y, N, C, H, W, O, KH, KW, sh, sw, ph, pw, 1);
}

/* avg_pool2d (op-set extension): the reference conv2d loop on the constant
 * depthwise rewrite — double sum over in-bounds taps of x * fl32(1/(KH*KW)) */
void orc_avg_pool2d(const float* x, float* y, int N, int C, int H, int W, int KH, int KW, int sh,
                    int sw, int ph, int pw) {
  int OH = (H + 2 * ph - KH) / sh + 1, OW = (W + 2 * pw - KW) / sw + 1;
  double wk = (double)(float)(1.0 / ((double)KH * KW));
  for (int64_t nc = 0; nc < (int64_t)N * C; ++nc)
    for (int64_t oh = 0; oh < OH; ++oh)
      for (int64_t ow = 0; ow < OW; ++ow) {
        double acc = 0.0;
        for (int64_t kh = 0; kh < KH; ++kh)
          for (int64_t kw = 0; kw < KW; ++kw) {
            int64_t ih = oh * sh - ph + kh, iw = ow * sw - pw + kw;
            if (ih < 0 || ih >= H || iw < 0 || iw >= W) continue;
            acc += (double)x[(nc * H + ih) * W + iw] * wk;
          }
        y[(nc * OH + oh) * OW + ow] = (float)acc;
      }
}

/* interpreter.cpp global_avg_pool2d: sequential double sum / (double)(H*W) */
void orc_global_avg_pool2d(const float* x, float* y, int NC, int HW) {
  for (int64_t i = 0; i < NC; ++i) {
    double acc = 0.0;
    for (int64_t k = 0; k < HW; ++k) acc += (double)x[i * HW + k];
    y[i] = (float)(acc / (double)HW);
  }
}

/* interpreter.cpp:244-263 */
int64_t orc_conv2d_int(const int32_t* x, const int32_t* w, const int32_t* bias, int32_t* y,
                       int N, int C, int H, int W, int O, int KH, int KW, int sh, int sw,
                       int ph, int pw, int64_t zp0, int64_t zp1, int64_t acc_min,
                       int64_t acc_max) {
  int OH = (H + 2 * ph - KH) / sh + 1, OW = (W + 2 * pw - KW) / sw + 1;
  int64_t flat = 0, first = -1;
  for (int64_t n = 0; n < N; ++n)
    for (int64_t o = 0; o < O; ++o)
      for (int64_t oh = 0; oh < OH; ++oh)
        for (int64_t ow = 0; ow < OW; ++ow, ++flat) {
          int64_t acc = 0;
          for (int64_t c = 0; c < C; ++c)
            for (int64_t kh = 0; kh < KH; ++kh)
              for (int64_t kw = 0; kw < KW; ++kw) {
                int64_t ih = oh * sh - ph + kh, iw = ow * sw - pw + kw;
                if (ih < 0 || ih >= H || iw < 0 || iw >= W) continue;
                acc += ((int64_t)x[((n * C + c) * H + ih) * W + iw] - zp0) *
                       ((int64_t)w[((o * C + c) * KH + kh) * KW + kw] - zp1);
              }
          if (bias) acc += bias[o];
          if (acc < acc_min || acc > acc_max) {
            if (first < 0) first = flat;
            acc = acc < acc_min ? acc_min : acc_max;
          }
          y[((n * O + o) * OH + oh) * OW + ow] = (int32_t)acc;
        }
  return first;
}

/* interpreter.cpp:32-37, :477-480 */
void orc_requantize(const int32_t* x, int32_t* y, int64_t n, int64_t mult, int shift,
                    int64_t in_zp, int64_t out_zp, int64_t qmin, int64_t qmax) {
  for (int64_t i = 0; i < n; ++i) {
    int64_t v = (int64_t)x[i] - in_zp;
    int64_t p = v * mult;
    int64_t r;
    if (shift == 0) {
      r = p;
    } else {
      int64_t nudge = (int64_t)1 << (shift - 1);
      r = p >= 0 ? (p + nudge) >> shift : -((-p + nudge) >> shift);
    }
    int64_t q = r + out_zp;
    y[i] = (int32_t)(q < qmin ? qmin : (q > qmax ? qmax : q));
  }
}
