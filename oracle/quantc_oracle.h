/* ORACLE TEST INFRASTRUCTURE — plain-C restatement of the reference's
 * arithmetic on the calibrate-and-search path.  Used only by tests/, smoke()
 * and bench.py's cpu_baseline leg, as a checker.  Each function cites the
 * reference lines it restates (paths under /root/reference/proj/src).
 * Pinned against the compiled reference (oracle/_ref) by
 * tests/test_oracle.py. */
#ifndef QUANTC_ORACLE_H_
#define QUANTC_ORACLE_H_

#include <stdint.h>

/* simulate.cpp:64-78 — has_acc/acc_lo/acc_hi already multiplied out */
float orc_sim_quant(float x, double threshold, int bit, int sign, int64_t zero_point,
                    int passthrough, int has_acc, double acc_lo, double acc_hi);
void orc_sim_quant_array(const float* x, float* y, int64_t n, double threshold, int bit,
                         int sign, int64_t zero_point, int passthrough, int has_acc,
                         double acc_lo, double acc_hi);

/* calibration.cpp:28-33 and :97-105 (absmax > 0 path; absmax <= 0 -> bin 0) */
int orc_bin_index(double a, double absmax, int bins);
void orc_histogram(const float* x, int64_t n, double absmax, int bins, int64_t* counts);

/* calibration.cpp:121-134 */
double orc_threshold_quantile(const int64_t* counts, int bins, double absmax, double q);

/* calibration.cpp:138-206 — returns best_i (threshold = absmax*best_i/bins) */
int orc_kl_best_index(const int64_t* counts, int bins, int target_bit, double* best_kl);

/* interpreter.cpp:210-236 (dense = conv with H=W=KH=KW=1) */
void orc_conv2d_grouped_f64acc(const float* x, const float* w, const float* bias, float* y,
                               int N, int C, int H, int W, int O, int KH, int KW, int sh, int sw,
                               int ph, int pw, int groups);
void orc_avg_pool2d(const float* x, float* y, int N, int C, int H, int W, int KH, int KW, int sh,
                    int sw, int ph, int pw);
void orc_global_avg_pool2d(const float* x, float* y, int NC, int HW);
void orc_conv2d_f64acc(const float* x, const float* w, const float* bias, float* y, int N,
                       int C, int H, int W, int O, int KH, int KW, int sh, int sw, int ph,
                       int pw);

/* interpreter.cpp:238-264 with clamp_or_trap :25-29; returns the first
 * overflowing flat index (trap semantics) or -1, output saturated */
int64_t orc_conv2d_int(const int32_t* x, const int32_t* w, const int32_t* bias, int32_t* y,
                       int N, int C, int H, int W, int O, int KH, int KW, int sh, int sw,
                       int ph, int pw, int64_t zp0, int64_t zp1, int64_t acc_min,
                       int64_t acc_max);

/* interpreter.cpp:32-37 and :464-482 */
void orc_requantize(const int32_t* x, int32_t* y, int64_t n, int64_t mult, int shift,
                    int64_t in_zp, int64_t out_zp, int64_t qmin, int64_t qmax);

#endif
