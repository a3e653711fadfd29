/*
 * quantc_cuda.h — the thin C-ABI between the quantc C++ host and the sm_100a
 * kernels (north_star: "The host side stays C++ and calls CUDA through a thin
 * C-ABI layer").  Plain device pointers, sizes and an explicit cudaStream_t
 * (passed as void*, NULL = the engine stream, (void*)1 = cudaStreamLegacy,
 * i.e. the legacy default stream); status codes as in
 * quantc_capi.h, message via qc_last_error().
 *
 * Each entry point replaces one hot loop of the reference CPU implementation:
 *   qcu_sim_quant        simulate.cpp:64-87     simulated_quantize over a tensor
 *   qcu_minmax           calibration.cpp:70-79  per-edge exact extrema
 *   qcu_histogram        calibration.cpp:97-105 |v| histogram against absmax
 *   qcu_kl_sweep         calibration.cpp:161-206 KL threshold sweep, many edges
 *   qcu_conv2d_f64acc    interpreter.cpp:210-236 fp32 conv/dense, double acc
 *   qcu_conv2d_int       interpreter.cpp:238-264 integer conv/dense + clamp/trap
 *   qcu_requantize       interpreter.cpp:464-482 fixed-point requantize
 *   qcu_gemm_s8          int8 x int8 -> int32 on tcgen05 with the fused
 *                        sim-quant conv epilogue (y = float(acc*scale+bias))
 */
#ifndef QUANTC_CUDA_H_
#define QUANTC_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#include "quantc_capi.h"

#ifdef __cplusplus
extern "C" {
#endif

/* x, y: float32 device buffers of n elements (y may alias x). */
int qcu_sim_quant(const float* x, float* y, int64_t n, const qc_qparams* p, void* stream);

/* out_minmax: 2 doubles on the device (min, max) of the n values. */
int qcu_minmax(const float* x, int64_t n, double* out_minmax, void* stream);

/* counts: `bins` uint64 on the device, accumulated (+=) */
int qcu_histogram(const float* x, int64_t n, double absmax, int bins, uint64_t* counts,
                  void* stream);

/* counts: [n_edges][bins] int64 on the device; best_i (int32) and best_kl
 * (double) per edge on the device.  threshold = absmax * best_i / bins. */
int qcu_kl_sweep(const int64_t* counts, int n_edges, int bins, int target_bit, int* best_i,
                 double* best_kl, void* stream);

/* NCHW x [N,C,H,W], OIHW w, bias [O] (may be NULL), y [N,O,OH,OW]; dense is
 * H=W=KH=KW=1. */
int qcu_conv2d_f64acc(const float* x, const float* w, const float* bias, float* y, int N, int C,
                      int H, int W, int O, int KH, int KW, int sh, int sw, int ph, int pw,
                      void* stream);

/* Op-set extension (no reference counterpart — the
 * semantics are those of the exact rewrites the reference does run,
 * fixtures.py / tests/test_rewrites.py):
 *   qcu_conv2d_grouped_f64acc  conv2d with `groups` (weight [O][C/G][KH][KW]),
 *                              the interpreter.cpp:210-236 double accumulator
 *                              over the group's channels
 *   qcu_avg_pool2d_f32         double sum of x * fl32(1/(KH*KW)) over in-bounds
 *                              taps (count_include_pad), one rounding */
int qcu_conv2d_grouped_f64acc(const float* x, const float* w, const float* bias, float* y, int N,
                              int C, int H, int W, int O, int KH, int KW, int sh, int sw, int ph,
                              int pw, int groups, void* stream);
int qcu_avg_pool2d_f32(const float* x, float* y, int N, int C, int H, int W, int KH, int KW,
                       int sh, int sw, int ph, int pw, void* stream);

/* int32-storage operands; acc_dtype QC_I16/QC_I32; trap != 0 reports the
 * lowest overflowing flat index through *overflow_flat (-1 if none). */
int qcu_conv2d_int(const int32_t* x, const int32_t* w, const int32_t* bias, int32_t* y, int N,
                   int C, int H, int W, int O, int KH, int KW, int sh, int sw, int ph, int pw,
                   int64_t zp0, int64_t zp1, int acc_dtype, int trap, int64_t* overflow_flat,
                   void* stream);

int qcu_requantize(const int32_t* x, int32_t* y, int64_t n, int64_t multiplier, int shift,
                   int64_t in_zp, int64_t out_zp, int64_t qmin, int64_t qmax, void* stream);

/* A [M][K], B [N][K] int8 row-major (K multiple of 128); y float NCHW with
 * OHW pixels per image: y[(m/OHW)*N + n][m%OHW] = float(acc*scale + bias[n]). */
int qcu_gemm_s8(const int8_t* A, const int8_t* B, int M, int N, int K, double scale,
                const float* bias, float* y, int OHW, void* stream);

/* per-row argmax of x [rows][cols] with the reference argmax_class
 * semantics (interpreter.cpp:533-541: first maximum, strict '>', NaN never
 * taken, NaN at index 0 wins); grouped > 0 runs the grouped-candidate kernel
 * over that many equal row groups */
int qcu_argmax_rows(const float* x, int rows, int64_t cols, int grouped, int64_t* out,
                    void* stream);
int qcu_synchronize(void* stream);
const char* qcu_last_error(void);
/* 1 when the tcgen05 path can run on the current device */
int qcu_tcgen05_available(void);
/* engine mode for sim-quant evaluation: 0 exact, 1 fast, 2 auto */
int qcu_set_engine_mode(int mode);
/* the engine's cudaStream_t (for CUDA-event timing of engine work) */
void* qcu_engine_stream(void);
/* per-GEMM CUDA-event profiling of the engine's tcgen05 launches */
int qcu_profile_enable(int on);
int qcu_profile_read(double* gemm_ms, int64_t* gemm_launches, double* gemm_ops,
                     double* gemm_bytes);
/* CandidateEvaluator::agreement_counts (B200 extension): per candidate, the
 * number of local calibration samples whose top-1 equals the fp32 reference;
 * the multi-GPU driver all-reduces these (loss = 1 - sum / N_total). */
int qc_evaluator_agreement(const qc_evaluator* e, const int* cands, size_t n_cands,
                           size_t n_slots, int64_t* counts);
/* Sharded calibration (B200 extension; quantc/device.hpp): pass 1 extrema of
 * the listed canonical edges over this process's shard, pass 2 histograms
 * against the GLOBAL absmax.  A multi-GPU driver all-reduces min/max between
 * the passes and sums the int64 counts after (paper_2103_14949_b200/parallel.py).
 * counts: n x bins. */
int qc_collect_extrema(const qc_graph* g, const qc_dataset* d, const int* edges, size_t n,
                       double* mins, double* maxs);
int qc_collect_histograms(const qc_graph* g, const qc_dataset* d, const int* edges, size_t n,
                          const double* absmax, int bins, int64_t* counts);
/* realize (SPEC.md realize module; the reference declares it without an
 * implementation): the simulated graph lowered under a strategy (the JSON of
 * qc_evaluator_strategy) into an integer graph for qc_eval_int. */
int qc_realize(const qc_graph* sim_g, const char* strategy_json, const qc_spec* spec,
               qc_graph** out);
/* realize.hpp helpers: fixed-point requantize parameters,
 * storage dtype (candidates as "int8,int16"; writes the dtype name), and the
 * integer clip bounds of rewrite_clip. */
int qc_requantize_params(double s_in, double s_out, int32_t* multiplier, int* shift);
int qc_choose_storage_dtype(int bit, const char* candidates_csv, int sign, char* out, size_t cap);
int qc_rewrite_clip(double min_f, double max_f, double s_out, int64_t zero_point,
                    const char* storage, int64_t* q_min, int64_t* q_max);
/* fp32 score rows of predict_top1 (samples x per-sample numel) under the
 * active engine mode (B200 extension; quantc/device.hpp predict_scores). */
int qc_predict_scores(const qc_graph* g, const qc_dataset* d, const int64_t* bind_nodes,
                      const qc_qparams* bind_params, size_t n_bind, float* out, size_t cap,
                      size_t* n_out, int64_t* per_sample);
/* host worker pool self-test (no GPU): sum of i over [0, n) through
 * quantc::parallel_for with `workers`; throw_at >= 0 makes that index throw
 * (the call then reports QC_ERR_INTERNAL with the lowest throwing index). */
int qcu_parallel_selftest(size_t n, int workers, int64_t throw_at, int64_t* sum);
/* counters since load: kernel launches issued by the engine, tcgen05 GEMMs */
int qcu_counters(int64_t* steps, int64_t* tcgen05_gemms, int64_t* f64_convs,
                 int64_t* fused_batches);
/* realized-graph integer conv/dense layers run on the CUDA-core backend
 * (int16 codes / int16 accumulator; kernels/conv_simt.cu) since load */
int qcu_simt_int_convs(int64_t* n);

/* ---- distributed hot path (quantc/comm.hpp, quantc/distributed.hpp) ------
 * One process per GPU.  A communicator is NCCL (libnccl.so.2 bound at run
 * time; the 128-byte unique id comes from one rank and is shared out of band)
 * or host callbacks over the caller's own transport (e.g. torch.distributed
 * gloo).  Every rank must make the same calls in the same order. */
typedef struct qc_comm qc_comm;
typedef int (*qc_comm_sum_i64_fn)(int64_t* data, size_t n, void* user);
typedef int (*qc_comm_f64_fn)(double* data, size_t n, int op /* 0 min, 1 max */, void* user);
typedef int (*qc_comm_gather_f64_fn)(const double* send, size_t n, double* recv, void* user);
int qc_comm_local(qc_comm** out);
int qc_comm_nccl_unique_id(char id[128]);
int qc_comm_nccl(int rank, int world, const char id[128], qc_comm** out);
int qc_comm_callbacks(int rank, int world, qc_comm_sum_i64_fn sum_i64, qc_comm_f64_fn minmax_f64,
                      qc_comm_gather_f64_fn gather_f64, void* user, qc_comm** out);
void qc_comm_free(qc_comm* c);
/* collect_stats over every rank's shard `d` (all-reduced extrema, then
 * histograms; EdgeStats.sample_count is the global count). */
int qc_collect_stats_dist(const qc_graph* g, const qc_dataset* d, qc_comm* comm, int bins,
                          const int* edges, size_t n_edges, qc_stats** out);
/* Why the fused int8 engine does ("") or does not run graph g under the
 * binding in the active engine mode (quantc/device.hpp fused_status). */
int qc_fused_status(const qc_graph* g, const int64_t* bind_nodes, const qc_qparams* bind_params,
                    size_t n_bind, char** why);
/* CandidateEvaluator::scores (B200 extension): fp32 output rows of each
 * candidate's forward, [n_cands x N x per_sample], `group` candidates per
 * grouped launch (0: default). */
int qc_evaluator_scores(const qc_evaluator* e, const int* cands, size_t n_cands, size_t n_slots,
                        int group, float* out, size_t cap, size_t* n_out, int64_t* per_sample);
/* The batched / speculative searches (search.hpp *_batched; results and
 * traces identical to qc_search).  Loss source: `fn` (a batch callback) when
 * non-NULL, else the evaluator: mode QC_LOSS_LOCAL (this process only),
 * QC_LOSS_SAMPLES (ev holds this rank's calibration shard; counts
 * all-reduced over comm) or QC_LOSS_CANDIDATES (ev holds the full set; each
 * batch split over ranks, losses all-gathered).  spec_stats (optional):
 * batches, evaluated, committed. */
typedef int (*qc_batch_loss_fn)(const int* cands, size_t n_cands, size_t n_slots, void* user,
                                double* losses);
enum { QC_LOSS_LOCAL = 0, QC_LOSS_SAMPLES = 1, QC_LOSS_CANDIDATES = 2 };
int qc_search_batched(int method, const int* edges, const int* lo, const int* hi, size_t n_slots,
                      qc_batch_loss_fn fn, void* user, const qc_evaluator* ev, qc_comm* comm,
                      int loss_mode, const qc_search_params* p, int width, int* best,
                      double* best_loss, int64_t* evaluations, char** trace_json,
                      int64_t* spec_stats);

#ifdef __cplusplus
}
#endif

#endif /* QUANTC_CUDA_H_ */
