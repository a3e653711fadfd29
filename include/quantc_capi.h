/*
 * quantc_capi.h — flat C-ABI over the quantc calibrate-and-search API.
 *
 * This is the foreign-function boundary a maintainer of the reference would
 * add to bind `quantc` from Python/Go/Java (the reference's CMakeLists.txt:12
 * names a "quantc python extension" that never shipped).  Every entry point
 * maps 1:1 onto a function of the reference's C++ API in
 * /root/reference/proj/include/quantc/<name>.hpp (cited per function below).
 *
 * The SAME binding source (paper_2103_14949_b200/csrc/host/capi.cpp) is
 * compiled twice:
 *   - against this repo's B200 implementation  -> libquantc_b200.so
 *   - against the reference sources (oracle)   -> oracle/_ref/libquantc_ref.so
 * so the C ABI is provably a drop-in for the reference path.
 *
 * Conventions
 *   - every function returns QC_OK (0) or a QC_ERR_* code; no exception
 *     crosses the ABI.  qc_last_error() returns the message of the last
 *     failure on the calling thread.
 *   - buffers are caller-allocated (pointer + capacity); functions write the
 *     required size to *n even when the capacity is too small (QC_ERR_BUFFER).
 *   - strings returned through char** are malloc'ed; release with qc_free().
 *   - dtypes are encoded as QC_F32..QC_I32 (reference dtype.hpp:13-19 order).
 */
#ifndef QUANTC_CAPI_H_
#define QUANTC_CAPI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (reference exception types) -------------- */
enum {
  QC_OK = 0,
  QC_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument (dtype.cpp:71, simulate.cpp:13) */
  QC_ERR_GRAPH = 2,            /* GraphError (graph.hpp:141) */
  QC_ERR_SPEC = 3,             /* SpecError (hwspec.hpp:47) */
  QC_ERR_TOPOLOGY = 4,         /* TopologyError (topology.hpp:30) */
  QC_ERR_CALIBRATION = 5,      /* CalibrationError (calibration.hpp:37) */
  QC_ERR_SEARCH = 6,           /* SearchError (search.hpp:26) */
  QC_ERR_EVAL = 7,             /* EvalError (interpreter.hpp:27) */
  QC_ERR_OVERFLOW = 8,         /* OverflowError (interpreter.hpp:32); see qc_last_overflow */
  QC_ERR_CUDA = 9,             /* device failure (B200 implementation only) */
  QC_ERR_BUFFER = 10,          /* caller buffer too small */
  QC_ERR_INTERNAL = 11         /* any other std::exception */
};

/* ---- dtypes (reference dtype.hpp:13-19) -------------------------------- */
enum { QC_F32 = 0, QC_I8 = 1, QC_U8 = 2, QC_I16 = 3, QC_I32 = 4, QC_NONE = -1 };

/* ---- opaque handles ----------------------------------------------------- */
typedef struct qc_graph qc_graph;         /* quantc::Graph (graph.hpp:87) */
typedef struct qc_spec qc_spec;           /* quantc::HardwareSpec (hwspec.hpp:30) */
typedef struct qc_topology qc_topology;   /* quantc::Topology (topology.hpp:16) */
typedef struct qc_dataset qc_dataset;     /* quantc::Dataset (interpreter.hpp:60-64) */
typedef struct qc_stats qc_stats;         /* quantc::CalibrationStats (calibration.hpp:31) */
typedef struct qc_evaluator qc_evaluator; /* quantc::CandidateEvaluator (search.hpp:100) */

/* quantc::QParams (simulate.hpp:33-45) as a POD. acc_dtype = QC_NONE when
 * the optional accumulator is disengaged. */
typedef struct qc_qparams {
  double threshold;
  int32_t bit;
  int32_t sign;
  int32_t in_dtype;
  int32_t out_dtype;
  int64_t zero_point;
  int32_t passthrough;
  int32_t acc_dtype;
  double acc_scale;
} qc_qparams;

/* ---- errors / memory ---------------------------------------------------- */
const char* qc_last_error(void);
/* OverflowError payload of the last QC_ERR_OVERFLOW (interpreter.hpp:35-37) */
void qc_last_overflow(int64_t* node, int64_t* flat_index, int64_t* value);
const char* qc_impl_name(void);
void qc_free(void* p);

/* ---- graph (graph.hpp) --------------------------------------------------
 * JSON: {"nodes":[{"id","op","attrs",("payload":{"dtype","shape","offset"})}],
 *        "edges":[{"src":[id,port],"dst":[id,port]}], "inputs":[..],
 *        "outputs":[[id,port]..]}; payload bytes live in `blob` (little-endian
 * float32 or int32 elements, the sidecar convention of SPEC.md graph-ir). */
int qc_graph_from_json(const char* json, const void* blob, size_t blob_len, qc_graph** out);
/* structure + attrs only (payload shapes/dtypes, no bytes) */
int qc_graph_to_json(const qc_graph* g, char** json_out);
/* the payload bytes the offsets of qc_graph_to_json refer to (int32/fp32
 * little-endian, in node order): with the JSON, qc_graph_from_json rebuilds
 * the graph in any library exporting this ABI */
int qc_graph_blob(const qc_graph* g, void* out, size_t cap, size_t* n);
void qc_graph_free(qc_graph* g);
int qc_graph_num_nodes(const qc_graph* g, size_t* n);
/* validate_graph (graph.hpp:131): JSON array of {"node","message"} */
int qc_validate_graph(const qc_graph* g, char** report_json);
/* traversal_order (graph.hpp:137) */
int qc_traversal_order(const qc_graph* g, int64_t* out, size_t cap, size_t* n);
/* edge_order (graph.hpp:141): 4 int64 per edge: src,src_port,dst,dst_port */
int qc_edge_order(const qc_graph* g, int64_t* out, size_t cap, size_t* n_edges);

/* ---- hardware spec (hwspec.hpp) ---------------------------------------- */
int qc_spec_parse(const char* text, qc_spec** out);          /* hwspec.hpp:54 */
void qc_spec_free(qc_spec* s);
int qc_spec_serialize(const qc_spec* s, char** text);         /* hwspec.hpp:55 */
int qc_classify_op(const qc_spec* s, const char* op, int* cls); /* 0 float,1 int,2 mixed */
int qc_candidate_dtypes(const qc_spec* s, const char* op, int port, int* out, size_t cap,
                        size_t* n);                             /* hwspec.hpp:60 */
/* match_signature (hwspec.hpp:65): *found=0 when no signature fits */
int qc_match_signature(const qc_spec* s, const char* op, const int* bits, const int* signs,
                       size_t n, int* found, int* in_dtypes, int* out_dtype);

/* ---- topology (topology.hpp) -------------------------------------------- */
int qc_generate_topology(const qc_graph* g, const qc_spec* s, qc_topology** out); /* :38 */
void qc_topology_free(qc_topology* t);
int qc_dump_topology(const qc_graph* g, const qc_topology* t, char** json);      /* :72 */
/* quantized vertex ids (qv set), ascending */
int qc_topology_qv(const qc_topology* t, int64_t* out, size_t cap, size_t* n);
int qc_insert_simulated_quantize(const qc_graph* g, const qc_topology* t, qc_graph** out);
int qc_searchable_edge_indices(const qc_topology* t, int* out, size_t cap, size_t* n);
int qc_simulated_edge_indices(const qc_graph* g, const qc_topology* t, int* out, size_t cap,
                              size_t* n);

/* ---- dataset (interpreter.hpp:60-64) ------------------------------------
 * n_samples samples of one float32 input each, packed contiguously; `labels`
 * may be NULL. */
int qc_dataset_create(const float* data, int64_t n_samples, const int64_t* sample_shape,
                      int ndim, const int64_t* labels, qc_dataset** out);
void qc_dataset_free(qc_dataset* d);

/* ---- simulate (simulate.hpp) -------------------------------------------- */
int qc_compute_scale(double threshold, int bit, int sign, double* out);
int qc_quant_bounds(int bit, int sign, int64_t* qmin, int64_t* qmax);
int qc_simulated_quantize_value(float x, const qc_qparams* p, float* out);
int qc_simulated_quantize(const float* x, int64_t n, const qc_qparams* p, float* out);
int qc_asymmetric_zero_point(double min_value, double range_threshold, int bit, int64_t* out);
int qc_noop_params(qc_qparams* out);

/* ---- calibration (calibration.hpp) -------------------------------------- */
int qc_collect_stats(const qc_graph* g, const qc_dataset* d, int bins, const int* edges,
                     size_t n_edges, int workers, qc_stats** out);          /* :48 */
/* build a CalibrationStats from raw per-edge arrays (stats file analogue) */
int qc_stats_create(qc_stats** out);
int qc_stats_set_edge(qc_stats* s, int edge, double min, double max, double absmax,
                      int64_t sample_count, const int64_t* counts, size_t bins);
void qc_stats_free(qc_stats* s);
int qc_stats_edges(const qc_stats* s, int* out, size_t cap, size_t* n);
int qc_stats_get(const qc_stats* s, int edge, double* min, double* max, double* absmax,
                 int64_t* sample_count, int64_t* counts, size_t cap, size_t* bins);
/* method: 0 max, 1 quantile, 2 kl (calibration.hpp:69-76) */
int qc_estimate_thresholds(const qc_stats* s, int method, double quantile, int kl_bits,
                           int pow2, int* edges_out, double* thresholds_out, size_t cap,
                           size_t* n);
int qc_threshold_max(double absmax, double* out);
int qc_threshold_quantile(const int64_t* counts, size_t bins, double absmax, double q,
                          double* out);
int qc_threshold_kl(const int64_t* counts, size_t bins, double absmax, int target_bit,
                    double* out);
int qc_round_pow2(double threshold, double* out);

/* ---- interpreter (interpreter.hpp) --------------------------------------
 * Single-input graphs. A SimBinding is passed as parallel arrays
 * (node ids, params); n_bind = 0 means "no binding". The first graph output
 * is returned (its shape through out_shape, rank through out_ndim). */
int qc_eval_fp32(const qc_graph* g, const float* input, const int64_t* shape, int ndim,
                 const int64_t* bind_nodes, const qc_qparams* bind_params, size_t n_bind,
                 float* out, size_t cap, size_t* n_out, int64_t* out_shape, int* out_ndim);
/* all node outputs of eval_fp32_values for the listed nodes, concatenated */
int qc_eval_fp32_values(const qc_graph* g, const float* input, const int64_t* shape, int ndim,
                        const int64_t* nodes, size_t n_nodes, float* out, size_t cap,
                        size_t* n_out);
/* eval_int (interpreter.hpp:54): mode 0 saturate, 1 trap; int outputs as int32 */
int qc_eval_int(const qc_graph* g, const float* input, const int64_t* shape, int ndim,
                int mode, int32_t* out, size_t cap, size_t* n_out, int* out_dtype);
int qc_predict_top1(const qc_graph* g, const qc_dataset* d, int workers,
                    const int64_t* bind_nodes, const qc_qparams* bind_params, size_t n_bind,
                    int64_t* out, size_t cap, size_t* n);

/* ---- search (search.hpp) ------------------------------------------------ */
int qc_evaluator_create(const qc_graph* sim_g, const qc_spec* spec, const qc_topology* t,
                        const int* thr_edges, const double* thr_values, size_t n_thr,
                        const qc_stats* stats, const qc_dataset* calib, int min_bit,
                        int workers, qc_evaluator** out);                     /* :102 */
void qc_evaluator_free(qc_evaluator* e);
/* SearchSpace ranges (search.hpp:41): edge index, lo, hi per slot */
int qc_evaluator_space(const qc_evaluator* e, int* edges, int* lo, int* hi, size_t cap,
                       size_t* n);
int qc_evaluator_refs(const qc_evaluator* e, int64_t* out, size_t cap, size_t* n);
int qc_evaluator_bind(const qc_evaluator* e, const int* cand, size_t n_slots,
                      int64_t* nodes_out, qc_qparams* params_out, size_t cap, size_t* n);
int qc_evaluator_loss(const qc_evaluator* e, const int* cand, size_t n_slots, double* out);
int qc_evaluator_losses(const qc_evaluator* e, const int* cands, size_t n_cands,
                        size_t n_slots, double* out);
int qc_evaluator_strategy(const qc_evaluator* e, const int* cand, size_t n_slots, char** json);
int qc_evaluator_evaluations(const qc_evaluator* e, int64_t* out);

/* LossFn seam (search.hpp:70). Return 0 and write *loss, nonzero to abort. */
typedef int (*qc_loss_fn)(const int* cand, size_t n_slots, void* user, double* loss);

enum { QC_SEARCH_GREEDY = 0, QC_SEARCH_ANNEAL = 1, QC_SEARCH_RANDOM = 2, QC_SEARCH_EXHAUSTIVE = 3 };
typedef struct qc_search_params {
  int32_t rounds;  /* greedy */
  double tol;      /* greedy */
  int32_t steps;   /* anneal */
  double t0;       /* anneal */
  double decay;    /* anneal */
  uint64_t seed;   /* anneal, random */
  int32_t n;       /* random */
  int64_t cap;     /* exhaustive */
} qc_search_params;

/* Runs one of greedy/anneal/random/exhaustive_search (search.hpp:75-95) over
 * the space given by (edges, lo, hi). The loss is `fn` when non-NULL, else
 * evaluator->loss. Writes best candidate / loss / evaluation count and the
 * trace as JSON {"header":{..},"records":[[iter,[bits..],loss,accepted],..]}. */
int qc_search(int method, const int* edges, const int* lo, const int* hi, size_t n_slots,
              qc_loss_fn fn, void* user, const qc_evaluator* ev, const qc_search_params* p,
              int* best, double* best_loss, int64_t* evaluations, char** trace_json);
/* space_size (search.hpp:72) as a decimal string */
int qc_space_size(const int* lo, const int* hi, size_t n_slots, char** decimal);

#ifdef __cplusplus
}
#endif

#endif /* QUANTC_CAPI_H_ */
