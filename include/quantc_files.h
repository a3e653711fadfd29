/* quantc_files.h — C ABI of the serialize.hpp file formats (B200 library).
 *
 * Drop-in for /root/reference/proj/include/quantc/serialize.hpp:18-56, which
 * the reference declares but does not implement; the reference oracle build
 * (which compiles the shared quantc_capi.h binding) therefore does not export
 * these.  Handles and error codes are those of quantc_capi.h. */
#ifndef QUANTC_FILES_H
#define QUANTC_FILES_H

#include "quantc_capi.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- files (serialize.hpp; reference proj/include/quantc/serialize.hpp) --
 * graph file: JSON + little-endian sidecar "<stem>.bin" next to it, payloads
 * referenced as {file, offset, dtype, shape}. */
int qc_graph_save(const qc_graph* g, const char* json_path);          /* :24 */
int qc_graph_load(const char* json_path, qc_graph** out);             /* :23 */
/* stats file: JSON keyed by edge index {min,max,absmax,bins,counts,samples}
 * + dataset/graph fingerprints */
int qc_stats_save(const qc_stats* s, const char* path);               /* :43 */
int qc_stats_load(const char* path, qc_stats** out);                  /* :42 */
/* FNV-1a 64 over the graph's canonical JSON + sidecar bytes (:51) */
int qc_fingerprint_graph(const qc_graph* g, uint64_t* out);
int qc_fnv1a64(const void* data, size_t size, uint64_t seed, uint64_t* out); /* :53 */
/* dataset manifest (serialize.hpp:27-28 load_dataset): single-input fp32
 * samples of one shape */
int qc_dataset_load(const char* manifest_path, qc_dataset** out, int64_t* n_samples);
/* fixtures (reference fixtures.hpp:55-60): write every committed fixture
 * under dir / regenerate and byte-compare (QC_ERR_* on a mismatch) */
int qc_fixtures_write_all(const char* dir);
int qc_fixtures_verify_committed(const char* dir);

#ifdef __cplusplus
}
#endif

#endif /* QUANTC_FILES_H */
