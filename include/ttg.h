/*
 * ttg.h — C ABI of the B200-native TT-ICE / TT-ICE* per-increment update.
 *
 * This is the drop-in boundary.  Plain pointers and sizes
 * only; no C++ or torch types cross it and no exception crosses it.  The C++
 * host mirror of the reference API (include/ttstream/*.hpp) and the Python
 * ctypes mirror (paper_2211_12487_b200/ttstream.py) both sit on top of it.
 *
 * Entry point  -> reference interface it replaces (reference = /root/reference/proj)
 *   ttg_bootstrap                     -> tt_ice_bootstrap          include/ttstream/tt_ice.hpp:48-49
 *                                        (tt_svd                   include/ttstream/tt_svd.hpp:13)
 *   ttg_tt_ice_update                 -> tt_ice_update             include/ttstream/tt_ice.hpp:38-39
 *   ttg_tt_ice_update_with_tolerances -> tt_ice_update_with_tolerances tt_ice.hpp:43-45
 *   ttg_tt_ice_star_update            -> tt_ice_star_update        include/ttstream/tt_ice_star.hpp:57-59
 *   ttg_per_obs_errors                -> per_obs_errors            include/ttstream/tt_ice_star.hpp:24
 *   ttg_project                       -> tt_project                include/ttstream/tensor_train.hpp:103
 *   ttg_reconstruct                   -> tt_reconstruct            include/ttstream/tensor_train.hpp:96-98
 *   ttg_tt_upload / ttg_tt_download_* -> TensorTrain ctor / accessors tensor_train.hpp:59-93
 *   status codes                      -> exception classes         include/ttstream/errors.hpp:9-55
 *
 * Semantics that differ from the reference by design:
 *   - a device train (ttg_tt) is updated IN PLACE; earlier observations'
 *     coefficients are never rewritten (Thm 3.3 holds bit-for-bit);
 *   - UpdateReport.seconds is wall time from CUDA events, not std::clock.
 */
#ifndef TTG_H_
#define TTG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TTG_MAX_CORES 32

/* Status codes map 1:1 onto ttstream::*Error (errors.hpp:9-55). */
enum ttg_status {
  TTG_OK = 0,
  TTG_E_DIMENSION = 1, /* DimensionError */
  TTG_E_NUMERIC = 2,   /* NumericError   */
  TTG_E_STATE = 3,     /* StateError     */
  TTG_E_FORMAT = 4,    /* FormatError    */
  TTG_E_INDEX = 5,     /* IndexError     */
  TTG_E_CONFIG = 6,    /* ConfigError    */
  TTG_E_RESOURCE = 7,  /* ResourceError  */
  TTG_E_CUDA = 8,      /* CUDA runtime failure (no reference analogue) */
  TTG_E_NCCL = 9,      /* NCCL failure (no reference analogue) */
  TTG_E_ARGUMENT = 10  /* null pointer / bad enum at the ABI */
};

/* Where a data pointer lives. */
enum ttg_where { TTG_HOST = 0, TTG_DEVICE = 1 };

/* SkipStatistic (tt_ice_star.hpp:9-12). */
enum ttg_skip_statistic { TTG_SKIP_MEAN = 0, TTG_SKIP_FULL_BATCH = 1 };

typedef struct ttg_ctx ttg_ctx;
typedef struct ttg_tt ttg_tt;

/* Mirrors UpdateReport (tt_ice.hpp:10-20) with fixed-size rank arrays. */
typedef struct ttg_report {
  int64_t increment_index;
  int64_t obs_in_batch;
  int64_t obs_used;
  int32_t n_ranks; /* D+1 entries used in the arrays below */
  int32_t tolerance_clamped;
  int64_t ranks_before[TTG_MAX_CORES + 1];
  int64_t ranks_after[TTG_MAX_CORES + 1];
  double eps_target;
  double batch_rel_error_estimate;
  double seconds; /* wall time (CUDA events) */
  int32_t guard_reorthogonalised; /* number of modes whose 1e-10 Gram guard fired */
  int32_t modes_updated;          /* modes whose basis grew */
  /* numerics of the truncated SVDs (truncated_svd.cpp:29-94 is one backward-stable
     BDCSVD; here a Gram eigen-solve with two fallbacks): */
  int32_t accurate_modes;         /* modes solved on the unsquared factor (TSQR + Jacobi) */
  int32_t raw_fallbacks;          /* modes whose raw-Gram result was recomputed from the explicit residual */
  int32_t gram_only_unstable;     /* modes where the accuracy test asked for the factor path and none
                                     applied (the result rests on the squared-condition Gram); 0 means
                                     every decision was taken at full resolution */
} ttg_report;

/* Mirrors HeuristicConfig (tt_ice_star.hpp:14-20). */
typedef struct ttg_heuristics {
  double occupancy_threshold; /* default 0.8 */
  int32_t skip_enabled;       /* default 1 */
  int32_t subselect_enabled;  /* default 1 */
  int32_t skip_statistic;     /* ttg_skip_statistic, default TTG_SKIP_MEAN */
  int32_t use_approx_tolerance; /* default 0 */
} ttg_heuristics;

void ttg_heuristics_default(ttg_heuristics* h);

/* ---- context ------------------------------------------------------------ */
/* One context per stream (single logical writer).  Calls on a
 * context are serialised on its CUDA stream. */
int ttg_ctx_create(int device, ttg_ctx** out);
/* Multi-GPU: one context per rank, batch axis sharded; Grams and scalars are
 * all-reduced, coefficient columns all-gathered over NCCL.  `nccl_id` is the
 * 128-byte ncclUniqueId produced by ttg_nccl_unique_id on rank 0.  Every
 * exchange of an NCCL context goes through NCCL, world 1 included. */
int ttg_nccl_unique_id(uint8_t out[128]);
int ttg_ctx_create_dist(int device, int rank, int world, const uint8_t nccl_id[128], ttg_ctx** out);
/* Multi-rank context whose exchanges go through caller-supplied HOST
 * collectives instead of NCCL (another transport, or several ranks sharing
 * one GPU in tests): the library copies the operand to host memory, calls the
 * function, and copies the result back.  allreduce: element-wise sum of `n`
 * doubles in place over all ranks; allgather: `bytes` from every rank,
 * concatenated in rank order into `recv` (world * bytes).  Both return 0 on
 * success; a nonzero return surfaces as TTG_E_NCCL. */
typedef int (*ttg_host_allreduce_fn)(void* user, double* buf, int64_t n);
typedef int (*ttg_host_allgather_fn)(void* user, const void* send, int64_t bytes, void* recv);
int ttg_ctx_create_hostcoll(int device, int rank, int world, ttg_host_allreduce_fn allreduce,
                            ttg_host_allgather_fn allgather, void* user, ttg_ctx** out);
void ttg_ctx_destroy(ttg_ctx* ctx);
/* ctx = NULL: the message of the calling thread's last context-free call (ttg_read_batch /
 * ttg_write_batch). */
const char* ttg_last_error(const ttg_ctx* ctx);
int ttg_ctx_rank(const ttg_ctx* ctx);
int ttg_ctx_world(const ttg_ctx* ctx);
/* cudaStream_t the context launches on (as void*), for event timing. */
void* ttg_ctx_stream(const ttg_ctx* ctx);
/* Number of ttg kernels launched by this context so far. */
int64_t ttg_ctx_launch_count(const ttg_ctx* ctx);
int ttg_ctx_synchronize(ttg_ctx* ctx);
/* Ordering against a caller's CUDA stream (cudaStream_t as void*; NULL = the
 * legacy default stream), no host synchronisation.  The context stream is
 * non-blocking, so a device increment produced on another stream must be
 * ordered before the update reads it (wait), and a device result written by
 * the context (ttg_reconstruct into device memory) before the caller's stream
 * reads it (join). */
int ttg_ctx_wait_stream(ttg_ctx* ctx, void* stream);
int ttg_ctx_join_stream(ttg_ctx* ctx, void* stream);
/* Per-kernel accounting.  Launch counts and ALGORITHMIC bytes / flops per
 * launch are always kept; device time (CUDA events on the
 * context stream around each launch) only while profiling is on. */
int ttg_ctx_set_profiling(ttg_ctx* ctx, int on);
void ttg_ctx_reset_stats(ttg_ctx* ctx);
int ttg_ctx_num_kernel_stats(ttg_ctx* ctx);
int ttg_ctx_kernel_stat(ttg_ctx* ctx, int idx, char* name, int name_len, int64_t* launches, double* ms,
                        double* bytes, double* flops);
/* Pre-map `bytes` of device memory into the context's stream-ordered workspace
 * pool, so workspace growth during a stream (ranks grow) never maps new
 * pages mid-update. */
int ttg_ctx_reserve(ttg_ctx* ctx, int64_t bytes);
/* Host<->device bytes moved by the context (H2D of host increments, D2H of
 * scalars/decisions). */
int ttg_ctx_io_bytes(const ttg_ctx* ctx, int64_t* h2d, int64_t* d2h);
/* Speculative sweeps (one host read per update instead of one per mode; no
 * reference counterpart -- the reference's loop tt_ice.cpp:71-117 is host code):
 * `sweeps` = update sweeps that sized launches from the previous update's ranks,
 * `redone` = those a device-side check rejected and that were repeated with a
 * host read per mode.  Results are identical either way. */
int ttg_ctx_spec_stats(const ttg_ctx* ctx, int64_t* sweeps, int64_t* redone);
/* Start copying a host increment (n doubles, ideally page-locked) to the
 * device on the context's copy stream, into one of two staging slots; the next
 * update / projection call given the same host pointer and size (where =
 * TTG_HOST) consumes the staged copy instead of copying, so the PCIe transfer
 * of increment k+1 overlaps the update of increment k.  The caller must not
 * modify y until that consuming call has returned.  No reference counterpart:
 * the in-memory analogue of the double-buffered stream reader
 * (stream_io.cpp:123-204, ttg_stream_*). */
int ttg_prefetch(ttg_ctx* ctx, const double* y, int64_t n);

/* ---- device train ------------------------------------------------------- */
/* Upload a host train: cores[i] is r_left[i]*n[i]*r_right[i] doubles,
 * first-index-fastest (TTCore layout, tensor_train.hpp:12-31). */
int ttg_tt_upload(ttg_ctx* ctx, int n_cores, const int64_t* r_left, const int64_t* n,
                  const int64_t* r_right, const double* const* cores, int64_t ortho_count,
                  const int64_t* bounds, int64_t n_bounds, ttg_tt** out);
void ttg_tt_destroy(ttg_tt* tt);
int ttg_tt_num_cores(const ttg_tt* tt);
/* ranks: n_cores+1 entries; modes: n_cores entries (last = local obs count). */
int ttg_tt_shape(const ttg_tt* tt, int64_t* ranks, int64_t* modes, int64_t* ortho_count,
                 int64_t* n_bounds);
int ttg_tt_bounds(const ttg_tt* tt, int64_t* bounds);
/* Copies core i (compact r_left*n*r_right, first-index-fastest) to host. */
int ttg_tt_download_core(ttg_ctx* ctx, const ttg_tt* tt, int i, double* out);

/* ---- the hot path ------------------------------------------------------- */
/* y: shape[0..ndim-1] (spatial modes + observation mode), first-index-fastest.
 * where: TTG_HOST (copied H2D inside the call) or TTG_DEVICE. */
int ttg_bootstrap(ttg_ctx* ctx, const double* y, int where, const int64_t* shape, int ndim,
                  double eps_des, ttg_tt** out, ttg_report* report);
int ttg_tt_ice_update(ttg_ctx* ctx, ttg_tt* tt, const double* y, int where,
                      const int64_t* shape, int ndim, double eps_des, ttg_report* report);
int ttg_tt_ice_update_with_tolerances(ttg_ctx* ctx, ttg_tt* tt, const double* y, int where,
                                      const int64_t* shape, int ndim, const double* deltas,
                                      int n_deltas, ttg_report* report);
int ttg_tt_ice_star_update(ttg_ctx* ctx, ttg_tt* tt, const double* y, int where,
                           const int64_t* shape, int ndim, double eps_des,
                           const ttg_heuristics* cfg, ttg_report* report);
/* errs: host array of shape[ndim-1] doubles. */
int ttg_per_obs_errors(ttg_ctx* ctx, const ttg_tt* tt, const double* y, int where,
                       const int64_t* shape, int ndim, double* errs);
/* coeffs: host array r_d x n_obs (first-index-fastest). */
int ttg_project(ttg_ctx* ctx, const ttg_tt* tt, const double* y, int where,
                const int64_t* shape, int ndim, double* coeffs);
/* out: (n_1..n_d, obs_end-obs_begin) dense reconstruction; where = host or device. */
int ttg_reconstruct(ttg_ctx* ctx, const ttg_tt* tt, int64_t obs_begin, int64_t obs_end,
                    double* out, int where);

/* ---- metrics (reference proj/include/ttstream/metrics.hpp) ---- */
/* compression_ratio, metrics.hpp:11 / metrics.cpp:7-11: (prod n_i * n_obs) / param_count. */
int ttg_compression_ratio(const ttg_tt* tt, double* cr);
/* rre, metrics.hpp:15-18 / metrics.cpp:34-38: ||x_ref - reconstruct(obs_begin, obs_end)|| / ||x_ref||,
 * computed on the device without materialising the reconstruction.  Zero-norm reference -> 0 and
 * *zero_reference = 1 (nullable).  x_ref shape: (n_1..n_d, obs_end - obs_begin). */
int ttg_rre(ttg_ctx* ctx, const ttg_tt* tt, const double* x_ref, int where, const int64_t* shape, int ndim,
            int64_t obs_begin, int64_t obs_end, double* rre, int* zero_reference);
/* rpe, metrics.hpp:24 / metrics.cpp:44-47: relative error of tt_expand(tt_project(unseen)). */
int ttg_rpe(ttg_ctx* ctx, const ttg_tt* tt, const double* unseen, int where, const int64_t* shape,
            int ndim, double* rpe, int* zero_reference);
/* TensorTrain::measure_ortho_count, tensor_train.cpp:135-146 (device Gram of each left unfolding). */
int ttg_tt_measure_ortho_count(ttg_ctx* ctx, const ttg_tt* tt, double tol, int64_t* count);

/* ---- TTC1 checkpoint (reference serialization.hpp:12-22) ---- */
/* serialize, serialization.cpp:68-87: strided D2H of the device train into the TTC1 image.
 * Call with buf = NULL to get *len; then with a buffer of cap >= *len. */
int ttg_tt_serialize(ttg_ctx* ctx, const ttg_tt* tt, uint8_t* buf, int64_t cap, int64_t* len);
/* deserialize, serialization.cpp:89-129: same validation and FormatError messages; the
 * orthonormality is re-measured on the device (tol 1e-10), not trusted from the file. */
int ttg_tt_deserialize(ttg_ctx* ctx, const uint8_t* buf, int64_t len, ttg_tt** out);
/* save_ttc / load_ttc, serialization.cpp:131-152. */
int ttg_tt_save_ttc(ttg_ctx* ctx, const ttg_tt* tt, const char* path);
int ttg_tt_load_ttc(ttg_ctx* ctx, const char* path, ttg_tt** out);

/* ---- TTB1 ingest (reference stream_io.hpp:57-65) ---- */
/* write_batch / read_batch, stream_io.cpp:123-187.  read: call with data = NULL to get ndim,
 * shape (int64_t[255] or NULL) and *count, then with a buffer of cap >= *count doubles. */
int ttg_write_batch(const char* path, const int64_t* shape, int ndim, const double* data);
int ttg_read_batch(const char* path, int64_t* shape, int* ndim, double* data, int64_t cap, int64_t* count);
/* A directory of .ttb increments in lexicographic order (list_stream, stream_io.cpp:189-204),
 * read by a host thread into pinned buffers and copied H2D on a side stream while the caller
 * updates on the previous increment.  ttg_stream_next returns a DEVICE pointer (pass it with
 * TTG_DEVICE) valid until the next call; the library stream already waits for its copy. */
typedef struct ttg_stream ttg_stream;
int ttg_stream_open(ttg_ctx* ctx, const char* dir, ttg_stream** out);
int64_t ttg_stream_count(const ttg_stream* s);
int ttg_stream_next(ttg_stream* s, const double** y, int64_t* shape, int* ndim);
int ttg_stream_close(ttg_stream* s);

#ifdef __cplusplus
}
#endif

#endif /* TTG_H_ */
