/*
 * pulsegrid_b200.h -- C ABI of the B200-native single-pulse search hot path.
 *
 * This is the drop-in boundary under the reference's C++ stage API
 * (/root/reference/proj/include/pulsegrid/, the *.hpp files).  The reference has no FFI of its
 * own; these entry points are what a maintainer binds to
 * replace, one for one:
 *
 *   pgb_generate_dm_trials  <- pulsegrid::generate_dm_trials   dedisp.hpp:53-54   (src/dedisp.cpp:28-70)
 *   pgb_delay_samples       <- pulsegrid::delay_samples        dedisp.hpp:48      (src/dedisp.cpp:13-18)
 *   pgb_adaptive_dm_step    <- pulsegrid::adaptive_dm_step     dedisp.hpp:51      (src/dedisp.cpp:20-26)
 *   pgb_set_plan            <- the DmTrialPlan argument of run_dm_loop (dedisp.hpp:17-25), uploaded once
 *   pgb_run_dm_loop_u8/_f32 <- pulsegrid::run_dm_loop          engine.hpp:61-62   (src/engine.cpp:85-265)
 *   pgb_dedisperse_*        <- pulsegrid::dedisperse / dedisperse_block  dedisp.hpp:61,71-74 (src/dedisp.cpp:133-218)
 *   pgb_link_grid           <- pulsegrid::link_grid            cluster.hpp:43     (src/cluster.cpp:99-146)
 *   pgb_search_file_u8      <- pulsegrid::execute_task's chunk loop + sort + link_grid
 *                              (src/pipeline.cpp:72-106), fed raw 8-bit payload bytes
 *
 * Conventions: plain pointers and sizes, no C++ types.  Every function returns a
 * pgb_status; on failure pgb_last_error() (thread-local) holds the message and the
 * status names the reference exception type the C++ layer rethrows
 * (errors.hpp:10-67).  A context owns one CUDA stream and its device arena; distinct
 * contexts may be used from distinct threads concurrently (run_dm_loop is
 * re-entrant in the reference, src/pipeline.cpp:182-194).  There is no CPU
 * fallback: without a usable sm_100 device pgb_create fails with PGB_ERR_NO_DEVICE.
 */
#ifndef PULSEGRID_B200_H
#define PULSEGRID_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PGB_ABI_VERSION 1

typedef enum pgb_status {
    PGB_OK = 0,
    PGB_ERR_CONFIG = 1,          /* pulsegrid::config_error            errors.hpp:65-67 */
    PGB_ERR_INVALID_RANGE = 2,   /* pulsegrid::invalid_range_error     errors.hpp:48-50 */
    PGB_ERR_CHUNK_TOO_SHORT = 3, /* pulsegrid::chunk_too_short_error   errors.hpp:51-56 */
    PGB_ERR_BUDGET = 4,          /* pulsegrid::budget_exhausted_error  errors.hpp:59-61 */
    PGB_ERR_DEGENERATE = 5,      /* pulsegrid::degenerate_series_error errors.hpp:44-46 */
    PGB_ERR_INVALID_PLAN = 6,    /* pulsegrid::invalid_plan_error      errors.hpp:24-26 */
    PGB_ERR_ARGUMENT = 7,        /* bad pointer / size (std::invalid_argument) */
    PGB_ERR_INSUFFICIENT = 8,    /* pulsegrid::insufficient_statistics_error errors.hpp:40-42 */
    PGB_ERR_READ = 9,            /* pulsegrid::read_error              errors.hpp:29-34 */
    PGB_ERR_NO_DEVICE = 100,     /* no sm_100 device visible */
    PGB_ERR_CUDA = 101,          /* CUDA runtime / kernel failure */
    PGB_ERR_OOM = 102            /* device allocation failed */
} pgb_status;

/* Byte-for-byte the layout of pulsegrid::Candidate (detect.hpp:14-25): 72 bytes. */
typedef struct pgb_candidate {
    float snr;
    uint32_t _pad0;
    uint64_t peak_sample;   /* absolute sample of the peak window start */
    double time_s;          /* peak_sample * tsamp */
    uint32_t width_index;   /* ordinal into the boxcar ladder */
    uint32_t _pad1;
    uint64_t width_samples; /* 2^width_index */
    uint32_t dm_trial;
    uint32_t _pad2;
    double dm;
    uint64_t begin_sample;  /* above-threshold run, inclusive */
    uint64_t end_sample;
} pgb_candidate;

/* pulsegrid::ChunkSpec (filterbank.hpp:48-55). */
typedef struct pgb_chunk_spec {
    uint64_t index;
    uint64_t start_sample;
    uint64_t length;
    uint64_t overlap;
    uint64_t valid_begin;
    uint64_t valid_end;
} pgb_chunk_spec;

/* The numeric fields of pulsegrid::EngineConfig (engine.hpp:25-35).  n_workers,
 * memory_budget and max_in_flight are accepted and validated like the reference
 * (src/engine.cpp:87-97); on the device they only bound the trial batch size,
 * which never changes results. */
typedef struct pgb_engine_config {
    uint32_t n_workers;
    float detect_thresh;
    double tsamp;
    uint64_t boxcar_max;      /* power of two */
    uint64_t baseline_window; /* samples; 0 disables baseline removal */
    uint64_t memory_budget;
    uint64_t max_in_flight;   /* 0 = derive from memory_budget */
} pgb_engine_config;

/* pulsegrid::LinkRadii (cluster.hpp:13-17). */
typedef struct pgb_link_radii {
    uint64_t sep_time;
    uint32_t sep_dm_trials;
    uint32_t sep_width;
} pgb_link_radii;

/* pulsegrid::ClusterResult (cluster.hpp:20-28); member_ids are returned in a flat
 * array, cluster k owning member_ids[member_offset, member_offset + members). */
typedef struct pgb_cluster {
    pgb_candidate representative;
    uint64_t members;
    uint64_t begin_sample;
    uint64_t end_sample;
    double dm_lo;
    double dm_hi;
    uint64_t member_offset;
} pgb_cluster;

/* The subset of pulsegrid::FilterbankHeader (filterbank.hpp:22-43) the plan uses. */
typedef struct pgb_header {
    double fch1;
    double foff;
    double tsamp;
    uint32_t nchans;
    uint32_t _pad;
} pgb_header;

typedef enum pgb_spacing { PGB_SPACING_LINEAR = 0, PGB_SPACING_ADAPTIVE = 1 } pgb_spacing;

/* RFI excision settings (SearchParams, pipeline.hpp:31-35; rfi.hpp:10-33). */
typedef struct pgb_rfi_config {
    int32_t narrowband;  /* flag_narrowband (src/rfi.cpp:32-68) */
    int32_t broadband;   /* flag_broadband (src/rfi.cpp:70-91) */
    double k_sigma;
    double k_mad;
    int32_t local_mean;  /* MaskPolicy::local_mean (1) or zero (0), src/rfi.cpp:93-139 */
    int32_t _pad;
} pgb_rfi_config;

typedef struct pgb_context pgb_context;

/* ---- library ---------------------------------------------------------------- */
int pgb_abi_version(void);
const char* pgb_last_error(void);
pgb_status pgb_device_count(int* count);

/* ---- DM plan (host arithmetic, bit-identical to the reference build) --------- */
int64_t pgb_delay_samples(double dm, const pgb_header* header, uint32_t channel);
double pgb_adaptive_dm_step(double tol, const pgb_header* header);
/* Two-call protocol: dms/delays may be NULL to query *ntrials.  delays is
 * [ntrials][nchans] row-major when non-NULL. */
pgb_status pgb_generate_dm_trials(double dm_lo, double dm_hi, const pgb_header* header,
                                  pgb_spacing spacing, double step_or_tol, double* dms,
                                  int64_t* delays, size_t capacity, size_t* ntrials);

/* ---- context ----------------------------------------------------------------- */
pgb_status pgb_create(int device, pgb_context** ctx);
pgb_status pgb_destroy(pgb_context* ctx);
/* Upload a plan: dms[ntrials], delays[ntrials][nchans] (int64, as DmTrialPlan holds). */
pgb_status pgb_set_plan(pgb_context* ctx, const double* dms, const int64_t* delays,
                        uint32_t ntrials, uint32_t nchans);
/* Restrict subsequent runs to trials [begin, end) of the plan (multi-GPU sharding;
 * default = all).  Candidate dm_trial values stay global plan ordinals. */
pgb_status pgb_set_trial_range(pgb_context* ctx, uint32_t begin, uint32_t end);

/* ---- run_dm_loop ------------------------------------------------------------- */
/* data: time-major [spec->length][nchans] samples (8-bit codes, or widened floats).
 * data_on_device != 0 means `data` is a device pointer on the context's device.
 * Results stay on the device until fetched; counts are returned here. */
pgb_status pgb_run_dm_loop_u8(pgb_context* ctx, const uint8_t* data, int data_on_device,
                              const pgb_chunk_spec* spec, const pgb_engine_config* cfg,
                              size_t* n_candidates, size_t* n_skipped);
pgb_status pgb_run_dm_loop_f32(pgb_context* ctx, const float* data, int data_on_device,
                               const pgb_chunk_spec* spec, const pgb_engine_config* cfg,
                               size_t* n_candidates, size_t* n_skipped);
/* Candidates sorted by (peak_sample, dm_trial, width_index), skipped trials ascending. */
pgb_status pgb_fetch_candidates(pgb_context* ctx, pgb_candidate* out, size_t capacity);
pgb_status pgb_fetch_skipped(pgb_context* ctx, uint64_t* out, size_t capacity);
/* Device pointer to the last run's sorted candidates (valid until the next run). */
pgb_status pgb_device_candidates(pgb_context* ctx, const pgb_candidate** dev_ptr, size_t* n);

/* ---- dedispersion only (dedisperse_block semantics, parity tests) ------------ */
/* out: [trial_end - trial_begin][out_stride] floats; row t holds the length
 * - trial_max_delay(t) valid samples.  Trials whose span exceeds the chunk raise
 * PGB_ERR_CHUNK_TOO_SHORT (src/dedisp.cpp:137-142). */
pgb_status pgb_dedisperse_u8(pgb_context* ctx, const uint8_t* data, uint64_t length,
                             uint32_t trial_begin, uint32_t trial_end, float* out,
                             uint64_t out_stride);
pgb_status pgb_dedisperse_f32(pgb_context* ctx, const float* data, uint64_t length,
                              uint32_t trial_begin, uint32_t trial_end, float* out,
                              uint64_t out_stride);

/* ---- link_grid --------------------------------------------------------------- */
/* Clusters of `cands` (any order).  Output identical to pulsegrid::link_grid:
 * clusters sorted by representative (peak_sample, dm_trial, width_index), member ids
 * ascending.  cands may be a device pointer (cands_on_device != 0), e.g. from
 * pgb_device_candidates or the file-level accumulator. */
pgb_status pgb_link_grid(pgb_context* ctx, const pgb_candidate* cands, int cands_on_device,
                         size_t n, const pgb_link_radii* radii, size_t* n_clusters);
pgb_status pgb_fetch_clusters(pgb_context* ctx, pgb_cluster* out, size_t capacity,
                              uint64_t* member_ids, size_t member_capacity);

/* ---- file-level search (execute_task's loop, raw u8 ingest) ------------------ */
/* payload: time-major 8-bit samples of the whole file, [nsamples][nchans], in host
 * memory (pinned or pageable; uploaded segment by segment on a copy stream that
 * overlaps the previous chunk's compute) or, with payload_on_device != 0, already
 * resident in device memory.  Runs every chunk of `chunks` (plan_chunks output) with
 * double-buffered H2D, accumulates candidates on the device, sorts them and
 * clusters them with link_grid (radii == NULL: stop after the sorted candidates, as a
 * multi-GPU trial shard does before the candidate gather).  Fetch with pgb_fetch_clusters /
 * pgb_fetch_file_candidates / pgb_fetch_file_skipped. */
pgb_status pgb_search_file_u8(pgb_context* ctx, const uint8_t* payload, int payload_on_device,
                              uint64_t nsamples, const pgb_chunk_spec* chunks, size_t nchunks,
                              const pgb_engine_config* cfg, const pgb_link_radii* radii,
                              const pgb_rfi_config* rfi, size_t* n_candidates,
                              size_t* n_clusters);

/* ---- RFI excision (next row f1: the reference runs it before run_dm_loop) ------- */
/* Flags (narrowband channels, broadband samples) and masks one time-major chunk
 * [length][nchans] (u8 codes or floats; host or device) into a float chunk, exactly
 * as flag_narrowband + flag_broadband + apply_mask do.  out_host (optional) receives
 * the cleaned chunk; the flags stay fetchable with pgb_fetch_rfi_flags. */
pgb_status pgb_rfi_clean(pgb_context* ctx, const void* data, int is_u8, int on_device,
                         uint64_t length, const pgb_rfi_config* rfi, float* out_host,
                         uint64_t* n_bad_channels, uint64_t* n_bad_samples);
pgb_status pgb_fetch_rfi_flags(pgb_context* ctx, uint8_t* bad_channels, uint8_t* bad_samples);
pgb_status pgb_fetch_file_candidates(pgb_context* ctx, pgb_candidate* out, size_t capacity);
/* (chunk index, trial) pairs, as FileOutcome::skipped_trials (pipeline.hpp:59). */
pgb_status pgb_fetch_file_skipped(pgb_context* ctx, uint64_t* chunk_trial_pairs,
                                  size_t capacity, size_t* n_pairs);

/* ---- bounded-memory streaming file search ------------------------------------ */
/* execute_task with the prefetching reader (src/pipeline.cpp:66-106,
 * src/filterbank.cpp:326-419): host and device memory stay at two chunks whatever the
 * file size.  Protocol: pgb_stream_begin(plan of chunks); for k = 0..nchunks-1 in
 * order: pgb_stream_buffer(k) -> read chunk k's [length][nchans] bytes into it ->
 * pgb_stream_push(k, NULL) (or push a caller-owned host pointer); pgb_stream_finish
 * sorts, clusters (radii == NULL: candidates only) and makes the results fetchable
 * with the pgb_fetch_file_* / pgb_fetch_clusters calls.  The upload of chunk k runs
 * on a copy stream while chunk k-1 computes; pgb_stream_buffer blocks only until the
 * buffer's previous upload (chunk k-2) has left it, and may be called for chunk k+1
 * from a reader thread while chunk k is being pushed. */
pgb_status pgb_stream_begin(pgb_context* ctx, uint64_t nsamples, const pgb_chunk_spec* chunks,
                            size_t nchunks, const pgb_engine_config* cfg,
                            const pgb_link_radii* radii, const pgb_rfi_config* rfi);
pgb_status pgb_stream_buffer(pgb_context* ctx, size_t chunk, uint8_t** host_buffer,
                             size_t* capacity);
pgb_status pgb_stream_push(pgb_context* ctx, size_t chunk, const uint8_t* bytes);
/* Optional: start chunk k's upload from its pinned buffer as soon as it is filled (a
 * reader thread may call it for chunk k+1 while chunk k is being pushed), so the copy
 * overlaps chunk k's compute instead of starting inside pgb_stream_push(k+1). */
pgb_status pgb_stream_upload(pgb_context* ctx, size_t chunk);
/* Optional, progressive: upload piece `part` of `nparts` (rows [r(part), r(part+1)) of
 * chunk k, r(j) = floor(floor(L*j/nparts)/64)*64 and r(nparts) = L, L the chunk length)
 * as soon as that piece of the stream buffer
 * is filled, from any thread and in any order (ok = 0: the piece could not be read).
 * Announce the pieces first (part = 0, ok = -1: nothing uploaded) before the push can
 * happen.  pgb_stream_push(k) then transposes and dedisperses the chunk's tiles piece by piece as
 * their rows arrive, so the first chunk's read overlaps its own compute; it fails with
 * PGB_ERR_READ if a piece was reported unread. */
pgb_status pgb_stream_upload_part(pgb_context* ctx, size_t chunk, size_t part, size_t nparts, int ok);
pgb_status pgb_stream_finish(pgb_context* ctx, size_t* n_candidates, size_t* n_clusters);

/* ---- multi-GPU payload fan-out ------------------------------------------------ */
/* One process per GPU: each rank uploads 1/N of the file from host memory and pulls
 * the other ranks' slices over NVLink from their device buffers (CUDA IPC), so the
 * host link carries each byte once.  NCCL stays reserved for the candidate gather. */
#define PGB_IPC_HANDLE_BYTES 64
pgb_status pgb_device_alloc(int device, size_t bytes, void** device_ptr);
pgb_status pgb_device_free(int device, void* device_ptr);
pgb_status pgb_ipc_get_handle(const void* device_ptr, void* handle /* PGB_IPC_HANDLE_BYTES */);
pgb_status pgb_ipc_open(int device, const void* handle, void** device_ptr);
pgb_status pgb_ipc_close(void* device_ptr);
/* Copy on the context's stream (any direction; peer device pointers included). */
pgb_status pgb_copy_async(pgb_context* ctx, void* dst, const void* src, size_t bytes);
pgb_status pgb_synchronize(pgb_context* ctx);

/* ---- instrumentation --------------------------------------------------------- */
/* Kernel launches issued by this context since creation (bench gpu_launches). */
pgb_status pgb_launch_count(pgb_context* ctx, uint64_t* launches);
/* Device time (ms) of the dominant kernel (dedispersion) summed over the last
 * run_dm_loop / search_file call, measured with CUDA events on the context stream,
 * and the number of dedispersion launches it covered. */
pgb_status pgb_last_dedisp_time(pgb_context* ctx, double* ms, uint64_t* launches,
                                uint64_t* channel_adds);
/* Device time (ms) of each stage of the last pgb_run_dm_loop_* call, measured with CUDA
 * events: ms[0] dedispersion, [1] baseline removal, [2] normalisation (robust RMS),
 * [3] boxcar ladder with the threshold runs, [4] run stitching + candidate order.  The
 * stages run batched over every trial of the chunk; the C++ drop-in amortises them over
 * the processed trials for TrialTiming (engine.hpp:16-23). */
pgb_status pgb_last_stage_times(pgb_context* ctx, double* ms /* [5] */);
/* Host time (ms) of the last file search's file-level sort + link_grid (FileOutcome
 * cluster_ms, pipeline.hpp:63). */
pgb_status pgb_last_cluster_ms(pgb_context* ctx, double* ms);
/* The context's CUDA stream (cudaStream_t), for callers that order their own work. */
pgb_status pgb_stream(pgb_context* ctx, void** stream);
/* Measured CUDA-core 32-bit add throughput of `device` (lane-adds/s): the roofline
 * denominator of the ALU-bound dedispersion kernel.  per_mode (optional, [3]):
 * integer-only, fp32-only, interleaved. */
pgb_status pgb_microbench_add_peak(int device, double* adds_per_s, double* per_mode);

#ifdef __cplusplus
}
#endif

#endif /* PULSEGRID_B200_H */
