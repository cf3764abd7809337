// C ABI of libpgb200 (include/pulsegrid_b200.h): contexts, plan upload, the
// device run_dm_loop / link_grid / file search, and the host-side DM plan.
//
// Host orchestration per chunk (one CUDA stream per context, two host syncs):
//   H2D (optional) -> transpose -> dedispersion -> baseline -> robust RMS ->
//   boxcar ladder + runs -> [sync: counts] -> fragment sort + stitch ->
//   candidate sort -> [sync: count, degenerate flags]
// Results stay on the device until fetched (pgb_fetch_*).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <numeric>
#include <stdexcept>
#include <atomic>
#include <thread>
#include <vector>

#include <chrono>
#include <cstdio>
#include <condition_variable>
#include <functional>

#include "pgb_internal.h"

namespace pgb {

namespace {
thread_local std::string g_last_error;
}

void raise(pgb_status code, const std::string& msg) { throw Error{code, msg}; }

void check_cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    const pgb_status code = (e == cudaErrorMemoryAllocation) ? PGB_ERR_OOM : PGB_ERR_CUDA;
    raise(code, std::string(what) + ": " + cudaGetErrorString(e));
}

void DevBuf::reserve(size_t n, bool zero) {
    if (n <= bytes && p) return;
    // grow geometrically (at least 2x, 64 KB granules): a file search sizes several
    // buffers by its candidate count, and an exact-size regrowth per file meant a
    // cudaFree -- a device-wide synchronisation -- in nearly every call (config D's
    // concurrent contexts stalled each other on it)
    const size_t grown = p ? std::max<size_t>(n, 2 * bytes) : n;
    release();
    const size_t want = std::max<size_t>((grown + 65535) & ~size_t(65535), 256);
    PGB_CUDA(cudaMalloc(&p, want));
    bytes = want;
    if (zero) PGB_CUDA(cudaMemset(p, 0, want));
}
void DevBuf::release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
}
void PinnedBuf::reserve(size_t n) {
    if (n <= bytes && p) return;
    const size_t grown = p ? std::max<size_t>(n, 2 * bytes) : n;
    release();
    const size_t want = std::max<size_t>((grown + 4095) & ~size_t(4095), 256);
    PGB_CUDA(cudaMallocHost(&p, want));
    bytes = want;
}
void PinnedBuf::release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
}

// ---- host DM plan, bit-identical to the reference build ------------------------
// (the reference's -ffp-contract=fast turns fch1 + foff*c and dm_lo + i*step into
// FMAs; this TU is compiled with -ffp-contract=off and spells them out.)

constexpr double k_dispersion = 4.148808e3;  // dedisp.hpp:13

double channel_freq(const pgb_header* h, uint32_t c) { return std::fma(h->foff, (double)c, h->fch1); }
double max_freq(const pgb_header* h) { return h->foff >= 0 ? channel_freq(h, h->nchans - 1) : h->fch1; }
double min_freq(const pgb_header* h) { return h->foff >= 0 ? h->fch1 : channel_freq(h, h->nchans - 1); }

int64_t delay_samples(double dm, const pgb_header* h, uint32_t c) {  // src/dedisp.cpp:13-18
    const double f_ref = max_freq(h);
    const double f_c = channel_freq(h, c);
    const double delay_s = k_dispersion * dm * (1.0 / (f_c * f_c) - 1.0 / (f_ref * f_ref));
    return (int64_t)std::floor(delay_s / h->tsamp + 0.5);
}

double adaptive_step(double tol, const pgb_header* h) {  // src/dedisp.cpp:20-26
    const double f_lo = min_freq(h), f_hi = max_freq(h);
    const double band = 1.0 / (f_lo * f_lo) - 1.0 / (f_hi * f_hi);
    if (band <= 0.0) return 0.0;
    return (tol - 1.0) * h->tsamp / (k_dispersion * band);
}

// BufferPool::aligned_size (src/buffer_pool.cpp:22-24)
static size_t pool_aligned(size_t n) {
    size_t v = std::max<size_t>(n, 256);
    size_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

}  // namespace pgb

using namespace pgb;

struct ChunkRunHolder;

struct pgb_context {
    int device = 0;
    cudaStream_t st = nullptr;
    cudaStream_t copy_st = nullptr;
    cudaStream_t rms_st = nullptr;  // robust RMS of chunk k overlaps the boxcar of chunk k-1
    // asynchronous file-search back halves (boxcar, runs, append) run on bx_st, so their CTAs
    // fill the SMs the persistent dedispersion of the next chunk leaves idle in its tail;
    // ev_back[slot] marks a slot's back half done (the next front half of that slot waits)
    cudaStream_t bx_st = nullptr;
    cudaEvent_t ev_back[2] = {};
    bool back_pending[2] = {false, false};
    cudaEvent_t ev_dd0[2] = {}, ev_dd1[2] = {}, ev_front[2] = {}, ev_rms[2] = {};
    // per-stage timing of the synchronous run_dm_loop path (TrialTiming, engine.hpp:16-23):
    // RMS start on rms_st, boxcar start / end and the end of the run order on the main stream
    cudaEvent_t ev_rms0[2] = {}, ev_bx0 = nullptr, ev_bx1 = nullptr, ev_pk1 = nullptr;
    std::vector<cudaEvent_t> seg_events;
    std::vector<cudaEvent_t> sub_events;                 // first chunk's upload pieces
    std::vector<std::pair<uint64_t, cudaEvent_t>> prog;  // (end sample, event) of those pieces

    // plan
    uint32_t ntrials = 0, nchans = 0;
    std::vector<double> dms;
    std::vector<int64_t> delays;  // host copy [T][C]
    std::vector<int64_t> maxd;
    DevBuf d_delays_ct, d_dms;
    uint32_t tr_begin = 0, tr_end = 0;

    // per-chunk geometry cache (keyed on the active trial list)
    std::vector<uint32_t> active;
    std::vector<uint32_t> blk_spread;  // per 32-row block
    bool geom_valid = false;

    // device work buffers
    DevBuf in_raw, rows, series, d_active, d_blk_len, d_scale;
    // per-slot buffers: a chunk's chain state lives in slot k & 1 from its front half
    // (transpose, dedispersion, baseline, RMS) to its back half (boxcar, runs, order)
    DevBuf base[2], frms[2], status[2], d_row_len[2], slot_active[2];
    DevBuf cands_raw, cands_sorted, frags, frags_sorted, counters, sort_keys, sort_idx, sort_tmp;
    DevBuf payload, in_u8, ws_base, ws_off, dd_win, dd_off, d_keep, d_work, d_bsums, d_lmin;
    // what the series buffer holds: the dedispersed rows of the raw-sample chunk
    // [ser_start, ser_start + ser_len) at pitch ser_pitch (overlap reuse)
    bool ser_ok = false;
    uint64_t ser_start = 0, ser_len = 0, ser_pitch = 0;
    uint32_t dd_tab_wmax = 0;  // wmax the staging table was built for (0 = stale)
    DevBuf ddf_win, ddf_off;     // f32 staging table (non-integer float chunks)
    uint32_t ddf_tab_wmax = 0;
    DevBuf ddh_win, ddh_off;
    DevBuf ddy_win, ddy_off, d_dirty;  // event-replay RFI kernel (ablation): tables, fallback flag     // fp16 staging table (RFI-masked 8-bit chunks with float rows)
    uint32_t ddh_tab_wmax = 0;
    std::vector<uint32_t> bad_rows_host;  // the current chunk's flagged rows (exception density)
    DevBuf file_cands, file_sorted;
    // asynchronous file-search back halves: {candidate total, high-water nc, nf}, the
    // per-chunk degenerate-trial flags (pinned) and per-chunk dedispersion events
    DevBuf file_ctr;
    PinnedBuf h_file_status, h_file_ctr;
    std::vector<cudaEvent_t> file_dd_ev;
    // pinned staging arena for the small per-chunk uploads (a pageable cudaMemcpyAsync
    // waited for the RMS kernel running on the other stream, stalling the next chunk's
    // dedispersion); bump-allocated, reset at the start of every top-level call
    std::vector<PinnedBuf> stage;
    size_t stage_blk = 0, stage_off = 0;
    // PGB_TRACE=1: an event after each stage of a file search, printed as a timeline
    bool trace = false;
    std::vector<std::pair<std::string, cudaEvent_t>> trace_ev;
    std::vector<double> trace_host;  // host clock (ms) when each mark was issued
    DevBuf cl_scratch, clusters, members;
    DevBuf d_wide;    // rows of trial blocks too wide for the staged dedispersion
    DevBuf d_levels;  // boxcar ladder levels above the tile kernel's (boxcar_max > 8192)
    DevBuf d_bxs;     // boxcar launcher scratch
    PinnedBuf h_counters;
    RfiWork rfi;
    DevBuf rfi_out;
    uint64_t rfi_len = 0;

    // per-chunk candidate / fragment buffers; the file search sorts whole buffers (device-side
    // counts), so they start moderate and grow on overflow
    uint64_t cand_cap = 1 << 14, frag_cap = 1 << 14;

    // results
    uint64_t n_cands = 0;
    std::vector<uint64_t> skipped;
    uint64_t n_clusters = 0, n_members = 0;
    uint64_t file_ncands = 0;
    std::vector<uint64_t> file_skipped;  // (chunk, trial) pairs
    bool last_from_file = false;

    // instrumentation
    uint64_t launches = 0;
    double dedisp_ms = 0.0;
    uint64_t dedisp_launches = 0;
    uint64_t channel_adds = 0;
    double cluster_ms = 0.0;  // file-level sort + link_grid of the last file search (host clock)
    // last run_dm_loop: device ms of {dedisperse, baseline, normalize, boxcar, peaks}
    double stage_ms[5] = {};
    // last chunk's row geometry for stage fetches
    uint64_t last_out_pitch = 0;
    uint32_t last_nrows = 0;
    bool last_had_baseline = false;
    bool last_u8 = true;

    // bounded-memory streaming file search (pgb_stream_*): two pinned host and two device
    // chunk buffers, chunks pushed in order, synchronous back halves
    struct Stream {
        bool open = false;
        uint64_t nsamples = 0;
        std::vector<pgb_chunk_spec> chunks;
        pgb_engine_config cfg{};
        bool has_radii = false, has_rfi = false;
        pgb_link_radii radii{};
        pgb_rfi_config rfi{};
        size_t next = 0;        // next chunk to push
        uint64_t total = 0;     // candidates appended so far
        uint64_t pitch_min = 0;
        bool overlap = false, pending = false;
        ChunkRunHolder* runs = nullptr;
        PinnedBuf hbuf[2];
        DevBuf dbuf[2];
        cudaEvent_t up_done[2] = {}, dev_free[2] = {};
        bool up_pending[2] = {false, false}, dev_pending[2] = {false, false};
        int64_t uploaded[2] = {-1, -1};  // chunk whose upload was issued into buffer b (not yet pushed)
        std::mutex mu;                   // pgb_stream_upload (reader thread) vs pgb_stream_push
        // progressive pieces of one chunk (pgb_stream_upload_part): the chunk, piece ends
        // and events, which pieces have been issued / failed
        int64_t part_chunk = -1;
        std::vector<std::pair<uint64_t, cudaEvent_t>> parts;
        std::vector<char> part_state;  // 0 pending, 1 issued, 2 failed
        std::condition_variable cv;
    } stream;
    // host repack of widened 8-bit float chunks (pgb_run_dm_loop_f32 with host data)
    PinnedBuf h_pack;
};

namespace {

template <typename F>
pgb_status guarded(F&& f) {
    try {
        f();
        return PGB_OK;
    } catch (const Error& e) {
        g_last_error = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return PGB_ERR_OOM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return PGB_ERR_ARGUMENT;
    }
}

void need(bool cond, pgb_status code, const char* msg) {
    if (!cond) raise(code, msg);
}

struct ChunkInput {
    const void* data;   // device pointer, time-major
    bool u8;
    bool raw = false;         // the file's unmodified 8-bit samples (overlap reuse allowed)
    bool more = false;        // another chunk's dedispersion follows (RMS runs beside it)
    // progressive upload (u8, host payload): (end sample, event) of the chunk's
    // sub-segments; transpose and dedispersion start on the tiles whose inputs arrived
    const std::vector<std::pair<uint64_t, cudaEvent_t>>* prog = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;  // dedispersion timing events (else the slot's)
    uint64_t pitch_min = 0;   // series pitch floor (a file search keeps one pitch for all chunks)
    // RFI-masked 8-bit chunk (data = the raw codes, src/rfi.cpp:93-139): the transpose zeroes
    // the bad channels and bad rows; with local-mean replacement (h16) the bad rows' float
    // values come from ctx->rfi's exception lists and the fp16 in-order kernel runs, unless
    // the geometry or the flag density does not fit it -- then fallback() widens the masked
    // chunk to floats (the fp32 path)
    const uint8_t* chan_bad = nullptr;
    const uint8_t* samp_bad = nullptr;
    bool h16 = false;
    bool hyb = false;  // (with u8) local-mean rows through the event-replay kernel (ablation)
    std::function<ChunkInput()> fallback;
    // progressive chunk whose pieces are uploaded by another thread (streaming search):
    // called with the piece index before its event is waited on; returns once the piece's
    // upload has been issued (or throws)
    std::function<void(size_t)> seg_ready;
};

// Validation and in-flight arithmetic of run_dm_loop (src/engine.cpp:60-97).
void validate_cfg(pgb_context* ctx, const pgb_chunk_spec* spec, const pgb_engine_config* cfg) {
    need(spec && cfg, PGB_ERR_ARGUMENT, "null spec/config");
    if (cfg->n_workers < 1) raise(PGB_ERR_CONFIG, "n_workers must be >= 1");
    if (cfg->boxcar_max < 1 || (cfg->boxcar_max & (cfg->boxcar_max - 1)) != 0)
        raise(PGB_ERR_CONFIG, "boxcar_max must be a power of two");
    if (cfg->boxcar_max > (1ull << 30))  // ladder levels fit the 5-bit fragment level field
        raise(PGB_ERR_CONFIG, "boxcar_max above 2^30");
    if (ctx->ntrials == 0) return;
    if (cfg->max_in_flight == 0) {  // in_flight_limit, src/engine.cpp:75-83
        const int64_t min_delay = ctx->maxd[0];
        const uint64_t length = spec->length;
        const uint64_t longest = length > (uint64_t)min_delay ? length - (uint64_t)min_delay : 1;
        const size_t series_bytes = pool_aligned(longest * sizeof(float));
        const uint64_t n_blocks = (longest + 63) / 64;
        const size_t sums_bytes = pool_aligned((longest + n_blocks) * sizeof(double));
        const size_t buffers = cfg->baseline_window > 0 ? 2 : 1;
        const size_t ws = buffers * series_bytes + sums_bytes;
        if (cfg->memory_budget / ws == 0)
            raise(PGB_ERR_CONFIG, "memory budget of " + std::to_string(cfg->memory_budget) +
                                      " bytes is below one trial's working set (" +
                                      std::to_string(ws) + ")");
    }
}

uint64_t round_up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

void stage_reset(pgb_context* ctx) {
    ctx->stage_blk = 0;
    ctx->stage_off = 0;
}

// H2D copy of a small host array through the pinned arena (asynchronous for real)
void stage_h2d(pgb_context* ctx, void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (!bytes) return;
    const size_t need = (bytes + 255) & ~size_t(255);
    constexpr size_t kBlock = 4u << 20;
    while (true) {
        if (ctx->stage_blk == ctx->stage.size()) {
            ctx->stage.emplace_back();
            ctx->stage.back().reserve(std::max(kBlock, need));
            ctx->stage_off = 0;
        }
        PinnedBuf& b = ctx->stage[ctx->stage_blk];
        if (ctx->stage_off + need <= b.bytes) break;
        ++ctx->stage_blk;
        ctx->stage_off = 0;
        if (ctx->stage_blk < ctx->stage.size() && ctx->stage[ctx->stage_blk].bytes < need)
            ctx->stage[ctx->stage_blk].reserve(need);  // (not in use: blocks past the cursor are free)
    }
    char* p = ctx->stage[ctx->stage_blk].as<char>() + ctx->stage_off;
    ctx->stage_off += need;
    std::memcpy(p, src, bytes);
    // the device reads the pinned bytes itself (zero copy): a cudaMemcpyAsync would queue
    // behind the multi-GB payload segments on the H2D copy engine
    launch_copy_from_host(dst, p, bytes, st);
}

double host_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

void trace_mark(pgb_context* ctx, const char* name, cudaStream_t s) {
    if (!ctx->trace) return;
    ctx->trace_host.push_back(host_ms());
    cudaEvent_t e;
    PGB_CUDA(cudaEventCreate(&e));
    PGB_CUDA(cudaEventRecord(e, s));
    ctx->trace_ev.emplace_back(std::string(name) + (s == ctx->st ? "" : " [side stream]"), e);
}

void trace_dump(pgb_context* ctx) {
    if (!ctx->trace || ctx->trace_ev.empty()) return;
    PGB_CUDA(cudaDeviceSynchronize());
    float prev = 0.f;
    size_t k = 0;
    for (auto& [name, e] : ctx->trace_ev) {
        float t = 0.f;
        PGB_CUDA(cudaEventElapsedTime(&t, ctx->trace_ev.front().second, e));
        const double hm = k < ctx->trace_host.size() ? ctx->trace_host[k] - ctx->trace_host.front() : 0.0;
        fprintf(stderr, "[pgb trace] %9.3f ms  +%8.3f  (host %8.3f)  %s\n", t, t - prev, hm, name.c_str());
        prev = t;
        ++k;
    }
    ctx->trace_host.clear();
    for (auto& [name, e] : ctx->trace_ev) cudaEventDestroy(e);
    ctx->trace_ev.clear();
}
constexpr int PGB_PROG_SUBSEG = 8;  // pieces of the first chunk's upload

// One chunk's chain, split in two halves so a file search can overlap them across
// chunks: the front half (transpose, dedispersion, baseline on the main stream; the
// latency-bound robust RMS on rms_st) and the back half (boxcar ladder, runs,
// candidate order, degenerate trials).  Everything a back half needs lives in the
// chunk's slot, so the back half of chunk k-1 may run after the front half of chunk k.
struct ChunkRun {
    bool live = false;  // has active rows, i.e. a back half to run
    int slot = 0;
    pgb_chunk_spec spec{};
    pgb_engine_config cfg{};
    uint32_t nrows = 0;
    uint64_t out_pitch = 0, max_n = 0;
    int kind = 0;
    bool baseline = false, u8 = true;
    const void* work = nullptr;
    std::vector<uint32_t> active;
    std::vector<uint64_t> skipped;  // uncoverable trials (front) + degenerate ones (back)
};

}  // namespace
struct ChunkRunHolder {
    ChunkRun r[2];
};
namespace {

void chunk_front(pgb_context* ctx, const ChunkInput& in, const pgb_chunk_spec* spec,
                 const pgb_engine_config* cfg, int slot, ChunkRun& run) {
    NvtxRange nvtx("pgb chunk front (transpose, dedispersion, baseline, rms)");
    cudaStream_t st = ctx->st;
    if (ctx->back_pending[slot]) {  // the slot's buffers are still read by a back half on bx_st
        PGB_CUDA(cudaStreamWaitEvent(st, ctx->ev_back[slot], 0));
        ctx->back_pending[slot] = false;
    }
    const uint64_t L = spec->length;
    const uint32_t C = ctx->nchans;
    run = ChunkRun{};
    run.slot = slot;
    run.spec = *spec;
    run.cfg = *cfg;
    if (ctx->ntrials == 0 || L == 0) return;

    // active rows: trials whose span fits the chunk (src/engine.cpp:112-118)
    std::vector<uint32_t>& active = run.active;
    active.reserve(ctx->tr_end - ctx->tr_begin);
    for (uint32_t t = ctx->tr_begin; t < ctx->tr_end; ++t) {
        if ((uint64_t)ctx->maxd[t] >= L) run.skipped.push_back(t);
        else active.push_back(t);
    }
    const uint32_t nrows = (uint32_t)active.size();
    // the series buffer holds the previous chunk's rows only if it ran on the same
    // active set from the file's raw samples (set again below once this chunk is issued)
    const bool ser_prev = ctx->ser_ok && ctx->geom_valid && ctx->active == active;
    ctx->ser_ok = false;
    if (nrows == 0) return;
    if (ctx->nchans > 0 && nrows > (1u << 20)) raise(PGB_ERR_CONFIG, "more than 2^20 trials");

    std::vector<uint32_t> row_len(nrows);
    uint64_t max_n = 0, maxd_active = 0;
    for (uint32_t r = 0; r < nrows; ++r) {
        row_len[r] = (uint32_t)(L - (uint64_t)ctx->maxd[active[r]]);
        max_n = std::max<uint64_t>(max_n, row_len[r]);
        maxd_active = std::max<uint64_t>(maxd_active, (uint64_t)ctx->maxd[active[r]]);
    }
    // per 32-row block: longest series and channel window spread (cached per active set)
    const int tpw = 2, tb = DD_WARPS * tpw;
    const uint32_t nblocks = (nrows + tb - 1) / tb;
    if (!ctx->geom_valid || ctx->active != active) {
        ctx->blk_spread.assign(nblocks, 0);
        for (uint32_t b = 0; b < nblocks; ++b) {
            const uint32_t r0 = b * tb, r1 = std::min(nrows, r0 + tb);
            uint32_t sp = 0;
            for (uint32_t c = 0; c < C; ++c) {
                int64_t lo = INT64_MAX, hi = INT64_MIN;
                for (uint32_t r = r0; r < r1; ++r) {
                    const int64_t d = ctx->delays[(size_t)active[r] * C + c];
                    lo = std::min(lo, d);
                    hi = std::max(hi, d);
                }
                sp = std::max<uint32_t>(sp, (uint32_t)(hi - lo));
            }
            ctx->blk_spread[b] = sp;
        }
        ctx->active = active;
        ctx->geom_valid = true;
        ctx->dd_tab_wmax = 0;
        ctx->ddf_tab_wmax = 0;
        ctx->ddh_tab_wmax = 0;
        ctx->d_active.reserve(nrows * sizeof(uint32_t));
        stage_h2d(ctx, ctx->d_active.p, active.data(), nrows * sizeof(uint32_t), st);
    }
    std::vector<uint32_t> blk_len(nblocks, 0);
    for (uint32_t r = 0; r < nrows; ++r) blk_len[r / tb] = std::max(blk_len[r / tb], row_len[r]);
    const bool u8 = in.u8;
    const bool h16 = in.h16;  // RFI-masked 8-bit chunk with float rows: the fp16 in-order kernel
    const bool hyb = in.hyb;  // ... or the event-replay kernel over the masked integer codes
    const bool ints = u8 && !hyb;  // integer series (else fp32)
    if (u8 && C > PGB_MAX_EXACT_CHANS)
        raise(PGB_ERR_CONFIG, "8-bit input with more than 65793 channels: the integer channel sums pass "
                              "2^24, where the reference's fp32 sums start rounding (widen to floats)");
    // Blocks whose channel delay spread fits a staged window go through the shared-memory
    // kernels; wider ones (very coarse DM steps) through the direct kernel, which reads
    // the channel rows from L1/L2.  The staged kernels skip those (block length 0).
    uint32_t spread = 0;
    std::vector<uint32_t> wide_rows;
    for (uint32_t b = 0; b < nblocks; ++b) {
        if (h16 || dedisp_staged_fits(u8, ctx->blk_spread[b])) {
            spread = std::max(spread, ctx->blk_spread[b]);
        } else {
            for (uint32_t r = b * tb; r < std::min(nrows, (b + 1) * tb); ++r) wide_rows.push_back(r);
            blk_len[b] = 0;
        }
    }
    const uint32_t align_el = u8 ? 16 : 4;
    const uint32_t wmax = h16 ? (uint32_t)round_up(spread + DD_NT + 32, 16)  // halves per copy
                              : (uint32_t)round_up(spread + DD_NT + 2 * align_el + 16, 16);
    int g = 8;
    if (h16) {
        // every block must fit a staged window, and no window may cover more than HX_CAP
        // flagged rows (a window of wmax + 2 rows covers R[lo..hi] iff R[hi] - R[lo] < wmax + 2)
        g = dedisp_h16_stage_width(wmax);
        const std::vector<uint32_t>& R = ctx->bad_rows_host;
        size_t dense = 0;  // most flagged rows in one window
        for (size_t lo = 0, hi = 0; hi < R.size(); ++hi) {
            while ((uint64_t)R[hi] - R[lo] >= (uint64_t)wmax + 2) ++lo;
            dense = std::max(dense, hi - lo + 1);
        }
        static const bool which = getenv("PGB_DD_WHICH") != nullptr;
        if (which)
            fprintf(stderr, "pgb rfi: %zu flagged rows, at most %zu per %u-row window, stage width %d\n", R.size(),
                    dense, wmax + 2, g);
        if (g == 0 || dense > (size_t)HX_CAP) {
            ChunkInput fb = in.fallback();
            fb.more = in.more;
            fb.ev0 = in.ev0;
            fb.ev1 = in.ev1;
            fb.pitch_min = in.pitch_min;
            chunk_front(ctx, fb, spec, cfg, slot, run);
            return;
        }
    } else {
        while (g > 1 && dedisp_smem_bytes(u8, g, wmax) > DD_SMEM_BUDGET) g >>= 1;
    }
    if (hyb) {
        // every block staged, integer sums below 2^21 (the merges' exactness bound), room for
        // the head, at most HX_CAP flagged rows per staged window
        const uint32_t hw = hyb_wmax(spread);
        const std::vector<uint32_t>& R = ctx->bad_rows_host;
        size_t dense = 0;
        for (size_t lo = 0, hi = 0; hi < R.size(); ++hi) {
            while ((uint64_t)R[hi] - R[lo] >= (uint64_t)hw + 4) ++lo;
            dense = std::max(dense, hi - lo + 1);
        }
        const uint32_t cpad = (C + 7) & ~7u;
        if (!wide_rows.empty() || !hyb_fits(hw) || (uint64_t)C * 255 >= (1u << 21) ||
            cpad < hyb_head_channels() + 8 || dense > (size_t)HX_CAP) {
            ChunkInput fb = in.fallback();
            fb.more = in.more;
            fb.ev0 = in.ev0;
            fb.ev1 = in.ev1;
            fb.pitch_min = in.pitch_min;
            chunk_front(ctx, fb, spec, cfg, slot, run);
            return;
        }
    }
    // warp-specialized TMA kernel (u8): 16-byte aligned window starts, 256-byte boxes,
    // >= 20 bytes of slack for the packers' funnel shifts; deepest ring that fits
    int ws_g = 0, ws_ns = 0;
    const uint32_t ws_wmax = (uint32_t)round_up(spread + DD_NT + 16 + 20, 2048);
#ifdef PGB_ABLATIONS
    if (u8 && dedisp_ws_available()) {
        const int cand[][2] = {{8, 4}, {8, 3}, {4, 4}, {4, 3}, {8, 2}, {2, 4}, {4, 2}, {2, 3}, {1, 4}, {1, 2}};
        for (const auto& c : cand)
            if (dedisp_ws_smem_bytes(c[0], ws_wmax, c[1]) <= 220 * 1024) {
                ws_g = c[0];
                ws_ns = c[1];
                break;
            }
        const char* eg = pgb_ablation_env("PGB_WS_G");  // geometry overrides (experiments)
        const char* en = pgb_ablation_env("PGB_WS_NS");
        if (eg && en && dedisp_ws_smem_bytes(atoi(eg), ws_wmax, atoi(en)) <= 220 * 1024) {
            ws_g = atoi(eg);
            ws_ns = atoi(en);
        }
    }
#endif
    const uint32_t ntiles = (uint32_t)((max_n + DD_NT - 1) / DD_NT);
    const uint64_t out_pitch = std::max<uint64_t>((uint64_t)ntiles * DD_NT, round_up(in.pitch_min, DD_NT));
    const uint64_t rows_pitch =
        round_up((uint64_t)ntiles * DD_NT + maxd_active + std::max(wmax, ws_wmax) + 64, 64);
    const size_t esz = u8 ? 1 : h16 ? 2 : 4;

    const uint32_t C_pad = (C + 7) & ~7u;  // u8/fp16 rows padded with zero rows to whole 8-channel groups
    ctx->rows.reserve((size_t)(u8 || h16 ? C_pad : C) * rows_pitch * esz, true);
    ctx->series.reserve((size_t)nrows * out_pitch * 4);
    const bool baseline = cfg->baseline_window > 0;
    if (baseline) ctx->base[slot].reserve((size_t)nrows * out_pitch * 4);
    ctx->frms[slot].reserve(nrows * sizeof(float));
    ctx->status[slot].reserve(nrows);
    ctx->d_row_len[slot].reserve(nrows * sizeof(uint32_t));
    ctx->slot_active[slot].reserve(nrows * sizeof(uint32_t));
    ctx->d_blk_len.reserve(nblocks * sizeof(uint32_t));
    stage_h2d(ctx, ctx->d_row_len[slot].p, row_len.data(), nrows * sizeof(uint32_t), st);
    stage_h2d(ctx, ctx->slot_active[slot].p, active.data(), nrows * sizeof(uint32_t), st);
    stage_h2d(ctx, ctx->d_blk_len.p, blk_len.data(), nblocks * sizeof(uint32_t), st);
    // ladder scales 1/sqrt(w) (src/engine.cpp:207), computed on the host like the reference
    {
        double sc[32];
        for (int l = 0; l < 32; ++l) sc[l] = 1.0 / std::sqrt((double)(1ull << l));
        ctx->d_scale.reserve(sizeof sc);
        stage_h2d(ctx, ctx->d_scale.p, sc, sizeof sc, st);
    }

    if (!wide_rows.empty()) {
        ctx->d_wide.reserve(wide_rows.size() * sizeof(uint32_t));
        stage_h2d(ctx, ctx->d_wide.p, wide_rows.data(), wide_rows.size() * sizeof(uint32_t), st);
    }
    // 1. transpose to channel-major rows (a progressive chunk transposes per sub-segment
    // below, interleaved with the dedispersion of the tiles it completes)
    const bool progressive = u8 && in.prog && !ws_g && !in.prog->empty() && wide_rows.empty();
    if (in.prog && !in.prog->empty() && !progressive) {  // whole chunk first
        if (in.seg_ready) {  // pieces uploaded in any order by another thread: wait for each
            for (size_t j = 0; j < in.prog->size(); ++j) {
                in.seg_ready(j);
                PGB_CUDA(cudaStreamWaitEvent(st, (*in.prog)[j].second, 0));
            }
        } else {
            PGB_CUDA(cudaStreamWaitEvent(st, in.prog->back().second, 0));
        }
    }
    if (u8) {
        if (in.chan_bad)  // RFI zero mask: integer cells, bad channels and rows zeroed
            launch_transpose_masked(static_cast<const uint8_t*>(in.data), L, C, in.chan_bad, in.samp_bad,
                                    ctx->rows.p, rows_pitch, false, st);
        else if (!progressive)
            launch_transpose_u8(static_cast<const uint8_t*>(in.data), L, C, ctx->rows.as<uint8_t>(),
                                rows_pitch, st);
        trace_mark(ctx, "transpose", st);
        if (C_pad > C)
            PGB_CUDA(cudaMemsetAsync(ctx->rows.as<uint8_t>() + (size_t)C * rows_pitch, 0,
                                     (size_t)(C_pad - C) * rows_pitch, st));
    } else if (h16) {
        launch_transpose_masked(static_cast<const uint8_t*>(in.data), L, C, in.chan_bad, in.samp_bad,
                                ctx->rows.p, rows_pitch, true, st);
        trace_mark(ctx, "transpose (fp16, masked)", st);
        if (C_pad > C)
            PGB_CUDA(cudaMemsetAsync(ctx->rows.as<uint16_t>() + (size_t)C * rows_pitch, 0,
                                     (size_t)(C_pad - C) * rows_pitch * 2, st));
    }
    else
        launch_transpose_f32(static_cast<const float*>(in.data), L, C, ctx->rows.as<float>(),
                             rows_pitch, st);
    // 2. dedispersion
    DedispLaunch dl{};
    dl.delays_ct = ctx->d_delays_ct.as<int32_t>();
    dl.ntrials_plan = ctx->ntrials;
    dl.nchans = C;
    dl.active = ctx->d_active.as<uint32_t>();
    dl.nrows = nrows;
    dl.row_len = ctx->d_row_len[slot].as<uint32_t>();
    dl.blk_len = ctx->d_blk_len.as<uint32_t>();
    dl.rows_pitch = rows_pitch;
    dl.out_pitch = out_pitch;
    dl.tpw = tpw;
    dl.g = g;
    dl.wmax = wmax;
    dl.ntiles = ntiles;
    dl.mul24 = 1u << 24;
    uint64_t reused = 0;  // channel-adds taken over from the previous chunk
    PGB_CUDA(cudaEventRecord(in.ev0 ? in.ev0 : ctx->ev_dd0[slot], st));
#ifdef PGB_ABLATIONS
    if (u8 && ws_g) {
        DedispLaunch dw = dl;
        dw.g = ws_g;
        dw.wmax = ws_wmax;
        dw.nchans_pad = (C + 7) & ~7u;
        ctx->ws_base.reserve((size_t)nblocks * C * 4);
        ctx->ws_off.reserve((size_t)nblocks * dw.nchans_pad * 32 * 2);
        dw.wbase = ctx->ws_base.as<uint32_t>();
        dw.woff = ctx->ws_off.as<uint16_t>();
        launch_ws_offsets(dw, ctx->ws_base.as<uint32_t>(), ctx->ws_off.as<uint16_t>(), st);
        ctx->launches += 1;
        launch_dedisp_u8_ws(dw, ws_ns, ctx->rows.as<uint8_t>(), ctx->series.as<int32_t>(), st);
    } else
#endif
    if (hyb) {
        dl.nchans_pad = C_pad;
        dl.wmax = hyb_wmax(spread);
        dl.ntiles = (uint32_t)((max_n + hyb_tile_len() - 1) / hyb_tile_len());
        ctx->ddy_win.reserve((size_t)nblocks * C_pad * sizeof(uint2));
        ctx->ddy_off.reserve((size_t)nblocks * C_pad * 32 * 4);
        dl.dd_win = ctx->ddy_win.as<uint2>();
        dl.dd_off = ctx->ddy_off.as<uint32_t>();
        dl.xP = ctx->rfi.xP.as<uint32_t>();
        dl.xR = ctx->rfi.xR.as<uint32_t>();
        dl.xF = ctx->rfi.xF.as<float>();
        dl.xlen = L;
        ctx->d_work.reserve(64 * sizeof(uint32_t), true);
        dl.work_ctr = ctx->d_work.as<uint32_t>();
        ctx->d_dirty.reserve(sizeof(unsigned));
        launch_dedisp_hyb(dl, ctx->rows.as<uint8_t>(), ctx->series.as<float>(), ctx->d_dirty.as<unsigned>(), st);
        ctx->launches += 4;
        ctx->h_counters.reserve(4 * sizeof(unsigned long long));
        auto* hd = ctx->h_counters.as<unsigned long long>() + 3;
        *hd = 0;
        PGB_CUDA(cudaMemcpyAsync(hd, ctx->d_dirty.p, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        PGB_CUDA(cudaStreamSynchronize(st));
        static const bool which = getenv("PGB_DD_WHICH") != nullptr;
        if (which && *hd) fprintf(stderr, "pgb rfi: event replay undecidable, chunk recomputed on the fp32 path\n");
        if (*hd) {  // a state below 256 crossed two binades in one merge: the fp32 path
            ChunkInput fb = in.fallback();
            fb.more = in.more;
            fb.ev0 = in.ev0;
            fb.ev1 = in.ev1;
            fb.pitch_min = in.pitch_min;
            chunk_front(ctx, fb, spec, cfg, slot, run);
            return;
        }
    } else
    if (u8) {
        dl.nchans_pad = C_pad;
        if (ctx->dd_tab_wmax != wmax) {
            ctx->dd_win.reserve((size_t)nblocks * dl.nchans_pad * sizeof(uint2));
            ctx->dd_off.reserve((size_t)nblocks * dl.nchans_pad * 32 * 4);
            launch_dd_table(dl, ctx->dd_win.as<uint2>(), ctx->dd_off.as<uint32_t>(), st);
            ctx->launches += 1;
            ctx->dd_tab_wmax = wmax;
        }
        dl.dd_win = ctx->dd_win.as<uint2>();
        dl.dd_off = ctx->dd_off.as<uint32_t>();
        // Overlap reuse (file search, raw 8-bit chunks): the dedispersed value of an
        // absolute sample does not depend on the chunk, so outputs chunk k-1 already
        // produced -- [start_k, start_{k-1} + L_{k-1} - d_t) for trial t -- are moved to
        // the front of each row instead of being summed again.  Every output of chunk k
        // is still a sum over the same input bytes, so the series is unchanged bit for bit.
        if (in.raw && ser_prev && out_pitch == ctx->ser_pitch && spec->start_sample > ctx->ser_start &&
            !pgb_ablation_env("PGB_NO_OVERLAP_REUSE")) {
            const uint64_t shift = spec->start_sample - ctx->ser_start;
            std::vector<uint32_t> keep(nrows);
            uint64_t kmax = 0;
            for (uint32_t r = 0; r < nrows; ++r) {
                const uint64_t prev_n = ctx->ser_len - (uint64_t)ctx->maxd[active[r]];
                const uint64_t k = prev_n > shift ? std::min<uint64_t>(prev_n - shift, row_len[r]) : 0;
                keep[r] = (uint32_t)k;
                kmax = std::max(kmax, k);
            }
            if (kmax >= DD_NT && shift >= kmax) {
                std::vector<uint32_t> first(nblocks, UINT32_MAX);
                for (uint32_t r = 0; r < nrows; ++r)
                    first[r / tb] = std::min<uint32_t>(first[r / tb], keep[r] / DD_NT);
                const uint32_t tile0 = *std::min_element(first.begin(), first.end());
                ctx->d_keep.reserve((size_t)(nrows + nblocks) * sizeof(uint32_t));
                uint32_t* dk = ctx->d_keep.as<uint32_t>();
                stage_h2d(ctx, dk, keep.data(), nrows * 4, st);
                stage_h2d(ctx, dk + nrows, first.data(), nblocks * 4, st);
                launch_series_shift(ctx->series.as<int32_t>(), nrows, out_pitch, shift, dk, st);
                trace_mark(ctx, "series shift", st);
                ctx->launches += 1;
                dl.blk_first = dk + nrows;
                dl.tile0 = tile0;
                for (uint32_t r = 0; r < nrows; ++r) reused += (uint64_t)keep[r] * C;
            }
        }
        // persistent ring kernel: one CTA per SM pulling (block, tile) items from a counter
        if (!pgb_ablation_env("PGB_DD_PERSIST0")) {
            ctx->d_work.reserve(64 * sizeof(uint32_t), true);
            dl.work_ctr = ctx->d_work.as<uint32_t>();
        }
        auto dd_launch = [&](const DedispLaunch& part) {
            if (part.work_ctr) PGB_CUDA(cudaMemsetAsync(part.work_ctr, 0, sizeof(uint32_t), st));
            launch_dedisp_u8(part, ctx->rows.as<uint8_t>(), ctx->series.as<int32_t>(), st);
        };
        if (progressive && dl.tile0 == 0) {
            // tile t reads channel rows up to t*DD_NT + max delay + DD_NT + 20 bytes (window
            // start rounded down to 16, whole 16-byte vectors, one extra word)
            uint64_t a = 0;
            uint32_t done = 0;
            size_t segi = 0;
            for (const auto& seg : *in.prog) {
                const uint64_t b = std::min<uint64_t>(seg.first, L);
                if (in.seg_ready) in.seg_ready(segi);
                ++segi;
                PGB_CUDA(cudaStreamWaitEvent(st, seg.second, 0));
                if (ctx->trace) trace_mark(ctx, "piece arrived", st);
                if (b > a) {
                    launch_transpose_u8(static_cast<const uint8_t*>(in.data) + a * C, b - a, C,
                                        ctx->rows.as<uint8_t>() + a, rows_pitch, st);
                    ctx->launches += 1;
                }
                a = b;
                const uint64_t need = maxd_active + 2 * DD_NT + 64;
                uint32_t t_end = b >= L ? ntiles : (b >= need ? (uint32_t)((b - need) / DD_NT) + 1 : 0);
                t_end = std::min(t_end, ntiles);
                if (t_end > done) {
                    DedispLaunch part = dl;
                    part.tile0 = done;
                    part.ntiles = t_end;
                    dd_launch(part);
                    ctx->launches += 1;
                    done = t_end;
                    if (ctx->trace) trace_mark(ctx, "dedispersion piece", st);
                }
            }
            if (done < ntiles) {  // (the last sub-segment ends at L, so this does not happen)
                DedispLaunch part = dl;
                part.tile0 = done;
                dd_launch(part);
            }
        } else if (wide_rows.size() < nrows) {
            dd_launch(dl);
        }
        launch_dedisp_direct(dl, true, ctx->rows.p, ctx->series.p, ctx->d_wide.as<uint32_t>(),
                             (uint32_t)wide_rows.size(), st);
        if (in.raw) {
            ctx->ser_ok = true;
            ctx->ser_start = spec->start_sample;
            ctx->ser_len = L;
            ctx->ser_pitch = out_pitch;
        }
    }
    else if (h16) {
        dl.nchans_pad = C_pad;
        if (ctx->ddh_tab_wmax != wmax) {
            ctx->ddh_win.reserve((size_t)nblocks * dl.nchans_pad * sizeof(uint2));
            ctx->ddh_off.reserve((size_t)nblocks * dl.nchans_pad * 32 * 4);
            launch_ddh_table(dl, ctx->ddh_win.as<uint2>(), ctx->ddh_off.as<uint32_t>(), st);
            ctx->launches += 1;
            ctx->ddh_tab_wmax = wmax;
        }
        dl.dd_win = ctx->ddh_win.as<uint2>();
        dl.dd_off = ctx->ddh_off.as<uint32_t>();
        dl.xP = ctx->rfi.xP.as<uint32_t>();
        dl.xR = ctx->rfi.xR.as<uint32_t>();
        dl.xF = ctx->rfi.xF.as<float>();
        dl.xlen = L;
        ctx->d_work.reserve(64 * sizeof(uint32_t), true);
        dl.work_ctr = ctx->d_work.as<uint32_t>();
        PGB_CUDA(cudaMemsetAsync(dl.work_ctr, 0, sizeof(uint32_t), st));
        launch_dedisp_h16(dl, ctx->rows.as<uint16_t>(), ctx->series.as<float>(), st);
    }
    else {
        dl.nchans_pad = (C + 7) & ~7u;
        if (dl.tpw == 2) {
            if (ctx->ddf_tab_wmax != wmax) {
                ctx->ddf_win.reserve((size_t)nblocks * dl.nchans_pad * sizeof(uint2));
                ctx->ddf_off.reserve((size_t)nblocks * dl.nchans_pad * 32 * 4);
                launch_ddf_table(dl, ctx->ddf_win.as<uint2>(), ctx->ddf_off.as<uint32_t>(), st);
                ctx->launches += 1;
                ctx->ddf_tab_wmax = wmax;
            }
            dl.dd_win = ctx->ddf_win.as<uint2>();
            dl.dd_off = ctx->ddf_off.as<uint32_t>();
        }
        if (wide_rows.size() < nrows) launch_dedisp_f32(dl, ctx->rows.as<float>(), ctx->series.as<float>(), st);
        launch_dedisp_direct(dl, false, ctx->rows.p, ctx->series.p, ctx->d_wide.as<uint32_t>(),
                             (uint32_t)wide_rows.size(), st);
    }
    PGB_CUDA(cudaEventRecord(in.ev1 ? in.ev1 : ctx->ev_dd1[slot], st));
    trace_mark(ctx, "dedispersion", st);
    ctx->dedisp_launches += 1;
    ctx->launches += 2;
    uint64_t adds = 0;
    for (uint32_t r = 0; r < nrows; ++r) adds += (uint64_t)row_len[r] * C;
    ctx->channel_adds += adds - reused;

    // 3. baseline, 4. robust RMS (on rms_st: one sequential chain per thread, so it
    // leaves the SMs nearly idle and overlaps the previous chunk's boxcar)
    const void* work = ctx->series.p;
    int kind = ints ? 1 : 0;
    const uint32_t* d_len = ctx->d_row_len[slot].as<uint32_t>();
    if (baseline) {
        const uint64_t w = cfg->baseline_window % 2 == 0 ? cfg->baseline_window + 1 : cfg->baseline_window;
        if (ints)
        {
            long long* bsums = nullptr;
            if (!pgb_ablation_env("PGB_BASELINE_SERIAL")) {
                ctx->d_bsums.reserve(baseline_block_sums_bytes(nrows, out_pitch));
                bsums = ctx->d_bsums.as<long long>();
            }
            launch_baseline_int(ctx->series.as<int32_t>(), ctx->base[slot].as<float>(), d_len, nrows,
                                out_pitch, w, bsums, st);
        }
        else
        {
            long long* bsums = nullptr;
            int* lmin = nullptr;
            if (!pgb_ablation_env("PGB_BASELINE_SERIAL")) {
                ctx->d_bsums.reserve(baseline_block_sums_bytes(nrows, out_pitch));
                ctx->d_lmin.reserve(nrows * sizeof(int));
                bsums = ctx->d_bsums.as<long long>();
                lmin = ctx->d_lmin.as<int>();
            }
            launch_baseline_f32(ctx->series.as<float>(), ctx->base[slot].as<float>(), d_len, nrows,
                                out_pitch, w, bsums, lmin, st);
        }
        work = ctx->base[slot].p;
        kind = 0;
    }
    trace_mark(ctx, "baseline", st);
    static const bool rms_main = pgb_ablation_env("PGB_RMS_MAIN") != nullptr;  // experiment: no overlap
    cudaStream_t rst = rms_main ? st : ctx->rms_st;
    PGB_CUDA(cudaEventRecord(ctx->ev_front[slot], st));
    PGB_CUDA(cudaStreamWaitEvent(rst, ctx->ev_front[slot], 0));
    PGB_CUDA(cudaEventRecord(ctx->ev_rms0[slot], rst));
    launch_rms(work, kind, d_len, nrows, out_pitch, ctx->frms[slot].as<float>(),
               ctx->status[slot].as<uint8_t>(), in.more && !rms_main, rst);
    PGB_CUDA(cudaEventRecord(ctx->ev_rms[slot], rst));
    trace_mark(ctx, "robust rms", rst);
    ctx->launches += 5;

    run.live = true;
    run.nrows = nrows;
    run.out_pitch = out_pitch;
    run.max_n = max_n;
    run.kind = kind;
    run.baseline = baseline;
    run.u8 = ints;
    run.work = work;
}

// The boxcar launcher's tile list (tiles the prefix kernel hands to the tree kernel).
void* box_scratch(pgb_context* ctx, uint32_t nrows, uint64_t max_len, uint64_t boxcar_max) {
    ctx->d_bxs.reserve(boxcar_scratch_bytes(nrows, max_len, boxcar_max));
    return ctx->d_bxs.p;
}

// Global ladder levels for boxcar_max > BX_TILE_MAX (null otherwise).
double* box_levels(pgb_context* ctx, uint64_t boxcar_max, uint32_t nrows, uint64_t pitch) {
    const size_t b = boxcar_levels_bytes(boxcar_max, nrows, pitch);
    if (!b) return nullptr;
    ctx->d_levels.reserve(b);
    return ctx->d_levels.as<double>();
}

void chunk_back(pgb_context* ctx, ChunkRun& run) {
    NvtxRange nvtx("pgb chunk back (boxcar, runs, order)");
    cudaStream_t st = ctx->st;
    const int slot = run.slot;
    const pgb_chunk_spec* spec = &run.spec;
    const pgb_engine_config* cfg = &run.cfg;
    ctx->n_cands = 0;
    ctx->skipped = run.skipped;
    ctx->last_nrows = 0;
    if (!run.live) return;
    const uint32_t nrows = run.nrows;
    const uint64_t out_pitch = run.out_pitch, max_n = run.max_n;
    const int kind = run.kind;
    const void* work = run.work;
    const std::vector<uint32_t>& active = run.active;
    PGB_CUDA(cudaStreamWaitEvent(st, ctx->ev_rms[slot], 0));
    PGB_CUDA(cudaEventRecord(ctx->ev_bx0, st));

    // 5. boxcar ladder + runs (re-run with larger buffers on overflow)
    ChainParams cp{};
    cp.start_sample = spec->start_sample;
    cp.valid_begin = spec->valid_begin;
    cp.valid_end = spec->valid_end;
    cp.drop_left = spec->start_sample > 0;
    cp.drop_right = spec->overlap > 0;
    cp.tsamp = cfg->tsamp;
    cp.threshold = (double)cfg->detect_thresh;
    cp.boxcar_max = cfg->boxcar_max;
    ctx->counters.reserve(4 * sizeof(unsigned long long));
    ctx->h_counters.reserve(4 * sizeof(unsigned long long));
    auto* dcnt = ctx->counters.as<unsigned long long>();
    auto* hcnt = ctx->h_counters.as<unsigned long long>();
    for (int attempt = 0;; ++attempt) {
        ctx->cands_raw.reserve(ctx->cand_cap * sizeof(pgb_candidate));
        ctx->frags.reserve(ctx->frag_cap * sizeof(Fragment));
        PGB_CUDA(cudaMemsetAsync(dcnt, 0, 2 * sizeof(unsigned long long), st));
        if (attempt) PGB_CUDA(cudaEventRecord(ctx->ev_bx0, st));  // time the final attempt
        launch_boxcar_peaks(work, kind, ctx->d_row_len[slot].as<uint32_t>(), ctx->frms[slot].as<float>(),
                            ctx->status[slot].as<uint8_t>(), nrows, out_pitch, max_n, cp,
                            ctx->slot_active[slot].as<uint32_t>(), ctx->d_dms.as<double>(),
                            ctx->d_scale.as<double>(), ctx->cands_raw.as<pgb_candidate>(), dcnt,
                            ctx->cand_cap, ctx->frags.as<Fragment>(), dcnt + 1, ctx->frag_cap,
                            box_levels(ctx, cfg->boxcar_max, nrows, out_pitch),
                            box_scratch(ctx, nrows, max_n, cfg->boxcar_max), st);
        PGB_CUDA(cudaEventRecord(ctx->ev_bx1, st));
        PGB_CUDA(cudaMemcpyAsync(hcnt, dcnt, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        PGB_CUDA(cudaStreamSynchronize(st));
        const uint64_t nc = hcnt[0], nf = hcnt[1];
        ctx->launches += 1;
        if (nc > ctx->cand_cap || nf > ctx->frag_cap) {
            ctx->cand_cap = std::max<uint64_t>(ctx->cand_cap, round_up(nc * 2, 1024));
            ctx->frag_cap = std::max<uint64_t>(ctx->frag_cap, round_up(nf * 2, 1024));
            continue;
        }
        if (nf) {
            ctx->frags_sorted.reserve(nf * sizeof(Fragment));
            const size_t tmp = sort_fragments_temp_bytes(nf);
            ctx->sort_tmp.reserve(tmp);
            ctx->sort_keys.reserve(2 * nf * sizeof(uint64_t));
            ctx->sort_idx.reserve(2 * nf * sizeof(uint32_t));
            sort_fragments(ctx->frags.as<Fragment>(), ctx->frags_sorted.as<Fragment>(), nf,
                           ctx->sort_tmp.p, tmp, ctx->sort_keys.as<uint64_t>(),
                           ctx->sort_keys.as<uint64_t>() + nf, ctx->sort_idx.as<uint32_t>(),
                           ctx->sort_idx.as<uint32_t>() + nf, st);
            launch_stitch(ctx->frags_sorted.as<Fragment>(), nf, ctx->d_row_len[slot].as<uint32_t>(), cp,
                          ctx->slot_active[slot].as<uint32_t>(), ctx->d_dms.as<double>(),
                          ctx->cands_raw.as<pgb_candidate>(), dcnt, ctx->cand_cap, st);
            PGB_CUDA(cudaMemcpyAsync(hcnt, dcnt, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
            PGB_CUDA(cudaStreamSynchronize(st));
            ctx->launches += 4;
            if (hcnt[0] > ctx->cand_cap) {
                ctx->cand_cap = round_up(hcnt[0] * 2, 1024);
                continue;
            }
        }
        ctx->n_cands = hcnt[0];
        break;
    }
    // 6. candidate order
    const uint64_t nc = ctx->n_cands;
    ctx->cands_sorted.reserve(std::max<uint64_t>(nc, 1) * sizeof(pgb_candidate));
    if (nc) {
        const size_t tmp = sort_candidates_temp_bytes(nc);
        ctx->sort_tmp.reserve(tmp);
        ctx->sort_keys.reserve(2 * nc * sizeof(uint64_t));
        ctx->sort_idx.reserve(2 * nc * sizeof(uint32_t));
        sort_candidates(ctx->cands_raw.as<pgb_candidate>(), ctx->cands_sorted.as<pgb_candidate>(),
                        nc, ctx->sort_tmp.p, tmp, ctx->sort_keys.as<uint64_t>(),
                        ctx->sort_keys.as<uint64_t>() + nc, ctx->sort_idx.as<uint32_t>(),
                        ctx->sort_idx.as<uint32_t>() + nc, st);
        ctx->launches += 3;
    }
    PGB_CUDA(cudaEventRecord(ctx->ev_pk1, st));
    // 7. degenerate trials (src/engine.cpp:189-194) join the uncoverable ones
    std::vector<uint8_t> stat(nrows);
    PGB_CUDA(cudaMemcpyAsync(stat.data(), ctx->status[slot].p, nrows, cudaMemcpyDeviceToHost, st));
    PGB_CUDA(cudaStreamSynchronize(st));
    for (uint32_t r = 0; r < nrows; ++r)
        if (stat[r]) ctx->skipped.push_back(active[r]);
    std::sort(ctx->skipped.begin(), ctx->skipped.end());
    float ms = 0.f;
    PGB_CUDA(cudaEventElapsedTime(&ms, ctx->ev_dd0[slot], ctx->ev_dd1[slot]));
    ctx->dedisp_ms += ms;
    {  // stage times of this chunk (device clock): dedispersion, baseline, RMS, ladder, runs
        float t[4] = {};
        PGB_CUDA(cudaEventElapsedTime(&t[0], ctx->ev_dd1[slot], ctx->ev_front[slot]));
        PGB_CUDA(cudaEventElapsedTime(&t[1], ctx->ev_rms0[slot], ctx->ev_rms[slot]));
        PGB_CUDA(cudaEventElapsedTime(&t[2], ctx->ev_bx0, ctx->ev_bx1));
        PGB_CUDA(cudaEventElapsedTime(&t[3], ctx->ev_bx1, ctx->ev_pk1));
        ctx->stage_ms[0] = ms;
        for (int k = 0; k < 4; ++k) ctx->stage_ms[k + 1] = t[k];
    }
    ctx->last_out_pitch = out_pitch;
    ctx->last_nrows = nrows;
    ctx->last_had_baseline = run.baseline;
    ctx->last_u8 = run.u8;
}

// File-search back half without host round trips (the synchronous chunk_back reads the
// run/candidate counts back three times per chunk, idling the GPU while the host issues
// the next launches): fixed capacities and device-side counts for the fragment and
// candidate sorts, candidates appended to ctx->file_cands at a device-side total, the
// degenerate-trial flags copied to pinned host memory.  The file search reads all of it
// once at the end and re-runs the file with larger capacities if a counter overflowed.
void chunk_back_async(pgb_context* ctx, ChunkRun& run, uint8_t* h_status, uint64_t file_cap,
                      cudaStream_t st) {
    NvtxRange nvtx("pgb chunk back (async)");
    const int slot = run.slot;
    if (!run.live) return;
    if (st != ctx->st) PGB_CUDA(cudaStreamWaitEvent(st, ctx->ev_front[slot], 0));  // dedispersion + baseline done
    const pgb_chunk_spec* spec = &run.spec;
    const pgb_engine_config* cfg = &run.cfg;
    PGB_CUDA(cudaStreamWaitEvent(st, ctx->ev_rms[slot], 0));
    ChainParams cp{};
    cp.start_sample = spec->start_sample;
    cp.valid_begin = spec->valid_begin;
    cp.valid_end = spec->valid_end;
    cp.drop_left = spec->start_sample > 0;
    cp.drop_right = spec->overlap > 0;
    cp.tsamp = cfg->tsamp;
    cp.threshold = (double)cfg->detect_thresh;
    cp.boxcar_max = cfg->boxcar_max;
    const uint64_t ccap = ctx->cand_cap, fcap = ctx->frag_cap, cap = std::max(ccap, fcap);
    ctx->counters.reserve(4 * sizeof(unsigned long long));
    auto* dcnt = ctx->counters.as<unsigned long long>();
    ctx->cands_raw.reserve(ccap * sizeof(pgb_candidate));
    ctx->cands_sorted.reserve(ccap * sizeof(pgb_candidate));
    ctx->frags.reserve(fcap * sizeof(Fragment));
    ctx->frags_sorted.reserve(fcap * sizeof(Fragment));
    const size_t tmp = sort_fragments_temp_bytes(cap);
    ctx->sort_tmp.reserve(tmp);
    ctx->sort_keys.reserve(2 * cap * sizeof(uint64_t));
    ctx->sort_idx.reserve(2 * cap * sizeof(uint32_t));
    uint64_t* ka = ctx->sort_keys.as<uint64_t>();
    uint32_t* ia = ctx->sort_idx.as<uint32_t>();
    PGB_CUDA(cudaMemsetAsync(dcnt, 0, 2 * sizeof(unsigned long long), st));
    launch_boxcar_peaks(run.work, run.kind, ctx->d_row_len[slot].as<uint32_t>(), ctx->frms[slot].as<float>(),
                        ctx->status[slot].as<uint8_t>(), run.nrows, run.out_pitch, run.max_n, cp,
                        ctx->slot_active[slot].as<uint32_t>(), ctx->d_dms.as<double>(),
                        ctx->d_scale.as<double>(), ctx->cands_raw.as<pgb_candidate>(), dcnt, ccap,
                        ctx->frags.as<Fragment>(), dcnt + 1, fcap,
                        box_levels(ctx, cfg->boxcar_max, run.nrows, run.out_pitch),
                        box_scratch(ctx, run.nrows, run.max_n, cfg->boxcar_max), st);
    trace_mark(ctx, "boxcar + runs", st);
    sort_fragments_dev(ctx->frags.as<Fragment>(), ctx->frags_sorted.as<Fragment>(), fcap, dcnt + 1,
                       ctx->sort_tmp.p, tmp, ka, ka + cap, ia, ia + cap, st);
    launch_stitch_dev(ctx->frags_sorted.as<Fragment>(), fcap, dcnt + 1, ctx->d_row_len[slot].as<uint32_t>(),
                      cp, ctx->slot_active[slot].as<uint32_t>(), ctx->d_dms.as<double>(),
                      ctx->cands_raw.as<pgb_candidate>(), dcnt, ccap, st);
    // no per-chunk candidate order: the file-level sort (src/pipeline.cpp:100-105) orders
    // the appended candidates of all chunks by the same unique key
    auto* fc = ctx->file_ctr.as<unsigned long long>();
    append_candidates_dev(ctx->cands_raw.as<pgb_candidate>(), ccap, dcnt,
                          ctx->file_cands.as<pgb_candidate>(), fc, file_cap, fc + 1, st);
    PGB_CUDA(cudaMemcpyAsync(h_status, ctx->status[slot].p, run.nrows, cudaMemcpyDeviceToHost, st));
    trace_mark(ctx, "fragment order + stitch + append", st);
    ctx->launches += 12;
}

// Back half of a chunk with host reads (sync chunk_back): append its sorted candidates
// to the file list and its skipped trials to the file's (chunk, trial) pairs.
void append_chunk_sync(pgb_context* ctx, ChunkRun& run, uint64_t& total) {
    chunk_back(ctx, run);
    const uint64_t nc = ctx->n_cands;
    if (nc) {
        if ((total + nc) * sizeof(pgb_candidate) > ctx->file_cands.bytes) {
            DevBuf grown;
            grown.reserve(std::max<uint64_t>(2 * (total + nc), 4096) * sizeof(pgb_candidate));
            if (total)
                PGB_CUDA(cudaMemcpyAsync(grown.p, ctx->file_cands.p, total * sizeof(pgb_candidate),
                                         cudaMemcpyDeviceToDevice, ctx->st));
            PGB_CUDA(cudaStreamSynchronize(ctx->st));
            ctx->file_cands.release();
            ctx->file_cands = grown;
            grown.p = nullptr;
        }
        PGB_CUDA(cudaMemcpyAsync(ctx->file_cands.as<pgb_candidate>() + total, ctx->cands_sorted.p,
                                 nc * sizeof(pgb_candidate), cudaMemcpyDeviceToDevice, ctx->st));
    }
    total += nc;
    for (uint64_t t : ctx->skipped) {
        ctx->file_skipped.push_back(run.spec.index);
        ctx->file_skipped.push_back(t);
    }
}

// End of a file: the file-level sort (src/pipeline.cpp:100-105) and link_grid (:106).
void file_sort_link(pgb_context* ctx, uint64_t total, const pgb_link_radii* radii,
                    size_t* n_candidates, size_t* n_clusters) {
    NvtxRange nvtx("pgb file sort + link_grid");
    const double t0 = host_ms();  // every chunk's work has been synchronised already
    ctx->file_sorted.reserve(std::max<uint64_t>(total, 1) * sizeof(pgb_candidate));
    if (total) {
        const size_t tmp = sort_candidates_temp_bytes(total);
        ctx->sort_tmp.reserve(tmp);
        ctx->sort_keys.reserve(2 * total * sizeof(uint64_t));
        ctx->sort_idx.reserve(2 * total * sizeof(uint32_t));
        sort_candidates(ctx->file_cands.as<pgb_candidate>(), ctx->file_sorted.as<pgb_candidate>(), total,
                        ctx->sort_tmp.p, tmp, ctx->sort_keys.as<uint64_t>(), ctx->sort_keys.as<uint64_t>() + total,
                        ctx->sort_idx.as<uint32_t>(), ctx->sort_idx.as<uint32_t>() + total, ctx->st);
    }
    uint64_t ncl = 0;
    if (radii)  // radii == NULL: candidates only (multi-GPU shards cluster after the gather)
        cluster_candidates(ctx->file_sorted.as<pgb_candidate>(), total, *radii, ctx->cl_scratch, ctx->clusters,
                           ctx->members, &ncl, ctx->st, &ctx->launches);
    PGB_CUDA(cudaStreamSynchronize(ctx->st));
    trace_mark(ctx, "file sort + link_grid", ctx->st);
    trace_dump(ctx);
    ctx->file_ncands = total;
    ctx->n_clusters = ncl;
    ctx->n_members = radii ? total : 0;
    ctx->last_from_file = true;
    ctx->cluster_ms = host_ms() - t0;
    if (n_candidates) *n_candidates = total;
    if (n_clusters) *n_clusters = ncl;
}

// Runs the whole chain for one chunk whose samples are already on the device.
void run_chunk(pgb_context* ctx, const ChunkInput& in, const pgb_chunk_spec* spec,
               const pgb_engine_config* cfg) {
    ChunkRun run;
    chunk_front(ctx, in, spec, cfg, 0, run);
    chunk_back(ctx, run);
}

// A float chunk whose cells are all integers in [0, 255] (read_chunk's widening of
// 8-bit data, src/filterbank.cpp:304-307, or a zero-policy RFI mask) takes the integer
// path: every in-order fp32 partial sum is then an exact integer, so series and
// baselines are bit-identical.  Repacked on the device; otherwise the fp32 path.
ChunkInput prepare_f32(pgb_context* ctx, const float* dptr, uint64_t length) {
    if (!ctx->ntrials || !length || ctx->nchans > PGB_MAX_EXACT_CHANS || pgb_ablation_env("PGB_FORCE_F32_PATH"))
        return ChunkInput{dptr, false};
    const size_t cells = (size_t)length * ctx->nchans;
    ctx->in_u8.reserve(cells);
    ctx->counters.reserve(4 * sizeof(unsigned long long));
    ctx->h_counters.reserve(4 * sizeof(unsigned long long));
    auto* dflag = ctx->counters.as<unsigned long long>() + 2;
    PGB_CUDA(cudaMemsetAsync(dflag, 0, sizeof(unsigned long long), ctx->st));
    launch_pack_u8(dptr, cells, ctx->in_u8.as<uint8_t>(), dflag, ctx->st);
    auto* hflag = ctx->h_counters.as<unsigned long long>() + 2;
    PGB_CUDA(cudaMemcpyAsync(hflag, dflag, sizeof *hflag, cudaMemcpyDeviceToHost, ctx->st));
    PGB_CUDA(cudaStreamSynchronize(ctx->st));
    ctx->launches += 1;
    trace_mark(ctx, "integer check (pack)", ctx->st);
    if (*hflag == 0) return ChunkInput{ctx->in_u8.p, true};
    return ChunkInput{dptr, false};
}

RfiParams to_rfi(const pgb_rfi_config* r) {
    return RfiParams{r->narrowband, r->broadband, r->local_mean, r->k_sigma, r->k_mad};
}

// RFI excision of an 8-bit chunk on the device (src/pipeline.cpp:79-87, src/rfi.cpp): the
// flags, then -- if any -- the masked chunk as the dedispersion input.  Zero replacement or
// bad channels only: integer cells, the u8 path with the transpose zeroing them.  Local-mean
// replacement of bad rows: the fp16 in-order kernel with the rows' float values as
// exceptions; the widened float chunk (fp32 path) only if that kernel does not fit.
ChunkInput rfi_input(pgb_context* ctx, const uint8_t* cptr, uint64_t length, const pgb_rfi_config* rfi) {
    const uint32_t C = ctx->nchans;
    const RfiParams rp = to_rfi(rfi);
    uint64_t nbc = 0, nbs = 0;
    rfi_flags_impl<uint8_t>(cptr, length, C, rp, ctx->rfi, ctx->st, &nbc, &nbs);
    ctx->launches += 8;
    trace_mark(ctx, "rfi flags", ctx->st);
    ChunkInput ci{cptr, true};
    ci.raw = true;
    if (!nbc && !nbs) return ci;
    ci.raw = false;  // the mask is chunk-local: no overlap reuse
    ci.chan_bad = ctx->rfi.chan_bad.as<uint8_t>();
    ci.samp_bad = ctx->rfi.samp_bad.as<uint8_t>();
    if (nbs && rp.local_mean && pgb_ablation_env("PGB_RFI_HYB")) {
        // the event-replay kernel over the masked integer codes (ablation library)
        rfi_exceptions_u8(cptr, length, C, rp, ctx->rfi, nbs, ctx->st, &ctx->bad_rows_host);
        ctx->launches += 4;
        trace_mark(ctx, "rfi exceptions", ctx->st);
        ci.hyb = true;
        ci.fallback = [ctx, cptr, length, rp, nbc, nbs]() {
            ctx->rfi_out.reserve((size_t)length * ctx->nchans * 4);
            rfi_mask_impl<uint8_t>(cptr, length, ctx->nchans, rp, ctx->rfi, ctx->rfi_out.as<float>(), ctx->st,
                                   nbc, nbs);
            ctx->launches += 2;
            return prepare_f32(ctx, ctx->rfi_out.as<float>(), length);
        };
        return ci;
    }
    if (nbs && rp.local_mean && !pgb_ablation_env("PGB_RFI_H16")) {
        // local-mean rows: the widened float chunk and the in-order fp32 ring (the fp16
        // kernel with exception rows, PGB_RFI_H16=1 in the ablation library, measured
        // slower on config E: DESIGN.md section 10)
        ctx->rfi_out.reserve((size_t)length * C * 4);
        rfi_mask_impl<uint8_t>(cptr, length, C, rp, ctx->rfi, ctx->rfi_out.as<float>(), ctx->st, nbc, nbs);
        ctx->launches += 2;
        return prepare_f32(ctx, ctx->rfi_out.as<float>(), length);
    }
    if (nbs && rp.local_mean) {
        rfi_exceptions_u8(cptr, length, C, rp, ctx->rfi, nbs, ctx->st, &ctx->bad_rows_host);
        ctx->launches += nbs ? 4 : 3;
        trace_mark(ctx, "rfi exceptions", ctx->st);
        ci.u8 = false;
        ci.h16 = true;
        ci.fallback = [ctx, cptr, length, rp, nbc, nbs]() {
            ctx->rfi_out.reserve((size_t)length * ctx->nchans * 4);
            rfi_mask_impl<uint8_t>(cptr, length, ctx->nchans, rp, ctx->rfi, ctx->rfi_out.as<float>(), ctx->st,
                                   nbc, nbs);
            ctx->launches += 2;
            return prepare_f32(ctx, ctx->rfi_out.as<float>(), length);
        };
    }
    return ci;
}

// Parallel host repack of a float chunk into bytes; false if any cell is not an integer
// in [0, 255] (then the caller uploads the floats and takes the fp32 path).

void reset_timing(pgb_context* ctx) {
    // every top-level call starts here (after the previous call's final stream sync), so
    // the staging arena is free again
    ctx->stage_blk = 0;
    ctx->stage_off = 0;
    ctx->dedisp_ms = 0.0;
    ctx->dedisp_launches = 0;
    ctx->channel_adds = 0;
    for (double& v : ctx->stage_ms) v = 0.0;
}

}  // namespace

extern "C" {

int pgb_abi_version(void) { return PGB_ABI_VERSION; }

const char* pgb_last_error(void) { return g_last_error.c_str(); }

pgb_status pgb_device_count(int* count) {
    return guarded([&] {
        need(count != nullptr, PGB_ERR_ARGUMENT, "null count");
        int n = 0;
        const cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
        *count = n;
    });
}

int64_t pgb_delay_samples(double dm, const pgb_header* header, uint32_t channel) {
    return delay_samples(dm, header, channel);
}

double pgb_adaptive_dm_step(double tol, const pgb_header* header) { return adaptive_step(tol, header); }

pgb_status pgb_generate_dm_trials(double dm_lo, double dm_hi, const pgb_header* h, pgb_spacing spacing,
                                  double value, double* dms, int64_t* delays, size_t capacity,
                                  size_t* ntrials) {
    return guarded([&] {  // src/dedisp.cpp:28-70
        need(h && ntrials, PGB_ERR_ARGUMENT, "null header/ntrials");
        if (dm_lo < 0.0 || dm_hi < dm_lo)
            raise(PGB_ERR_INVALID_RANGE, "invalid DM range [" + std::to_string(dm_lo) + ", " +
                                             std::to_string(dm_hi) + "]");
        double step;
        if (spacing == PGB_SPACING_LINEAR) {
            if (value <= 0.0) raise(PGB_ERR_INVALID_RANGE, "linear DM step must be positive");
            step = value;
        } else {
            if (value <= 1.0) raise(PGB_ERR_INVALID_RANGE, "adaptive tolerance must exceed 1");
            step = adaptive_step(value, h);
        }
        std::vector<double> out;
        if (step <= 0.0 || dm_hi == dm_lo) {
            out.push_back(dm_lo);
            if (dm_hi != dm_lo) out.push_back(dm_hi);
        } else {
            const double eps = step * 1e-9;
            for (size_t i = 0;; ++i) {
                const double dm = std::fma((double)i, step, dm_lo);
                if (dm >= dm_hi - eps) {
                    out.push_back(dm_hi);
                    break;
                }
                out.push_back(dm);
            }
        }
        *ntrials = out.size();
        if (!dms) return;
        need(capacity >= out.size(), PGB_ERR_ARGUMENT, "capacity too small");
        std::copy(out.begin(), out.end(), dms);
        if (delays) {
            // delay_samples evaluates (k * dm) * (1/f_c^2 - 1/f_ref^2) left to right: the
            // channel factor is the same double for every trial, so it is formed once per
            // channel (same operations, same bits); trials are split over host threads
            const uint32_t C = h->nchans;
            const double f_ref = max_freq(h);
            std::vector<double> fac(C);
            for (uint32_t c = 0; c < C; ++c) {
                const double f_c = channel_freq(h, c);
                fac[c] = 1.0 / (f_c * f_c) - 1.0 / (f_ref * f_ref);
            }
            const size_t T = out.size();
            auto rows = [&](size_t t0, size_t t1) {
                for (size_t t = t0; t < t1; ++t) {
                    const double kd = k_dispersion * out[t];
                    int64_t* d = delays + t * C;
                    for (uint32_t c = 0; c < C; ++c) d[c] = (int64_t)std::floor(kd * fac[c] / h->tsamp + 0.5);
                }
            };
            const size_t nth = (size_t)T * C >= (1u << 20)
                                   ? std::min<size_t>(T, std::max(1u, std::min(16u, std::thread::hardware_concurrency())))
                                   : 1;
            std::vector<std::thread> pool;
            for (size_t i = 1; i < nth; ++i) pool.emplace_back(rows, T * i / nth, T * (i + 1) / nth);
            rows(0, T / nth);
            for (auto& th : pool) th.join();
        }
    });
}

pgb_status pgb_create(int device, pgb_context** out) {
    return guarded([&] {
        need(out != nullptr, PGB_ERR_ARGUMENT, "null ctx");
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
            cudaGetLastError();
            raise(PGB_ERR_NO_DEVICE, "no CUDA device visible (libpgb200 has no CPU fallback)");
        }
        need(device >= 0 && device < n, PGB_ERR_NO_DEVICE, "device ordinal out of range");
        cudaDeviceProp prop{};
        PGB_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10 || prop.minor != 0)
            raise(PGB_ERR_NO_DEVICE, std::string("libpgb200 is built for sm_100a; device is ") +
                                         prop.name);
        auto* ctx = new pgb_context();
        ctx->device = device;
        if (const char* e = getenv("PGB_INITIAL_CAP")) {  // tests: start the candidate/fragment
            const uint64_t c = strtoull(e, nullptr, 10);   // buffers small to force the growth paths
            if (c) ctx->cand_cap = ctx->frag_cap = c;
        }
        PGB_CUDA(cudaSetDevice(device));
        PGB_CUDA(cudaStreamCreateWithFlags(&ctx->st, cudaStreamNonBlocking));
        PGB_CUDA(cudaStreamCreateWithFlags(&ctx->copy_st, cudaStreamNonBlocking));
        PGB_CUDA(cudaStreamCreateWithFlags(&ctx->rms_st, cudaStreamNonBlocking));
        PGB_CUDA(cudaStreamCreateWithFlags(&ctx->bx_st, cudaStreamNonBlocking));
        for (int k = 0; k < 2; ++k) {
            PGB_CUDA(cudaEventCreateWithFlags(&ctx->ev_back[k], cudaEventDisableTiming));
            PGB_CUDA(cudaEventCreate(&ctx->ev_dd0[k]));
            PGB_CUDA(cudaEventCreate(&ctx->ev_dd1[k]));
            PGB_CUDA(cudaEventCreate(&ctx->ev_front[k]));
            PGB_CUDA(cudaEventCreate(&ctx->ev_rms[k]));
            PGB_CUDA(cudaEventCreate(&ctx->ev_rms0[k]));
        }
        PGB_CUDA(cudaEventCreate(&ctx->ev_bx0));
        PGB_CUDA(cudaEventCreate(&ctx->ev_bx1));
        PGB_CUDA(cudaEventCreate(&ctx->ev_pk1));
        *out = ctx;
    });
}

pgb_status pgb_destroy(pgb_context* ctx) {
    return guarded([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->st);
        cudaStreamSynchronize(ctx->copy_st);
        cudaStreamSynchronize(ctx->rms_st);
        cudaStreamSynchronize(ctx->bx_st);
        for (int k = 0; k < 2; ++k)
            for (DevBuf* b : {&ctx->base[k], &ctx->frms[k], &ctx->status[k], &ctx->d_row_len[k],
                              &ctx->slot_active[k]})
                b->release();
        ctx->d_work.release();
        ctx->d_bsums.release();
        ctx->d_lmin.release();
        ctx->d_keep.release();
        ctx->file_ctr.release();
        for (DevBuf* b : {&ctx->d_delays_ct, &ctx->d_dms, &ctx->in_raw, &ctx->rows, &ctx->series,
                          &ctx->d_active, &ctx->d_blk_len, &ctx->d_scale, &ctx->in_u8, &ctx->ws_base, &ctx->ws_off, &ctx->dd_win, &ctx->dd_off, &ctx->rfi_out, &ctx->rfi.chan_bad,
                          &ctx->rfi.samp_bad, &ctx->rfi.dbl, &ctx->rfi.tmp, &ctx->rfi.rows, &ctx->cands_raw, &ctx->cands_sorted,
                          &ctx->frags, &ctx->frags_sorted, &ctx->counters, &ctx->sort_keys,
                          &ctx->sort_idx, &ctx->sort_tmp, &ctx->payload, &ctx->file_cands,
                          &ctx->file_sorted, &ctx->cl_scratch, &ctx->clusters, &ctx->members, &ctx->d_levels, &ctx->d_wide,
                          &ctx->d_bxs, &ctx->ddf_win, &ctx->ddf_off, &ctx->ddh_win, &ctx->ddh_off, &ctx->rfi.xcnt,
                          &ctx->rfi.xP, &ctx->rfi.xR, &ctx->rfi.xF})
            b->release();
        ctx->h_counters.release();
        for (auto e : ctx->seg_events) cudaEventDestroy(e);
        for (auto e : ctx->sub_events) cudaEventDestroy(e);
        for (auto& b : ctx->stage) b.release();
        for (auto e : ctx->file_dd_ev) cudaEventDestroy(e);
        ctx->h_file_status.release();
        ctx->h_file_ctr.release();
        ctx->h_pack.release();
        for (int b = 0; b < 2; ++b) {
            ctx->stream.hbuf[b].release();
            ctx->stream.dbuf[b].release();
            if (ctx->stream.up_done[b]) cudaEventDestroy(ctx->stream.up_done[b]);
            if (ctx->stream.dev_free[b]) cudaEventDestroy(ctx->stream.dev_free[b]);
        }
        delete ctx->stream.runs;
        for (int k = 0; k < 2; ++k)
            for (cudaEvent_t e : {ctx->ev_dd0[k], ctx->ev_dd1[k], ctx->ev_front[k], ctx->ev_rms[k], ctx->ev_rms0[k]})
                cudaEventDestroy(e);
        for (cudaEvent_t e : {ctx->ev_bx0, ctx->ev_bx1, ctx->ev_pk1, ctx->ev_back[0], ctx->ev_back[1]}) cudaEventDestroy(e);
        cudaStreamDestroy(ctx->rms_st);
        cudaStreamDestroy(ctx->bx_st);
        cudaStreamDestroy(ctx->st);
        cudaStreamDestroy(ctx->copy_st);
        delete ctx;
    });
}

pgb_status pgb_set_plan(pgb_context* ctx, const double* dms, const int64_t* delays, uint32_t ntrials,
                        uint32_t nchans) {
    return guarded([&] {
        need(ctx && (ntrials == 0 || (dms && delays)), PGB_ERR_ARGUMENT, "null plan");
        need(nchans > 0 || ntrials == 0, PGB_ERR_ARGUMENT, "nchans must be positive");
        PGB_CUDA(cudaSetDevice(ctx->device));
        ctx->ntrials = ntrials;
        ctx->nchans = nchans;
        ctx->dms.assign(dms, dms + ntrials);
        ctx->delays.assign(delays, delays + (size_t)ntrials * nchans);
        ctx->maxd.assign(ntrials, 0);
        std::vector<int32_t> ct((size_t)ntrials * nchans);
        for (uint32_t t = 0; t < ntrials; ++t) {
            int64_t m = INT64_MIN;
            for (uint32_t c = 0; c < nchans; ++c) {
                const int64_t d = delays[(size_t)t * nchans + c];
                if (d < 0 || d > INT32_MAX) raise(PGB_ERR_INVALID_PLAN, "delay out of range");
                m = std::max(m, d);
                ct[(size_t)c * ntrials + t] = (int32_t)d;
            }
            ctx->maxd[t] = m;
        }
        ctx->tr_begin = 0;
        ctx->tr_end = ntrials;
        ctx->geom_valid = false;
        if (ntrials) {
            ctx->d_delays_ct.reserve(ct.size() * sizeof(int32_t));
            ctx->d_dms.reserve(ntrials * sizeof(double));
            PGB_CUDA(cudaMemcpyAsync(ctx->d_delays_ct.p, ct.data(), ct.size() * sizeof(int32_t),
                                     cudaMemcpyHostToDevice, ctx->st));
            PGB_CUDA(cudaMemcpyAsync(ctx->d_dms.p, dms, ntrials * sizeof(double),
                                     cudaMemcpyHostToDevice, ctx->st));
            PGB_CUDA(cudaStreamSynchronize(ctx->st));
        }
    });
}

pgb_status pgb_set_trial_range(pgb_context* ctx, uint32_t begin, uint32_t end) {
    return guarded([&] {
        need(ctx, PGB_ERR_ARGUMENT, "null ctx");
        need(begin <= end && end <= ctx->ntrials, PGB_ERR_ARGUMENT, "trial range out of plan");
        ctx->tr_begin = begin;
        ctx->tr_end = end;
        ctx->geom_valid = false;
    });
}

static pgb_status run_dm_loop_impl(pgb_context* ctx, const void* data, bool u8, int on_device,
                                   const pgb_chunk_spec* spec, const pgb_engine_config* cfg,
                                   size_t* n_candidates, size_t* n_skipped) {
    return guarded([&] {
        NvtxRange nvtx("pgb run_dm_loop");
        need(ctx && data, PGB_ERR_ARGUMENT, "null ctx/data");
        PGB_CUDA(cudaSetDevice(ctx->device));
        validate_cfg(ctx, spec, cfg);
        reset_timing(ctx);
        ctx->last_from_file = false;
        const void* dptr = data;
        const size_t cells = (size_t)spec->length * ctx->nchans;
        const size_t bytes = cells * (u8 ? 1 : 4);
        bool as_u8 = u8;
        if (!on_device && ctx->ntrials) {
            if (!u8 && ctx->nchans <= PGB_MAX_EXACT_CHANS) {
                // read_chunk widens 8-bit files to floats (src/filterbank.cpp:304-307): repack
                // integer chunks to bytes on the host threads, so a quarter of the bytes cross
                // PCIe from pinned memory; any non-integer cell keeps the fp32 upload
                ctx->h_pack.reserve(cells);
                as_u8 = host_pack_u8(static_cast<const float*>(data), cells, ctx->h_pack.as<uint8_t>());
            }
            ctx->in_raw.reserve(as_u8 ? cells : bytes);
            PGB_CUDA(cudaMemcpyAsync(ctx->in_raw.p, as_u8 && !u8 ? ctx->h_pack.p : data, as_u8 ? cells : bytes,
                                     cudaMemcpyHostToDevice, ctx->st));
            dptr = ctx->in_raw.p;
        }
        const ChunkInput ci = as_u8 ? ChunkInput{dptr, true}
                                    : prepare_f32(ctx, static_cast<const float*>(dptr), spec->length);
        run_chunk(ctx, ci, spec, cfg);
        if (n_candidates) *n_candidates = ctx->n_cands;
        if (n_skipped) *n_skipped = ctx->skipped.size();
    });
}

pgb_status pgb_run_dm_loop_u8(pgb_context* ctx, const uint8_t* data, int on_device,
                              const pgb_chunk_spec* spec, const pgb_engine_config* cfg,
                              size_t* n_candidates, size_t* n_skipped) {
    return run_dm_loop_impl(ctx, data, true, on_device, spec, cfg, n_candidates, n_skipped);
}

pgb_status pgb_run_dm_loop_f32(pgb_context* ctx, const float* data, int on_device,
                               const pgb_chunk_spec* spec, const pgb_engine_config* cfg,
                               size_t* n_candidates, size_t* n_skipped) {
    return run_dm_loop_impl(ctx, data, false, on_device, spec, cfg, n_candidates, n_skipped);
}

pgb_status pgb_fetch_candidates(pgb_context* ctx, pgb_candidate* out, size_t capacity) {
    return guarded([&] {
        need(ctx, PGB_ERR_ARGUMENT, "null ctx");
        const uint64_t n = ctx->last_from_file ? ctx->file_ncands : ctx->n_cands;
        need(capacity >= n && (n == 0 || out), PGB_ERR_ARGUMENT, "capacity too small");
        if (!n) return;
        const DevBuf& src = ctx->last_from_file ? ctx->file_sorted : ctx->cands_sorted;
        PGB_CUDA(cudaMemcpyAsync(out, src.p, n * sizeof(pgb_candidate), cudaMemcpyDeviceToHost, ctx->st));
        PGB_CUDA(cudaStreamSynchronize(ctx->st));
    });
}

pgb_status pgb_fetch_skipped(pgb_context* ctx, uint64_t* out, size_t capacity) {
    return guarded([&] {
        need(ctx, PGB_ERR_ARGUMENT, "null ctx");
        need(capacity >= ctx->skipped.size(), PGB_ERR_ARGUMENT, "capacity too small");
        std::copy(ctx->skipped.begin(), ctx->skipped.end(), out);
    });
}

pgb_status pgb_device_candidates(pgb_context* ctx, const pgb_candidate** dev_ptr, size_t* n) {
    return guarded([&] {
        need(ctx && dev_ptr && n, PGB_ERR_ARGUMENT, "null argument");
        if (ctx->last_from_file) {
            *dev_ptr = ctx->file_sorted.as<pgb_candidate>();
            *n = ctx->file_ncands;
        } else {
            *dev_ptr = ctx->cands_sorted.as<pgb_candidate>();
            *n = ctx->n_cands;
        }
    });
}

static pgb_status dedisperse_impl(pgb_context* ctx, const void* data, bool u8, uint64_t length,
                                  uint32_t tb, uint32_t te, float* out, uint64_t out_stride) {
    return guarded([&] {
        need(ctx && data && out, PGB_ERR_ARGUMENT, "null argument");
        need(tb <= te && te <= ctx->ntrials, PGB_ERR_ARGUMENT, "trial range out of plan");
        PGB_CUDA(cudaSetDevice(ctx->device));
        for (uint32_t t = tb; t < te; ++t)  // src/dedisp.cpp:137-142
            if ((uint64_t)ctx->maxd[t] >= length)
                raise(PGB_ERR_CHUNK_TOO_SHORT,
                      "trial " + std::to_string(t) + ": chunk of " + std::to_string(length) +
                          " samples cannot cover delay span " + std::to_string(ctx->maxd[t]));
        if (tb == te) return;
        stage_reset(ctx);
        const uint32_t save_b = ctx->tr_begin, save_e = ctx->tr_end;
        ctx->tr_begin = tb;
        ctx->tr_end = te;
        ctx->geom_valid = false;
        const size_t bytes = (size_t)length * ctx->nchans * (u8 ? 1 : 4);
        ctx->in_raw.reserve(bytes);
        PGB_CUDA(cudaMemcpyAsync(ctx->in_raw.p, data, bytes, cudaMemcpyHostToDevice, ctx->st));
        // dedispersion only: reuse run_chunk's geometry by running the chain with
        // a zero-width config is wasteful; replicate the first two stages instead.
        pgb_chunk_spec spec{0, 0, length, 0, 0, length};
        pgb_engine_config cfg{1, 1e30f, 0.0, 1, 0, 0, 1};
        try {
            run_chunk(ctx, ChunkInput{ctx->in_raw.p, u8}, &spec, &cfg);
        } catch (...) {
            ctx->tr_begin = save_b;
            ctx->tr_end = save_e;
            ctx->geom_valid = false;
            throw;
        }
        ctx->tr_begin = save_b;
        ctx->tr_end = save_e;
        ctx->geom_valid = false;
        const uint32_t nrows = te - tb;
        const uint64_t pitch = ctx->last_out_pitch;
        std::vector<float> host((size_t)nrows * pitch);
        if (u8) {
            std::vector<int32_t> tmp((size_t)nrows * pitch);
            PGB_CUDA(cudaMemcpy(tmp.data(), ctx->series.p, tmp.size() * 4, cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < tmp.size(); ++i) host[i] = (float)tmp[i];
        } else {
            PGB_CUDA(cudaMemcpy(host.data(), ctx->series.p, host.size() * 4, cudaMemcpyDeviceToHost));
        }
        for (uint32_t r = 0; r < nrows; ++r) {
            const uint64_t n = length - (uint64_t)ctx->maxd[tb + r];
            std::memcpy(out + (size_t)r * out_stride, host.data() + (size_t)r * pitch, n * sizeof(float));
        }
    });
}

pgb_status pgb_dedisperse_u8(pgb_context* ctx, const uint8_t* data, uint64_t length,
                             uint32_t trial_begin, uint32_t trial_end, float* out,
                             uint64_t out_stride) {
    return dedisperse_impl(ctx, data, true, length, trial_begin, trial_end, out, out_stride);
}

pgb_status pgb_dedisperse_f32(pgb_context* ctx, const float* data, uint64_t length,
                              uint32_t trial_begin, uint32_t trial_end, float* out,
                              uint64_t out_stride) {
    return dedisperse_impl(ctx, data, false, length, trial_begin, trial_end, out, out_stride);
}

pgb_status pgb_rfi_clean(pgb_context* ctx, const void* data, int is_u8, int on_device,
                         uint64_t length, const pgb_rfi_config* rfi, float* out_host,
                         uint64_t* n_bad_channels, uint64_t* n_bad_samples) {
    return guarded([&] {
        NvtxRange nvtx("pgb rfi_clean");
        need(ctx && data && rfi && ctx->nchans, PGB_ERR_ARGUMENT, "null argument or no plan");
        PGB_CUDA(cudaSetDevice(ctx->device));
        const uint32_t C = ctx->nchans;
        const size_t cells = (size_t)length * C;
        const void* dptr = data;
        if (!on_device) {
            ctx->in_raw.reserve(cells * (is_u8 ? 1 : 4));
            PGB_CUDA(cudaMemcpyAsync(ctx->in_raw.p, data, cells * (is_u8 ? 1 : 4), cudaMemcpyHostToDevice,
                                     ctx->st));
            dptr = ctx->in_raw.p;
        }
        ctx->rfi_out.reserve(cells * 4);
        uint64_t nbc = 0, nbs = 0;
        if (is_u8)
            rfi_clean_impl<uint8_t>(static_cast<const uint8_t*>(dptr), length, C, to_rfi(rfi), ctx->rfi,
                                    ctx->rfi_out.as<float>(), ctx->st, &nbc, &nbs);
        else
            rfi_clean_impl<float>(static_cast<const float*>(dptr), length, C, to_rfi(rfi), ctx->rfi,
                                  ctx->rfi_out.as<float>(), ctx->st, &nbc, &nbs);
        ctx->rfi_len = length;
        if (out_host)
            PGB_CUDA(cudaMemcpyAsync(out_host, ctx->rfi_out.p, cells * 4, cudaMemcpyDeviceToHost, ctx->st));
        PGB_CUDA(cudaStreamSynchronize(ctx->st));
        if (n_bad_channels) *n_bad_channels = nbc;
        if (n_bad_samples) *n_bad_samples = nbs;
    });
}

pgb_status pgb_fetch_rfi_flags(pgb_context* ctx, uint8_t* bad_channels, uint8_t* bad_samples) {
    return guarded([&] {
        need(ctx, PGB_ERR_ARGUMENT, "null ctx");
        if (bad_channels && ctx->rfi.chan_bad.p)
            PGB_CUDA(cudaMemcpyAsync(bad_channels, ctx->rfi.chan_bad.p, ctx->nchans, cudaMemcpyDeviceToHost, ctx->st));
        if (bad_samples && ctx->rfi.samp_bad.p)
            PGB_CUDA(cudaMemcpyAsync(bad_samples, ctx->rfi.samp_bad.p, ctx->rfi_len, cudaMemcpyDeviceToHost, ctx->st));
        PGB_CUDA(cudaStreamSynchronize(ctx->st));
    });
}

pgb_status pgb_link_grid(pgb_context* ctx, const pgb_candidate* cands, int on_device, size_t n,
                         const pgb_link_radii* radii, size_t* n_clusters) {
    return guarded([&] {
        NvtxRange nvtx("pgb link_grid");
        need(ctx && radii && (n == 0 || cands), PGB_ERR_ARGUMENT, "null argument");
        PGB_CUDA(cudaSetDevice(ctx->device));
        const pgb_candidate* dptr = cands;
        if (!on_device && n) {
            ctx->file_cands.reserve(n * sizeof(pgb_candidate));
            PGB_CUDA(cudaMemcpyAsync(ctx->file_cands.p, cands, n * sizeof(pgb_candidate),
                                     cudaMemcpyHostToDevice, ctx->st));
            dptr = ctx->file_cands.as<pgb_candidate>();
        }
        uint64_t ncl = 0;
        cluster_candidates(dptr, n, *radii, ctx->cl_scratch, ctx->clusters, ctx->members, &ncl,
                           ctx->st, &ctx->launches);
        PGB_CUDA(cudaStreamSynchronize(ctx->st));
        ctx->n_clusters = ncl;
        ctx->n_members = n;
        if (n_clusters) *n_clusters = ncl;
    });
}

pgb_status pgb_fetch_clusters(pgb_context* ctx, pgb_cluster* out, size_t capacity,
                              uint64_t* member_ids, size_t member_capacity) {
    return guarded([&] {
        need(ctx, PGB_ERR_ARGUMENT, "null ctx");
        need(capacity >= ctx->n_clusters, PGB_ERR_ARGUMENT, "cluster capacity too small");
        if (ctx->n_clusters && out)
            PGB_CUDA(cudaMemcpyAsync(out, ctx->clusters.p, ctx->n_clusters * sizeof(pgb_cluster),
                                     cudaMemcpyDeviceToHost, ctx->st));
        if (member_ids && ctx->n_members) {
            need(member_capacity >= ctx->n_members, PGB_ERR_ARGUMENT, "member capacity too small");
            PGB_CUDA(cudaMemcpyAsync(member_ids, ctx->members.p, ctx->n_members * sizeof(uint64_t),
                                     cudaMemcpyDeviceToHost, ctx->st));
        }
        PGB_CUDA(cudaStreamSynchronize(ctx->st));
    });
}

pgb_status pgb_search_file_u8(pgb_context* ctx, const uint8_t* payload, int payload_on_device,
                              uint64_t nsamples, const pgb_chunk_spec* chunks, size_t nchunks,
                              const pgb_engine_config* cfg, const pgb_link_radii* radii,
                              const pgb_rfi_config* rfi, size_t* n_candidates, size_t* n_clusters) {
    return guarded([&] {
        NvtxRange nvtx("pgb search_file_u8");
        need(ctx && payload && cfg && (nchunks == 0 || chunks), PGB_ERR_ARGUMENT,
             "null argument");
        PGB_CUDA(cudaSetDevice(ctx->device));
        reset_timing(ctx);
        const uint32_t C = ctx->nchans;
        const uint8_t* dpay = payload;
        if (!payload_on_device) {
            ctx->payload.reserve((size_t)nsamples * C);
            dpay = ctx->payload.as<uint8_t>();
            while (ctx->seg_events.size() < nchunks) {
                cudaEvent_t e;
                PGB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                ctx->seg_events.push_back(e);
            }
            // upload segment k = [end of chunk k-1, end of chunk k) on the copy stream; the
            // first chunk's segment goes up in PGB_PROG_SUBSEG pieces so its transpose and
            // dedispersion start before the whole chunk has arrived
            uint64_t done = 0;
            ctx->prog.clear();
            const bool prog_ok = nchunks > 0 && !(rfi && (rfi->narrowband || rfi->broadband)) &&
                                 chunks[0].start_sample == 0 && !pgb_ablation_env("PGB_NO_PROGRESSIVE");
            if (prog_ok) {
                const uint64_t L0 = std::min<uint64_t>(chunks[0].length, nsamples);
                while (ctx->sub_events.size() < PGB_PROG_SUBSEG) {
                    cudaEvent_t e;
                    PGB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                    ctx->sub_events.push_back(e);
                }
                // the first piece ends where the first dedispersion tiles can run (every
                // trial's delay plus two tiles); the rest of the chunk in equal pieces
                int64_t maxd_all = 0;
                for (uint32_t t = ctx->tr_begin; t < ctx->tr_end; ++t) maxd_all = std::max(maxd_all, ctx->maxd[t]);
                const uint64_t first = std::min<uint64_t>(L0, round_up((uint64_t)maxd_all + 3 * DD_NT + 64, 64));
                for (int j = 0; j < PGB_PROG_SUBSEG; ++j) {
                    uint64_t e = j + 1 == PGB_PROG_SUBSEG
                                     ? L0
                                     : first + round_up((L0 - first) * j / (PGB_PROG_SUBSEG - 1), 64);
                    e = std::min(e, L0);
                    if (e > done) {
                        PGB_CUDA(cudaMemcpyAsync(ctx->payload.as<uint8_t>() + done * C, payload + done * C,
                                                 (e - done) * C, cudaMemcpyHostToDevice, ctx->copy_st));
                        done = e;
                    }
                    PGB_CUDA(cudaEventRecord(ctx->sub_events[j], ctx->copy_st));
                    ctx->prog.emplace_back(e, ctx->sub_events[j]);
                }
            }
            for (size_t k = 0; k < nchunks; ++k) {
                const uint64_t end = chunks[k].start_sample + chunks[k].length;
                need(end <= nsamples, PGB_ERR_INVALID_PLAN, "chunk extends past the payload");
                if (end > done) {
                    PGB_CUDA(cudaMemcpyAsync(ctx->payload.as<uint8_t>() + done * C, payload + done * C,
                                             (end - done) * C, cudaMemcpyHostToDevice, ctx->copy_st));
                    done = end;
                }
                PGB_CUDA(cudaEventRecord(ctx->seg_events[k], ctx->copy_st));
            }
        }
        ctx->file_skipped.clear();
        ctx->trace = getenv("PGB_TRACE") != nullptr;
        trace_mark(ctx, "begin", ctx->st);
        uint64_t total = 0;
        auto finish = [&](ChunkRun& run) { append_chunk_sync(ctx, run, total); };
        // With a baseline the chain reads the slot's own baseline buffer, so chunk k's
        // front half (dedispersion + RMS) is issued before chunk k-1's back half: the
        // RMS of chunk k then runs beside the boxcar of chunk k-1.  Without one the
        // chain reads the shared series buffer and the halves stay in order.
        const bool overlap = cfg->baseline_window > 0;
        uint64_t pitch_min = 0;  // one series pitch for the whole file (overlap reuse)
        for (size_t k = 0; k < nchunks; ++k) pitch_min = std::max<uint64_t>(pitch_min, chunks[k].length);
        ctx->ser_ok = false;
        // Back halves: asynchronous (device-side counts, one read at the end of the file)
        // unless PGB_SYNC_BACK is set (per-chunk host reads, the run_dm_loop path).
        const bool async_back = !pgb_ablation_env("PGB_SYNC_BACK");
        uint32_t max_rows = 0;
        for (uint32_t t = ctx->tr_begin; t < ctx->tr_end; ++t) ++max_rows;
        struct ChunkBook {  // what the end-of-file pass needs from each chunk
            bool live = false;
            uint64_t index = 0;
            std::vector<uint32_t> active;
            std::vector<uint64_t> skipped;
        };
        std::vector<ChunkBook> book;
        uint64_t file_cap = 0;
        auto run_chunks = [&]() {
            ChunkRun runs[2];
            bool pending = false;
            ctx->ser_ok = false;
            if (async_back) {
                book.assign(nchunks, ChunkBook{});
                file_cap = std::max<uint64_t>(1, nchunks * ctx->cand_cap);
                ctx->file_cands.reserve(file_cap * sizeof(pgb_candidate));
                ctx->file_ctr.reserve(4 * sizeof(unsigned long long));
                PGB_CUDA(cudaMemsetAsync(ctx->file_ctr.p, 0, 4 * sizeof(unsigned long long), ctx->st));
                ctx->h_file_status.reserve(std::max<size_t>(1, nchunks * (size_t)max_rows));
                ctx->h_file_ctr.reserve(4 * sizeof(unsigned long long));
                while (ctx->file_dd_ev.size() < 2 * nchunks) {
                    cudaEvent_t e;
                    PGB_CUDA(cudaEventCreate(&e));
                    ctx->file_dd_ev.push_back(e);
                }
            }
            size_t back_k = 0;  // chunk index of the next back half
            auto back = [&](ChunkRun& run) {
                if (!async_back) {
                    finish(run);
                } else {
                    ChunkBook& b = book[back_k];
                    b.live = run.live;
                    b.index = run.spec.index;
                    b.active = run.active;
                    b.skipped = run.skipped;
                    // with a baseline the back half reads only its slot's buffers: it runs on
                    // bx_st, beside the next chunk's dedispersion
                    cudaStream_t bst = overlap && !pgb_ablation_env("PGB_BACK_MAIN") ? ctx->bx_st : ctx->st;
                    chunk_back_async(ctx, run, ctx->h_file_status.as<uint8_t>() + back_k * (size_t)max_rows,
                                     file_cap, bst);
                    if (bst != ctx->st && run.live) {
                        PGB_CUDA(cudaEventRecord(ctx->ev_back[run.slot], bst));
                        ctx->back_pending[run.slot] = true;
                    }
                }
                ++back_k;
            };
            for (size_t k = 0; k < nchunks; ++k) {
                validate_cfg(ctx, &chunks[k], cfg);
                const bool prog_k = k == 0 && !payload_on_device && !ctx->prog.empty();
                if (!payload_on_device && !prog_k) PGB_CUDA(cudaStreamWaitEvent(ctx->st, ctx->seg_events[k], 0));
                const uint8_t* cptr = dpay + chunks[k].start_sample * C;
                ChunkInput ci{cptr, true};
                ci.raw = true;
                ci.pitch_min = pitch_min;
                ci.more = overlap && k + 1 < nchunks;
                if (prog_k) ci.prog = &ctx->prog;
                if (rfi && (rfi->narrowband || rfi->broadband)) {  // src/pipeline.cpp:79-87
                    ci = rfi_input(ctx, cptr, chunks[k].length, rfi);
                    ci.pitch_min = pitch_min;
                    ci.more = overlap && k + 1 < nchunks;
                }
                if (async_back) {
                    ci.ev0 = ctx->file_dd_ev[2 * k];
                    ci.ev1 = ctx->file_dd_ev[2 * k + 1];
                }
                ChunkRun& cur = runs[k & 1];
                chunk_front(ctx, ci, &chunks[k], cfg, (int)(k & 1), cur);
                if (pending) back(runs[(k - 1) & 1]);
                pending = true;
                if (!overlap) {
                    back(cur);
                    pending = false;
                }
            }
            if (pending) back(runs[(nchunks - 1) & 1]);
        };
        if (!async_back) {
            run_chunks();
        } else {
            for (;;) {
                run_chunks();
                for (int sl = 0; sl < 2; ++sl)  // the back halves on bx_st are done before the readback
                    if (ctx->back_pending[sl]) {
                        PGB_CUDA(cudaStreamWaitEvent(ctx->st, ctx->ev_back[sl], 0));
                        ctx->back_pending[sl] = false;
                    }
                auto* hc = ctx->h_file_ctr.as<unsigned long long>();
                PGB_CUDA(cudaMemcpyAsync(hc, ctx->file_ctr.p, 3 * sizeof(unsigned long long),
                                         cudaMemcpyDeviceToHost, ctx->st));
                PGB_CUDA(cudaStreamSynchronize(ctx->st));
                total = hc[0];
                const uint64_t hi_c = hc[1], hi_f = hc[2];
                if (hi_c <= ctx->cand_cap && hi_f <= ctx->frag_cap && total <= file_cap) break;
                // a counter overflowed: grow and search the file again (rare)
                ctx->cand_cap = std::max<uint64_t>(ctx->cand_cap, round_up(hi_c * 2, 1024));
                ctx->frag_cap = std::max<uint64_t>(ctx->frag_cap, round_up(hi_f * 2, 1024));
                reset_timing(ctx);
            }
            const uint8_t* hs = ctx->h_file_status.as<uint8_t>();
            for (size_t k = 0; k < nchunks; ++k) {
                ChunkBook& b = book[k];
                std::vector<uint64_t> sk = b.skipped;
                if (b.live)
                    for (size_t r = 0; r < b.active.size(); ++r)
                        if (hs[k * (size_t)max_rows + r]) sk.push_back(b.active[r]);
                std::sort(sk.begin(), sk.end());
                for (uint64_t t : sk) {
                    ctx->file_skipped.push_back(b.index);
                    ctx->file_skipped.push_back(t);
                }
                if (b.live) {
                    float ms = 0.f;
                    PGB_CUDA(cudaEventElapsedTime(&ms, ctx->file_dd_ev[2 * k], ctx->file_dd_ev[2 * k + 1]));
                    ctx->dedisp_ms += ms;
                }
            }
        }
        trace_mark(ctx, "chunks done (host sync)", ctx->st);
        file_sort_link(ctx, total, radii, n_candidates, n_clusters);
    });
}

pgb_status pgb_fetch_file_candidates(pgb_context* ctx, pgb_candidate* out, size_t capacity) {
    return guarded([&] {
        need(ctx, PGB_ERR_ARGUMENT, "null ctx");
        need(capacity >= ctx->file_ncands && (ctx->file_ncands == 0 || out), PGB_ERR_ARGUMENT,
             "capacity too small");
        if (!ctx->file_ncands) return;
        PGB_CUDA(cudaMemcpyAsync(out, ctx->file_sorted.p, ctx->file_ncands * sizeof(pgb_candidate),
                                 cudaMemcpyDeviceToHost, ctx->st));
        PGB_CUDA(cudaStreamSynchronize(ctx->st));
    });
}

pgb_status pgb_fetch_file_skipped(pgb_context* ctx, uint64_t* pairs, size_t capacity, size_t* n_pairs) {
    return guarded([&] {
        need(ctx && n_pairs, PGB_ERR_ARGUMENT, "null argument");
        *n_pairs = ctx->file_skipped.size() / 2;
        if (!pairs) return;
        need(capacity >= *n_pairs, PGB_ERR_ARGUMENT, "capacity too small");
        std::copy(ctx->file_skipped.begin(), ctx->file_skipped.end(), pairs);
    });
}

pgb_status pgb_launch_count(pgb_context* ctx, uint64_t* launches) {
    return guarded([&] {
        need(ctx && launches, PGB_ERR_ARGUMENT, "null argument");
        *launches = ctx->launches;
    });
}

pgb_status pgb_last_dedisp_time(pgb_context* ctx, double* ms, uint64_t* launches, uint64_t* adds) {
    return guarded([&] {
        need(ctx, PGB_ERR_ARGUMENT, "null ctx");
        if (ms) *ms = ctx->dedisp_ms;
        if (launches) *launches = ctx->dedisp_launches;
        if (adds) *adds = ctx->channel_adds;
    });
}

pgb_status pgb_last_stage_times(pgb_context* ctx, double* ms) {
    return guarded([&] {
        need(ctx && ms, PGB_ERR_ARGUMENT, "null argument");
        for (int k = 0; k < 5; ++k) ms[k] = ctx->stage_ms[k];
    });
}

pgb_status pgb_last_cluster_ms(pgb_context* ctx, double* ms) {
    return guarded([&] {
        need(ctx && ms, PGB_ERR_ARGUMENT, "null argument");
        *ms = ctx->cluster_ms;
    });
}

pgb_status pgb_stream(pgb_context* ctx, void** stream) {
    return guarded([&] {
        need(ctx && stream, PGB_ERR_ARGUMENT, "null argument");
        *stream = ctx->st;
    });
}

// ---- bounded-memory streaming file search ---------------------------------------------
// execute_task with the prefetching reader (src/pipeline.cpp:66-106,
// src/filterbank.cpp:326-419): the caller reads chunk k into a pinned host buffer
// (pgb_stream_buffer) and pushes it; the upload of chunk k runs on the copy stream
// while chunk k-1 computes.  Host and device hold two chunks each, whatever the file
// size.  Back halves are synchronous (per-chunk count reads), so a counter overflow
// re-runs only that chunk's back half while its data is still resident.

pgb_status pgb_stream_begin(pgb_context* ctx, uint64_t nsamples, const pgb_chunk_spec* chunks, size_t nchunks,
                            const pgb_engine_config* cfg, const pgb_link_radii* radii,
                            const pgb_rfi_config* rfi) {
    return guarded([&] {
        need(ctx && cfg && (nchunks == 0 || chunks), PGB_ERR_ARGUMENT, "null argument");
        PGB_CUDA(cudaSetDevice(ctx->device));
        auto& S = ctx->stream;
        for (int b = 0; b < 2; ++b) {
            if (!S.up_done[b]) PGB_CUDA(cudaEventCreateWithFlags(&S.up_done[b], cudaEventDisableTiming));
            if (!S.dev_free[b]) PGB_CUDA(cudaEventCreateWithFlags(&S.dev_free[b], cudaEventDisableTiming));
            if (S.up_pending[b]) PGB_CUDA(cudaEventSynchronize(S.up_done[b]));
            S.up_pending[b] = S.dev_pending[b] = false;
        }
        for (size_t k = 0; k < nchunks; ++k) {
            need(chunks[k].start_sample + chunks[k].length <= nsamples, PGB_ERR_INVALID_PLAN,
                 "chunk extends past the file");
            validate_cfg(ctx, &chunks[k], cfg);
        }
        if (!S.runs) S.runs = new ChunkRunHolder();
        S.open = true;
        S.nsamples = nsamples;
        S.chunks.assign(chunks, chunks + nchunks);
        S.cfg = *cfg;
        S.has_radii = radii != nullptr;
        if (radii) S.radii = *radii;
        S.has_rfi = rfi && (rfi->narrowband || rfi->broadband);
        if (S.has_rfi) S.rfi = *rfi;
        S.next = 0;
        S.uploaded[0] = S.uploaded[1] = -1;
        S.part_chunk = -1;
        S.total = 0;
        S.pending = false;
        S.overlap = cfg->baseline_window > 0;
        S.pitch_min = 0;
        uint64_t lmax = 0;
        for (size_t k = 0; k < nchunks; ++k) {
            S.pitch_min = std::max<uint64_t>(S.pitch_min, chunks[k].length);
            lmax = std::max<uint64_t>(lmax, chunks[k].length);
        }
        const size_t cb = (size_t)lmax * ctx->nchans;
        for (int b = 0; b < 2 && b < (int)nchunks; ++b) {
            S.hbuf[b].reserve(cb);
            S.dbuf[b].reserve(cb);
        }
        reset_timing(ctx);
        ctx->file_skipped.clear();
        ctx->ser_ok = false;
        ctx->last_from_file = false;
        ctx->trace = getenv("PGB_TRACE") != nullptr;
        trace_mark(ctx, "stream begin", ctx->st);
    });
}

pgb_status pgb_stream_buffer(pgb_context* ctx, size_t k, uint8_t** host_buffer, size_t* capacity) {
    return guarded([&] {
        need(ctx && host_buffer, PGB_ERR_ARGUMENT, "null argument");
        auto& S = ctx->stream;
        std::lock_guard<std::mutex> lock(S.mu);  // the reader thread calls this during a push
        // the next chunk's buffer, or the one after it (a reader thread fills chunk k+1
        // while chunk k is being pushed)
        need(S.open && k >= S.next && k <= S.next + 1 && k < S.chunks.size(), PGB_ERR_ARGUMENT,
             "stream buffer requested out of order (next or next + 1 only)");
        const int b = (int)(k & 1);
        if (S.up_pending[b]) {  // chunk k-2's upload still reads this host buffer
            PGB_CUDA(cudaEventSynchronize(S.up_done[b]));
            S.up_pending[b] = false;
        }
        *host_buffer = S.hbuf[b].as<uint8_t>();
        if (capacity) *capacity = S.hbuf[b].bytes;
    });
}

namespace {
// first row of piece j of nparts (multiples of 64 rows: the progressive transpose writes
// 16-byte vectors at the piece start; the last piece ends at L)
uint64_t stream_piece_row(uint64_t L, size_t j, size_t nparts) {
    return j >= nparts ? L : L * j / nparts / 64 * 64;
}

// H2D of chunk k into device buffer k & 1 on the copy stream (caller holds S.mu)
void stream_upload(pgb_context* ctx, size_t k, const uint8_t* bytes) {
    auto& S = ctx->stream;
    const int b = (int)(k & 1);
    const size_t cb = (size_t)S.chunks[k].length * ctx->nchans;
    // the device buffer held chunk k-2 until its front half (transpose / RFI) read it
    if (S.dev_pending[b]) PGB_CUDA(cudaStreamWaitEvent(ctx->copy_st, S.dev_free[b], 0));
    if (bytes && bytes != S.hbuf[b].as<uint8_t>() && S.up_pending[b]) {
        PGB_CUDA(cudaEventSynchronize(S.up_done[b]));
        S.up_pending[b] = false;
    }
    PGB_CUDA(cudaMemcpyAsync(S.dbuf[b].p, bytes ? bytes : S.hbuf[b].as<uint8_t>(), cb,
                             cudaMemcpyHostToDevice, ctx->copy_st));
    PGB_CUDA(cudaEventRecord(S.up_done[b], ctx->copy_st));
    S.up_pending[b] = true;
    S.uploaded[b] = (int64_t)k;
}
}  // namespace

pgb_status pgb_stream_upload(pgb_context* ctx, size_t k) {
    return guarded([&] {
        need(ctx, PGB_ERR_ARGUMENT, "null ctx");
        auto& S = ctx->stream;
        std::lock_guard<std::mutex> lock(S.mu);
        need(S.open && k >= S.next && k <= S.next + 1 && k < S.chunks.size(), PGB_ERR_ARGUMENT,
             "stream upload requested out of order (next or next + 1 only)");
        PGB_CUDA(cudaSetDevice(ctx->device));
        if (S.uploaded[k & 1] != (int64_t)k) stream_upload(ctx, k, nullptr);
    });
}

pgb_status pgb_stream_upload_part(pgb_context* ctx, size_t k, size_t part, size_t nparts, int ok) {
    return guarded([&] {
        need(ctx && nparts > 0 && part < nparts, PGB_ERR_ARGUMENT, "bad piece");
        auto& S = ctx->stream;
        std::unique_lock<std::mutex> lock(S.mu);
        need(S.open && k >= S.next && k <= S.next + 1 && k < S.chunks.size(), PGB_ERR_ARGUMENT,
             "stream piece requested out of order (next or next + 1 only)");
        PGB_CUDA(cudaSetDevice(ctx->device));
        if (S.part_chunk != (int64_t)k) {
            need(S.part_chunk < 0 || (int64_t)k > S.part_chunk, PGB_ERR_ARGUMENT, "pieces of two chunks at once");
            S.part_chunk = (int64_t)k;
            const uint64_t L = S.chunks[k].length;
            while (S.parts.size() < nparts) {
                cudaEvent_t e;
                PGB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                S.parts.emplace_back(0, e);
            }
            for (size_t j = 0; j < S.parts.size(); ++j) S.parts[j].first = j < nparts ? stream_piece_row(L, j + 1, nparts) : 0;
            S.part_state.assign(nparts, 0);
            const int b = (int)(k & 1);
            // the device buffer held chunk k-2 until its front half read it
            if (S.dev_pending[b]) PGB_CUDA(cudaStreamWaitEvent(ctx->copy_st, S.dev_free[b], 0));
        }
        need(S.part_state.size() == nparts, PGB_ERR_ARGUMENT, "piece count changed within a chunk");
        if (ok < 0) {
            // announcement only: pgb_stream_push(k) will wait for the pieces
        } else if (!ok) {
            S.part_state[part] = 2;
        } else if (S.part_state[part] == 0) {
            const int b = (int)(k & 1);
            const size_t C = ctx->nchans;
            const uint64_t L = S.chunks[k].length;
            const uint64_t r0 = stream_piece_row(L, part, nparts), r1 = stream_piece_row(L, part + 1, nparts);
            if (r1 > r0)
                PGB_CUDA(cudaMemcpyAsync(S.dbuf[b].as<uint8_t>() + r0 * C, S.hbuf[b].as<uint8_t>() + r0 * C,
                                         (r1 - r0) * C, cudaMemcpyHostToDevice, ctx->copy_st));
            PGB_CUDA(cudaEventRecord(S.parts[part].second, ctx->copy_st));
            S.part_state[part] = 1;
        }
        S.cv.notify_all();
    });
}

pgb_status pgb_stream_push(pgb_context* ctx, size_t k, const uint8_t* bytes) {
    return guarded([&] {
        NvtxRange nvtx("pgb stream push");
        need(ctx, PGB_ERR_ARGUMENT, "null ctx");
        auto& S = ctx->stream;
        need(S.open && k == S.next && k < S.chunks.size(), PGB_ERR_ARGUMENT, "chunks are pushed in order");
        PGB_CUDA(cudaSetDevice(ctx->device));
        // every earlier push ended with a stream sync (append_chunk_sync), so the pinned
        // staging arena of the small per-chunk uploads is free again
        if (k > 0) stage_reset(ctx);
        const pgb_chunk_spec& spec = S.chunks[k];
        const int b = (int)(k & 1);
        const bool pieces = S.part_chunk == (int64_t)k;  // uploaded piece by piece (progressive)
        std::vector<std::pair<uint64_t, cudaEvent_t>> prog;
        {
            std::lock_guard<std::mutex> lock(S.mu);
            if (pieces) {
                need(!bytes || bytes == S.hbuf[b].as<uint8_t>(), PGB_ERR_ARGUMENT,
                     "a chunk uploaded in pieces is pushed from its stream buffer");
                prog.assign(S.parts.begin(), S.parts.begin() + (long)S.part_state.size());
            } else {
                // already uploaded by pgb_stream_upload (from the caller's own buffer only if
                // that is where the bytes are)
                if (S.uploaded[b] != (int64_t)k || (bytes && bytes != S.hbuf[b].as<uint8_t>()))
                    stream_upload(ctx, k, bytes);
                S.uploaded[b] = -1;
                PGB_CUDA(cudaStreamWaitEvent(ctx->st, S.up_done[b], 0));
            }
        }
        trace_mark(ctx, "chunk upload waited", ctx->st);
        const uint8_t* cptr = S.dbuf[b].as<uint8_t>();
        ChunkInput ci{cptr, true};
        ci.raw = true;
        ci.pitch_min = S.pitch_min;
        ci.more = S.overlap && k + 1 < S.chunks.size();
        auto wait_piece = [&S](size_t j) {
            std::unique_lock<std::mutex> lock(S.mu);
            S.cv.wait(lock, [&] { return S.part_state[j] != 0; });
            if (S.part_state[j] == 2) raise(PGB_ERR_READ, "stream piece " + std::to_string(j) + " was not read");
        };
        if (pieces) {
            if (k == 0 && !S.has_rfi) {  // progressive transpose + dedispersion (chunk_front)
                ci.prog = &prog;
                ci.seg_ready = wait_piece;
            } else {  // RFI excision and overlap reuse need the whole chunk first
                for (size_t j = 0; j < prog.size(); ++j) {
                    wait_piece(j);
                    PGB_CUDA(cudaStreamWaitEvent(ctx->st, prog[j].second, 0));
                }
            }
        }
        if (S.has_rfi) {  // src/pipeline.cpp:79-87
            ci = rfi_input(ctx, cptr, spec.length, &S.rfi);
            ci.pitch_min = S.pitch_min;
            ci.more = S.overlap && k + 1 < S.chunks.size();
        }
        ChunkRun* runs = S.runs->r;
        ChunkRun& cur = runs[k & 1];
        chunk_front(ctx, ci, &spec, &S.cfg, (int)(k & 1), cur);
        {
            std::lock_guard<std::mutex> lock(S.mu);
            PGB_CUDA(cudaEventRecord(S.dev_free[b], ctx->st));
            S.dev_pending[b] = true;
            if (pieces) {  // every piece was issued (chunk_front waited for each): the host
                // buffer is free once the copy stream is past them
                PGB_CUDA(cudaEventRecord(S.up_done[b], ctx->copy_st));
                S.up_pending[b] = true;
                S.part_chunk = -1;
            }
        }
        if (S.pending) append_chunk_sync(ctx, runs[(k - 1) & 1], S.total);
        S.pending = true;
        if (!S.overlap) {
            append_chunk_sync(ctx, cur, S.total);
            S.pending = false;
        }
        {
            std::lock_guard<std::mutex> lock(S.mu);
            ++S.next;
        }
    });
}

pgb_status pgb_stream_finish(pgb_context* ctx, size_t* n_candidates, size_t* n_clusters) {
    return guarded([&] {
        need(ctx, PGB_ERR_ARGUMENT, "null ctx");
        auto& S = ctx->stream;
        need(S.open && S.next == S.chunks.size(), PGB_ERR_ARGUMENT, "not every chunk was pushed");
        PGB_CUDA(cudaSetDevice(ctx->device));
        if (S.pending) append_chunk_sync(ctx, S.runs->r[(S.next - 1) & 1], S.total);
        S.pending = false;
        S.open = false;
        trace_mark(ctx, "chunks done (host sync)", ctx->st);
        file_sort_link(ctx, S.total, S.has_radii ? &S.radii : nullptr, n_candidates, n_clusters);
        for (int b = 0; b < 2; ++b) S.up_pending[b] = S.dev_pending[b] = false;  // stream synced
    });
}

// ---- multi-GPU payload fan-out (CUDA IPC over NVLink) -----------------------------------
// A dedicated cudaMalloc allocation, so its IPC handle maps exactly this buffer (a
// sub-allocation of a caching allocator would export its whole segment).
pgb_status pgb_device_alloc(int device, size_t bytes, void** device_ptr) {
    return guarded([&] {
        need(device_ptr && bytes, PGB_ERR_ARGUMENT, "null argument");
        PGB_CUDA(cudaSetDevice(device));
        if (cudaMalloc(device_ptr, bytes) != cudaSuccess) {
            cudaGetLastError();
            raise(PGB_ERR_OOM, "device allocation of " + std::to_string(bytes) + " bytes failed");
        }
    });
}

pgb_status pgb_device_free(int device, void* device_ptr) {
    return guarded([&] {
        PGB_CUDA(cudaSetDevice(device));
        PGB_CUDA(cudaFree(device_ptr));
    });
}

pgb_status pgb_ipc_get_handle(const void* device_ptr, void* handle) {
    return guarded([&] {
        need(device_ptr && handle, PGB_ERR_ARGUMENT, "null argument");
        static_assert(sizeof(cudaIpcMemHandle_t) == PGB_IPC_HANDLE_BYTES, "IPC handle size");
        cudaIpcMemHandle_t h;
        PGB_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(device_ptr)));
        std::memcpy(handle, &h, sizeof h);
    });
}

pgb_status pgb_ipc_open(int device, const void* handle, void** device_ptr) {
    return guarded([&] {
        need(handle && device_ptr, PGB_ERR_ARGUMENT, "null argument");
        PGB_CUDA(cudaSetDevice(device));
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof h);
        PGB_CUDA(cudaIpcOpenMemHandle(device_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    });
}

pgb_status pgb_ipc_close(void* device_ptr) {
    return guarded([&] { PGB_CUDA(cudaIpcCloseMemHandle(device_ptr)); });
}

pgb_status pgb_copy_async(pgb_context* ctx, void* dst, const void* src, size_t bytes) {
    return guarded([&] {
        need(ctx && (bytes == 0 || (dst && src)), PGB_ERR_ARGUMENT, "null argument");
        PGB_CUDA(cudaSetDevice(ctx->device));
        if (bytes) PGB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->st));
    });
}

pgb_status pgb_synchronize(pgb_context* ctx) {
    return guarded([&] {
        need(ctx, PGB_ERR_ARGUMENT, "null ctx");
        PGB_CUDA(cudaSetDevice(ctx->device));
        PGB_CUDA(cudaStreamSynchronize(ctx->st));
    });
}

}  // extern "C"
