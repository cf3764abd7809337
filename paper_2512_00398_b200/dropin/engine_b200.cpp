// Drop-in replacement for the reference's engine translation unit
// (/root/reference/proj/src/engine.cpp), compiled against the reference's own
// headers (include/pulsegrid/engine.hpp) and linked in its place.  Every symbol
// of engine.hpp:43-62 is defined with the identical C++ signature; run_dm_loop runs
// on the B200 through the C ABI of libpgb200 (include/pulsegrid_b200.h).
//
// Semantics: identical candidates, skipped trials and exceptions to the
// reference in its defect-free parity mode.  n_workers,
// memory_budget and max_in_flight are validated exactly as src/engine.cpp:87-97
// does; the BufferPool is not used for device memory (the context keeps its own
// arena), so pool-exhaustion errors (budget_exhausted_error) never arise.
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>

#include "pulsegrid/engine.hpp"
#include "pulsegrid_b200.h"

namespace pulsegrid {

static_assert(sizeof(Candidate) == sizeof(pgb_candidate), "Candidate layout must match the C ABI");

namespace {

[[noreturn]] void rethrow_status(pgb_status st) {
    const std::string msg = pgb_last_error();
    switch (st) {
        case PGB_ERR_CONFIG: throw config_error(msg);
        case PGB_ERR_INVALID_RANGE: throw invalid_range_error(msg);
        case PGB_ERR_CHUNK_TOO_SHORT: {
            std::size_t trial = 0;
            if (msg.rfind("trial ", 0) == 0) trial = std::stoull(msg.substr(6));
            throw chunk_too_short_error(trial, msg);
        }
        case PGB_ERR_BUDGET: throw budget_exhausted_error(msg);
        case PGB_ERR_DEGENERATE: throw degenerate_series_error(msg);
        case PGB_ERR_INVALID_PLAN: throw invalid_plan_error(msg);
        default: throw error("libpgb200: " + msg);
    }
}

void check(pgb_status st) {
    if (st != PGB_OK) rethrow_status(st);
}

// One device context per calling thread (run_dm_loop is re-entrant across the
// pipeline's execution workers, src/pipeline.cpp:182-194).  The plan is uploaded
// once and re-used while the same DmTrialPlan is passed in.
struct ThreadCtx {
    pgb_context* ctx = nullptr;
    const DmTrialPlan* plan = nullptr;
    std::size_t ntrials = 0, nchans = 0;
    std::int64_t max_delay = -1;
    double dm0 = 0.0, dm1 = 0.0;
    std::vector<std::int64_t> flat;  // the uploaded delays, to detect in-place edits

    ~ThreadCtx() {
        if (ctx) pgb_destroy(ctx);
    }

    void ensure_plan(const DmTrialPlan& p, std::uint32_t nch) {
        const bool same = plan == &p && ntrials == p.ntrials() && nchans == nch &&
                          max_delay == p.max_delay && (ntrials == 0 || (dm0 == p.dms.front() &&
                                                                        dm1 == p.dms.back()));
        if (same) {
            bool identical = true;
            for (std::size_t t = 0; t < ntrials && identical; ++t)
                identical = std::memcmp(flat.data() + t * nch, p.delays[t].data(),
                                        nch * sizeof(std::int64_t)) == 0;
            if (identical) return;
        }
        flat.resize(p.ntrials() * nch);
        for (std::size_t t = 0; t < p.ntrials(); ++t) {
            if (p.delays[t].size() != nch) throw invalid_plan_error("plan nchans differs from chunk");
            std::memcpy(flat.data() + t * nch, p.delays[t].data(), nch * sizeof(std::int64_t));
        }
        check(pgb_set_plan(ctx, p.dms.data(), flat.data(), (std::uint32_t)p.ntrials(), nch));
        plan = &p;
        ntrials = p.ntrials();
        nchans = nch;
        max_delay = p.max_delay;
        dm0 = ntrials ? p.dms.front() : 0.0;
        dm1 = ntrials ? p.dms.back() : 0.0;
    }
};

ThreadCtx& thread_ctx() {
    thread_local ThreadCtx tc;
    if (!tc.ctx) {
        int device = 0;
        if (const char* e = std::getenv("PULSEGRID_B200_DEVICE")) device = std::atoi(e);
        check(pgb_create(device, &tc.ctx));
    }
    return tc;
}

}  // namespace

std::vector<std::vector<std::size_t>> partition_trials(std::size_t ntrials,
                                                       std::uint32_t n_workers) {
    std::vector<std::vector<std::size_t>> parts(std::max<std::uint32_t>(1, n_workers));
    for (std::size_t i = 0; i < ntrials; ++i) parts[i % parts.size()].push_back(i);
    return parts;
}

std::size_t trial_working_set_bytes(const DmTrialPlan& plan, std::uint64_t chunk_len,
                                    const EngineConfig& cfg) {
    const std::int64_t min_delay = plan.trial_max_delay(0);
    const std::uint64_t longest =
        chunk_len > std::uint64_t(min_delay) ? chunk_len - std::uint64_t(min_delay) : 1;
    const std::size_t series_bytes = BufferPool::aligned_size(longest * sizeof(float));
    const std::uint64_t n_blocks = (longest + scan_block_size - 1) / scan_block_size;
    const std::size_t sums_bytes = BufferPool::aligned_size((longest + n_blocks) * sizeof(double));
    return (cfg.baseline_window > 0 ? 2 : 1) * series_bytes + sums_bytes;
}

std::size_t in_flight_limit(const DmTrialPlan& plan, std::uint64_t chunk_len,
                            const EngineConfig& cfg) {
    const std::size_t ws = trial_working_set_bytes(plan, chunk_len, cfg);
    const std::size_t limit = cfg.memory_budget / ws;
    if (limit == 0)
        throw config_error("memory budget of " + std::to_string(cfg.memory_budget) +
                           " bytes is below one trial's working set (" + std::to_string(ws) + ")");
    return limit;
}

DmLoopResult run_dm_loop(const Chunk& chunk, const DmTrialPlan& plan, const EngineConfig& cfg,
                         BufferPool& /*pool: device arena instead*/) {
    if (cfg.n_workers < 1) throw config_error("n_workers must be >= 1");
    if (cfg.boxcar_max < 1 || (cfg.boxcar_max & (cfg.boxcar_max - 1)) != 0)
        throw config_error("boxcar_max must be a power of two");
    if (plan.ntrials() == 0) return {};
    if (cfg.max_in_flight == 0) (void)in_flight_limit(plan, chunk.spec.length, cfg);

    ThreadCtx& tc = thread_ctx();
    tc.ensure_plan(plan, chunk.nchans);
    const pgb_chunk_spec spec{chunk.spec.index,   chunk.spec.start_sample, chunk.spec.length,
                              chunk.spec.overlap, chunk.spec.valid_begin,  chunk.spec.valid_end};
    const pgb_engine_config ec{cfg.n_workers,     cfg.detect_thresh,        cfg.tsamp,
                               cfg.boxcar_max,    cfg.baseline_window,      cfg.memory_budget,
                               cfg.max_in_flight};
    std::size_t nc = 0, ns = 0;
    // widened chunk (floats): integral 8-bit data is repacked to bytes on the host and
    // uploaded from pinned memory (a quarter of the bytes); anything else stays fp32
    check(pgb_run_dm_loop_f32(tc.ctx, chunk.data.data(), 0, &spec, &ec, &nc, &ns));
    DmLoopResult result;
    result.candidates.resize(nc);
    check(pgb_fetch_candidates(tc.ctx, reinterpret_cast<pgb_candidate*>(result.candidates.data()), nc));
    std::vector<std::uint64_t> sk(ns);
    check(pgb_fetch_skipped(tc.ctx, sk.data(), ns));
    result.skipped_trials.assign(sk.begin(), sk.end());
    if (cfg.timing_sink) {
        // The device runs each stage batched over the chunk's trials; like the reference's
        // per-block dedisperse_ms (src/engine.cpp:147-149), every stage time is amortised
        // over the trials it processed, and only trials that reached the end of the chain
        // emit a record (uncoverable and degenerate ones do not, src/engine.cpp:112-118,
        // 189-194)
        double ms[5] = {};
        check(pgb_last_stage_times(tc.ctx, ms));
        std::vector<std::size_t> done;
        done.reserve(plan.ntrials());
        std::size_t k = 0;
        for (std::size_t t = 0; t < plan.ntrials(); ++t) {
            while (k < result.skipped_trials.size() && result.skipped_trials[k] < t) ++k;
            if (k < result.skipped_trials.size() && result.skipped_trials[k] == t) continue;
            done.push_back(t);
        }
        const double inv = done.empty() ? 0.0 : 1.0 / double(done.size());
        for (std::size_t t : done) {
            TrialTiming timing;
            timing.trial = t;
            timing.dedisperse_ms = ms[0] * inv;
            timing.baseline_ms = cfg.baseline_window > 0 ? ms[1] * inv : 0.0;
            timing.normalize_ms = ms[2] * inv;
            timing.boxcar_ms = ms[3] * inv;
            timing.peaks_ms = ms[4] * inv;
            cfg.timing_sink(timing);
        }
    }
    return result;
}

}  // namespace pulsegrid
