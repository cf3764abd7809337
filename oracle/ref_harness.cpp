// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// C ABI over the *unmodified* reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  The reference
// ships no FFI; the tests, tests/golden/make_golden.py and bench.py's
// cpu_baseline / --impl reference arm drive the reference's own public API
// through these shims, using the same plain-C record layouts as the product ABI
// (include/pulsegrid_b200.h) so results compare field by field.
//
// Parity mode: run_dm_loop with max_in_flight == n_workers gives block size 1
// (src/engine.cpp:95-97), which sidesteps the straggler-loop defect of
// dedisperse_block (src/dedisp.cpp:188-195) and equals the
// naive definition for every worker count.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../include/pulsegrid_b200.h"
#include "pulsegrid/cluster.hpp"
#include "pulsegrid/cluster_io.hpp"
#include "pulsegrid/dedisp.hpp"
#include "pulsegrid/detect.hpp"
#include "pulsegrid/engine.hpp"
#include "pulsegrid/filterbank.hpp"
#include "pulsegrid/pipeline.hpp"
#include "pulsegrid/rfi.hpp"
#include "pulsegrid/synth.hpp"

using namespace pulsegrid;

static_assert(sizeof(pgb_candidate) == sizeof(Candidate), "Candidate layout");
static_assert(offsetof(pgb_candidate, peak_sample) == offsetof(Candidate, peak_sample));
static_assert(offsetof(pgb_candidate, time_s) == offsetof(Candidate, time_s));
static_assert(offsetof(pgb_candidate, width_index) == offsetof(Candidate, width_index));
static_assert(offsetof(pgb_candidate, width_samples) == offsetof(Candidate, width_samples));
static_assert(offsetof(pgb_candidate, dm_trial) == offsetof(Candidate, dm_trial));
static_assert(offsetof(pgb_candidate, dm) == offsetof(Candidate, dm));
static_assert(offsetof(pgb_candidate, begin_sample) == offsetof(Candidate, begin_sample));
static_assert(offsetof(pgb_candidate, end_sample) == offsetof(Candidate, end_sample));

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const config_error*>(&e)) return PGB_ERR_CONFIG;
    if (dynamic_cast<const invalid_range_error*>(&e)) return PGB_ERR_INVALID_RANGE;
    if (dynamic_cast<const chunk_too_short_error*>(&e)) return PGB_ERR_CHUNK_TOO_SHORT;
    if (dynamic_cast<const budget_exhausted_error*>(&e)) return PGB_ERR_BUDGET;
    if (dynamic_cast<const degenerate_series_error*>(&e)) return PGB_ERR_DEGENERATE;
    if (dynamic_cast<const invalid_plan_error*>(&e)) return PGB_ERR_INVALID_PLAN;
    return PGB_ERR_ARGUMENT;
}

FilterbankHeader to_header(const pgb_header* h) {
    FilterbankHeader fh;
    fh.source_name = "pgref";
    fh.fch1 = h->fch1;
    fh.foff = h->foff;
    fh.tsamp = h->tsamp;
    fh.nchans = h->nchans;
    fh.nbits = 8;
    fh.tstart = 60000.0;
    return fh;
}

DmTrialPlan to_plan(const double* dms, const int64_t* delays, uint32_t ntrials, uint32_t nchans) {
    DmTrialPlan plan;
    plan.dms.assign(dms, dms + ntrials);
    plan.delays.resize(ntrials);
    for (uint32_t t = 0; t < ntrials; ++t) {
        plan.delays[t].assign(delays + size_t(t) * nchans, delays + size_t(t + 1) * nchans);
        for (auto d : plan.delays[t]) plan.max_delay = std::max(plan.max_delay, d);
    }
    return plan;
}

EngineConfig to_cfg(const pgb_engine_config* c) {
    EngineConfig cfg;
    cfg.n_workers = c->n_workers;
    cfg.tsamp = c->tsamp;
    cfg.detect_thresh = c->detect_thresh;
    cfg.boxcar_max = c->boxcar_max;
    cfg.baseline_window = c->baseline_window;
    cfg.memory_budget = c->memory_budget;
    cfg.max_in_flight = c->max_in_flight;
    return cfg;
}

ChunkSpec to_spec(const pgb_chunk_spec* s) {
    ChunkSpec spec;
    spec.index = s->index;
    spec.start_sample = s->start_sample;
    spec.length = s->length;
    spec.overlap = s->overlap;
    spec.valid_begin = s->valid_begin;
    spec.valid_end = s->valid_end;
    return spec;
}

template <typename T>
T* dup(const std::vector<T>& v) {
    T* p = static_cast<T*>(std::malloc(std::max<size_t>(1, v.size() * sizeof(T))));
    if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
    return p;
}

int export_clusters(const std::vector<ClusterResult>& clusters, pgb_cluster** out, size_t* n_out,
                    uint64_t** members_out) {
    std::vector<pgb_cluster> cs(clusters.size());
    std::vector<uint64_t> members;
    for (size_t k = 0; k < clusters.size(); ++k) {
        const auto& c = clusters[k];
        std::memcpy(&cs[k].representative, &c.representative, sizeof(Candidate));
        cs[k].members = c.members;
        cs[k].begin_sample = c.begin_sample;
        cs[k].end_sample = c.end_sample;
        cs[k].dm_lo = c.dm_lo;
        cs[k].dm_hi = c.dm_hi;
        cs[k].member_offset = members.size();
        for (auto id : c.member_ids) members.push_back(id);
    }
    *out = dup(cs);
    *n_out = cs.size();
    *members_out = dup(members);
    return PGB_OK;
}

}  // namespace

extern "C" {

const char* pgref_last_error() { return g_err.c_str(); }
void pgref_free(void* p) { std::free(p); }

int64_t pgref_delay_samples(double dm, const pgb_header* h, uint32_t channel) {
    return delay_samples(dm, to_header(h), channel);
}

double pgref_adaptive_dm_step(double tol, const pgb_header* h) {
    return adaptive_dm_step(tol, to_header(h));
}

int pgref_generate_dm_trials(double dm_lo, double dm_hi, const pgb_header* h, int spacing,
                             double value, double* dms, int64_t* delays, size_t cap,
                             size_t* ntrials) {
    try {
        DmSpacing sp = spacing == PGB_SPACING_LINEAR ? DmSpacing{LinearSpacing{value}}
                                                     : DmSpacing{AdaptiveSpacing{value}};
        auto plan = generate_dm_trials(dm_lo, dm_hi, to_header(h), sp);
        *ntrials = plan.ntrials();
        if (dms) {
            if (cap < plan.ntrials()) throw std::invalid_argument("capacity");
            for (size_t t = 0; t < plan.ntrials(); ++t) {
                dms[t] = plan.dms[t];
                if (delays)
                    std::memcpy(delays + t * h->nchans, plan.delays[t].data(),
                                h->nchans * sizeof(int64_t));
            }
        }
        return PGB_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// run_dm_loop on a widened float chunk.  parity != 0 forces max_in_flight =
// n_workers (block size 1); parity == 0 runs the shipped default (defective).
int pgref_run_dm_loop_f32(const float* data, const pgb_chunk_spec* spec, uint32_t nchans,
                          const double* dms, const int64_t* delays, uint32_t ntrials,
                          const pgb_engine_config* c, int parity, pgb_candidate** cands,
                          size_t* ncands, uint64_t** skipped, size_t* nskipped, double* ms) {
    try {
        Chunk chunk;
        chunk.spec = to_spec(spec);
        chunk.nchans = nchans;
        chunk.data.assign(data, data + spec->length * nchans);
        auto plan = to_plan(dms, delays, ntrials, nchans);
        auto cfg = to_cfg(c);
        if (parity) cfg.max_in_flight = cfg.n_workers;
        BufferPool pool(std::max<size_t>(cfg.memory_budget, size_t(1) << 20));
        const auto t0 = std::chrono::steady_clock::now();
        auto result = run_dm_loop(chunk, plan, cfg, pool);
        const auto t1 = std::chrono::steady_clock::now();
        if (ms) *ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        std::vector<pgb_candidate> out(result.candidates.size());
        if (!out.empty()) std::memcpy(out.data(), result.candidates.data(), out.size() * sizeof(Candidate));
        *cands = dup(out);
        *ncands = out.size();
        std::vector<uint64_t> sk(result.skipped_trials.begin(), result.skipped_trials.end());
        *skipped = dup(sk);
        *nskipped = sk.size();
        return PGB_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int pgref_run_dm_loop_u8(const uint8_t* data, const pgb_chunk_spec* spec, uint32_t nchans,
                         const double* dms, const int64_t* delays, uint32_t ntrials,
                         const pgb_engine_config* c, int parity, pgb_candidate** cands,
                         size_t* ncands, uint64_t** skipped, size_t* nskipped, double* ms) {
    // read_chunk's 8-bit widening, src/filterbank.cpp:304-307
    std::vector<float> f(spec->length * nchans);
    for (size_t i = 0; i < f.size(); ++i) f[i] = float(data[i]);
    return pgref_run_dm_loop_f32(f.data(), spec, nchans, dms, delays, ntrials, c, parity, cands,
                                 ncands, skipped, nskipped, ms);
}

// Single-trial dedispersion (the naive-definition reference, src/dedisp.cpp:200-218).
int pgref_dedisperse(const float* data, uint64_t length, uint32_t nchans, const double* dms,
                     const int64_t* delays, uint32_t ntrials, uint32_t trial, float* out,
                     uint64_t* n_out) {
    try {
        Chunk chunk;
        chunk.spec.length = length;
        chunk.spec.valid_end = length;
        chunk.nchans = nchans;
        chunk.data.assign(data, data + length * nchans);
        auto plan = to_plan(dms, delays, ntrials, nchans);
        auto series = dedisperse(chunk, plan, trial);
        std::memcpy(out, series.values.data(), series.values.size() * sizeof(float));
        *n_out = series.values.size();
        return PGB_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// The shipped multi-trial block path (exhibits the straggler defect for >1 tile).
int pgref_dedisperse_block(const float* data, uint64_t length, uint32_t nchans,
                           const double* dms, const int64_t* delays, uint32_t ntrials,
                           const uint64_t* trials, uint32_t ntr, float* out, uint64_t stride) {
    try {
        Chunk chunk;
        chunk.spec.length = length;
        chunk.spec.valid_end = length;
        chunk.nchans = nchans;
        chunk.data.assign(data, data + length * nchans);
        auto plan = to_plan(dms, delays, ntrials, nchans);
        auto rows = transpose_chunk(chunk);
        std::vector<size_t> idx(trials, trials + ntr);
        std::vector<float*> ptrs(ntr);
        for (uint32_t b = 0; b < ntr; ++b) ptrs[b] = out + size_t(b) * stride;
        dedisperse_block(rows, length, nchans, plan, idx, ptrs);
        return PGB_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int pgref_remove_baseline(const float* x, uint64_t n, uint64_t window, float* out) {
    try {
        remove_baseline_into(std::span<const float>(x, n), window, std::span<float>(out, n));
        return PGB_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int pgref_normalize_to_sums(const float* x, uint64_t n, double* sums, double* maxima,
                            double* rms) {
    try {
        const uint64_t nb = (n + scan_block_size - 1) / scan_block_size;
        *rms = normalize_to_sums(std::span<const float>(x, n), std::span<double>(sums, n),
                                 std::span<double>(maxima, nb));
        return PGB_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// find_peaks (detect.hpp:211) on a caller-provided S/N series.
int pgref_find_peaks(const double* snr, uint64_t n, double threshold, uint32_t width_index,
                     uint64_t start_sample, double tsamp, uint32_t dm_trial, double dm,
                     uint64_t valid_begin, uint64_t valid_end, int drop_left, int drop_right,
                     pgb_candidate** cands, size_t* ncands) {
    try {
        PeakMeta meta;
        meta.start_sample = start_sample;
        meta.tsamp = tsamp;
        meta.dm_trial = dm_trial;
        meta.dm = dm;
        meta.valid_begin = valid_begin;
        meta.valid_end = valid_end;
        meta.drop_left_edge_run = drop_left != 0;
        meta.drop_right_edge_run = drop_right != 0;
        auto cs = find_peaks(std::span<const double>(snr, n), threshold, width_index, meta);
        std::vector<pgb_candidate> out(cs.size());
        if (!out.empty()) std::memcpy(out.data(), cs.data(), out.size() * sizeof(Candidate));
        *cands = dup(out);
        *ncands = out.size();
        return PGB_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int pgref_link_grid(const pgb_candidate* cands, size_t n, const pgb_link_radii* r, int reference,
                    pgb_cluster** out, size_t* nclusters, uint64_t** members, double* ms) {
    try {
        std::vector<Candidate> cs(n);
        if (n) std::memcpy(cs.data(), cands, n * sizeof(Candidate));
        LinkRadii radii{r->sep_time, r->sep_dm_trials, r->sep_width};
        const auto t0 = std::chrono::steady_clock::now();
        auto clusters = reference ? link_reference(cs, radii) : link_grid(cs, radii);
        const auto t1 = std::chrono::steady_clock::now();
        if (ms) *ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        return export_clusters(clusters, out, nclusters, members);
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// .cand text of a cluster list (src/cluster_io.cpp:11-34).
int pgref_write_candidates(const pgb_cluster* clusters, size_t n, char** text, size_t* len) {
    try {
        std::vector<ClusterResult> cs(n);
        for (size_t k = 0; k < n; ++k) {
            std::memcpy(&cs[k].representative, &clusters[k].representative, sizeof(Candidate));
            cs[k].members = clusters[k].members;
            cs[k].begin_sample = clusters[k].begin_sample;
            cs[k].end_sample = clusters[k].end_sample;
            cs[k].dm_lo = clusters[k].dm_lo;
            cs[k].dm_hi = clusters[k].dm_hi;
        }
        std::ostringstream os;
        write_candidates(cs, os);
        const std::string s = os.str();
        *text = static_cast<char*>(std::malloc(s.size() + 1));
        std::memcpy(*text, s.c_str(), s.size() + 1);
        *len = s.size();
        return PGB_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int pgref_plan_chunks(uint64_t nsamples, uint64_t chunk_len, uint64_t overlap, pgb_chunk_spec* out,
                      size_t cap, size_t* n) {
    try {
        auto specs = plan_chunks(nsamples, chunk_len, overlap);
        *n = specs.size();
        if (out) {
            if (cap < specs.size()) throw std::invalid_argument("capacity");
            for (size_t k = 0; k < specs.size(); ++k)
                out[k] = {specs[k].index,   specs[k].start_sample, specs[k].length,
                          specs[k].overlap, specs[k].valid_begin,  specs[k].valid_end};
        }
        return PGB_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Deterministic reference noise (src/synth.cpp:46-53) and injection (:55-70).
int pgref_generate_noise(const pgb_header* h, uint64_t nsamples, float mean, float sigma,
                         uint64_t seed, float* out) {
    try {
        auto g = generate_noise(to_header(h), nsamples, mean, sigma, seed);
        std::memcpy(out, g.data(), g.size() * sizeof(float));
        return PGB_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int pgref_inject_pulse(float* grid, uint64_t nsamples, const pgb_header* h, double dm, double t0,
                       uint64_t width, float amplitude) {
    try {
        inject_pulse(std::span<float>(grid, nsamples * h->nchans), to_header(h),
                     PulseSpec{dm, t0, width, amplitude});
        return PGB_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

double pgref_amplitude_for_snr(double snr, double sigma, uint32_t nchans, uint64_t width) {
    return amplitude_for_snr(snr, sigma, nchans, width);
}

uint32_t pgref_quantize_code(float value, double offset, double scale, uint32_t nbits) {
    return quantize_code(value, QuantSpec{offset, scale}, nbits);
}

int pgref_write_filterbank(const char* path, const pgb_header* h, uint32_t nbits,
                           const float* samples, uint64_t nsamples) {
    try {
        auto fh = to_header(h);
        fh.nbits = nbits;
        std::ofstream out(path, std::ios::binary);
        write_filterbank(fh, std::span<const float>(samples, nsamples * h->nchans), out);
        return out ? PGB_OK : PGB_ERR_ARGUMENT;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// flag_narrowband + flag_broadband + apply_mask on one widened chunk
// (src/rfi.cpp:32-139; execute_task's order, src/pipeline.cpp:79-87).  `data` is
// cleaned in place; bad channel / sample masks are returned as 0/1 bytes.
int pgref_rfi(float* data, uint64_t length, uint32_t nchans, int narrowband, int broadband,
              double k_sigma, double k_mad, int local_mean, uint8_t* bad_ch, uint8_t* bad_s) {
    try {
        Chunk chunk;
        chunk.spec.length = length;
        chunk.spec.valid_end = length;
        chunk.nchans = nchans;
        chunk.data.assign(data, data + length * nchans);
        RfiMask mask;
        mask.replacement = local_mean ? MaskPolicy::local_mean : MaskPolicy::zero;
        if (narrowband) mask.bad_channels = flag_narrowband(chunk, k_mad);
        if (broadband) mask.bad_samples = flag_broadband(chunk, k_sigma);
        if (!mask.bad_channels.empty() || !mask.bad_samples.empty()) apply_mask(chunk, mask);
        std::memcpy(data, chunk.data.data(), length * nchans * sizeof(float));
        std::memset(bad_ch, 0, nchans);
        std::memset(bad_s, 0, length);
        for (auto c : mask.bad_channels) bad_ch[c] = 1;
        for (auto s : mask.bad_samples) bad_s[s] = 1;
        return PGB_OK;
    } catch (const insufficient_statistics_error& e) {
        g_err = e.what();
        return PGB_ERR_INSUFFICIENT;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Search parameters for the file-level run (pipeline.hpp:17-38), flattened.
struct pgref_search_params {
    double dm_lo, dm_hi, dm_step;
    uint32_t n_workers;
    float detect_thresh;
    uint64_t boxcar_max;
    double baseline_len_s;
    uint64_t nsamps_chunk;
    int rfi_narrowband, rfi_broadband;
    double k_sigma, k_mad;
    int parity;
    pgb_link_radii radii;
};

// create_task + execute_task on a file (src/pipeline.cpp:32-119): writes the
// reference .cand file and reports the stage timings.
int pgref_execute_file(const char* path, const char* out_path, const pgref_search_params* p,
                       double* stage_ms /*[6]: wall read rfi dm_loop cluster write*/,
                       size_t* n_clusters) {
    try {
        SearchParams params;
        params.dm_lo = p->dm_lo;
        params.dm_hi = p->dm_hi;
        params.spacing = LinearSpacing{p->dm_step};
        params.engine.n_workers = p->n_workers;
        params.engine.detect_thresh = p->detect_thresh;
        params.engine.boxcar_max = p->boxcar_max;
        params.engine.radii = LinkRadii{p->radii.sep_time, p->radii.sep_dm_trials, p->radii.sep_width};
        if (p->parity) params.engine.max_in_flight = p->n_workers;
        params.baseline_len_s = p->baseline_len_s;
        params.nsamps_chunk = p->nsamps_chunk;
        params.rfi_narrowband = p->rfi_narrowband != 0;
        params.rfi_broadband = p->rfi_broadband != 0;
        params.k_sigma = p->k_sigma;
        params.k_mad = p->k_mad;
        auto task = create_task(path, params, out_path);
        BufferPool pool(params.engine.memory_budget);
        auto outcome = execute_task(task, pool);
        if (stage_ms) {
            stage_ms[0] = outcome.wall_ms;
            stage_ms[1] = outcome.read_ms;
            stage_ms[2] = outcome.rfi_ms;
            stage_ms[3] = outcome.dm_loop_ms;
            stage_ms[4] = outcome.cluster_ms;
            stage_ms[5] = outcome.write_ms;
        }
        *n_clusters = outcome.candidates;
        return PGB_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// execute_task's body (src/pipeline.cpp:61-119) on a file, returning the structured
// results instead of only the .cand text: the sorted file-level candidate list, the
// link_grid clusters (+ flat member ids), the (chunk, trial) skipped pairs and the
// .cand text.  Chunks are read synchronously (FilterbankReader::read_chunk; the
// prefetching reader returns identical chunks) so memory stays at one chunk.
int pgref_search_file(const char* path, const pgref_search_params* p, pgb_candidate** cands,
                      size_t* ncands, pgb_cluster** clusters, size_t* nclusters,
                      uint64_t** members, uint64_t** skipped /* pairs */, size_t* nskipped,
                      char** cand_text, size_t* cand_len, double* stage_ms /*[4] read rfi loop cluster*/) {
    try {
        SearchParams params;
        params.dm_lo = p->dm_lo;
        params.dm_hi = p->dm_hi;
        params.spacing = LinearSpacing{p->dm_step};
        params.engine.n_workers = p->n_workers;
        params.engine.detect_thresh = p->detect_thresh;
        params.engine.boxcar_max = p->boxcar_max;
        params.engine.radii = LinkRadii{p->radii.sep_time, p->radii.sep_dm_trials, p->radii.sep_width};
        if (p->parity) params.engine.max_in_flight = p->n_workers;
        params.baseline_len_s = p->baseline_len_s;
        params.nsamps_chunk = p->nsamps_chunk;
        params.rfi_narrowband = p->rfi_narrowband != 0;
        params.rfi_broadband = p->rfi_broadband != 0;
        params.k_sigma = p->k_sigma;
        params.k_mad = p->k_mad;
        auto task = create_task(path, params, "/dev/null");
        BufferPool pool(task.engine.memory_budget);
        FilterbankReader reader(path);
        using clk = std::chrono::steady_clock;
        auto ms = [](clk::time_point a) {
            return std::chrono::duration<double, std::milli>(clk::now() - a).count();
        };
        double st[4] = {0, 0, 0, 0};
        std::vector<Candidate> all;
        std::vector<uint64_t> sk;
        for (const auto& spec : task.chunks) {
            auto t0 = clk::now();
            Chunk chunk = reader.read_chunk(spec);
            st[0] += ms(t0);
            t0 = clk::now();
            RfiMask mask;
            mask.replacement = task.params.replacement;
            if (task.params.rfi_narrowband) mask.bad_channels = flag_narrowband(chunk, task.params.k_mad);
            if (task.params.rfi_broadband) mask.bad_samples = flag_broadband(chunk, task.params.k_sigma);
            if (!mask.bad_channels.empty() || !mask.bad_samples.empty()) apply_mask(chunk, mask);
            st[1] += ms(t0);
            t0 = clk::now();
            DmLoopResult r = run_dm_loop(chunk, task.plan, task.engine, pool);
            st[2] += ms(t0);
            all.insert(all.end(), r.candidates.begin(), r.candidates.end());
            for (auto t : r.skipped_trials) {
                sk.push_back(chunk.spec.index);
                sk.push_back(t);
            }
        }
        auto t0 = clk::now();
        std::sort(all.begin(), all.end(), [](const Candidate& a, const Candidate& b) {
            if (a.peak_sample != b.peak_sample) return a.peak_sample < b.peak_sample;
            if (a.dm_trial != b.dm_trial) return a.dm_trial < b.dm_trial;
            return a.width_index < b.width_index;
        });
        auto cl = link_grid(all, task.engine.radii);
        st[3] = ms(t0);
        if (stage_ms) std::memcpy(stage_ms, st, sizeof st);
        std::vector<pgb_candidate> out(all.size());
        if (!out.empty()) std::memcpy(out.data(), all.data(), out.size() * sizeof(Candidate));
        *cands = dup(out);
        *ncands = out.size();
        *skipped = dup(sk);
        *nskipped = sk.size() / 2;
        std::ostringstream os;
        write_candidates(cl, os);
        const std::string s = os.str();
        *cand_text = static_cast<char*>(std::malloc(s.size() + 1));
        std::memcpy(*cand_text, s.c_str(), s.size() + 1);
        *cand_len = s.size();
        return export_clusters(cl, clusters, nclusters, members);
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Chunk plan create_task would build (overlap = max_delay + boxcar_max,
// src/pipeline.cpp:50-57) and the baseline window it resolves (:22-28).
int pgref_create_task_plan(const char* path, const pgref_search_params* p, pgb_chunk_spec* out,
                           size_t cap, size_t* nchunks, uint64_t* baseline_window) {
    try {
        SearchParams params;
        params.dm_lo = p->dm_lo;
        params.dm_hi = p->dm_hi;
        params.spacing = LinearSpacing{p->dm_step};
        params.engine.boxcar_max = p->boxcar_max;
        params.baseline_len_s = p->baseline_len_s;
        params.nsamps_chunk = p->nsamps_chunk;
        auto task = create_task(path, params, "/dev/null");
        *nchunks = task.chunks.size();
        *baseline_window = task.engine.baseline_window;
        if (out) {
            if (cap < task.chunks.size()) throw std::invalid_argument("capacity");
            for (size_t k = 0; k < task.chunks.size(); ++k) {
                const auto& s = task.chunks[k];
                out[k] = {s.index, s.start_sample, s.length, s.overlap, s.valid_begin, s.valid_end};
            }
        }
        return PGB_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
