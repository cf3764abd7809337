/*
 * pg_oracle.c -- plain-C restatement of the reference single-pulse search hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see pg_oracle.h).  Compiled with -ffp-contract=off;
 * every place where the reference build contracts a multiply-add (GCC's default
 * -ffp-contract=fast under -march=native, proj/CMakeLists.txt:12-17) is written as
 * an explicit fma() here, so the restatement is bit-identical to that build.
 * Parity pinned against the compiled reference (tests/test_oracle.py) and the
 * reference tests' known answers (tests/golden/).
 */
#include "pg_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define K_DISPERSION 4.148808e3 /* include/pulsegrid/dedisp.hpp:13 */
#define SCAN_BLOCK 64           /* include/pulsegrid/detect.hpp:219 (no effect on results) */

void pgo_free(void* p) { free(p); }

/* FilterbankHeader::channel_freq (filterbank.hpp:35): fch1 + foff*c, contracted. */
static double channel_freq(const pgb_header* h, uint32_t c) { return fma(h->foff, (double)c, h->fch1); }
/* max_freq / min_freq (src/filterbank.cpp:10-16) */
static double max_freq(const pgb_header* h) { return h->foff >= 0 ? channel_freq(h, h->nchans - 1) : h->fch1; }
static double min_freq(const pgb_header* h) { return h->foff >= 0 ? h->fch1 : channel_freq(h, h->nchans - 1); }

/* delay_samples, src/dedisp.cpp:13-18 */
int64_t pgo_delay_samples(double dm, const pgb_header* h, uint32_t channel) {
    const double f_ref = max_freq(h);
    const double f_c = channel_freq(h, channel);
    const double delay_s = K_DISPERSION * dm * (1.0 / (f_c * f_c) - 1.0 / (f_ref * f_ref));
    return (int64_t)floor(delay_s / h->tsamp + 0.5);
}

/* adaptive_dm_step, src/dedisp.cpp:20-26 */
double pgo_adaptive_dm_step(double tol, const pgb_header* h) {
    const double f_lo = min_freq(h);
    const double f_hi = max_freq(h);
    const double band = 1.0 / (f_lo * f_lo) - 1.0 / (f_hi * f_hi);
    if (band <= 0.0) return 0.0;
    return (tol - 1.0) * h->tsamp / (K_DISPERSION * band);
}

/* generate_dm_trials, src/dedisp.cpp:28-70 */
int pgo_generate_dm_trials(double dm_lo, double dm_hi, const pgb_header* h, int spacing,
                           double value, double* dms, int64_t* delays, size_t cap,
                           size_t* ntrials) {
    if (dm_lo < 0.0 || dm_hi < dm_lo) return PGB_ERR_INVALID_RANGE;
    double step;
    if (spacing == PGB_SPACING_LINEAR) {
        if (value <= 0.0) return PGB_ERR_INVALID_RANGE;
        step = value;
    } else {
        if (value <= 1.0) return PGB_ERR_INVALID_RANGE;
        step = pgo_adaptive_dm_step(value, h);
    }
    size_t n = 0;
    /* count first, then fill (two-call protocol like the product ABI) */
    for (int pass = 0; pass < 2; ++pass) {
        n = 0;
        if (step <= 0.0 || dm_hi == dm_lo) {
            if (pass && dms) dms[n] = dm_lo;
            ++n;
            if (dm_hi != dm_lo) {
                if (pass && dms) dms[n] = dm_hi;
                ++n;
            }
        } else {
            const double eps = step * 1e-9;
            for (size_t i = 0;; ++i) {
                const double dm = fma((double)i, step, dm_lo); /* dm_lo + i*step, contracted */
                if (dm >= dm_hi - eps) {
                    if (pass && dms) dms[n] = dm_hi;
                    ++n;
                    break;
                }
                if (pass && dms) dms[n] = dm;
                ++n;
            }
        }
        if (!pass) {
            *ntrials = n;
            if (!dms) return PGB_OK;
            if (cap < n) return PGB_ERR_ARGUMENT;
        }
    }
    if (delays)
        for (size_t t = 0; t < n; ++t)
            for (uint32_t c = 0; c < h->nchans; ++c)
                delays[t * h->nchans + c] = pgo_delay_samples(dms[t], h, c);
    return PGB_OK;
}

static int64_t trial_max_delay(const int64_t* d, uint32_t nchans) {
    int64_t m = d[0];
    for (uint32_t c = 1; c < nchans; ++c)
        if (d[c] > m) m = d[c];
    return m;
}

/* dedisperse (src/dedisp.cpp:200-218) == tests/oracles.hpp:16-26: fp32 adds from
 * 0.0f in ascending channel order. */
void pgo_dedisperse(const float* data, uint64_t length, uint32_t nchans, const int64_t* delays,
                    float* out) {
    const uint64_t n = length - (uint64_t)trial_max_delay(delays, nchans);
    for (uint64_t i = 0; i < n; ++i) {
        float acc = 0.0f;
        for (uint32_t c = 0; c < nchans; ++c)
            acc += data[(i + (uint64_t)delays[c]) * nchans + c];
        out[i] = acc;
    }
}

/* remove_baseline_into, src/detect.cpp:8-55 */
void pgo_remove_baseline(const float* x, uint64_t n, uint64_t window, float* out) {
    if (n == 0) return;
    if (window < 1) window = 1;
    if (window % 2 == 0) ++window;
    const uint64_t h = window / 2;
    if (h >= n - 1) { /* global mean path, :16-32 */
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        uint64_t i = 0;
        for (; i + 4 <= n; i += 4) {
            a0 += x[i + 0];
            a1 += x[i + 1];
            a2 += x[i + 2];
            a3 += x[i + 3];
        }
        for (; i < n; ++i) a0 += x[i];
        const float mean = (float)(((a0 + a1) + (a2 + a3)) / (double)n);
        for (uint64_t j = 0; j < n; ++j) out[j] = x[j] - mean;
        return;
    }
    double sum = 0.0;
    uint64_t count = n < h + 1 ? n : h + 1;
    for (uint64_t j = 0; j < count; ++j) sum += x[j];
    for (uint64_t i = 0; i < n; ++i) {
        const double inv = 1.0 / (double)count;
        out[i] = (float)fma(-sum, inv, (double)x[i]); /* :45, contracted to fnmadd */
        if (i + 1 + h < n) {
            sum += x[i + 1 + h];
            ++count;
        }
        if (i >= h) {
            sum -= x[i - h];
            --count;
        }
    }
}

/* sum_squares / sum_squares_cut, src/detect.cpp:67-108 (4 chains + tail into a0) */
static double sum_squares(const float* x, uint64_t n) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    uint64_t i = 0;
    for (; i + 4 <= n; i += 4) {
        a0 += (double)x[i + 0] * (double)x[i + 0];
        a1 += (double)x[i + 1] * (double)x[i + 1];
        a2 += (double)x[i + 2] * (double)x[i + 2];
        a3 += (double)x[i + 3] * (double)x[i + 3];
    }
    for (; i < n; ++i) a0 += (double)x[i] * (double)x[i];
    return (a0 + a1) + (a2 + a3);
}

static double sum_squares_cut(const float* x, uint64_t n, float cut, uint64_t* kept) {
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    uint64_t k = 0;
    uint64_t i = 0;
    for (; i + 4 <= n; i += 4)
        for (int j = 0; j < 4; ++j)
            if (fabsf(x[i + j]) <= cut) {
                a[j] += (double)x[i + j] * (double)x[i + j];
                ++k;
            }
    for (; i < n; ++i)
        if (fabsf(x[i]) <= cut) {
            a[0] += (double)x[i] * (double)x[i];
            ++k;
        }
    *kept = k;
    return (a[0] + a[1]) + (a[2] + a[3]);
}

/* normalize_to_sums, src/detect.cpp:193-214 (block maxima omitted: they only skip work) */
int pgo_normalize_to_sums(const float* x, uint64_t n, double* sums, double* rms_out) {
    if (n < 2) return PGB_ERR_DEGENERATE;
    const double sumsq = sum_squares(x, n);
    const double rms0 = sqrt(sumsq / (double)n);
    if (rms0 == 0.0) return PGB_ERR_DEGENERATE;
    const float cut = (float)(3.0 * rms0);
    uint64_t kept = 0;
    const double kept_sumsq = sum_squares_cut(x, n, cut, &kept);
    const double rms = kept ? sqrt(kept_sumsq / (double)kept) : rms0;
    if (rms == 0.0) return PGB_ERR_DEGENERATE;
    const float frms = (float)rms;
    for (uint64_t i = 0; i < n; ++i) sums[i] = (double)(x[i] / frms);
    *rms_out = rms;
    return PGB_OK;
}

typedef struct cand_vec {
    pgb_candidate* v;
    size_t n, cap;
} cand_vec;

static void push(cand_vec* cv, const pgb_candidate* c) {
    if (cv->n == cv->cap) {
        cv->cap = cv->cap ? 2 * cv->cap : 256;
        cv->v = (pgb_candidate*)realloc(cv->v, cv->cap * sizeof(pgb_candidate));
    }
    cv->v[cv->n++] = *c;
}

typedef struct peak_meta {
    uint64_t start_sample, valid_begin, valid_end;
    double tsamp, dm;
    uint32_t dm_trial;
    int drop_left, drop_right;
} peak_meta;

/* scan_peaks, src/detect.cpp:223-296: one candidate per maximal run of
 * sums[i]*scale > threshold, at the first maximum. */
static void scan_peaks(const double* sums, uint64_t n, double scale, double threshold,
                       uint32_t width_index, uint64_t width, const peak_meta* meta, cand_vec* out) {
    int in_run = 0;
    uint64_t run_begin = 0, peak_at = 0;
    double peak_val = 0.0;
    for (uint64_t i = 0; i <= n; ++i) {
        const int above = i < n && sums[i] * scale > threshold;
        const double v = i < n ? sums[i] * scale : 0.0;
        if (above) {
            if (!in_run) {
                in_run = 1;
                run_begin = i;
                peak_at = i;
                peak_val = v;
            } else if (v > peak_val) {
                peak_at = i;
                peak_val = v;
            }
        } else if (in_run) {
            const uint64_t run_end = i - 1;
            in_run = 0;
            if (meta->drop_left && run_begin == 0) continue;
            if (meta->drop_right && run_end == n - 1) continue;
            const uint64_t abs_peak = meta->start_sample + peak_at;
            if (abs_peak < meta->valid_begin || abs_peak >= meta->valid_end) continue;
            pgb_candidate c;
            memset(&c, 0, sizeof c);
            c.snr = (float)peak_val;
            c.peak_sample = abs_peak;
            c.time_s = (double)abs_peak * meta->tsamp;
            c.width_index = width_index;
            c.width_samples = width;
            c.dm_trial = meta->dm_trial;
            c.dm = meta->dm;
            c.begin_sample = meta->start_sample + run_begin;
            c.end_sample = meta->start_sample + run_end;
            push(out, &c);
        }
    }
}

static int cand_cmp(const void* pa, const void* pb) {
    const pgb_candidate* a = (const pgb_candidate*)pa;
    const pgb_candidate* b = (const pgb_candidate*)pb;
    if (a->peak_sample != b->peak_sample) return a->peak_sample < b->peak_sample ? -1 : 1;
    if (a->dm_trial != b->dm_trial) return a->dm_trial < b->dm_trial ? -1 : 1;
    if (a->width_index != b->width_index) return a->width_index < b->width_index ? -1 : 1;
    return 0;
}

void pgo_sort_candidates(pgb_candidate* c, size_t n) { qsort(c, n, sizeof *c, cand_cmp); }

/* run_dm_loop, src/engine.cpp:85-265, restated sequentially (results are
 * independent of n_workers and the in-flight limit in parity mode). */
int pgo_run_dm_loop_f32(const float* data, const pgb_chunk_spec* spec, uint32_t nchans,
                        const double* dms, const int64_t* delays, uint32_t ntrials,
                        const pgb_engine_config* cfg, pgb_candidate** cands, size_t* ncands,
                        uint64_t** skipped, size_t* nskipped) {
    if (cfg->n_workers < 1) return PGB_ERR_CONFIG;                                   /* :87 */
    if (cfg->boxcar_max < 1 || (cfg->boxcar_max & (cfg->boxcar_max - 1))) return PGB_ERR_CONFIG; /* :88-89 */
    const uint64_t length = spec->length;
    cand_vec out = {0, 0, 0};
    uint64_t* sk = (uint64_t*)malloc((ntrials + 1) * sizeof(uint64_t));
    size_t nsk = 0;
    float* series = (float*)malloc((length + 1) * sizeof(float));
    float* base = (float*)malloc((length + 1) * sizeof(float));
    double* sums = (double*)malloc((length + 1) * sizeof(double));
    for (uint32_t t = 0; t < ntrials; ++t) {
        const int64_t* d = delays + (size_t)t * nchans;
        const uint64_t span = (uint64_t)trial_max_delay(d, nchans);
        if (span >= length) { /* :114-115 */
            sk[nsk++] = t;
            continue;
        }
        const uint64_t n = length - span;
        pgo_dedisperse(data, length, nchans, d, series);
        const float* work = series;
        if (cfg->baseline_window > 0) { /* :161-168 */
            pgo_remove_baseline(series, n, cfg->baseline_window, base);
            work = base;
        }
        peak_meta meta; /* :170-178 */
        meta.start_sample = spec->start_sample;
        meta.tsamp = cfg->tsamp;
        meta.dm_trial = t;
        meta.dm = dms[t];
        meta.valid_begin = spec->valid_begin;
        meta.valid_end = spec->valid_end;
        meta.drop_left = spec->start_sample > 0;
        meta.drop_right = spec->overlap > 0;
        double rms;
        if (pgo_normalize_to_sums(work, n, sums, &rms) != PGB_OK) { /* :189-194 */
            sk[nsk++] = t;
            continue;
        }
        uint32_t widx = 0;
        for (uint64_t w = 1; w <= cfg->boxcar_max && w <= n; w <<= 1, ++widx) { /* :197-212 */
            const uint64_t m = n - w + 1;
            if (w > 1) /* boxcar_double_step, src/detect.cpp:216-221 */
                for (uint64_t i = 0; i < m; ++i) sums[i] += sums[i + w / 2];
            const double inv_sqrt_w = 1.0 / sqrt((double)w);
            scan_peaks(sums, m, inv_sqrt_w, (double)cfg->detect_thresh, widx, w, &meta, &out);
        }
    }
    free(series);
    free(base);
    free(sums);
    pgo_sort_candidates(out.v, out.n); /* :257-262 */
    *cands = out.v ? out.v : (pgb_candidate*)malloc(sizeof(pgb_candidate));
    *ncands = out.n;
    *skipped = sk; /* trials visited in ascending order: already sorted (:263) */
    *nskipped = nsk;
    return PGB_OK;
}

int pgo_run_dm_loop_u8(const uint8_t* data, const pgb_chunk_spec* spec, uint32_t nchans,
                       const double* dms, const int64_t* delays, uint32_t ntrials,
                       const pgb_engine_config* cfg, pgb_candidate** cands, size_t* ncands,
                       uint64_t** skipped, size_t* nskipped) {
    const size_t cells = (size_t)spec->length * nchans;
    float* f = (float*)malloc((cells + 1) * sizeof(float));
    for (size_t i = 0; i < cells; ++i) f[i] = (float)data[i]; /* src/filterbank.cpp:304-307 */
    const int rc = pgo_run_dm_loop_f32(f, spec, nchans, dms, delays, ntrials, cfg, cands, ncands,
                                       skipped, nskipped);
    free(f);
    return rc;
}

/* ---- link_grid (src/cluster.cpp:99-146) ------------------------------------ */

static size_t dsu_find(size_t* parent, size_t x) {
    while (parent[x] != x) {
        parent[x] = parent[parent[x]];
        x = parent[x];
    }
    return x;
}

static void dsu_unite(size_t* parent, size_t a, size_t b) { /* :22-27 */
    a = dsu_find(parent, a);
    b = dsu_find(parent, b);
    if (a != b) {
        if (a > b) parent[a] = b;
        else parent[b] = a;
    }
}

/* linked, src/cluster.cpp:77-88 */
static int linked(const pgb_candidate* a, const pgb_candidate* b, const pgb_link_radii* r) {
    const uint64_t dt = a->peak_sample > b->peak_sample ? a->peak_sample - b->peak_sample
                                                        : b->peak_sample - a->peak_sample;
    const uint64_t wmax = a->width_samples > b->width_samples ? a->width_samples : b->width_samples;
    if (dt > r->sep_time * wmax) return 0;
    const uint32_t ddm = a->dm_trial > b->dm_trial ? a->dm_trial - b->dm_trial : b->dm_trial - a->dm_trial;
    if (ddm > r->sep_dm_trials) return 0;
    const uint32_t dw = a->width_index > b->width_index ? a->width_index - b->width_index
                                                        : b->width_index - a->width_index;
    return dw <= r->sep_width;
}

/* better_representative, src/cluster.cpp:33-37 */
static int better(const pgb_candidate* a, const pgb_candidate* b) {
    if (a->snr != b->snr) return a->snr > b->snr;
    if (a->peak_sample != b->peak_sample) return a->peak_sample < b->peak_sample;
    return a->dm_trial < b->dm_trial;
}

static const pgb_candidate* g_sort_base;
static int by_peak(const void* pa, const void* pb) {
    const size_t a = *(const size_t*)pa, b = *(const size_t*)pb;
    const uint64_t x = g_sort_base[a].peak_sample, y = g_sort_base[b].peak_sample;
    if (x != y) return x < y ? -1 : 1;
    return a < b ? -1 : (a > b);
}

static int cluster_cmp(const void* pa, const void* pb) {
    const pgb_cluster* a = (const pgb_cluster*)pa;
    const pgb_cluster* b = (const pgb_cluster*)pb;
    const int c = cand_cmp(&a->representative, &b->representative);
    if (c) return c;
    return a->member_offset < b->member_offset ? -1 : (a->member_offset > b->member_offset);
}

int pgo_link_grid(const pgb_candidate* cands, size_t n, const pgb_link_radii* r,
                  pgb_cluster** clusters_out, size_t* nclusters, uint64_t** members_out) {
    *clusters_out = (pgb_cluster*)malloc((n + 1) * sizeof(pgb_cluster));
    *members_out = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
    *nclusters = 0;
    if (n == 0) return PGB_OK;
    /* Same linking closure as the grid (cell edge = maximal linking distance,
     * :102-108): any linked pair is within sep_time*wmax_all samples, so a scan
     * over candidates sorted by peak_sample finds every linked pair. */
    uint64_t wmax = 1;
    for (size_t i = 0; i < n; ++i)
        if (cands[i].width_samples > wmax) wmax = cands[i].width_samples;
    const uint64_t reach = r->sep_time * wmax;
    size_t* order = (size_t*)malloc(n * sizeof(size_t));
    size_t* parent = (size_t*)malloc(n * sizeof(size_t));
    for (size_t i = 0; i < n; ++i) order[i] = parent[i] = i;
    g_sort_base = cands;
    qsort(order, n, sizeof(size_t), by_peak);
    for (size_t a = 0; a < n; ++a)
        for (size_t b = a + 1; b < n; ++b) {
            const pgb_candidate* ca = &cands[order[a]];
            const pgb_candidate* cb = &cands[order[b]];
            if (cb->peak_sample - ca->peak_sample > reach) break;
            if (linked(ca, cb, r)) dsu_unite(parent, order[a], order[b]);
        }
    /* collect, :39-73: clusters in first-seen order, members ascending */
    size_t* root_to_cluster = (size_t*)malloc(n * sizeof(size_t));
    size_t* count = (size_t*)calloc(n + 1, sizeof(size_t));
    for (size_t i = 0; i < n; ++i) root_to_cluster[i] = (size_t)-1;
    size_t nc = 0;
    pgb_cluster* cs = *clusters_out;
    size_t* cluster_of = (size_t*)malloc(n * sizeof(size_t));
    for (size_t i = 0; i < n; ++i) {
        const size_t root = dsu_find(parent, i);
        size_t k = root_to_cluster[root];
        const pgb_candidate* c = &cands[i];
        if (k == (size_t)-1) {
            k = root_to_cluster[root] = nc++;
            cs[k].representative = *c;
            cs[k].members = 1;
            cs[k].begin_sample = c->begin_sample;
            cs[k].end_sample = c->end_sample;
            cs[k].dm_lo = cs[k].dm_hi = c->dm;
        } else {
            if (better(c, &cs[k].representative)) cs[k].representative = *c;
            cs[k].members++;
            if (c->begin_sample < cs[k].begin_sample) cs[k].begin_sample = c->begin_sample;
            if (c->end_sample > cs[k].end_sample) cs[k].end_sample = c->end_sample;
            if (c->dm < cs[k].dm_lo) cs[k].dm_lo = c->dm;
            if (c->dm > cs[k].dm_hi) cs[k].dm_hi = c->dm;
        }
        cluster_of[i] = k;
        count[k]++;
    }
    /* member offsets in first-seen cluster order, then sort clusters (:65-72) */
    size_t off = 0;
    for (size_t k = 0; k < nc; ++k) {
        cs[k].member_offset = off;
        off += count[k];
        count[k] = 0;
    }
    for (size_t i = 0; i < n; ++i) {
        const size_t k = cluster_of[i];
        (*members_out)[cs[k].member_offset + count[k]++] = i;
    }
    qsort(cs, nc, sizeof(pgb_cluster), cluster_cmp);
    *nclusters = nc;
    free(order);
    free(parent);
    free(root_to_cluster);
    free(count);
    free(cluster_of);
    return PGB_OK;
}

/* write_candidates, src/cluster_io.cpp:11-34: sorted by representative
 * (peak_sample, dm_trial); fixed printf format. */
static int cand_line_cmp(const void* pa, const void* pb) {
    const pgb_cluster* a = *(const pgb_cluster* const*)pa;
    const pgb_cluster* b = *(const pgb_cluster* const*)pb;
    if (a->representative.peak_sample != b->representative.peak_sample)
        return a->representative.peak_sample < b->representative.peak_sample ? -1 : 1;
    if (a->representative.dm_trial != b->representative.dm_trial)
        return a->representative.dm_trial < b->representative.dm_trial ? -1 : 1;
    return a < b ? -1 : (a > b);
}

size_t pgo_format_candidates(const pgb_cluster* clusters, size_t n, char* buf, size_t cap) {
    const pgb_cluster** order = (const pgb_cluster**)malloc((n + 1) * sizeof(*order));
    for (size_t k = 0; k < n; ++k) order[k] = &clusters[k];
    qsort(order, n, sizeof(*order), cand_line_cmp);
    size_t len = 0;
    char line[256];
    for (size_t k = 0; k < n; ++k) {
        const pgb_candidate* r = &order[k]->representative;
        const int w = snprintf(line, sizeof line, "%.2f\t%llu\t%.9f\t%u\t%u\t%.3f\t%llu\t%llu\t%llu\n",
                               (double)r->snr, (unsigned long long)r->peak_sample, r->time_s,
                               r->width_index, r->dm_trial, r->dm,
                               (unsigned long long)order[k]->members,
                               (unsigned long long)order[k]->begin_sample,
                               (unsigned long long)order[k]->end_sample);
        if (buf && len + (size_t)w < cap) memcpy(buf + len, line, (size_t)w + 1);
        len += (size_t)w;
    }
    free(order);
    return len;
}

/* plan_chunks, src/filterbank.cpp:239-272 */
int pgo_plan_chunks(uint64_t nsamples, uint64_t chunk_len, uint64_t overlap, pgb_chunk_spec* out,
                    size_t cap, size_t* n) {
    if (nsamples == 0 || chunk_len == 0 || overlap >= chunk_len) return PGB_ERR_INVALID_PLAN;
    size_t k = 0;
    if (chunk_len >= nsamples) {
        if (out && cap >= 1) out[0] = (pgb_chunk_spec){0, 0, nsamples, 0, 0, nsamples};
        *n = 1;
        return PGB_OK;
    }
    const uint64_t stride = chunk_len - overlap;
    for (uint64_t start = 0;; start += stride) {
        pgb_chunk_spec s;
        s.index = k;
        s.start_sample = start;
        s.valid_begin = start;
        const int last = start + chunk_len >= nsamples;
        s.length = last ? nsamples - start : chunk_len;
        s.overlap = last ? 0 : overlap;
        s.valid_end = last ? nsamples : start + stride;
        if (out && k < cap) out[k] = s;
        ++k;
        if (last) break;
    }
    *n = k;
    return PGB_OK;
}
