// Drop-in replacement for the reference's cluster translation unit
// (/root/reference/proj/src/cluster.cpp): linked / link_reference / link_grid with
// the signatures of include/pulsegrid/cluster.hpp:33-43.  The grouping runs on the
// B200 (libpgb200 pgb_link_grid): same clusters, representatives, extents and
// member ids as the reference, clusters sorted by the representative's
// (peak_sample, dm_trial, width_index).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "pulsegrid/cluster.hpp"
#include "pulsegrid_b200.h"

namespace pulsegrid {

namespace {

struct ClusterCtx {
    pgb_context* ctx = nullptr;
    ~ClusterCtx() {
        if (ctx) pgb_destroy(ctx);
    }
};

pgb_context* cluster_ctx() {
    thread_local ClusterCtx c;
    if (!c.ctx) {
        int device = 0;
        if (const char* e = std::getenv("PULSEGRID_B200_DEVICE")) device = std::atoi(e);
        if (pgb_create(device, &c.ctx) != PGB_OK)
            throw error(std::string("libpgb200: ") + pgb_last_error());
    }
    return c.ctx;
}

std::vector<ClusterResult> device_link(std::span<const Candidate> cands, const LinkRadii& radii) {
    if (cands.empty()) return {};
    pgb_context* ctx = cluster_ctx();
    const pgb_link_radii r{radii.sep_time, radii.sep_dm_trials, radii.sep_width};
    std::size_t ncl = 0;
    if (pgb_link_grid(ctx, reinterpret_cast<const pgb_candidate*>(cands.data()), 0, cands.size(), &r,
                      &ncl) != PGB_OK)
        throw error(std::string("libpgb200: ") + pgb_last_error());
    std::vector<pgb_cluster> cl(ncl);
    std::vector<std::uint64_t> members(cands.size());
    if (pgb_fetch_clusters(ctx, cl.data(), ncl, members.data(), members.size()) != PGB_OK)
        throw error(std::string("libpgb200: ") + pgb_last_error());
    std::vector<ClusterResult> out(ncl);
    for (std::size_t k = 0; k < ncl; ++k) {
        static_assert(sizeof(Candidate) == sizeof(pgb_candidate));
        std::memcpy(static_cast<void*>(&out[k].representative), &cl[k].representative, sizeof(Candidate));
        out[k].members = cl[k].members;
        out[k].begin_sample = cl[k].begin_sample;
        out[k].end_sample = cl[k].end_sample;
        out[k].dm_lo = cl[k].dm_lo;
        out[k].dm_hi = cl[k].dm_hi;
        out[k].member_ids.assign(members.begin() + cl[k].member_offset,
                                 members.begin() + cl[k].member_offset + cl[k].members);
    }
    return out;
}

}  // namespace

bool linked(const Candidate& a, const Candidate& b, const LinkRadii& radii) {
    const std::uint64_t dt = a.peak_sample > b.peak_sample ? a.peak_sample - b.peak_sample
                                                           : b.peak_sample - a.peak_sample;
    const std::uint64_t wmax = std::max(a.width_samples, b.width_samples);
    if (dt > radii.sep_time * wmax) return false;
    const std::uint32_t ddm = a.dm_trial > b.dm_trial ? a.dm_trial - b.dm_trial : b.dm_trial - a.dm_trial;
    if (ddm > radii.sep_dm_trials) return false;
    const std::uint32_t dw = a.width_index > b.width_index ? a.width_index - b.width_index
                                                           : b.width_index - a.width_index;
    return dw <= radii.sep_width;
}

// The reference computes the same partition by an O(N^2) pair scan; its output
// equals link_grid's (cluster.hpp:29-41), so both go to the device.
std::vector<ClusterResult> link_reference(std::span<const Candidate> cands, const LinkRadii& radii) {
    return device_link(cands, radii);
}

std::vector<ClusterResult> link_grid(std::span<const Candidate> cands, const LinkRadii& radii) {
    return device_link(cands, radii);
}

}  // namespace pulsegrid
