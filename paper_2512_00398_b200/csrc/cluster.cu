// Device candidate merging with link_grid semantics (src/cluster.cpp:99-146).
//
// The reference's output is a function of the connected components of the
// `linked` graph (:77-88), the representative order (:33-37 plus first-seen), and
// the final sort by the representative's (peak_sample, dm_trial, width_index)
// (:65-72).  The device version reproduces exactly that:
//   1. cell keys (peak / (sep_time*wmax_all), trial / sep_dm, widx / sep_width),
//      radix-sorted; every candidate scans the 27 neighbour cells by binary search
//      (any linked pair lies in the same or an adjacent cell, :106-108);
//   2. lock-free union-find (CAS hooking of the larger root under the smaller);
//   3. representative = atomicMax of (order-preserving snr bits << 32 | ~rank),
//      rank = position in the stable order by (peak_sample, dm_trial, input index)
//      -- exactly better_representative's tie chain with first-seen last;
//   4. extents by atomic min/max; members grouped by a stable sort on the root,
//      so each cluster's member ids are ascending like collect() (:39-73);
//   5. clusters sorted by the representative's packed (peak, trial, width) key.
#include <cub/device/device_radix_sort.cuh>

#include <cstdlib>

#include "pgb_internal.h"

namespace pgb {

namespace {

struct Radii {
    uint64_t sep_time;
    uint32_t sep_dm;
    uint32_t sep_w;
};

__device__ __forceinline__ uint32_t ord_f32(float f) {
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ uint64_t ord_f64(double d) {
    const uint64_t b = (uint64_t)__double_as_longlong(d);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double unord_f64(uint64_t u) {
    const uint64_t b = (u & 0x8000000000000000ull) ? (u & 0x7fffffffffffffffull) : ~u;
    return __longlong_as_double((long long)b);
}

__device__ __forceinline__ uint64_t cell_key(uint64_t kt, uint64_t kd, uint64_t kw) {
    return kt << 24 | kd << 5 | kw;
}

// Largest width (cell extent) and the key-packing limits every later stage relies on:
// dm_trial < 2^20, width_index < 32, peak_sample < 2^39 (sort keys peak<<25|trial<<5|width
// and peak<<20|trial); bad != 0 makes pgb_link_grid fail with PGB_ERR_ARGUMENT.
__global__ void wmax_kernel(const pgb_candidate* __restrict__ c, uint64_t n,
                            unsigned long long* wmax, unsigned long long* bad) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t w = 1;
    unsigned long long out = 0;
    if (i < n) {
        const pgb_candidate a = c[i];
        w = a.width_samples;
        out = (a.dm_trial >= (1u << 20)) | (a.width_index >= 32u) | (a.peak_sample >= (1ull << 39));
    }
    for (int o = 16; o; o >>= 1) w = max(w, (uint64_t)__shfl_xor_sync(0xffffffffu, w, o));
    out = __any_sync(0xffffffffu, out != 0);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(wmax, (unsigned long long)w);
        if (out) atomicOr(bad, 1ull);
    }
}

struct CellGeom {
    const unsigned long long* wmax;
    Radii r;
    __device__ uint64_t cell_t() const {
        const uint64_t ct = r.sep_time * (uint64_t)*wmax;
        return ct ? ct : 1;
    }
    __device__ uint32_t cell_dm() const { return r.sep_dm ? r.sep_dm : 1; }
    __device__ uint32_t cell_w() const { return r.sep_w ? r.sep_w : 1; }
};

__global__ void init_kernel(const pgb_candidate* __restrict__ c, uint64_t n, CellGeom g,
                            uint64_t* cell_keys, uint32_t* cell_idx, uint64_t* rank_keys,
                            uint32_t* rank_idx, uint32_t* parent, unsigned long long* repkey,
                            unsigned long long* cnt, unsigned long long* bmin,
                            unsigned long long* emax, unsigned long long* dlo,
                            unsigned long long* dhi) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const pgb_candidate a = c[i];
    cell_keys[i] = cell_key(a.peak_sample / g.cell_t(), a.dm_trial / g.cell_dm(),
                            a.width_index / g.cell_w());
    cell_idx[i] = (uint32_t)i;
    rank_keys[i] = a.peak_sample << 20 | a.dm_trial;  // stable sort keeps input order on ties
    rank_idx[i] = (uint32_t)i;
    parent[i] = (uint32_t)i;
    repkey[i] = 0;
    cnt[i] = 0;
    bmin[i] = ~0ull;
    emax[i] = 0;
    dlo[i] = ~0ull;
    dhi[i] = 0;
}

__device__ __forceinline__ bool linked(const pgb_candidate& a, const pgb_candidate& b,
                                       const Radii& r) {
    const uint64_t dt = a.peak_sample > b.peak_sample ? a.peak_sample - b.peak_sample
                                                      : b.peak_sample - a.peak_sample;
    const uint64_t wmax = a.width_samples > b.width_samples ? a.width_samples : b.width_samples;
    if (dt > r.sep_time * wmax) return false;
    const uint32_t ddm = a.dm_trial > b.dm_trial ? a.dm_trial - b.dm_trial : b.dm_trial - a.dm_trial;
    if (ddm > r.sep_dm) return false;
    const uint32_t dw = a.width_index > b.width_index ? a.width_index - b.width_index
                                                      : b.width_index - a.width_index;
    return dw <= r.sep_w;
}

__device__ uint32_t uf_find(uint32_t* parent, uint32_t x) {
    for (;;) {
        const uint32_t p = ((volatile uint32_t*)parent)[x];
        if (p == x) return x;
        const uint32_t gp = ((volatile uint32_t*)parent)[p];
        if (gp != p) ((volatile uint32_t*)parent)[x] = gp;  // path halving (ancestor only)
        x = gp;
    }
}

__device__ void uf_unite(uint32_t* parent, uint32_t a, uint32_t b) {
    for (;;) {
        a = uf_find(parent, a);
        b = uf_find(parent, b);
        if (a == b) return;
        if (a > b) {
            const uint32_t t = a;
            a = b;
            b = t;
        }
        const uint32_t old = atomicCAS(&parent[b], b, a);  // parent[max] = min, :26
        if (old == b) return;
        b = old;
    }
}

__device__ __forceinline__ uint64_t lower_bound(const uint64_t* k, uint64_t n, uint64_t key) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (k[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void link_kernel(const pgb_candidate* __restrict__ c, uint64_t n, CellGeom g,
                            const uint64_t* __restrict__ skeys, const uint32_t* __restrict__ sidx,
                            uint32_t* parent) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const pgb_candidate a = c[i];
    const int64_t kt = (int64_t)(a.peak_sample / g.cell_t());
    const int64_t kd = (int64_t)(a.dm_trial / g.cell_dm());
    const int64_t kw = (int64_t)(a.width_index / g.cell_w());
    for (int64_t dt = -1; dt <= 1; ++dt) {
        if (kt + dt < 0) continue;
        for (int64_t dd = -1; dd <= 1; ++dd) {
            if (kd + dd < 0) continue;
            for (int64_t dw = -1; dw <= 1; ++dw) {
                if (kw + dw < 0) continue;
                const uint64_t key = cell_key(kt + dt, kd + dd, kw + dw);
                uint64_t p = lower_bound(skeys, n, key);
                for (; p < n && skeys[p] == key; ++p) {
                    const uint32_t j = sidx[p];
                    if (j > i && linked(a, c[j], g.r)) uf_unite(parent, (uint32_t)i, j);
                }
            }
        }
    }
}

// Default linking: one warp per candidate, the lanes split the members of each of the
// 27 neighbour cells, the forest in global memory, CTAs across the whole GPU.  A bright
// pulse puts hundreds to thousands of mutually linked candidates into a few cells; with
// one thread per candidate walking them serially (below) a 1896-candidate config-A file
// took 2.35 ms, a one-CTA shared-memory forest did not help (the walks, not the loads,
// are serial).  Pairs are tested once (j > i); roots are compared before the box test.
__global__ void __launch_bounds__(256)
    link_warp_kernel(const pgb_candidate* __restrict__ c, uint64_t n, CellGeom g,
                     const uint64_t* __restrict__ skeys, const uint32_t* __restrict__ sidx,
                     uint32_t* parent) {
    const uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (i >= n) return;
    const pgb_candidate a = c[i];
    const int64_t kt = (int64_t)(a.peak_sample / g.cell_t());
    const int64_t kd = (int64_t)(a.dm_trial / g.cell_dm());
    const int64_t kw = (int64_t)(a.width_index / g.cell_w());
    for (int64_t dt = -1; dt <= 1; ++dt) {
        if (kt + dt < 0) continue;
        for (int64_t dd = -1; dd <= 1; ++dd) {
            if (kd + dd < 0) continue;
            for (int64_t dw = -1; dw <= 1; ++dw) {
                if (kw + dw < 0) continue;
                const uint64_t key = cell_key(kt + dt, kd + dd, kw + dw);
                const uint64_t p0 = lower_bound(skeys, n, key);
                for (uint64_t p = p0 + lane; p < n && skeys[p] == key; p += 32) {
                    const uint32_t j = sidx[p];
                    if (j <= i || uf_find(parent, (uint32_t)i) == uf_find(parent, j)) continue;
                    if (linked(a, c[j], g.r)) uf_unite(parent, (uint32_t)i, j);
                }
            }
        }
    }
}

// Small sets (n <= LINK_SMEM_MAX): the same linking with the union-find forest in
// shared memory, one CTA.  The global version's finds are chains of uncached L2 loads
// (~0.5 us each), which made a config-B link_grid (~600 candidates in a few dense
// cells) take ~1.9 ms; here a find is a few shared-memory loads.  The hooking rule
// (parent[max] = min) and therefore the forest's roots are the same.
constexpr uint32_t LINK_SMEM_MAX = 12288;

__device__ uint32_t suf_find(uint32_t* parent, uint32_t x) {
    for (;;) {
        const uint32_t p = ((volatile uint32_t*)parent)[x];
        if (p == x) return x;
        const uint32_t gp = ((volatile uint32_t*)parent)[p];
        if (gp != p) ((volatile uint32_t*)parent)[x] = gp;
        x = gp;
    }
}

__device__ void suf_unite(uint32_t* parent, uint32_t a, uint32_t b) {
    for (;;) {
        a = suf_find(parent, a);
        b = suf_find(parent, b);
        if (a == b) return;
        if (a > b) {
            const uint32_t t = a;
            a = b;
            b = t;
        }
        const uint32_t old = atomicCAS(&parent[b], b, a);
        if (old == b) return;
        b = old;
    }
}

__global__ void __launch_bounds__(1024)
    link_smem_kernel(const pgb_candidate* __restrict__ c, uint32_t n, CellGeom g,
                     const uint64_t* __restrict__ skeys, const uint32_t* __restrict__ sidx,
                     uint32_t* parent_out) {
    __shared__ uint32_t parent[LINK_SMEM_MAX];
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) parent[i] = i;
    __syncthreads();
    // one thread per candidate.  In a dense group (a bright pulse: hundreds of mutually
    // linked candidates) most pairs are already in one set, so the root comparison comes
    // first and the candidate record is only read for pairs in different sets.
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const pgb_candidate a = c[i];
        const int64_t kt = (int64_t)(a.peak_sample / g.cell_t());
        const int64_t kd = (int64_t)(a.dm_trial / g.cell_dm());
        const int64_t kw = (int64_t)(a.width_index / g.cell_w());
        for (int64_t dt = -1; dt <= 1; ++dt) {
            if (kt + dt < 0) continue;
            for (int64_t dd = -1; dd <= 1; ++dd) {
                if (kd + dd < 0) continue;
                for (int64_t dw = -1; dw <= 1; ++dw) {
                    if (kw + dw < 0) continue;
                    const uint64_t key = cell_key(kt + dt, kd + dd, kw + dw);
                    uint64_t p = lower_bound(skeys, n, key);
                    for (; p < n && skeys[p] == key; ++p) {
                        const uint32_t j = sidx[p];
                        if (j <= i || suf_find(parent, i) == suf_find(parent, j)) continue;
                        if (linked(a, c[j], g.r)) suf_unite(parent, i, j);
                    }
                }
            }
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) parent_out[i] = suf_find(parent, i);
}

// Up to LINK_SMEM2_MAX candidates: everything the linking reads -- the link fields, the
// sorted cell keys and indices, the forest -- is staged in shared memory (40 B per
// candidate), so the serial per-candidate cell walks (hundreds of members for a bright
// pulse) run at shared-memory latency instead of L1/L2 latency.
constexpr uint32_t LINK_SMEM2_MAX = 5120;

__global__ void __launch_bounds__(1024)
    link_smem2_kernel(const pgb_candidate* __restrict__ c, uint32_t n, CellGeom g,
                      const uint64_t* __restrict__ skeys, const uint32_t* __restrict__ sidx,
                      uint32_t* parent_out) {
    extern __shared__ __align__(16) unsigned char lsm[];
    uint64_t* s_peak = reinterpret_cast<uint64_t*>(lsm);
    uint64_t* s_ws = s_peak + n;
    uint64_t* s_key = s_ws + n;
    uint32_t* s_trial = reinterpret_cast<uint32_t*>(s_key + n);
    uint32_t* s_widx = s_trial + n;
    uint32_t* s_sidx = s_widx + n;
    uint32_t* parent = s_sidx + n;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const pgb_candidate a = c[i];
        s_peak[i] = a.peak_sample;
        s_ws[i] = a.width_samples;
        s_trial[i] = a.dm_trial;
        s_widx[i] = a.width_index;
        s_key[i] = skeys[i];
        s_sidx[i] = sidx[i];
        parent[i] = i;
    }
    __syncthreads();
    const uint64_t ct = g.cell_t();
    const uint32_t cd = g.cell_dm(), cw = g.cell_w();
    const Radii r = g.r;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint64_t pi = s_peak[i], wi = s_ws[i];
        const uint32_t ti = s_trial[i], xi = s_widx[i];
        const int64_t kt = (int64_t)(pi / ct), kd = (int64_t)(ti / cd), kw = (int64_t)(xi / cw);
        for (int64_t dt = -1; dt <= 1; ++dt) {
            if (kt + dt < 0) continue;
            for (int64_t dd = -1; dd <= 1; ++dd) {
                if (kd + dd < 0) continue;
                for (int64_t dw = -1; dw <= 1; ++dw) {
                    if (kw + dw < 0) continue;
                    const uint64_t key = cell_key(kt + dt, kd + dd, kw + dw);
                    uint32_t lo = 0, hi = n;
                    while (lo < hi) {
                        const uint32_t mid = (lo + hi) >> 1;
                        if (s_key[mid] < key) lo = mid + 1;
                        else hi = mid;
                    }
                    for (uint32_t p = lo; p < n && s_key[p] == key; ++p) {
                        const uint32_t j = s_sidx[p];
                        if (j <= i || suf_find(parent, i) == suf_find(parent, j)) continue;
                        // linked() on the staged fields (src/cluster.cpp:77-88)
                        const uint64_t pj = s_peak[j];
                        const uint64_t dtm = pi > pj ? pi - pj : pj - pi;
                        const uint64_t wm = wi > s_ws[j] ? wi : s_ws[j];
                        if (dtm > r.sep_time * wm) continue;
                        const uint32_t tj = s_trial[j], xj = s_widx[j];
                        if ((ti > tj ? ti - tj : tj - ti) > r.sep_dm) continue;
                        if ((xi > xj ? xi - xj : xj - xi) > r.sep_w) continue;
                        suf_unite(parent, i, j);
                    }
                }
            }
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) parent_out[i] = suf_find(parent, i);
}

__global__ void rank_kernel(const uint32_t* __restrict__ sorted_idx, uint64_t n, uint32_t* rank) {
    const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) rank[sorted_idx[p]] = (uint32_t)p;
}

__global__ void aggregate_kernel(const pgb_candidate* __restrict__ c, uint64_t n, uint32_t* parent,
                                 const uint32_t* __restrict__ rank, uint32_t* root_of,
                                 unsigned long long* repkey, unsigned long long* cnt,
                                 unsigned long long* bmin, unsigned long long* emax,
                                 unsigned long long* dlo, unsigned long long* dhi) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t r = uf_find(parent, (uint32_t)i);
    root_of[i] = r;
    const pgb_candidate a = c[i];
    atomicMax(&repkey[r], (unsigned long long)ord_f32(a.snr) << 32 | (0xffffffffu - rank[i]));
    atomicAdd(&cnt[r], 1ull);
    atomicMin(&bmin[r], (unsigned long long)a.begin_sample);
    atomicMax(&emax[r], (unsigned long long)a.end_sample);
    atomicMin(&dlo[r], (unsigned long long)ord_f64(a.dm));
    atomicMax(&dhi[r], (unsigned long long)ord_f64(a.dm));
}

__global__ void root_keys_kernel(const uint32_t* __restrict__ root_of, uint64_t n, uint32_t* keys,
                                 uint32_t* idx) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        keys[i] = root_of[i];
        idx[i] = (uint32_t)i;
    }
}

__global__ void segments_kernel(const uint32_t* __restrict__ sorted_roots,
                                const uint32_t* __restrict__ sorted_members, uint64_t n,
                                uint64_t* member_start, uint64_t* members_out,
                                uint32_t* cluster_roots, unsigned long long* ncl) {
    const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    members_out[p] = sorted_members[p];
    const uint32_t r = sorted_roots[p];
    if (p == 0 || sorted_roots[p - 1] != r) {
        member_start[r] = p;
        const unsigned long long k = atomicAdd(ncl, 1ull);
        cluster_roots[k] = r;
    }
}

__global__ void build_clusters_kernel(const pgb_candidate* __restrict__ c,
                                      const uint32_t* __restrict__ cluster_roots,
                                      const unsigned long long* __restrict__ ncl_p,
                                      const uint32_t* __restrict__ rank_to_idx,
                                      const unsigned long long* repkey,
                                      const unsigned long long* cnt, const unsigned long long* bmin,
                                      const unsigned long long* emax, const unsigned long long* dlo,
                                      const unsigned long long* dhi,
                                      const uint64_t* __restrict__ member_start, pgb_cluster* out,
                                      uint64_t* keys, uint32_t* idx) {
    const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= *ncl_p) return;
    const uint32_t r = cluster_roots[k];
    const uint32_t rank = 0xffffffffu - (uint32_t)(repkey[r] & 0xffffffffull);
    const pgb_candidate rep = c[rank_to_idx[rank]];
    pgb_cluster o;
    o.representative = rep;
    o.members = cnt[r];
    o.begin_sample = bmin[r];
    o.end_sample = emax[r];
    o.dm_lo = unord_f64(dlo[r]);
    o.dm_hi = unord_f64(dhi[r]);
    o.member_offset = member_start[r];
    out[k] = o;
    keys[k] = rep.peak_sample << 25 | (uint64_t)rep.dm_trial << 5 | rep.width_index;
    idx[k] = (uint32_t)k;
}

__global__ void gather_clusters_kernel(const pgb_cluster* __restrict__ in,
                                       const uint32_t* __restrict__ idx,
                                       const unsigned long long* __restrict__ ncl_p,
                                       pgb_cluster* __restrict__ out) {
    const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < *ncl_p) out[k] = in[idx[k]];
}

unsigned nblk(uint64_t n) { return (unsigned)((n + 255) / 256); }

template <typename T>
T* carve(char*& p, uint64_t count) {
    T* r = reinterpret_cast<T*>(p);
    p += ((count * sizeof(T) + 255) / 256) * 256;
    return r;
}

}  // namespace

void cluster_candidates(const pgb_candidate* cands, uint64_t n, const pgb_link_radii& radii,
                        DevBuf& scratch, DevBuf& out_clusters, DevBuf& out_members,
                        uint64_t* nclusters, cudaStream_t st, uint64_t* launches) {
    *nclusters = 0;
    if (n == 0) return;
    if (n >= (1ull << 31)) raise(PGB_ERR_ARGUMENT, "too many candidates to cluster (>= 2^31)");
    size_t sort_tmp = 0;
    {
        cub::DoubleBuffer<uint64_t> k(nullptr, nullptr);
        cub::DoubleBuffer<uint32_t> v(nullptr, nullptr);
        PGB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, k, v, (int)n));
        size_t t2 = 0;
        cub::DoubleBuffer<uint32_t> k2(nullptr, nullptr);
        PGB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t2, k2, v, (int)n));
        sort_tmp = std::max(sort_tmp, t2);
    }
    const uint64_t per = 4 * 8 + 6 * 4 + 7 * 8 + 8 + sizeof(pgb_cluster);
    scratch.reserve(n * per + 40 * 256 + sort_tmp + 4096);
    out_clusters.reserve(n * sizeof(pgb_cluster));
    out_members.reserve(n * sizeof(uint64_t));

    char* p = scratch.as<char>();
    auto* wmax = carve<unsigned long long>(p, 3);
    auto* ncl = wmax + 1;
    auto* bad = wmax + 2;
    auto* keys_a = carve<uint64_t>(p, n);
    auto* keys_b = carve<uint64_t>(p, n);
    auto* rkeys_a = carve<uint64_t>(p, n);
    auto* rkeys_b = carve<uint64_t>(p, n);
    auto* idx_a = carve<uint32_t>(p, n);
    auto* idx_b = carve<uint32_t>(p, n);
    auto* ridx_a = carve<uint32_t>(p, n);
    auto* ridx_b = carve<uint32_t>(p, n);
    auto* parent = carve<uint32_t>(p, n);
    auto* rank = carve<uint32_t>(p, n);
    auto* repkey = carve<unsigned long long>(p, n);
    auto* cnt = carve<unsigned long long>(p, n);
    auto* bmin = carve<unsigned long long>(p, n);
    auto* emax = carve<unsigned long long>(p, n);
    auto* dlo = carve<unsigned long long>(p, n);
    auto* dhi = carve<unsigned long long>(p, n);
    auto* member_start = carve<uint64_t>(p, n);
    auto* root_of = carve<uint32_t>(p, n);
    auto* croots = carve<uint32_t>(p, n);
    auto* cl_tmp = carve<pgb_cluster>(p, n);
    void* cub_tmp = carve<char>(p, sort_tmp);

    const Radii r{radii.sep_time, radii.sep_dm_trials, radii.sep_width};
    PGB_CUDA(cudaMemsetAsync(wmax, 0, 3 * sizeof(unsigned long long), st));
    wmax_kernel<<<nblk(n), 256, 0, st>>>(cands, n, wmax, bad);
    const CellGeom g{wmax, r};
    init_kernel<<<nblk(n), 256, 0, st>>>(cands, n, g, keys_a, idx_a, rkeys_a, ridx_a, parent,
                                         repkey, cnt, bmin, emax, dlo, dhi);
    // 1. cell sort, 2. linking
    cub::DoubleBuffer<uint64_t> ck(keys_a, keys_b);
    cub::DoubleBuffer<uint32_t> cv(idx_a, idx_b);
    PGB_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp, sort_tmp, ck, cv, (int)n, 0, 64, st));
    const int link_mode = [] {  // ablation: PGB_LINK_GLOBAL / PGB_LINK_SMEM1 / PGB_LINK_SMEM2
        if (pgb_ablation_env("PGB_LINK_GLOBAL")) return 2;
        if (pgb_ablation_env("PGB_LINK_SMEM1")) return 1;
        if (pgb_ablation_env("PGB_LINK_SMEM2")) return 3;
        return 0;
    }();
    if (link_mode == 0) {
        link_warp_kernel<<<(unsigned)((n * 32 + 255) / 256), 256, 0, st>>>(cands, n, g, ck.Current(),
                                                                            cv.Current(), parent);
    } else if (n <= LINK_SMEM2_MAX && link_mode == 3) {
        const size_t smem = (size_t)40 * n;
        PGB_CUDA(cudaFuncSetAttribute(link_smem2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(40 * LINK_SMEM2_MAX)));
        link_smem2_kernel<<<1, 1024, smem, st>>>(cands, (uint32_t)n, g, ck.Current(), cv.Current(), parent);
    } else if (n <= LINK_SMEM_MAX && link_mode != 2)
        link_smem_kernel<<<1, 1024, 0, st>>>(cands, (uint32_t)n, g, ck.Current(), cv.Current(), parent);
    else
        link_kernel<<<nblk(n), 256, 0, st>>>(cands, n, g, ck.Current(), cv.Current(), parent);
    // 3. ranks by (peak, trial, input index); representative and extents
    cub::DoubleBuffer<uint64_t> rk(rkeys_a, rkeys_b);
    cub::DoubleBuffer<uint32_t> rv(ridx_a, ridx_b);
    PGB_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp, sort_tmp, rk, rv, (int)n, 0, 64, st));
    const uint32_t* rank_to_idx = rv.Current();
    rank_kernel<<<nblk(n), 256, 0, st>>>(rank_to_idx, n, rank);
    aggregate_kernel<<<nblk(n), 256, 0, st>>>(cands, n, parent, rank, root_of, repkey, cnt, bmin,
                                              emax, dlo, dhi);
    // 4. members grouped by root (stable sort => ascending ids inside each cluster)
    uint32_t* kA = reinterpret_cast<uint32_t*>(keys_a);
    uint32_t* kB = reinterpret_cast<uint32_t*>(keys_b);
    root_keys_kernel<<<nblk(n), 256, 0, st>>>(root_of, n, kA, idx_a);
    cub::DoubleBuffer<uint32_t> mk(kA, kB);
    cub::DoubleBuffer<uint32_t> mv(idx_a, idx_b);
    PGB_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp, sort_tmp, mk, mv, (int)n, 0, 32, st));
    segments_kernel<<<nblk(n), 256, 0, st>>>(mk.Current(), mv.Current(), n, member_start,
                                             out_members.as<uint64_t>(), croots, ncl);
    // 5. cluster records keyed by the representative, sorted
    build_clusters_kernel<<<nblk(n), 256, 0, st>>>(cands, croots, ncl, rank_to_idx, repkey, cnt,
                                                   bmin, emax, dlo, dhi, member_start, cl_tmp,
                                                   keys_a, idx_a);
    PGB_CUDA(cudaGetLastError());
    unsigned long long h_cnt[2] = {0, 0};  // ncl, bad
    PGB_CUDA(cudaMemcpyAsync(h_cnt, ncl, sizeof h_cnt, cudaMemcpyDeviceToHost, st));
    PGB_CUDA(cudaStreamSynchronize(st));
    if (h_cnt[1])
        raise(PGB_ERR_ARGUMENT, "link_grid: candidate fields beyond the device key packing "
                                "(dm_trial < 2^20, width_index < 32, peak_sample < 2^39)");
    const unsigned long long h_ncl = h_cnt[0];
    *nclusters = h_ncl;
    cub::DoubleBuffer<uint64_t> sk(keys_a, keys_b);
    cub::DoubleBuffer<uint32_t> sv(idx_a, idx_b);
    if (h_ncl > 1)
        PGB_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp, sort_tmp, sk, sv, (int)h_ncl, 0, 64, st));
    gather_clusters_kernel<<<nblk(h_ncl), 256, 0, st>>>(cl_tmp, sv.Current(), ncl,
                                                        out_clusters.as<pgb_cluster>());
    PGB_CUDA(cudaGetLastError());
    if (launches) *launches += 12;
}

}  // namespace pgb
