// Exact integer sweep with event replay for RFI-masked 8-bit chunks with local-mean rows
// (ablation library, PGB_RFI_HYB=1, tools/fp32_chain_model.py).
//
// The reference sums each output's channels in ascending order in fp32
// (/root/reference/proj/src/dedisp.cpp:146-160) over a chunk whose flagged rows carry
// float local means (src/rfi.cpp:115-139).  Here the flagged cells are staged as 0 and the
// SWAR integer accumulation of the u8 ring kernel runs unchanged; every output keeps its
// fp32 chain value s in shared memory, and
//   * a flagged cell v at channel c of output o (an "event") first merges o's integer
//     partial through c into s, then adds v: s = fl(merge(s, P) + v);
//   * at every flush of the packed accumulators the rest of each output's partial is
//     merged: s = merge(s, P).
// merge(s, n) -- s followed by integer cells summing to n -- is fl(s + n) when s is an
// integer or at most one binade is crossed, else (s + n) with the fraction of s rounded to
// the ulp of every binade crossed in order; it is exact for s >= 256 (no cell <= 255 can
// skip a binade there).  The first K channels run in a plain in-order fp32 head kernel;
// an output whose state is below 256 and not an integer when a merge crosses two binades
// sets `dirty` and the host recomputes the chunk on the fp32 path.
//
// Tile: 32 trials x 512 outputs (the states take 64 KB of shared memory), 16 warps, 8
// channels per stage through a 3-slot mbarrier ring; events of a stage are collected per
// lane while scanning the stage's exception rows and then processed lane-parallel.
#include <cstdio>
#include <cstdlib>

#include "mbarrier.cuh"
#include "pgb_internal.h"

namespace pgb {

namespace {

constexpr int Y_NT = 512;            // outputs per tile
constexpr int Y_NS = 3;              // ring slots
constexpr int Y_G = 8;               // channels per stage
constexpr int Y_TB = 32;             // trials per block
constexpr uint32_t Y_HEAD = 64;      // channels of the in-order fp32 head

struct YExc {
    uint32_t pos;  // flagged row - window start (bytes)
    float val;
};

size_t hyb_smem_bytes(uint32_t wmax) {
    return (size_t)Y_NS * Y_G * 4 * wmax           // ring [NS][G][4 copies][wmax]
           + (size_t)Y_NS * Y_G * Y_TB * 4         // offsets
           + (size_t)Y_NS * Y_G * 4                // exception counts (24 words: 8-byte aligned end)
           + (size_t)Y_NS * Y_G * HX_CAP * 8       // exception lists
           + (size_t)Y_TB * Y_NT * 4               // fp32 chain states
           + 2 * Y_NS * 8;                         // mbarriers
}

#ifdef PGB_ABLATIONS  // the kernels ship in the ablation library only
constexpr int Y_WORDS = Y_NT / 128;  // 4-byte words per lane per trial
constexpr int Y_TPW = 2;             // trials per warp
constexpr int Y_Q = 4;               // events queued per lane before they are processed

__device__ __forceinline__ uint32_t ymin(uint32_t v) {
    for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ uint32_t ymax(uint32_t v) {
    for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// dd_table_kernel for 512-output tiles
__global__ void hyb_table_kernel(const DedispLaunch p, uint2* __restrict__ win, uint32_t* __restrict__ off) {
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t blk = gw / p.nchans_pad, c = gw % p.nchans_pad;
    const uint32_t nblocks = (p.nrows + 31) / 32;
    if (blk >= nblocks) return;
    const uint32_t row0 = blk * 32, nrows_blk = min(32u, p.nrows - row0);
    const uint32_t row = row0 + min((uint32_t)lane, nrows_blk - 1);
    const uint32_t d = c < p.nchans ? (uint32_t)__ldg(p.delays_ct + (size_t)c * p.ntrials_plan + p.active[row]) : 0;
    const uint32_t dmin = ymin(d), dmax = ymax(d);
    const uint32_t a = dmin & ~15u;
    const uint32_t o = d - a;
    off[(size_t)gw * 32 + lane] = (o & 3) * p.wmax + (o >> 2) * 4;
    if (lane == 0) win[gw] = make_uint2(a, (((dmax - a) & ~3u) + Y_NT - 1) / 16 + 1);
}

// exact fp32 chain: state s (>= +0) followed by integer cells summing to n
__device__ __forceinline__ float chain_merge(float s, uint32_t n, bool& ok) {
    if (n == 0) return s;
    const float r = __fadd_rn(s, __uint2float_rn(n));  // n < 2^24: exact operand
    if (s == truncf(s)) return r;                       // integer state: every partial sum exact
    const int es = (int)(__float_as_uint(s) >> 23), er = (int)(__float_as_uint(r) >> 23);
    if (er - es <= 1) return r;                         // at most one binade crossed: one rounding
    if (s < 256.0f) {                                   // a cell may skip a binade: undecidable
        ok = false;
        return r;
    }
    const float a = truncf(s);
    float fr = __fsub_rn(s, a);                          // exact
    const float whole = __fadd_rn(a, __uint2float_rn(n));  // exact integer
    for (int e = es + 1;; ++e) {                        // e: biased exponent of the next binade
        const float lo = __int_as_float(e << 23);
        if ((double)whole + (double)fr < (double)lo) break;
        const float m = __fmul_rn(lo, 1.5f);            // ulp(m) = ulp of [lo, 2 lo)
        fr = __fsub_rn(__fadd_rn(fr, m), m);            // round the fraction to that ulp (RNE)
    }
    return __fadd_rn(whole, fr);                        // exact
}

// In-order fp32 head over channels [0, K): s = sum of the masked codes plus, at flagged
// rows, their float values (fl(s + 0) = s, so the pair is the reference's fl(s + v)).
__global__ void __launch_bounds__(256) hyb_head_kernel(const DedispLaunch p, const uint8_t* __restrict__ rows,
                                                       float* __restrict__ out, uint32_t K,
                                                       unsigned* __restrict__ dirty) {
    const uint32_t row = blockIdx.y;
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= p.ntiles * (uint32_t)Y_NT) return;
    const uint32_t trial = p.active[row];
    float s = 0.0f;
    for (uint32_t c = 0; c < K; ++c) {
        const uint32_t d = __ldg(p.delays_ct + (size_t)c * p.ntrials_plan + trial);
        const uint64_t r = (uint64_t)t + d;
        s = __fadd_rn(s, (float)rows[(size_t)c * p.rows_pitch + r]);
        if (r < p.xlen) {
            const uint32_t k0 = __ldg(p.xP + r);
            if (__ldg(p.xP + r + 1) != k0) s = __fadd_rn(s, __ldg(p.xF + (size_t)k0 * p.nchans + c));
        }
    }
    out[(size_t)row * p.out_pitch + t] = s;
    if (t < p.row_len[row] && s != truncf(s) && s < 256.0f) atomicOr(dirty, 1u);
}

template <int VPT>
__device__ __forceinline__ void hyb_tile(const DedispLaunch& p, const uint8_t* __restrict__ rows,
                                         float* __restrict__ out, unsigned* __restrict__ dirty,
                                         const uint32_t blk, const uint32_t tile) {
    constexpr int G = Y_G, NS = Y_NS, TB = Y_TB, TPW = Y_TPW, NW = DD_WARPS;
    constexpr uint32_t D = NS - 1;
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t W = p.wmax;
    uint8_t* buf = smem;                                                        // [NS][G][4][W]
    uint32_t* offs = reinterpret_cast<uint32_t*>(smem + (size_t)NS * G * 4 * W);  // [NS][G][TB]
    uint32_t* xcnt = offs + NS * G * TB;                                         // [NS][G]
    YExc* xl = reinterpret_cast<YExc*>(xcnt + NS * G);                            // [NS][G][HX_CAP]
    float* S = reinterpret_cast<float*>(xl + NS * G * HX_CAP);                   // [TB][Y_NT]
    uint64_t* full = reinterpret_cast<uint64_t*>(S + TB * Y_NT);                 // [NS]
    uint64_t* empty = full + NS;                                                 // [NS]

    const uint32_t row0 = blk * TB;
    const uint32_t nrows_blk = min((uint32_t)TB, p.nrows - row0);
    const uint64_t i0 = (uint64_t)tile * Y_NT;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t g_first = Y_HEAD / G;
    const uint32_t nst = p.nchans_pad / G - g_first;  // stages of this kernel
    constexpr int wpc = NW / G;
    const int my_cs = warp / wpc;
    const uint32_t my_t = (uint32_t)((warp % wpc) * 32 + lane);
    constexpr uint32_t vstride = (uint32_t)wpc * 32;
    const uint32_t* offtab = p.dd_off + (size_t)blk * p.nchans_pad * TB;
    const uint2* wintab = p.dd_win + (size_t)blk * p.nchans_pad;
    const uint8_t* rows_i0 = rows + i0;
    const bool offs_thread = (int)threadIdx.x < G * TB / 4;
    const bool xthread = my_t < (uint32_t)HX_CAP;

    // chain states after the head
    for (uint32_t idx = threadIdx.x; idx < (uint32_t)(TB * Y_NT / 4); idx += NW * 32) {
        const uint32_t r = idx / (Y_NT / 4), j4 = idx % (Y_NT / 4);
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (r < nrows_blk) v = reinterpret_cast<const float4*>(out + (size_t)(row0 + r) * p.out_pitch + i0)[j4];
        reinterpret_cast<float4*>(S)[idx] = v;
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            ring_init(full + s, NW);
            ring_init(empty + s, NW);
        }
    }
    __syncthreads();

    uint4 v0[VPT];
    uint32_t v1[VPT];
    uint4 ov = make_uint4(0, 0, 0, 0);
    uint32_t xr = 0, xn = 0;
    float xv = 0.0f;
    auto pref = [&](uint2 wv) {  // flagged rows before the window's first byte and its end
        uint2 pk = make_uint2(0, 0);
        if (xthread) {
            const uint64_t s = i0 + wv.x, e = s + 16ull * wv.y + 4;
            pk.x = __ldg(p.xP + min(s, p.xlen));
            pk.y = __ldg(p.xP + min(e, p.xlen));
        }
        return pk;
    };
    auto load_stage = [&](uint32_t k, uint2 wv, uint2 pk) {  // k: kernel stage index
        const uint32_t c = (g_first + k) * G + my_cs;
        const uint8_t* src = rows_i0 + (size_t)c * p.rows_pitch + wv.x;
#pragma unroll
        for (int q = 0; q < VPT; ++q) {
            const uint32_t vi = my_t + q * vstride;
            if (vi < wv.y) {
                v0[q] = __ldg(reinterpret_cast<const uint4*>(src + 16 * vi));
                v1[q] = __ldg(reinterpret_cast<const uint32_t*>(src + 16 * vi + 16));
            }
        }
        if (offs_thread) ov = __ldg(reinterpret_cast<const uint4*>(offtab + (size_t)(g_first + k) * G * TB) + threadIdx.x);
        if (xthread) {
            xn = c < p.nchans ? min(pk.y - pk.x, (uint32_t)HX_CAP) : 0u;
            if (my_t < xn) {
                const uint32_t q = pk.x + my_t;
                xr = (uint32_t)(__ldg(p.xR + q) - (i0 + wv.x));
                xv = __ldg(p.xF + (size_t)q * p.nchans + c);
            }
        }
    };
    auto store_stage = [&](int slot, uint2 wv) {
        uint8_t* base = buf + (size_t)((slot * G + my_cs) * 4) * W;
#pragma unroll
        for (int q = 0; q < VPT; ++q) {
            const uint32_t vi = my_t + q * vstride;
            if (vi < wv.y) {
                uint8_t* dst = base + 16 * vi;
                const uint32_t w[5] = {v0[q].x, v0[q].y, v0[q].z, v0[q].w, v1[q]};
                *reinterpret_cast<uint4*>(dst) = v0[q];
#pragma unroll
                for (int s = 1; s < 4; ++s) {
                    const uint32_t sel = (uint32_t)(s | (s + 1) << 4 | (s + 2) << 8 | (s + 3) << 12);
                    uint4 sh;
                    sh.x = __byte_perm(w[0], w[1], sel);
                    sh.y = __byte_perm(w[1], w[2], sel);
                    sh.z = __byte_perm(w[2], w[3], sel);
                    sh.w = __byte_perm(w[3], w[4], sel);
                    *reinterpret_cast<uint4*>(dst + (size_t)s * W) = sh;
                }
            }
        }
        if (offs_thread) reinterpret_cast<uint4*>(offs + slot * G * TB)[threadIdx.x] = ov;
        if (xthread) {
            if (my_t < xn) xl[(slot * G + my_cs) * HX_CAP + my_t] = YExc{xr, xv};
            if (my_t == 0) xcnt[slot * G + my_cs] = xn;
        }
        __syncwarp();
        if (lane == 0) ring_arrive(full + slot);
    };

    uint32_t E[TPW][Y_WORDS], H[TPW][Y_WORDS];
    const uint32_t one = p.mul24 >> 24;
#pragma unroll
    for (int u = 0; u < TPW; ++u)
#pragma unroll
        for (int m = 0; m < Y_WORDS; ++m) E[u][m] = H[u][m] = 0;

    auto valid = [&](int u, uint32_t j) {
        const uint32_t r = row0 + warp * TPW + u;
        return (uint32_t)(warp * TPW + u) < nrows_blk && i0 + j < p.row_len[r];
    };
    auto flush = [&]() {
#pragma unroll
        for (int u = 0; u < TPW; ++u) {
            float* srow = S + (warp * TPW + u) * Y_NT;
#pragma unroll
            for (int m = 0; m < Y_WORDS; ++m) {
                const uint32_t k = E[u][m];
                const uint32_t b1 = k & 0xffffu, b3 = k >> 16;
                const uint32_t r = H[u][m] - (b1 << 8) - (b3 << 24);  // B0 + 2^16 B2
                const uint32_t j = 4 * (lane + 32 * m);
                float4 s4 = *reinterpret_cast<float4*>(srow + j);
                bool ok = true;
                s4.x = chain_merge(s4.x, r & 0xffffu, ok);
                s4.y = chain_merge(s4.y, b1, ok);
                s4.z = chain_merge(s4.z, r >> 16, ok);
                s4.w = chain_merge(s4.w, b3, ok);
                *reinterpret_cast<float4*>(srow + j) = s4;
                if (!ok && valid(u, j)) atomicOr(dirty, 1u);  // (a longer output is valid only if j is)
                E[u][m] = H[u][m] = 0;
            }
        }
    };

    // one event: output j of trial u at stage channel cs, flagged value val
    auto event = [&](uint32_t ev, int slot, const uint32_t* offb, const uint8_t* bufb) {
        const uint32_t cs = ev & 7, e = (ev >> 3) & 15, u = (ev >> 7) & 1, j = ev >> 8;
        const uint32_t m = j >> 7, b = j & 3;
        uint32_t K = 0, T = 0;
#pragma unroll
        for (int uu = 0; uu < TPW; ++uu)
#pragma unroll
            for (int mm = 0; mm < Y_WORDS; ++mm)
                if (uu == (int)u && mm == (int)m) {
                    K = E[uu][mm];
                    T = H[uu][mm];
                }
        const uint32_t b1 = K & 0xffffu, b3 = K >> 16;
        const uint32_t r = T - (b1 << 8) - (b3 << 24);
        uint32_t P = b == 0 ? (r & 0xffffu) : b == 1 ? b1 : b == 2 ? (r >> 16) : b3;
        for (uint32_t c2 = cs + 1; c2 < (uint32_t)G; ++c2)  // the stage's later channels
            P -= bufb[(size_t)c2 * 4 * W + offb[c2 * TB + u] + 128 * m + b];
        float* sp = S + (warp * TPW + u) * Y_NT + j;
        bool ok = true;
        float s = chain_merge(*sp, P, ok);
        s = __fadd_rn(s, xl[(slot * G + cs) * HX_CAP + e].val);
        *sp = s;
        if (!ok && valid((int)u, j)) atomicOr(dirty, 1u);
        const uint32_t dT = P << (8 * b), dK = (b & 1) ? P << (16 * (b >> 1)) : 0u;
#pragma unroll
        for (int uu = 0; uu < TPW; ++uu)
#pragma unroll
            for (int mm = 0; mm < Y_WORDS; ++mm)
                if (uu == (int)u && mm == (int)m) {
                    E[uu][mm] -= dK;
                    H[uu][mm] -= dT;
                }
    };

    // prologue: kernel stages 0 .. D-1 into slots 0 .. D-1
    for (uint32_t k = 0; k < D && k < nst; ++k) {
        const uint2 w = __ldg(wintab + (g_first + k) * G + my_cs);
        load_stage(k, w, pref(w));
        store_stage((int)k, w);
    }
    uint2 wnext = nst > D ? __ldg(wintab + (size_t)(g_first + D) * G + my_cs) : make_uint2(0, 0);
    uint2 pknext = pref(wnext);
    const uint32_t stages_per_flush = DD_FLUSH_CH / G;
    int slot = 0, slot2 = (int)D;
    uint32_t ph = 0, ph_prev = 0;

    for (uint32_t k0 = 0; k0 < nst; k0 += stages_per_flush) {
        const uint32_t k1 = min(k0 + stages_per_flush, nst);
        for (uint32_t k = k0; k < k1; ++k) {
            const bool pre = k + D < nst;
            const uint2 wstage = wnext;
            if (pre) {
                load_stage(k + D, wstage, pknext);
                if (k + D + 1 < nst) wnext = __ldg(wintab + (size_t)(g_first + k + D + 1) * G + my_cs);
            }
            ring_wait(full + slot, ph);
            const uint32_t* offb = offs + slot * G * TB + warp * TPW;
            const uint8_t* bufb = buf + (size_t)slot * G * 4 * W + 4 * lane;
#pragma unroll
            for (int cs = 0; cs < G; cs += 2) {
#pragma unroll
                for (int u = 0; u < TPW; ++u) {
                    const uint8_t* s0 = bufb + (size_t)cs * 4 * W + offb[cs * TB + u];
                    const uint8_t* s1 = bufb + (size_t)(cs + 1) * 4 * W + offb[(cs + 1) * TB + u];
#pragma unroll
                    for (int m = 0; m < Y_WORDS; ++m) {
                        const uint32_t w0 = *reinterpret_cast<const uint32_t*>(s0 + 128 * m);
                        const uint32_t w1 = *reinterpret_cast<const uint32_t*>(s1 + 128 * m);
                        uint32_t h = H[u][m];
                        E[u][m] += __byte_perm(w0, 0u, 0x4341) + __byte_perm(w1, 0u, 0x4341);
                        asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(h) : "r"(w0), "r"(one));
                        asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(h) : "r"(w1), "r"(one));
                        H[u][m] = h;
                    }
                }
            }
            // events: scan the stage's flagged rows, queue this lane's, process lane-parallel
            {
                const uint32_t* xc = xcnt + slot * G;
                uint32_t q[Y_Q];
                int nq = 0;
                auto drain = [&]() {
#pragma unroll
                    for (int i = 0; i < Y_Q; ++i)
                        if (i < nq) event(q[i], slot, offb, bufb);
                    nq = 0;
                };
                for (int cs = 0; cs < G; ++cs) {
                    const uint32_t n = xc[cs];
                    if (n == 0) continue;
                    const YExc* xe = xl + (slot * G + cs) * HX_CAP;
                    uint32_t o[TPW];
#pragma unroll
                    for (int u = 0; u < TPW; ++u) {
                        const uint32_t off = offb[cs * TB + u];
                        const uint32_t qd = (off >= W) + (off >= 2 * W) + (off >= 3 * W);
                        o[u] = off - qd * W + qd;  // delay - window start
                    }
                    for (uint32_t e = 0; e < n; ++e) {
                        const uint32_t pos = xe[e].pos;
#pragma unroll
                        for (int u = 0; u < TPW; ++u) {
                            const uint32_t j = pos - o[u];
                            if (j < (uint32_t)Y_NT && (int)((j >> 2) & 31) == lane) {
                                if (nq == Y_Q) drain();
                                const uint32_t ev = (uint32_t)cs | e << 3 | (uint32_t)u << 7 | j << 8;
#pragma unroll
                                for (int i = 0; i < Y_Q; ++i)
                                    if (i == nq) q[i] = ev;
                                ++nq;
                            }
                        }
                    }
                }
                drain();
            }
            __syncwarp();
            if (lane == 0) ring_arrive(empty + slot);
            if (pre) {
                if (k + D + 1 < nst) pknext = pref(wnext);
                if (k >= 1) ring_wait(empty + slot2, ph_prev);  // slot2 last held stage k-1
                store_stage(slot2, wstage);
            }
            ph_prev = ph;
            if (++slot == NS) {
                slot = 0;
                ph ^= 1;
            }
            if (++slot2 == NS) slot2 = 0;
        }
        flush();
    }
    __syncthreads();  // every lane's states are final
    for (uint32_t idx = threadIdx.x; idx < (uint32_t)(TB * Y_NT / 4); idx += NW * 32) {
        const uint32_t r = idx / (Y_NT / 4), j4 = idx % (Y_NT / 4);
        if (r < nrows_blk)
            reinterpret_cast<float4*>(out + (size_t)(row0 + r) * p.out_pitch + i0)[j4] =
                reinterpret_cast<const float4*>(S)[idx];
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            ring_inval(full + s);
            ring_inval(empty + s);
        }
    }
}

template <int VPT>
__global__ void __launch_bounds__(DD_THREADS, 1)
    dedisp_hyb_kernel(const DedispLaunch p, const uint8_t* __restrict__ rows, float* __restrict__ out,
                      unsigned* __restrict__ dirty) {
    __shared__ uint32_t s_item;
    const uint32_t nblocks = (p.nrows + 31) / 32;
    const uint32_t items = nblocks * p.ntiles;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_item = atomicAdd(p.work_ctr, 1u);
        __syncthreads();
        const uint32_t item = s_item;
        if (item >= items) return;
        const uint32_t blk = item % nblocks, tile = item / nblocks;
        if ((uint64_t)tile * Y_NT >= p.blk_len[blk]) continue;
        hyb_tile<VPT>(p, rows, out, dirty, blk, tile);
    }
}
#endif

}  // namespace

uint32_t hyb_wmax(uint32_t spread) { return (uint32_t)((spread + Y_NT + 2 * 16 + 16 + 15) / 16 * 16); }
uint32_t hyb_tile_len() { return Y_NT; }
uint32_t hyb_head_channels() { return Y_HEAD; }
bool hyb_fits(uint32_t wmax) { return hyb_smem_bytes(wmax) <= 227 * 1024; }

void launch_dedisp_hyb(const DedispLaunch& p, const uint8_t* rows, float* out, unsigned* dirty, cudaStream_t st) {
#ifndef PGB_ABLATIONS
    (void)p, (void)rows, (void)out, (void)dirty, (void)st;
    raise(PGB_ERR_CONFIG, "the event-replay RFI kernel is in the ablation library only");
#else
    if (!p.dd_off || !p.work_ctr || !p.xP || p.nchans_pad < Y_HEAD + Y_G)
        raise(PGB_ERR_CONFIG, "event-replay dedispersion launch without its tables");
    {  // 512-output tile tables
        const uint64_t warps = (uint64_t)((p.nrows + 31) / 32) * p.nchans_pad;
        hyb_table_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(p, const_cast<uint2*>(p.dd_win),
                                                                             const_cast<uint32_t*>(p.dd_off));
    }
    PGB_CUDA(cudaMemsetAsync(dirty, 0, sizeof(unsigned), st));
    hyb_head_kernel<<<dim3((p.ntiles * Y_NT + 255) / 256, p.nrows), 256, 0, st>>>(p, rows, out, Y_HEAD, dirty);
    PGB_CUDA(cudaMemsetAsync(p.work_ctr, 0, sizeof(uint32_t), st));
    const size_t smem = hyb_smem_bytes(p.wmax);
    const uint32_t vstride = 32u * (DD_WARPS / Y_G);
    const int vpt = (int)((p.wmax / 16 + vstride - 1) / vstride);
    int dev = 0, nsm = 0;
    PGB_CUDA(cudaGetDevice(&dev));
    PGB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    static const bool which = getenv("PGB_DD_WHICH") != nullptr;
#define PGB_HYB(V_)                                                                                \
    if (vpt <= V_) {                                                                               \
        PGB_CUDA(cudaFuncSetAttribute(dedisp_hyb_kernel<V_>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                      (int)smem));                                                 \
        dedisp_hyb_kernel<V_><<<nsm, DD_THREADS, smem, st>>>(p, rows, out, dirty);                 \
        PGB_CUDA(cudaGetLastError());                                                              \
        if (which) fprintf(stderr, "pgb dedisp: hyb-ring G=8 VPT=%d\n", V_);                      \
        return;                                                                                    \
    }
    PGB_HYB(1) PGB_HYB(2) PGB_HYB(4)
#undef PGB_HYB
    raise(PGB_ERR_CONFIG, "no event-replay dedispersion kernel for this staging geometry");
#endif
}

}  // namespace pgb
