// Brute-force incoherent dedispersion for sm_100a.
//
// Semantics: out[t][i] = sum over channels c (ascending) of x[c][i + d_t(c)], the
// naive definition the reference's single-trial path computes
// (/root/reference/proj/src/dedisp.cpp:200-218, tests/oracles.hpp:16-26).
//
// Layout: the chunk is first transposed to channel-major rows (the reference's
// transpose_chunk, src/dedisp.cpp:116-131, but on 8-bit codes: 1 byte/cell).
// A CTA owns a tile of TB consecutive (active) trials x DD_NT consecutive
// outputs and streams the channels through shared memory G at a time,
// double-buffered.  For channel c the tile needs the window
// x[c][i0 + min_t d_t(c) .. i0 + max_t d_t(c) + DD_NT), staged once and read by all
// TB trials.
//
// u8 path (integer, exact): the staged window is stored as four byte-shifted
// copies so every (trial, channel) reads 4 consecutive samples with one aligned,
// bank-conflict-free 32-bit LDS.  The 4 bytes are accumulated SWAR-style in two
// 32-bit registers per word:
//     E += w & 0x00FF00FF          (samples 0 and 2 in u16 lanes; LOP3 + IADD3)
//     H += w >> 8  (= mad.hi(w, 2^24, H), samples 1..3 overlapped; fma pipe)
// which splits the adds across the ALU and FMA pipes.  Every 256 channels the
// lanes are decoded (B0 = E&0xFFFF, B2 = E>>16, t = H - (B2<<8), B1 = t&0xFFFF,
// B3 = t>>16; exact because each lane sum < 2^16 and H < 2^32) and added into the
// int32 output, which stays L2-resident between flushes.  Integer sums of 8-bit
// codes are exact, and for every north-star config (<= 8192 channels) they are
// below 2^24, so float(sum) equals the reference's in-order fp32 sum bit for bit.
//
// f32 path (non-integer chunks, e.g. after local-mean RFI replacement): the
// window is staged once with cp.async and every output accumulates the
// channels in ascending order with IEEE __fadd_rn, reproducing the reference's
// rounding sequence exactly.
#include <cuda_pipeline.h>

#include <cstdlib>
#include <type_traits>

#include <cstdio>

#include "mbarrier.cuh"
#include "pgb_internal.h"

namespace pgb {

namespace {

__device__ __forceinline__ uint32_t warp_min_u32(uint32_t v) {
    for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ uint32_t warp_max_u32(uint32_t v) {
    for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Per-stage bookkeeping.  Warp w < G owns channel slot w of a stage and lane r
// trial r of the block.  The delays of stage g+1 are fetched from global memory
// one full stage ahead (stage_delay) so their latency hides behind compute; the
// offsets (window start and per-trial smem offset) are then derived from the
// register copy (stage_offsets) right before the stage is staged.
template <int TB>
__device__ __forceinline__ uint32_t stage_delay(const DedispLaunch& p, uint32_t gi,
                                                const uint32_t* trial_ids) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t c = gi * p.g + warp;
    if (warp >= p.g || lane >= TB || c >= p.nchans) return 0;
    return (uint32_t)__ldg(p.delays_ct + (size_t)c * p.ntrials_plan + trial_ids[lane]);
}

template <bool U8, int TB>
__device__ __forceinline__ void stage_offsets(const DedispLaunch& p, uint32_t d, int b,
                                              uint64_t i0, uint64_t* abase, uint32_t* offs) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp >= p.g) return;
    const uint32_t dmin = warp_min_u32(lane < TB ? d : 0xffffffffu);
    const uint64_t align = U8 ? 16 : 4;  // 16-byte aligned global window start
    const uint64_t a = (i0 + dmin) & ~(align - 1);
    const int slot = b * p.g + warp;
    if (lane == 0) abase[slot] = a;
    if (lane < TB) {
        const uint32_t o = (uint32_t)(i0 + d - a);
        uint32_t off;
        if (U8) off = (uint32_t)((slot * 4 + (o & 3)) * p.wmax + (o >> 2) * 4);  // byte offset
        else off = (uint32_t)(slot * p.wmax + o);                               // float index
        offs[slot * TB + lane] = off;
    }
}

constexpr int U8_VPT = 4;  // max 16-byte vectors per thread per stage (host guarantees)

#ifdef PGB_ABLATIONS  // per-stage-offset kernel (HMODE ablations)
// HMODE selects how the odd samples are accumulated (ablation):
//   0: H += w >> 8 via __umulhi -> ptxas emits LEA.HI (ALU pipe)
//   1: H += hi(w * 2^24) via mad.hi (IMAD.HI on the FMA pipe; needs a 64-bit addend pair)
//   2: S += w as a 64-bit sum via mad.wide (IMAD.WIDE, FMA pipe); decode from S - E
//   3: as 0, but E accumulates with IMAD (FMA pipe) instead of IADD3 (ALU pipe)
template <int TPW, int HMODE>
__global__ void __launch_bounds__(DD_THREADS, 1)
    dedisp_u8_kernel(const DedispLaunch p, const uint8_t* __restrict__ rows,
                     int32_t* __restrict__ out, const uint32_t* __restrict__ blk_len) {
    constexpr int TB = DD_WARPS * TPW;
    extern __shared__ __align__(16) uint8_t smem[];
    const int G = p.g;
    const uint32_t W = p.wmax;  // bytes per copy
    uint8_t* buf = smem;                                              // [2][G][4][W]
    uint32_t* offs = reinterpret_cast<uint32_t*>(smem + (size_t)2 * G * 4 * W);  // [2][G][TB]
    uint64_t* abase = reinterpret_cast<uint64_t*>(offs + 2 * G * TB);            // [2][G]
    __shared__ uint32_t trial_ids[32];

    // trial blocks vary fastest across the grid so the CTAs in flight share time
    // tiles of the channel rows through L2
    const uint32_t blk = blockIdx.x;
    const uint32_t row0 = blk * TB;
    const uint32_t nrows_blk = min((uint32_t)TB, p.nrows - row0);
    const uint32_t tile = blockIdx.y + p.tile0;
    if (p.blk_first && tile < p.blk_first[blk]) return;  // shifted in from the previous chunk
    const uint64_t i0 = (uint64_t)tile * DD_NT;
    if (i0 >= blk_len[blk]) return;  // every trial of the block is shorter than this tile
    if (threadIdx.x < 32)
        trial_ids[threadIdx.x] = p.active[row0 + min((uint32_t)threadIdx.x, nrows_blk - 1)];
    __syncthreads();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t nstages = (p.nchans + G - 1) / G;
    // staging map without divisions: DD_WARPS / G warps per channel slot
    const int wpc = DD_WARPS / G;
    const int my_cs = warp / wpc;
    const uint32_t my_t = (uint32_t)((warp % wpc) * 32 + lane);
    const uint32_t vstride = (uint32_t)wpc * 32;
    const uint32_t vec_per_ch = W / 16;
    const uint32_t k24 = p.mul24;  // 1 << 24 from the host: keeps H on the FMA pipe (IMAD.HI)

    uint4 v0[U8_VPT];
    uint32_t v1[U8_VPT];

    auto load_stage = [&](uint32_t gi, int b) {
        const uint32_t c = min(gi * G + my_cs, p.nchans - 1);
        const uint8_t* src = rows + (size_t)c * p.rows_pitch + abase[b * G + my_cs];
#pragma unroll
        for (int k = 0; k < U8_VPT; ++k) {
            const uint32_t vi = my_t + k * vstride;
            if (vi < vec_per_ch) {
                v0[k] = __ldg(reinterpret_cast<const uint4*>(src + 16 * vi));
                v1[k] = __ldg(reinterpret_cast<const uint32_t*>(src + 16 * vi + 16));
            }
        }
    };
    auto store_stage = [&](int b) {
        uint8_t* base = buf + (size_t)((b * G + my_cs) * 4) * W;
#pragma unroll
        for (int k = 0; k < U8_VPT; ++k) {
            const uint32_t vi = my_t + k * vstride;
            if (vi < vec_per_ch) {
                uint8_t* dst = base + 16 * vi;
                const uint32_t w[5] = {v0[k].x, v0[k].y, v0[k].z, v0[k].w, v1[k]};
                *reinterpret_cast<uint4*>(dst) = v0[k];
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
    };

    using HT = typename std::conditional<HMODE == 2, unsigned long long, uint32_t>::type;
    uint32_t E[TPW][DD_WORDS];
    HT H[TPW][DD_WORDS];
    const uint32_t one = p.mul24 >> 24;  // 1, opaque to the compiler
#pragma unroll
    for (int u = 0; u < TPW; ++u)
#pragma unroll
        for (int m = 0; m < DD_WORDS; ++m) E[u][m] = H[u][m] = 0;
    bool first_flush = true;

    auto flush = [&]() {
#pragma unroll
        for (int u = 0; u < TPW; ++u) {
            const uint32_t r = warp * TPW + u;
            if (r < nrows_blk) {
                int32_t* dst = out + (size_t)(row0 + r) * p.out_pitch + i0;
#pragma unroll
                for (int m = 0; m < DD_WORDS; ++m) {
                    const uint32_t q = lane + 32 * m;
                    const uint32_t e = E[u][m];
                    const uint32_t b0 = e & 0xffffu, b2 = e >> 16;
                    uint32_t t;
                    if (HMODE == 2) {
                        const unsigned long long d = H[u][m] - e;  // 2^8 B1 + 2^24 B3
                        t = (uint32_t)((d >> 8) & 0xffffu) | (uint32_t)(d >> 24) << 16;
                    } else {
                        t = (uint32_t)H[u][m] - (b2 << 8);  // B1 + 2^16 B3
                    }
                    int4 val = make_int4((int)b0, (int)(t & 0xffffu), (int)b2, (int)(t >> 16));
                    int4* pd = reinterpret_cast<int4*>(dst + 4 * q);
                    if (!first_flush) {
                        const int4 old = *pd;
                        val.x += old.x;
                        val.y += old.y;
                        val.z += old.z;
                        val.w += old.w;
                    }
                    *pd = val;
                }
            }
#pragma unroll
            for (int m = 0; m < DD_WORDS; ++m) E[u][m] = H[u][m] = 0;
        }
        first_flush = false;
    };

    // prologue: stage 0 offsets and data; delays of stage 1 in flight
    uint32_t dnext = stage_delay<TB>(p, 0, trial_ids);
    stage_offsets<true, TB>(p, dnext, 0, i0, abase, offs);
    dnext = nstages > 1 ? stage_delay<TB>(p, 1, trial_ids) : 0;
    __syncthreads();
    load_stage(0, 0);
    store_stage(0);
    const uint32_t stages_per_flush = DD_FLUSH_CH / G;

    for (uint32_t gi = 0; gi < nstages; ++gi) {
        const int b = gi & 1;
        const bool more = gi + 1 < nstages;
        if (more) {
            stage_offsets<true, TB>(p, dnext, b ^ 1, i0, abase, offs);
            if (gi + 2 < nstages) dnext = stage_delay<TB>(p, gi + 2, trial_ids);
        }
        __syncthreads();
        if (more) load_stage(gi + 1, b ^ 1);

        const uint32_t c0 = gi * G;
        const int nch = (int)min((uint32_t)G, p.nchans - c0);
        const uint32_t* offb = offs + b * G * TB;
#pragma unroll 2
        for (int cs = 0; cs < nch; ++cs) {
#pragma unroll
            for (int u = 0; u < TPW; ++u) {
                const uint8_t* src = buf + offb[cs * TB + warp * TPW + u] + 4 * lane;
#pragma unroll
                for (int m = 0; m < DD_WORDS; ++m) {
                    const uint32_t w = *reinterpret_cast<const uint32_t*>(src + 128 * m);
                    if (HMODE == 3) {  // E on the FMA pipe (IMAD), H on the ALU pipe (LEA.HI)
                        uint32_t e = E[u][m];
                        asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(e) : "r"(w & 0x00ff00ffu), "r"(one));
                        E[u][m] = e;
                    } else {
                        E[u][m] += w & 0x00ff00ffu;  // samples 0 and 2 (LOP3 + IADD3, ALU pipe)
                    }
                    if (HMODE == 0 || HMODE == 3) {
                        H[u][m] += __umulhi(w, 1u << 24);
                    } else if (HMODE == 1) {
                        uint32_t h = (uint32_t)H[u][m];
                        asm("mad.hi.u32 %0, %1, %2, %0;" : "+r"(h) : "r"(w), "r"(k24));
                        H[u][m] = h;
                    } else {
                        unsigned long long h = H[u][m];
                        asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(h) : "r"(w), "r"(one));
                        H[u][m] = h;
                    }
                }
            }
        }
        if (more) store_stage(b ^ 1);
        if ((gi + 1) % stages_per_flush == 0 || !more) flush();
        __syncthreads();
    }
}

#endif  // PGB_ABLATIONS
// ---- mbarrier ring variant ---------------------------------------------------------
// Same tile, table, staging layout and SWAR accumulation as dedisp_u8_tab_kernel, but the
// CTA-wide barrier per stage is replaced by per-slot mbarriers over a 3-slot ring:
//   iteration g: issue the global loads of stage g+2 -> wait full[g%3] -> add stage g ->
//   arrive empty[g%3] -> wait empty of stage g-1 (the slot stage g+2 reuses) -> shift and
//   store stage g+2 -> arrive full[(g+2)%3].
// A warp only waits for the others to have finished stage g-1, so warps drift up to a
// stage apart instead of meeting at every stage (the barrier cost ~7 ms of 51 per
// config-B chunk: timing experiment "no barrier").
constexpr int RING_NS = 3;

#ifdef PGB_ABLATIONS
// Warp-drift stress (PGB_RING_JITTER=seed, ablation library only): a pseudo-random eighth of
// the (CTA, warp, stage, site) points sleep up to ~2 us, so warps reach the ring's full /
// empty handshakes in scrambled orders and up to the ring's depth apart.  The tests run it
// against the product path bit for bit (racecheck cannot model mbarrier ordering).
__device__ __forceinline__ void ring_jitter(uint32_t seed, uint32_t gi, uint32_t site) {
    if (!seed) return;
    uint32_t h = seed ^ (blockIdx.x * 0x9E3779B9u) ^ ((threadIdx.x >> 5) * 0x85EBCA6Bu) ^
                 (gi * 0xC2B2AE35u) ^ (site * 0x27D4EB2Fu);
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    h *= 0x297A2D39u;
    h ^= h >> 15;
    if ((h & 7) == 0) __nanosleep((h >> 16) & 2047);
}
#define PGB_RING_JITTER(gi, site) ring_jitter(p.jitter, (gi), (site))
#else
#define PGB_RING_JITTER(gi, site) ((void)0)
#endif

// MODE bits: 8 (default, G >= 2) = channel pairs, every word accumulated as K += PRMT(w0) +
// PRMT(w1) (one IADD3) and T += w0, w1 (two IMADs): 2.5 instructions per word-add, ALU 1.5 /
// FMA 1 (16 with 8: T by IADD3 on even words, ALU-heavier; ablation).  4 = odd words accumulate K += (w >> 8) & 0x00ff00ff (one PRMT) and
// T += w (IMAD), even words E += w & 0x00ff00ff (LOP3 + IMAD) and H += w >> 8 (LEA.HI): the
// ALU and FMA pipes (equal rate) then carry 3 + 3 instructions per word pair instead of
// 4 + 2.  Flush: B1 = K & 0xffff, B3 = K >> 16, T - 2^8 B1 - 2^24 B3 = B0 + 2^16 B2 (mod
// 2^32, exact for <= 256 channels).  Ablations: 1 = byte shifts of the staged copies on
// the FMA pipe (mul.hi + mad.lo funnel) instead of PRMT on the ALU pipe; 2 = per-(channel,
// trial) shared-memory addresses formed with IMAD (FMA pipe) instead of IADD (ALU pipe)
// One (trial block, time tile) of the ring kernel; the whole CTA calls it.
// NW = warps per CTA (16: two trials per warp; 32: one trial per warp, ablation).
template <int G, int VPT, int MODE, int NS = RING_NS, int NW = DD_WARPS>
__device__ __forceinline__ void ring_tile(const DedispLaunch& p, const uint8_t* __restrict__ rows,
                                          int32_t* __restrict__ out, const uint32_t* __restrict__ blk_len,
                                          const uint32_t blk, const uint32_t tile) {
    constexpr int TPW = 32 / NW;
    constexpr int TB = NW * TPW;
    static_assert(TB == 32, "table layout assumes 32-trial blocks");
    static_assert(NS == 2 || NS == 3, "ring depth");
    constexpr uint32_t D = NS - 1;  // stages loaded ahead
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t W = p.wmax;  // bytes per copy
    uint8_t* buf = smem;                                                           // [NS][G][4][W]
    uint32_t* offs = reinterpret_cast<uint32_t*>(smem + (size_t)NS * G * 4 * W);  // [NS][G][TB]
    uint64_t* full = reinterpret_cast<uint64_t*>(offs + NS * G * TB);              // [NS]
    uint64_t* empty = full + NS;                                                   // [NS]

    const uint32_t row0 = blk * TB;
    const uint32_t nrows_blk = min((uint32_t)TB, p.nrows - row0);
    const uint64_t i0 = (uint64_t)tile * DD_NT;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t nstages = p.nchans_pad / G;
    constexpr int wpc = NW / G;
    const int my_cs = warp / wpc;
    const uint32_t my_t = (uint32_t)((warp % wpc) * 32 + lane);
    constexpr uint32_t vstride = (uint32_t)wpc * 32;
    const uint32_t* offtab = p.dd_off + (size_t)blk * p.nchans_pad * TB;
    const uint2* wintab = p.dd_win + (size_t)blk * p.nchans_pad;
    const uint8_t* rows_i0 = rows + i0;
    constexpr bool kOffs = true;
    const bool offs_thread = (int)threadIdx.x < G * TB / 4;
    const uint32_t kshift[3] = {p.mul24, p.mul24 >> 8, p.mul24 >> 16};  // 2^24, 2^16, 2^8 (run time)

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

    auto load_stage = [&](uint32_t gi, uint2 wv) {
        const uint8_t* src = rows_i0 + (size_t)(gi * G + my_cs) * p.rows_pitch + wv.x;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            const uint32_t vi = my_t + k * vstride;
            if (vi < wv.y) {
                v0[k] = __ldg(reinterpret_cast<const uint4*>(src + 16 * vi));
                v1[k] = __ldg(reinterpret_cast<const uint32_t*>(src + 16 * vi + 16));
            }
        }
        if (kOffs && offs_thread)
            ov = __ldg(reinterpret_cast<const uint4*>(offtab + (size_t)gi * G * TB) + threadIdx.x);
    };
    auto store_stage = [&](int slot, uint2 wv) {
        uint8_t* base = buf + (size_t)((slot * G + my_cs) * 4) * W;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            const uint32_t vi = my_t + k * vstride;
            if (vi < wv.y) {
                uint8_t* dst = base + 16 * vi;
                const uint32_t w[5] = {v0[k].x, v0[k].y, v0[k].z, v0[k].w, v1[k]};
                *reinterpret_cast<uint4*>(dst) = v0[k];
#pragma unroll
                for (int s = 1; s < 4; ++s) {
                    uint4 sh;
                    if (MODE & 1) {  // (lo >> 8s) + hi * 2^(32-8s), both on the FMA pipe
                        const uint32_t km = kshift[s - 1];
                        uint32_t q[4];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            uint32_t t;
                            asm("mul.hi.u32 %0, %1, %2;" : "=r"(t) : "r"(w[j]), "r"(km));
                            asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(t) : "r"(w[j + 1]), "r"(km));
                            q[j] = t;
                        }
                        sh = make_uint4(q[0], q[1], q[2], q[3]);
                    } else {
                        const uint32_t sel = (uint32_t)(s | (s + 1) << 4 | (s + 2) << 8 | (s + 3) << 12);
                        sh.x = __byte_perm(w[0], w[1], sel);
                        sh.y = __byte_perm(w[1], w[2], sel);
                        sh.z = __byte_perm(w[2], w[3], sel);
                        sh.w = __byte_perm(w[3], w[4], sel);
                    }
                    *reinterpret_cast<uint4*>(dst + (size_t)s * W) = sh;
                }
            }
        }
        if (kOffs && offs_thread) reinterpret_cast<uint4*>(offs + slot * G * TB)[threadIdx.x] = ov;
        __syncwarp();
        if (lane == 0) ring_arrive(full + slot);
    };

    uint32_t E[TPW][DD_WORDS], H[TPW][DD_WORDS];
    const uint32_t one = p.mul24 >> 24;  // 1, opaque to the compiler (keeps E on IMAD)
#pragma unroll
    for (int u = 0; u < TPW; ++u)
#pragma unroll
        for (int m = 0; m < DD_WORDS; ++m) E[u][m] = H[u][m] = 0;
    bool first_flush = true;

    auto flush = [&]() {
#pragma unroll
        for (int u = 0; u < TPW; ++u) {
            const uint32_t r = warp * TPW + u;
            if (r < nrows_blk) {
                int32_t* dst = out + (size_t)(row0 + r) * p.out_pitch + i0;
#pragma unroll
                for (int m = 0; m < DD_WORDS; ++m) {
                    const uint32_t e = E[u][m];
                    int4 val;
                    if (((MODE & 4) && (m & 1)) || ((MODE & 8) && G >= 2)) {  // e = B1 + 2^16 B3, H = sum mod 2^32
                        const uint32_t b1 = e & 0xffffu, b3 = e >> 16;
                        const uint32_t r = H[u][m] - (b1 << 8) - (b3 << 24);  // B0 + 2^16 B2
                        val = make_int4((int)(r & 0xffffu), (int)b1, (int)(r >> 16), (int)b3);
                    } else {
                        const uint32_t b0 = e & 0xffffu, b2 = e >> 16;
                        const uint32_t t = H[u][m] - (b2 << 8);  // B1 + 2^16 B3
                        val = make_int4((int)b0, (int)(t & 0xffffu), (int)b2, (int)(t >> 16));
                    }
                    int4* pd = reinterpret_cast<int4*>(dst + 4 * (lane + 32 * m));
                    if (!first_flush) {
                        const int4 old = *pd;
                        val.x += old.x;
                        val.y += old.y;
                        val.z += old.z;
                        val.w += old.w;
                    }
                    *pd = val;
                }
            }
#pragma unroll
            for (int m = 0; m < DD_WORDS; ++m) E[u][m] = H[u][m] = 0;
        }
        first_flush = false;
    };

    // prologue: stages 0 .. D-1 into slots 0 .. D-1 (full phase 0 of each)
    {
        const uint2 w0 = __ldg(wintab + my_cs);
        load_stage(0, w0);
        store_stage(0, w0);
        if (D > 1 && nstages > 1) {
            const uint2 w1 = __ldg(wintab + G + my_cs);
            load_stage(1, w1);
            store_stage(1, w1);
        }
    }
    uint2 wnext = nstages > D ? __ldg(wintab + (size_t)D * G + my_cs) : make_uint2(0, 0);
    const uint32_t stages_per_flush = DD_FLUSH_CH / G;
    int slot = 0, slot2 = (int)D;     // gi % NS, (gi + D) % NS
    uint32_t ph = 0, ph_prev = 0;     // parity of stage gi's use of its slot; of stage gi-1's

    // flush periods outside, their stages inside: the accumulators stay in place across the
    // inner loop's back edge (a flush test inside one flat loop cost 16 register moves per stage)
    for (uint32_t g0 = 0; g0 < nstages; g0 += stages_per_flush) {
    const uint32_t g1 = min(g0 + stages_per_flush, nstages);
    for (uint32_t gi = g0; gi < g1; ++gi) {
        PGB_RING_JITTER(gi, 0);
        const bool pre = gi + D < nstages;
        const uint2 wstage = wnext;
        if (pre) {
            load_stage(gi + D, wstage);
            if (gi + D + 1 < nstages) wnext = __ldg(wintab + (size_t)(gi + D + 1) * G + my_cs);
        }
        ring_wait(full + slot, ph);
        const uint32_t* offb = offs + slot * G * TB + warp * TPW;
        const uint8_t* bufb = buf + (size_t)slot * G * 4 * W + 4 * lane;
        const uint32_t bufo = (uint32_t)slot * G * 4 * W + 4 * lane;  // byte offset of bufb in smem
        if constexpr ((MODE & 8) && G >= 2) {
            // channel pairs, every word as (K, T): K += PRMT(w0) + PRMT(w1) (IADD3), T += w0,
            // w1 (two IMADs; with MODE 16 one IADD3 on even words): 2.5 instructions per word
#pragma unroll
            for (int cs = 0; cs < G; cs += 2) {
#pragma unroll
                for (int u = 0; u < TPW; ++u) {
                    const uint8_t* s0 = bufb + (size_t)cs * 4 * W + offb[cs * TB + u];
                    const uint8_t* s1 = bufb + (size_t)(cs + 1) * 4 * W + offb[(cs + 1) * TB + u];
#pragma unroll
                    for (int m = 0; m < DD_WORDS; ++m) {
                        const uint32_t w0 = *reinterpret_cast<const uint32_t*>(s0 + 128 * m);
                        const uint32_t w1 = *reinterpret_cast<const uint32_t*>(s1 + 128 * m);
                        uint32_t h = H[u][m];
                        E[u][m] += __byte_perm(w0, 0u, 0x4341) + __byte_perm(w1, 0u, 0x4341);
                        if ((MODE & 16) && !(m & 1)) {
                            h += w0 + w1;
                        } else {
                            asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(h) : "r"(w0), "r"(one));
                            asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(h) : "r"(w1), "r"(one));
                        }
                        H[u][m] = h;
                    }
                }
            }
        } else
#pragma unroll
        for (int cs = 0; cs < G; ++cs) {
#pragma unroll
            for (int u = 0; u < TPW; ++u) {
                const uint8_t* src;
                if (MODE & 2)  // off * 1 + base: one IMAD (FMA pipe) instead of an IADD (ALU)
                    src = smem + (offb[cs * TB + u] * one + (bufo + (uint32_t)cs * 4 * W));
                else
                    src = bufb + (size_t)cs * 4 * W + offb[cs * TB + u];
#pragma unroll
                for (int m = 0; m < DD_WORDS; ++m) {
                    const uint32_t w = *reinterpret_cast<const uint32_t*>(src + 128 * m);
                    uint32_t e = E[u][m], h = H[u][m];
                    if ((MODE & 4) && (m & 1)) {
                        // K += bytes 1,3 in 16-bit lanes (one PRMT, ALU); T += w (IMAD, FMA pipe)
                        asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(e) : "r"(__byte_perm(w, 0u, 0x4341)), "r"(one));
                        asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(h) : "r"(w), "r"(one));
                    } else {
                        asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(e) : "r"(w & 0x00ff00ffu), "r"(one));
                        h += __umulhi(w, 1u << 24);  // LEA.HI, ALU pipe
                    }
                    E[u][m] = e;
                    H[u][m] = h;
                }
            }
        }
        __syncwarp();
        if (lane == 0) ring_arrive(empty + slot);
        PGB_RING_JITTER(gi, 1);
        if (pre) {
            // slot2 last held stage gi-1: every warp must be done adding it
            if (gi >= 1) ring_wait(empty + slot2, ph_prev);
            store_stage(slot2, wstage);
        }
        // advance ring indices: stage gi+1 uses slot (gi+1)%NS, use count (gi+1)/NS
        ph_prev = ph;
        if (++slot == NS) { slot = 0; ph ^= 1; }
        if (++slot2 == NS) slot2 = 0;
    }
    flush();
    }
    // the barriers are re-initialised for the next (block, tile) item: invalidate them
    // once every warp is past its last wait on them
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            ring_inval(full + s);
            ring_inval(empty + s);
        }
    }
}

#ifdef PGB_ABLATIONS  // grid-launched ring (the product launches the persistent one)
template <int G, int VPT, int MODE, int NS = RING_NS>
__global__ void __launch_bounds__(DD_THREADS, 1)
    dedisp_u8_ring_kernel(const DedispLaunch p, const uint8_t* __restrict__ rows,
                          int32_t* __restrict__ out, const uint32_t* __restrict__ blk_len) {
    const uint32_t blk = blockIdx.x;
    const uint32_t tile = blockIdx.y + p.tile0;
    if (p.blk_first && tile < p.blk_first[blk]) return;  // shifted in from the previous chunk
    if ((uint64_t)tile * DD_NT >= blk_len[blk]) return;
    ring_tile<G, VPT, MODE, NS>(p, rows, out, blk_len, blk, tile);
}

#endif  // PGB_ABLATIONS
// Persistent variant: one CTA per SM takes (block, tile) items from a counter in the
// grid's order (blocks fastest), so the last wave is not quantised to whole CTAs of a
// 7-55-wave grid (the tail is ~1 % of a launch with 8192 CTAs, several % with 1024).
template <int G, int VPT, int NS = RING_NS, int MODE = 0, int NW = DD_WARPS>
__global__ void __launch_bounds__(NW * 32, 1)
    dedisp_u8_ring_persist_kernel(const DedispLaunch p, const uint8_t* __restrict__ rows,
                                  int32_t* __restrict__ out, const uint32_t* __restrict__ blk_len) {
    __shared__ uint32_t s_item;
    const uint32_t nblocks = (p.nrows + 31) / 32;
    const uint32_t items = nblocks * (p.ntiles - p.tile0);
    for (;;) {
        __syncthreads();  // every warp is done with the previous item (and with s_item)
        if (threadIdx.x == 0) s_item = atomicAdd(p.work_ctr, 1u);
        __syncthreads();
        const uint32_t item = s_item;
        if (item >= items) return;
        const uint32_t blk = item % nblocks, tile = p.tile0 + item / nblocks;
        if (p.blk_first && tile < p.blk_first[blk]) continue;
        if ((uint64_t)tile * DD_NT >= blk_len[blk]) continue;
        ring_tile<G, VPT, MODE, NS, NW>(p, rows, out, blk_len, blk, tile);
    }
}

#ifdef PGB_ABLATIONS
// Two CTAs per SM (PGB_DD_2CTA=1): the same ring tile capped at 64 registers so 32 warps
// share an SM (latency hiding) -- the stage width is halved to fit two rings in shared memory.
template <int G, int VPT>
__global__ void __launch_bounds__(DD_THREADS, 2)
    dedisp_u8_ring_persist2_kernel(const DedispLaunch p, const uint8_t* __restrict__ rows,
                                   int32_t* __restrict__ out, const uint32_t* __restrict__ blk_len) {
    __shared__ uint32_t s_item;
    const uint32_t nblocks = (p.nrows + 31) / 32;
    const uint32_t items = nblocks * (p.ntiles - p.tile0);
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_item = atomicAdd(p.work_ctr, 1u);
        __syncthreads();
        const uint32_t item = s_item;
        if (item >= items) return;
        const uint32_t blk = item % nblocks, tile = p.tile0 + item / nblocks;
        if (p.blk_first && tile < p.blk_first[blk]) continue;
        if ((uint64_t)tile * DD_NT >= blk_len[blk]) continue;
        ring_tile<G, VPT, 8, RING_NS, DD_WARPS>(p, rows, out, blk_len, blk, tile);
    }
}
#endif

// Tile-independent staging geometry of the u8 kernel, one warp per (trial block,
// channel): the window of channel c for a block starts at i0 + (min_t d_t(c) & ~15)
// (i0 is a multiple of DD_NT, so 16-byte aligned) and trial t reads it at
// o_t = d_t(c) - start, i.e. at byte (o_t & 3) * W + (o_t >> 2) * 4 of the channel's
// 4-copy slot.  Vectors: enough 16-byte groups for the furthest trial's 1024 bytes.
__global__ void dd_table_kernel(const DedispLaunch p, uint2* __restrict__ win, uint32_t* __restrict__ off) {
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t blk = gw / p.nchans_pad, c = gw % p.nchans_pad;
    const uint32_t nblocks = (p.nrows + 31) / 32;
    if (blk >= nblocks) return;
    const uint32_t row0 = blk * 32, nrows_blk = min(32u, p.nrows - row0);
    const uint32_t row = row0 + min((uint32_t)lane, nrows_blk - 1);
    // channels past nchans are zero rows (the kernel always runs whole 8-channel groups)
    const uint32_t d = c < p.nchans ? (uint32_t)__ldg(p.delays_ct + (size_t)c * p.ntrials_plan + p.active[row]) : 0;
    const uint32_t dmin = warp_min_u32(d), dmax = warp_max_u32(d);
    const uint32_t a = dmin & ~15u;
    const uint32_t o = d - a;
    off[(size_t)gw * 32 + lane] = (o & 3) * p.wmax + (o >> 2) * 4;
    if (lane == 0)
        win[gw] = make_uint2(a, (((dmax - a) & ~3u) + DD_NT - 1) / 16 + 1);
}

#ifdef PGB_ABLATIONS  // CTA-barrier table kernel (SF ablations)
// Table-driven u8 kernel (default).  Same tile, staging layout and SWAR accumulation as
// dedisp_u8_kernel<.., 3>, but the per-stage offsets come from dd_table_kernel:
//   * the per-trial offsets of stage g+1 are copied into shared memory with cp.async
//     while stage g computes (no per-stage delay loads, shuffles or offset math);
//   * each channel stages only its own window (min..max delay of the block + 1024),
//     not the widest channel's;
//   * one barrier per stage;
//   * G (channels per stage) and VPT (16-byte vectors per staging thread) are compile
//     time and the channel rows are padded with zero rows to a multiple of 8, so a
//     stage is straight-line code (no loop-carried register shuffles, no dead
//     predicated loads).
template <int G, int VPT, int SF>
__global__ void __launch_bounds__(DD_THREADS, 1)
    dedisp_u8_tab_kernel(const DedispLaunch p, const uint8_t* __restrict__ rows,
                         int32_t* __restrict__ out, const uint32_t* __restrict__ blk_len) {
    // timing experiments (builds with -DPGB_DD_EXPERIMENTS only; results are wrong):
    // 4 = no adds, 8 = no staging, 16 = no flush, 32 = no barrier
    constexpr int XP = SF & ~3;
    constexpr int TPW = 2;
    constexpr int TB = DD_WARPS * TPW;
    static_assert(TB == 32, "table layout assumes 32-trial blocks");
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t W = p.wmax;  // bytes per copy
    uint8_t* buf = smem;                                                          // [2][G][4][W]
    uint32_t* offs = reinterpret_cast<uint32_t*>(smem + (size_t)2 * G * 4 * W);  // [2][G][TB]

    const uint32_t blk = blockIdx.x;
    const uint32_t row0 = blk * TB;
    const uint32_t nrows_blk = min((uint32_t)TB, p.nrows - row0);
    const uint32_t tile = blockIdx.y + p.tile0;
    if (p.blk_first && tile < p.blk_first[blk]) return;  // shifted in from the previous chunk
    const uint64_t i0 = (uint64_t)tile * DD_NT;
    if (i0 >= blk_len[blk]) return;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t nstages = p.nchans_pad / G;
    constexpr int wpc = DD_WARPS / G;
    const int my_cs = warp / wpc;
    const uint32_t my_t = (uint32_t)((warp % wpc) * 32 + lane);
    constexpr uint32_t vstride = (uint32_t)wpc * 32;
    const uint32_t* offtab = p.dd_off + (size_t)blk * p.nchans_pad * TB;
    const uint2* wintab = p.dd_win + (size_t)blk * p.nchans_pad;
    const uint8_t* rows_i0 = rows + i0;
    const uint32_t kshift[3] = {p.mul24, p.mul24 >> 8, p.mul24 >> 16};  // 2^24, 2^16, 2^8 (run time)

    uint4 v0[VPT];
    uint32_t v1[VPT];

    auto fetch_offs = [&](uint32_t gi, int b) {
        if ((int)threadIdx.x < G * TB / 4)
            __pipeline_memcpy_async(offs + b * G * TB + 4 * threadIdx.x,
                                    offtab + (size_t)gi * G * TB + 4 * threadIdx.x, 16);
        __pipeline_commit();
    };
    auto load_stage = [&](uint32_t gi, uint2 wv) {
        const uint8_t* src = rows_i0 + (size_t)(gi * G + my_cs) * p.rows_pitch + wv.x;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            const uint32_t vi = my_t + k * vstride;
            if (vi < wv.y) {
                v0[k] = __ldg(reinterpret_cast<const uint4*>(src + 16 * vi));
                v1[k] = __ldg(reinterpret_cast<const uint32_t*>(src + 16 * vi + 16));
            }
        }
    };
    auto store_stage = [&](int b, uint2 wv) {
        uint8_t* base = buf + (size_t)((b * G + my_cs) * 4) * W;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            const uint32_t vi = my_t + k * vstride;
            if (vi < wv.y) {
                uint8_t* dst = base + 16 * vi;
                const uint32_t w[5] = {v0[k].x, v0[k].y, v0[k].z, v0[k].w, v1[k]};
                *reinterpret_cast<uint4*>(dst) = v0[k];
#pragma unroll
                for (int s = 1; s < 4; ++s) {
                    uint4 sh;
                    if (SF & 1) {  // funnel shift on the FMA pipe: (lo >> 8s) + hi * 2^(32-8s)
                        const uint32_t k = kshift[s - 1];
                        uint32_t q[4];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            uint32_t t;
                            asm("mul.hi.u32 %0, %1, %2;" : "=r"(t) : "r"(w[j]), "r"(k));
                            asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(t) : "r"(w[j + 1]), "r"(k));
                            q[j] = t;
                        }
                        sh = make_uint4(q[0], q[1], q[2], q[3]);
                    } else {
                        const uint32_t sel = (uint32_t)(s | (s + 1) << 4 | (s + 2) << 8 | (s + 3) << 12);
                        sh.x = __byte_perm(w[0], w[1], sel);
                        sh.y = __byte_perm(w[1], w[2], sel);
                        sh.z = __byte_perm(w[2], w[3], sel);
                        sh.w = __byte_perm(w[3], w[4], sel);
                    }
                    *reinterpret_cast<uint4*>(dst + (size_t)s * W) = sh;
                }
            }
        }
    };

    uint32_t E[TPW][DD_WORDS], H[TPW][DD_WORDS];
    const uint32_t one = p.mul24 >> 24;  // 1, opaque to the compiler (keeps E on IMAD)
#pragma unroll
    for (int u = 0; u < TPW; ++u)
#pragma unroll
        for (int m = 0; m < DD_WORDS; ++m) E[u][m] = H[u][m] = 0;
    bool first_flush = true;

    auto flush = [&]() {
#pragma unroll
        for (int u = 0; u < TPW; ++u) {
            const uint32_t r = warp * TPW + u;
            if (r < nrows_blk) {
                int32_t* dst = out + (size_t)(row0 + r) * p.out_pitch + i0;
#pragma unroll
                for (int m = 0; m < DD_WORDS; ++m) {
                    const uint32_t e = E[u][m];
                    const uint32_t b0 = e & 0xffffu, b2 = e >> 16;
                    const uint32_t t = H[u][m] - (b2 << 8);  // B1 + 2^16 B3
                    int4 val = make_int4((int)b0, (int)(t & 0xffffu), (int)b2, (int)(t >> 16));
                    int4* pd = reinterpret_cast<int4*>(dst + 4 * (lane + 32 * m));
                    if (!first_flush) {
                        const int4 old = *pd;
                        val.x += old.x;
                        val.y += old.y;
                        val.z += old.z;
                        val.w += old.w;
                    }
                    *pd = val;
                }
            }
#pragma unroll
            for (int m = 0; m < DD_WORDS; ++m) E[u][m] = H[u][m] = 0;
        }
        first_flush = false;
    };

    // prologue: stage 0 offsets and data; stage 1 window in flight
    uint2 wnext = __ldg(wintab + my_cs);
    fetch_offs(0, 0);
    load_stage(0, wnext);
    store_stage(0, wnext);
    wnext = nstages > 1 ? __ldg(wintab + G + my_cs) : make_uint2(0, 0);
    __pipeline_wait_prior(0);
    __syncthreads();
    const uint32_t stages_per_flush = DD_FLUSH_CH / G;
    uint32_t since_flush = 0;

    for (uint32_t gi = 0; gi < nstages; ++gi) {
        const int b = gi & 1;
        const bool more = gi + 1 < nstages;
        const uint2 wstage = wnext;
        if (more) {
            fetch_offs(gi + 1, b ^ 1);
            if (!(XP & 8)) load_stage(gi + 1, wstage);
            if (gi + 2 < nstages) wnext = __ldg(wintab + (size_t)(gi + 2) * G + my_cs);
        }
        const uint32_t* offb = offs + b * G * TB + warp * TPW;
        const uint8_t* bufb = buf + (size_t)b * G * 4 * W + 4 * lane;
#pragma unroll
        for (int cs = 0; cs < ((XP & 4) ? 0 : G); ++cs) {
#pragma unroll
            for (int u = 0; u < TPW; ++u) {
                const uint8_t* src = bufb + (size_t)cs * 4 * W + offb[cs * TB + u];
#pragma unroll
                for (int m = 0; m < DD_WORDS; ++m) {
                    const uint32_t w = *reinterpret_cast<const uint32_t*>(src + 128 * m);
                    uint32_t e = E[u][m];
                    asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(e) : "r"(w & 0x00ff00ffu), "r"(one));
                    E[u][m] = e;
                    if ((SF & 2) && (m & 1)) {  // odd words: H on the FMA pipe (IMAD.HI)
                        uint32_t h = H[u][m];
                        asm("mad.hi.u32 %0, %1, %2, %0;" : "+r"(h) : "r"(w), "r"(kshift[0]));
                        H[u][m] = h;
                    } else {
                        H[u][m] += __umulhi(w, 1u << 24);  // LEA.HI, ALU pipe
                    }
                }
            }
        }
        if (more && !(XP & 8)) store_stage(b ^ 1, wstage);
        if (++since_flush == stages_per_flush || !more) {
            if (!(XP & 16)) flush();
            since_flush = 0;
        }
        __pipeline_wait_prior(0);
        if (!(XP & 32)) __syncthreads();
    }
}

#endif  // PGB_ABLATIONS
template <int TPW>
__global__ void __launch_bounds__(DD_THREADS, 1)
    dedisp_f32_kernel(const DedispLaunch p, const float* __restrict__ rows,
                      float* __restrict__ out, const uint32_t* __restrict__ blk_len) {
    constexpr int TB = DD_WARPS * TPW;
    extern __shared__ __align__(16) uint8_t smem[];
    const int G = p.g;
    const uint32_t W = p.wmax;  // floats per window
    float* buf = reinterpret_cast<float*>(smem);                               // [2][G][W]
    uint32_t* offs = reinterpret_cast<uint32_t*>(smem + (size_t)2 * G * W * 4);  // [2][G][TB]
    uint64_t* abase = reinterpret_cast<uint64_t*>(offs + 2 * G * TB);
    __shared__ uint32_t trial_ids[32];

    const uint32_t blk = blockIdx.x;
    const uint32_t row0 = blk * TB;
    const uint32_t nrows_blk = min((uint32_t)TB, p.nrows - row0);
    const uint64_t i0 = (uint64_t)blockIdx.y * DD_NT;
    if (i0 >= blk_len[blk]) return;
    if (threadIdx.x < 32)
        trial_ids[threadIdx.x] = p.active[row0 + min((uint32_t)threadIdx.x, nrows_blk - 1)];
    __syncthreads();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t nstages = (p.nchans + G - 1) / G;
    const int wpc = DD_WARPS / G;
    const int my_cs = warp / wpc;
    const uint32_t my_t = (uint32_t)((warp % wpc) * 32 + lane);
    const uint32_t vstride = (uint32_t)wpc * 32;
    const uint32_t vec_per_ch = W / 4;

    auto issue_stage = [&](uint32_t gi, int b) {
        const uint32_t c = min(gi * G + my_cs, p.nchans - 1);
        const float* src = rows + (size_t)c * p.rows_pitch + abase[b * G + my_cs];
        float* dst = buf + (size_t)(b * G + my_cs) * W;
        for (uint32_t vi = my_t; vi < vec_per_ch; vi += vstride)
            __pipeline_memcpy_async(dst + 4 * vi, src + 4 * vi, 16);
        __pipeline_commit();
    };

    float acc[TPW][DD_FOUT];
#pragma unroll
    for (int u = 0; u < TPW; ++u)
#pragma unroll
        for (int m = 0; m < DD_FOUT; ++m) acc[u][m] = 0.0f;  // the reference starts from +0.0f

    uint32_t dnext = stage_delay<TB>(p, 0, trial_ids);
    stage_offsets<false, TB>(p, dnext, 0, i0, abase, offs);
    dnext = nstages > 1 ? stage_delay<TB>(p, 1, trial_ids) : 0;
    __syncthreads();
    issue_stage(0, 0);

    for (uint32_t gi = 0; gi < nstages; ++gi) {
        const int b = gi & 1;
        const bool more = gi + 1 < nstages;
        if (more) {
            stage_offsets<false, TB>(p, dnext, b ^ 1, i0, abase, offs);
            if (gi + 2 < nstages) dnext = stage_delay<TB>(p, gi + 2, trial_ids);
        }
        __pipeline_wait_prior(0);
        __syncthreads();
        if (more) issue_stage(gi + 1, b ^ 1);

        const uint32_t c0 = gi * G;
        const int nch = (int)min((uint32_t)G, p.nchans - c0);
        const uint32_t* offb = offs + b * G * TB;
        for (int cs = 0; cs < nch; ++cs) {
#pragma unroll
            for (int u = 0; u < TPW; ++u) {
                const float* src = buf + offb[cs * TB + warp * TPW + u] + lane;
#pragma unroll
                for (int m = 0; m < DD_FOUT; ++m) acc[u][m] = __fadd_rn(acc[u][m], src[32 * m]);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < TPW; ++u) {
        const uint32_t r = warp * TPW + u;
        if (r < nrows_blk) {
            float* dst = out + (size_t)(row0 + r) * p.out_pitch + i0;
#pragma unroll
            for (int m = 0; m < DD_FOUT; ++m) dst[lane + 32 * m] = acc[u][m];
        }
    }
}

// ---- f32 ring (non-integer chunks) ------------------------------------------------
// Table for the f32 kernels, one warp per (trial block, channel): window start
// i0 + (min delay & ~3) (16-byte aligned) and its length in float4 vectors; per trial the
// float offset into the channel's window.  Channels past nchans get empty windows.
__global__ void ddf_table_kernel(const DedispLaunch p, uint2* __restrict__ win, uint32_t* __restrict__ off) {
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t blk = gw / p.nchans_pad, c = gw % p.nchans_pad;
    const uint32_t nblocks = (p.nrows + 31) / 32;
    if (blk >= nblocks) return;
    const uint32_t row0 = blk * 32, nrows_blk = min(32u, p.nrows - row0);
    const uint32_t row = row0 + min((uint32_t)lane, nrows_blk - 1);
    const bool live = c < p.nchans;
    const uint32_t d = live ? (uint32_t)__ldg(p.delays_ct + (size_t)c * p.ntrials_plan + p.active[row]) : 0;
    const uint32_t dmin = warp_min_u32(d), dmax = warp_max_u32(d);
    const uint32_t a = dmin & ~3u;
    off[(size_t)gw * 32 + lane] = d - a;
    if (lane == 0) win[gw] = make_uint2(a, live ? (dmax - a + DD_NT + 3) / 4 : 0);
}

// Same channel-ordered IEEE fp32 sums as dedisp_f32_kernel, staged through a 4-slot
// ring filled by cp.async: every thread's copies of a stage arrive on the slot's `full`
// mbarrier when they land (cp.async.mbarrier.arrive.noinc), warps arrive on `empty`
// after adding a stage, and a stage is issued three stages ahead.  No CTA barrier and no
// staging registers.
constexpr int FRING_NS = 4;

__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sh_addr(bar)) : "memory");
}

template <int G>
__global__ void __launch_bounds__(DD_THREADS, 1)
    dedisp_f32_ring_kernel(const DedispLaunch p, const float* __restrict__ rows,
                           float* __restrict__ out, const uint32_t* __restrict__ blk_len) {
    constexpr int TPW = 2, TB = DD_WARPS * TPW, NS = FRING_NS, D = NS - 1;
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t W = p.wmax;  // floats per channel window
    float* buf = reinterpret_cast<float*>(smem);                                        // [NS][G][W]
    uint32_t* offs = reinterpret_cast<uint32_t*>(smem + (size_t)NS * G * W * 4);       // [NS][G][TB]
    uint64_t* full = reinterpret_cast<uint64_t*>(offs + NS * G * TB);                  // [NS]
    uint64_t* empty = full + NS;                                                        // [NS]

    const uint32_t blk = blockIdx.x;
    const uint32_t row0 = blk * TB;
    const uint32_t nrows_blk = min((uint32_t)TB, p.nrows - row0);
    const uint64_t i0 = (uint64_t)blockIdx.y * DD_NT;
    if (i0 >= blk_len[blk]) return;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t C = p.nchans;
    const uint32_t nstages = (C + G - 1) / G;
    constexpr int wpc = DD_WARPS / G;
    const int my_cs = warp / wpc;
    const uint32_t my_t = (uint32_t)((warp % wpc) * 32 + lane);
    constexpr uint32_t vstride = (uint32_t)wpc * 32;
    const uint32_t* offtab = p.dd_off + (size_t)blk * p.nchans_pad * TB;
    const uint2* wintab = p.dd_win + (size_t)blk * p.nchans_pad;
    const float* rows_i0 = rows + i0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            ring_init(full + s, DD_THREADS);
            ring_init(empty + s, DD_WARPS);
        }
    }
    __syncthreads();

    auto issue = [&](uint32_t gi, int slot) {
        const uint32_t c = gi * G + my_cs;
        if (c < C) {
            const uint2 wv = __ldg(wintab + c);
            const float* src = rows_i0 + (size_t)c * p.rows_pitch + wv.x;
            float* dst = buf + (size_t)(slot * G + my_cs) * W;
            for (uint32_t vi = my_t; vi < wv.y; vi += vstride)
                __pipeline_memcpy_async(dst + 4 * vi, src + 4 * vi, 16);
        }
        if ((int)threadIdx.x < G * TB / 4)
            __pipeline_memcpy_async(offs + slot * G * TB + 4 * threadIdx.x,
                                    offtab + (size_t)gi * G * TB + 4 * threadIdx.x, 16);
        cp_async_arrive(full + slot);
    };

    float acc[TPW][DD_FOUT];
#pragma unroll
    for (int u = 0; u < TPW; ++u)
#pragma unroll
        for (int m = 0; m < DD_FOUT; ++m) acc[u][m] = 0.0f;  // the reference starts from +0.0f

    for (int d = 0; d < D; ++d)
        if ((uint32_t)d < nstages) issue(d, d);
    int slot = 0;
    uint32_t ph = 0;
    for (uint32_t gi = 0; gi < nstages; ++gi) {
        ring_wait(full + slot, ph);
        const uint32_t c0 = gi * G;
        const int nch = (int)min((uint32_t)G, C - c0);
        const uint32_t* offb = offs + slot * G * TB + warp * TPW;
        const float* bufb = buf + (size_t)slot * G * W + lane;
        for (int cs = 0; cs < nch; ++cs) {
#pragma unroll
            for (int u = 0; u < TPW; ++u) {
                const float* src = bufb + (size_t)cs * W + offb[cs * TB + u];
#pragma unroll
                for (int m = 0; m < DD_FOUT; ++m) acc[u][m] = __fadd_rn(acc[u][m], src[32 * m]);
            }
        }
        __syncwarp();
        if (lane == 0) ring_arrive(empty + slot);
        if (gi + D < nstages) {
            // the slot of stage gi+D last held stage gi-1 (gi >= 1): all warps must be done
            const uint32_t nxt = gi + D;
            const int s2 = (int)(nxt % NS);
            if (gi >= 1) ring_wait(empty + s2, ((gi - 1) / NS) & 1);
            issue(nxt, s2);
        }
        if (++slot == NS) {
            slot = 0;
            ph ^= 1;
        }
    }
#pragma unroll
    for (int u = 0; u < TPW; ++u) {
        const uint32_t r = warp * TPW + u;
        if (r < nrows_blk) {
            float* dst = out + (size_t)(row0 + r) * p.out_pitch + i0;
#pragma unroll
            for (int m = 0; m < DD_FOUT; ++m) dst[lane + 32 * m] = acc[u][m];
        }
    }
}

// Overlap reuse: chunk k's first keep[r] outputs of row r are chunk k-1's outputs
// [shift, shift + keep[r]) (same absolute samples, same input bytes), moved in place.
__global__ void series_shift_kernel(int32_t* __restrict__ series, uint64_t pitch, uint64_t shift,
                                    const uint32_t* __restrict__ keep) {
    int32_t* row = series + (size_t)blockIdx.x * pitch;  // rows on x (any trial count)
    const uint32_t n = keep[blockIdx.x];
    for (uint32_t i = blockIdx.y * blockDim.x + threadIdx.x; i < n; i += gridDim.y * blockDim.x)
        row[i] = row[shift + i];
}

// ---- transposes ---------------------------------------------------------------

// u8 [length][nchans] -> rows [nchans][pitch]; tiles of TT samples x 64 channels, 256
// threads, TT/64 16-byte loads and stores per thread (TT = 256 keeps 16 KB per CTA in
// flight: the 64 x 64 tile left the copy at ~55 % of HBM bandwidth, latency-bound on
// bytes in flight).
template <int TT>
__global__ void __launch_bounds__(256) transpose_u8_kernel(const uint8_t* __restrict__ in, uint64_t length,
                                                            uint32_t nchans, uint8_t* __restrict__ rows,
                                                            uint64_t pitch) {
    constexpr int R = TT / 64;  // rows (and output vectors) per thread
    __shared__ uint8_t tile[TT][64 + 4];
    const uint64_t t0 = (uint64_t)blockIdx.x * TT;
    const uint32_t c0 = blockIdx.y * 64;
    const int tid = threadIdx.x;
    const bool full = (t0 + TT <= length) && (c0 + 64 <= nchans) && (nchans % 16 == 0);
    if (full) {
        const int cv = (tid & 3) * 16;
        uint4 v[R];
#pragma unroll
        for (int k = 0; k < R; ++k)
            v[k] = __ldg(reinterpret_cast<const uint4*>(in + (t0 + (tid >> 2) + 64 * k) * nchans + c0 + cv));
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const int r = (tid >> 2) + 64 * k;
            *reinterpret_cast<uint32_t*>(&tile[r][cv]) = v[k].x;
            *reinterpret_cast<uint32_t*>(&tile[r][cv + 4]) = v[k].y;
            *reinterpret_cast<uint32_t*>(&tile[r][cv + 8]) = v[k].z;
            *reinterpret_cast<uint32_t*>(&tile[r][cv + 12]) = v[k].w;
        }
    } else {
        for (int k = tid; k < TT * 64; k += blockDim.x) {
            const int r = k >> 6, c = k & 63;
            tile[r][c] = (t0 + r < length && c0 + c < nchans) ? in[(t0 + r) * nchans + c0 + c] : 0;
        }
    }
    __syncthreads();
    // write: thread -> (channel c, R runs of 16 consecutive samples)
    const int c = tid >> 2;
    if (c0 + c < nchans) {
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const int tv = ((tid & 3) + 4 * k) * 16;
            uint32_t w[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                w[q] = (uint32_t)tile[tv + 4 * q][c] | (uint32_t)tile[tv + 4 * q + 1][c] << 8 |
                       (uint32_t)tile[tv + 4 * q + 2][c] << 16 | (uint32_t)tile[tv + 4 * q + 3][c] << 24;
            uint8_t* dst = rows + (uint64_t)(c0 + c) * pitch + t0 + tv;
            if (t0 + tv + 16 <= pitch)
                *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
}

__global__ void transpose_f32_kernel(const float* __restrict__ in, uint64_t length,
                                     uint32_t nchans, float* __restrict__ rows, uint64_t pitch) {
    __shared__ float tile[32][33];
    const uint64_t t0 = (uint64_t)blockIdx.x * 32;
    const uint32_t c0 = blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int r = ty; r < 32; r += 8) {
        const uint64_t t = t0 + r;
        tile[r][tx] = (t < length && c0 + tx < nchans) ? __ldg(in + t * nchans + c0 + tx) : 0.0f;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const uint32_t c = c0 + r;
        if (c < nchans && t0 + tx < pitch) rows[(uint64_t)c * pitch + t0 + tx] = tile[tx][r];
    }
}

__global__ void pack_u8_kernel(const float* __restrict__ in, size_t cells, uint8_t* __restrict__ out,
                               unsigned long long* not_u8) {
    const size_t n4 = cells / 4;
    bool bad = false;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
         i += (size_t)gridDim.x * blockDim.x) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(in) + i);
        const float f[4] = {v.x, v.y, v.z, v.w};
        uint32_t w = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const bool ok = f[k] >= 0.0f && f[k] <= 255.0f && f[k] == truncf(f[k]);
            bad |= !ok;
            w |= (ok ? (uint32_t)f[k] : 0u) << (8 * k);
        }
        reinterpret_cast<uint32_t*>(out)[i] = w;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0)
        for (size_t i = 4 * n4; i < cells; ++i) {
            const float f = in[i];
            const bool ok = f >= 0.0f && f <= 255.0f && f == truncf(f);
            bad |= !ok;
            out[i] = ok ? (uint8_t)f : 0;
        }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(not_u8, 1ull);
}

// ---- direct fallback for wide trial blocks -------------------------------------------
// A 32-trial block whose channel delay spread is so wide that no staged window fits in
// shared memory (e.g. DM steps of tens over a 4096-channel L-band: a block spread of
// 27k samples) is dedispersed straight from the channel rows in global memory (L1/L2):
// one CTA per (trial, DD_NT-output tile), a thread per 4 consecutive outputs, channels
// ascending.  u8: two aligned words and a funnel shift per (thread, channel), the same
// exact SWAR lanes (bytes 0/2 and 1/3 in u16 lanes, decoded every 256 channels).
// f32: in-order __fadd_rn per output, the reference's rounding sequence.
__global__ void __launch_bounds__(256)
    dedisp_u8_direct_kernel(const DedispLaunch p, const uint8_t* __restrict__ rows, int32_t* __restrict__ out,
                            const uint32_t* __restrict__ wide_rows) {
    const uint32_t r = wide_rows[blockIdx.x];
    const uint32_t tile = blockIdx.y + p.tile0;
    if (p.blk_first && tile < p.blk_first[r / 32]) return;  // shifted in from the previous chunk
    if ((uint64_t)tile * DD_NT >= p.row_len[r]) return;
    const uint32_t t = p.active[r];
    const uint64_t i = (uint64_t)tile * DD_NT + 4 * threadIdx.x;
    const uint8_t* base = rows + i;
    uint32_t E = 0, H = 0;
    int4 acc = make_int4(0, 0, 0, 0);
    for (uint32_t c0 = 0; c0 < p.nchans; c0 += DD_FLUSH_CH) {
        const uint32_t c1 = min(p.nchans, c0 + (uint32_t)DD_FLUSH_CH);
#pragma unroll 4
        for (uint32_t c = c0; c < c1; ++c) {
            const uint32_t d = (uint32_t)__ldg(p.delays_ct + (size_t)c * p.ntrials_plan + t);
            const uintptr_t a = reinterpret_cast<uintptr_t>(base + (size_t)c * p.rows_pitch + d);
            const uint32_t* w2 = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
            const uint32_t w = __funnelshift_r(__ldg(w2), __ldg(w2 + 1), (uint32_t)(a & 3) * 8);
            E += w & 0x00ff00ffu;
            H += (w >> 8) & 0x00ff00ffu;
        }
        acc.x += (int)(E & 0xffffu);
        acc.y += (int)(H & 0xffffu);
        acc.z += (int)(E >> 16);
        acc.w += (int)(H >> 16);
        E = H = 0;
    }
    *reinterpret_cast<int4*>(out + (size_t)r * p.out_pitch + i) = acc;
}

__global__ void __launch_bounds__(256)
    dedisp_f32_direct_kernel(const DedispLaunch p, const float* __restrict__ rows, float* __restrict__ out,
                             const uint32_t* __restrict__ wide_rows) {
    const uint32_t r = wide_rows[blockIdx.x];
    const uint32_t tile = blockIdx.y + p.tile0;
    if ((uint64_t)tile * DD_NT >= p.row_len[r]) return;
    const uint32_t t = p.active[r];
    const uint64_t i0 = (uint64_t)tile * DD_NT + threadIdx.x;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};  // outputs i0 + 256 k: coalesced across the warp
    for (uint32_t c = 0; c < p.nchans; ++c) {
        const uint32_t d = (uint32_t)__ldg(p.delays_ct + (size_t)c * p.ntrials_plan + t);
        const float* src = rows + (size_t)c * p.rows_pitch + i0 + d;
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[k] = __fadd_rn(acc[k], __ldg(src + 256 * k));  // src/dedisp.cpp:146-160
    }
    float* dst = out + (size_t)r * p.out_pitch + i0;
#pragma unroll
    for (int k = 0; k < 4; ++k) dst[256 * k] = acc[k];
}

}  // namespace

void launch_pack_u8(const float* in, size_t cells, uint8_t* out, unsigned long long* not_u8,
                    cudaStream_t st) {
    pack_u8_kernel<<<148 * 8, 256, 0, st>>>(in, cells, out, not_u8);
    PGB_CUDA(cudaGetLastError());
}

size_t dedisp_smem_bytes(bool u8, int g, uint32_t wmax) {
    const int tb = 32;
    const size_t staged = u8 ? (size_t)2 * g * 4 * wmax : (size_t)2 * g * wmax * 4;
    return staged + (size_t)2 * g * tb * 4 + (size_t)2 * g * 8;
}

int num_sms() {
    static const int n = [] {
        int dev = 0, v = 0;
        PGB_CUDA(cudaGetDevice(&dev));
        PGB_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
        return v;
    }();
    return n;
}

// PGB_DD_WHICH=1: print each u8 dedispersion launch's kernel choice to stderr (tests)
void dd_which(const char* kind, int g, int vpt, int mode) {
    static const bool on = getenv("PGB_DD_WHICH") != nullptr;
    if (on) fprintf(stderr, "pgb dedisp: %s G=%d VPT=%d mode=%d\n", kind, g, vpt, mode);
}

size_t ring_smem_bytes(int g, uint32_t wmax, int ns = RING_NS) {
    return (size_t)ns * g * 4 * wmax + (size_t)ns * g * 32 * 4 + 2 * ns * sizeof(uint64_t);
}

#ifdef PGB_ABLATIONS
void launch_dedisp_u8_ablation(const DedispLaunch& p0, const uint8_t* rows, int32_t* out, cudaStream_t st) {
    DedispLaunch p = p0;
    {
        const char* j = pgb_ablation_env("PGB_RING_JITTER");
        p.jitter = j ? (uint32_t)strtoul(j, nullptr, 10) : 0u;
    }
    const size_t smem = dedisp_smem_bytes(true, p.g, p.wmax);
    const int tb = DD_WARPS * p.tpw;
    dim3 grid((p.nrows + tb - 1) / tb, p.ntiles - p.tile0);
    static const int mode = [] {
        const char* e = pgb_ablation_env("PGB_DD_HMODE");
        return e ? atoi(e) : 3;
    }();
    static const bool v1 = [] {  // PGB_DD_V1=1: per-stage offset kernel (ablation)
        const char* e = pgb_ablation_env("PGB_DD_V1");
        return e && *e && *e != '0';
    }();
    static const int sf = [] {  // variant bits: 1 = staging shifts on the FMA pipe (ablation),
        // 2 = odd-word H accumulation on the FMA pipe (IMAD.HI) to balance ALU/FMA
        const char* e = pgb_ablation_env("PGB_DD_SFMA");
        const char* h = pgb_ablation_env("PGB_DD_HHI");
        int v = (e && *e == '1' ? 1 : 0) | (h && *h == '1' ? 2 : 0);
#ifdef PGB_DD_EXPERIMENTS
        if (const char* x = pgb_ablation_env("PGB_DD_EXPERIMENT")) v |= atoi(x) & ~3;
#endif
        return v;
    }();
    static const bool ring = [] {  // PGB_DD_RING=0: CTA-barrier kernel instead of the mbarrier ring
        const char* e = pgb_ablation_env("PGB_DD_RING");
        return !(e && *e == '0');
    }();
    static const int rmode = [] {  // PGB_RING_MODE: ring accumulation / ablation bits (see the kernel)
        const char* e = pgb_ablation_env("PGB_RING_MODE");
        return e ? atoi(e) & 31 : 8;  // default: channel-paired (K, T) accumulation (8)
    }();
    static const int nw32 = [] {  // PGB_DD_WARPS=32: 1024-thread ring, one trial per warp
        const char* e = pgb_ablation_env("PGB_DD_WARPS");
        return e && atoi(e) == 32;
    }();
    static const bool two = [] {  // PGB_DD_2CTA=1: two 64-register CTAs per SM
        const char* e = pgb_ablation_env("PGB_DD_2CTA");
        return e && *e == '1';
    }();
    if (two && p.tpw == 2 && p.dd_off && p.work_ctr) {
        int g = 8;
        while (g > 1 && ring_smem_bytes(g, p.wmax) > 112 * 1024) g >>= 1;
        const size_t rsm = ring_smem_bytes(g, p.wmax);
        const int vpt = (int)((p.wmax / 16 + 32u * (DD_WARPS / g) - 1) / (32u * (DD_WARPS / g)));
        if (rsm <= 112 * 1024 && g >= p.g / 2) {
#define PGB_RING2C(G_, V_)                                                                         \
    if (g == G_ && vpt <= V_) {                                                                    \
        PGB_CUDA(cudaFuncSetAttribute(dedisp_u8_ring_persist2_kernel<G_, V_>,                      \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm));     \
        dedisp_u8_ring_persist2_kernel<G_, V_><<<2 * num_sms(), DD_THREADS, rsm, st>>>(p, rows, out, p.blk_len); \
        dd_which("ring3-persist-2cta", G_, V_, 8);                                                 \
        PGB_CUDA(cudaGetLastError());                                                              \
        return;                                                                                    \
    }
            PGB_RING2C(4, 1) PGB_RING2C(4, 2) PGB_RING2C(4, 4) PGB_RING2C(8, 1) PGB_RING2C(8, 2)
#undef PGB_RING2C
        }
    }
    if (ring && !v1 && !sf && p.tpw == 2 && p.dd_off && nw32 && p.work_ctr) {
        int g = 8;
        while (g > 1 && ring_smem_bytes(g, p.wmax) > 227 * 1024) g >>= 1;
        const size_t rsm = ring_smem_bytes(g, p.wmax);
        const int vpt = (int)((p.wmax / 16 + 32u * (32 / g) - 1) / (32u * (32 / g)));
        if (rsm <= 227 * 1024 && g >= p.g) {
#define PGB_RING32(G_, V_)                                                                           \
    if (g == G_ && vpt <= V_) {                                                                      \
        PGB_CUDA(cudaFuncSetAttribute(dedisp_u8_ring_persist_kernel<G_, V_, RING_NS, 8, 32>,         \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm));       \
        dedisp_u8_ring_persist_kernel<G_, V_, RING_NS, 8, 32><<<num_sms(), 1024, rsm, st>>>(         \
            p, rows, out, p.blk_len);                                                                \
        dd_which("ring3-persist-1024", G_, V_, 8);                                                   \
        PGB_CUDA(cudaGetLastError());                                                                \
        return;                                                                                      \
    }
            PGB_RING32(8, 1) PGB_RING32(8, 2) PGB_RING32(8, 4)
            PGB_RING32(4, 1) PGB_RING32(4, 2) PGB_RING32(4, 4)
#undef PGB_RING32
        }
    }
    if (ring && !v1 && !sf && p.tpw == 2 && p.dd_off) {
        int g = 8;
        while (g > 1 && ring_smem_bytes(g, p.wmax) > 227 * 1024) g >>= 1;
        const size_t rsm = ring_smem_bytes(g, p.wmax);
        const uint32_t vstride = 32u * (DD_WARPS / g);
        const int vpt = (int)((p.wmax / 16 + vstride - 1) / vstride);
        const bool pers = p.work_ctr && (rmode == 0 || rmode == 4 || rmode == 8 || rmode == 24);  // PGB_DD_PERSIST0 clears work_ctr
        // the 3-slot ring needs 1.5x the shared memory of the double-buffered kernel; when
        // that forces fewer channels per stage (wide windows, e.g. config C) a 2-slot ring
        // at the wider stage is faster (below; the 3-slot ring at G = 4: 18.4 T adds/s on C)
        if (rsm <= 227 * 1024 && g >= p.g) {
#define PGB_RINGK(G_, V_, M_)                                                                     \
    if (g == G_ && vpt <= V_ && rmode == M_) {                                                    \
        if (pers) {                                                                               \
            PGB_CUDA(cudaFuncSetAttribute(dedisp_u8_ring_persist_kernel<G_, V_, RING_NS, M_>,     \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm)); \
            dedisp_u8_ring_persist_kernel<G_, V_, RING_NS, M_><<<num_sms(), DD_THREADS, rsm, st>>>( \
                p, rows, out, p.blk_len);                                                         \
        } else {                                                                                  \
            PGB_CUDA(cudaFuncSetAttribute(dedisp_u8_ring_kernel<G_, V_, M_>,                      \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm)); \
            dedisp_u8_ring_kernel<G_, V_, M_><<<grid, DD_THREADS, rsm, st>>>(p, rows, out, p.blk_len); \
        }                                                                                         \
        dd_which(pers ? "ring3-persist" : "ring3-grid", G_, V_, M_);                              \
        PGB_CUDA(cudaGetLastError());                                                             \
        return;                                                                                   \
    }
            PGB_RINGK(8, 1, 4) PGB_RINGK(8, 2, 4) PGB_RINGK(8, 4, 4) PGB_RINGK(8, 2, 24)
#define PGB_RING(G_, V_) PGB_RINGK(G_, V_, 0) PGB_RINGK(G_, V_, 8)
            PGB_RING(8, 1) PGB_RING(8, 2) PGB_RING(8, 4)
            PGB_RING(4, 1) PGB_RING(4, 2) PGB_RING(4, 4)
            PGB_RING(2, 1) PGB_RING(2, 2) PGB_RING(2, 4)
            PGB_RING(1, 1) PGB_RING(1, 2) PGB_RING(1, 4)
#undef PGB_RING
            // ablations (grid launch): 1 staging shifts on the FMA pipe, 2 IMAD addressing, 3 both
            if (!pers) { PGB_RINGK(8, 2, 1) PGB_RINGK(8, 2, 2) PGB_RINGK(8, 2, 3) }
#undef PGB_RINGK
        }
        // wide windows: a 2-slot ring at the double-buffered kernel's stage width (one
        // stage of drift between warps instead of a CTA barrier per stage)
        const size_t rsm2 = ring_smem_bytes(p.g, p.wmax, 2);
        const uint32_t vstride2 = 32u * (DD_WARPS / p.g);
        const int vpt2 = (int)((p.wmax / 16 + vstride2 - 1) / vstride2);
        if (pers && rsm2 <= 227 * 1024 && !pgb_ablation_env("PGB_DD_RING2_OFF")) {
#define PGB_RING2(G_, V_, M_)                                                                     \
    if (p.g == G_ && vpt2 <= V_ && rmode == M_) {                                                 \
        PGB_CUDA(cudaFuncSetAttribute(dedisp_u8_ring_persist_kernel<G_, V_, 2, M_>,               \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm2));   \
        dedisp_u8_ring_persist_kernel<G_, V_, 2, M_><<<num_sms(), DD_THREADS, rsm2, st>>>(        \
            p, rows, out, p.blk_len);                                                             \
        dd_which("ring2-persist", G_, V_, M_);                                                    \
        PGB_CUDA(cudaGetLastError());                                                             \
        return;                                                                                   \
    }
            PGB_RING2(8, 1, 0) PGB_RING2(8, 2, 0) PGB_RING2(8, 4, 0)
            PGB_RING2(4, 1, 0) PGB_RING2(4, 2, 0) PGB_RING2(4, 4, 0)
            PGB_RING2(8, 1, 8) PGB_RING2(8, 2, 8) PGB_RING2(8, 4, 8)
            PGB_RING2(4, 1, 8) PGB_RING2(4, 2, 8) PGB_RING2(4, 4, 8)
#undef PGB_RING2
        }
    }
    if (!v1 && p.tpw == 2 && p.dd_off) {
        // vectors per staging thread: ceil(max window vectors / (32 * warps per channel))
        const uint32_t vstride = 32u * (DD_WARPS / p.g);
        const int vpt = (int)((p.wmax / 16 + vstride - 1) / vstride);
#define PGB_TAB3(G_, V_, S_)                                                                      \
    if (p.g == G_ && vpt <= V_ && sf == S_) {                                                     \
        PGB_CUDA(cudaFuncSetAttribute(dedisp_u8_tab_kernel<G_, V_, S_>,                           \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));   \
        dedisp_u8_tab_kernel<G_, V_, S_><<<grid, DD_THREADS, smem, st>>>(p, rows, out, p.blk_len);\
        dd_which("barrier", G_, V_, S_);                                                          \
        PGB_CUDA(cudaGetLastError());                                                             \
        return;                                                                                   \
    }
#define PGB_TAB(G_, V_) PGB_TAB3(G_, V_, 0) PGB_TAB3(G_, V_, 1)
        PGB_TAB3(8, 2, 2) PGB_TAB3(8, 2, 3)
#ifdef PGB_DD_EXPERIMENTS
        PGB_TAB3(8, 2, 4) PGB_TAB3(8, 2, 8) PGB_TAB3(8, 2, 40) PGB_TAB3(8, 2, 24) PGB_TAB3(8, 2, 56)
        PGB_TAB3(8, 2, 32) PGB_TAB3(8, 2, 16) PGB_TAB3(8, 2, 48)
#endif
        PGB_TAB(8, 1) PGB_TAB(8, 2) PGB_TAB(8, 4)
        PGB_TAB(4, 1) PGB_TAB(4, 2) PGB_TAB(4, 4)
        PGB_TAB(2, 1) PGB_TAB(2, 2) PGB_TAB(2, 4)
        PGB_TAB(1, 1) PGB_TAB(1, 2) PGB_TAB(1, 4)
#undef PGB_TAB
#undef PGB_TAB3
        raise(PGB_ERR_CONFIG, "no dedispersion kernel for this staging geometry");
    }
#define PGB_DD(TPW, M)                                                                          \
    do {                                                                                        \
        PGB_CUDA(cudaFuncSetAttribute(dedisp_u8_kernel<TPW, M>,                                 \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        dedisp_u8_kernel<TPW, M><<<grid, DD_THREADS, smem, st>>>(p, rows, out, p.blk_len);      \
    } while (0)
    if (p.tpw == 2) {
        if (mode == 1) PGB_DD(2, 1);
        else if (mode == 3) PGB_DD(2, 3);
        else if (mode == 2) PGB_DD(2, 2);
        else PGB_DD(2, 0);
    } else {
        PGB_DD(1, 0);
    }
#undef PGB_DD
    PGB_CUDA(cudaGetLastError());
}

#endif  // PGB_ABLATIONS

// Product dispatch: the persistent mbarrier-ring kernel with channel-paired SWAR
// accumulation (MODE 8), 3 slots at the widest stage that fits, else 2 slots at the
// host's stage width (wide windows, e.g. config C).  The host's geometry (G from the
// shared-memory budget, at most 4 vectors per staging thread, dedisp_staged_fits)
// guarantees one of the two fits; blocks beyond it take launch_dedisp_direct.
void launch_dedisp_u8(const DedispLaunch& p, const uint8_t* rows, int32_t* out, cudaStream_t st) {
#ifdef PGB_ABLATIONS
    launch_dedisp_u8_ablation(p, rows, out, st);
    return;
#endif
    if (p.tpw != 2 || !p.dd_off || !p.work_ctr) raise(PGB_ERR_CONFIG, "dedispersion launch without its staging table");
    int g = 8;
    while (g > 1 && ring_smem_bytes(g, p.wmax) > 227 * 1024) g >>= 1;
    const size_t rsm = ring_smem_bytes(g, p.wmax);
    const int vpt = (int)((p.wmax / 16 + 32u * (DD_WARPS / g) - 1) / (32u * (DD_WARPS / g)));
    if (rsm <= 227 * 1024 && g >= p.g) {
#define PGB_RING3(G_, V_)                                                                         \
    if (g == G_ && vpt <= V_) {                                                                   \
        PGB_CUDA(cudaFuncSetAttribute(dedisp_u8_ring_persist_kernel<G_, V_, RING_NS, 8>,          \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm));    \
        dedisp_u8_ring_persist_kernel<G_, V_, RING_NS, 8><<<num_sms(), DD_THREADS, rsm, st>>>(    \
            p, rows, out, p.blk_len);                                                             \
        dd_which("ring3-persist", G_, V_, 8);                                                     \
        PGB_CUDA(cudaGetLastError());                                                             \
        return;                                                                                   \
    }
        PGB_RING3(8, 1) PGB_RING3(8, 2) PGB_RING3(8, 4)
        PGB_RING3(4, 1) PGB_RING3(4, 2) PGB_RING3(4, 4)
        PGB_RING3(2, 1) PGB_RING3(2, 2) PGB_RING3(2, 4)
        PGB_RING3(1, 1) PGB_RING3(1, 2) PGB_RING3(1, 4)
#undef PGB_RING3
    }
    const size_t rsm2 = ring_smem_bytes(p.g, p.wmax, 2);
    const int vpt2 = (int)((p.wmax / 16 + 32u * (DD_WARPS / p.g) - 1) / (32u * (DD_WARPS / p.g)));
    if (rsm2 <= 227 * 1024) {
#define PGB_RING2(G_, V_)                                                                         \
    if (p.g == G_ && vpt2 <= V_) {                                                                \
        PGB_CUDA(cudaFuncSetAttribute(dedisp_u8_ring_persist_kernel<G_, V_, 2, 8>,                \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm2));   \
        dedisp_u8_ring_persist_kernel<G_, V_, 2, 8><<<num_sms(), DD_THREADS, rsm2, st>>>(         \
            p, rows, out, p.blk_len);                                                             \
        dd_which("ring2-persist", G_, V_, 8);                                                     \
        PGB_CUDA(cudaGetLastError());                                                             \
        return;                                                                                   \
    }
        PGB_RING2(8, 1) PGB_RING2(8, 2) PGB_RING2(8, 4)
        PGB_RING2(4, 1) PGB_RING2(4, 2) PGB_RING2(4, 4)
        PGB_RING2(2, 1) PGB_RING2(2, 2) PGB_RING2(2, 4)
        PGB_RING2(1, 1) PGB_RING2(1, 2) PGB_RING2(1, 4)
#undef PGB_RING2
    }
    raise(PGB_ERR_CONFIG, "no dedispersion kernel for this staging geometry");
}

void launch_dd_table(const DedispLaunch& p, uint2* win, uint32_t* off, cudaStream_t st) {
    const uint64_t warps = (uint64_t)((p.nrows + 31) / 32) * p.nchans_pad;
    dd_table_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(p, win, off);
    PGB_CUDA(cudaGetLastError());
}

size_t fring_smem_bytes(int g, uint32_t wmax) {
    return (size_t)FRING_NS * g * wmax * 4 + (size_t)FRING_NS * g * 32 * 4 + 2 * FRING_NS * sizeof(uint64_t);
}

void launch_ddf_table(const DedispLaunch& p, uint2* win, uint32_t* off, cudaStream_t st) {
    const uint64_t warps = (uint64_t)((p.nrows + 31) / 32) * p.nchans_pad;
    ddf_table_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(p, win, off);
    PGB_CUDA(cudaGetLastError());
}

void launch_dedisp_f32(const DedispLaunch& p, const float* rows, float* out, cudaStream_t st) {
    const size_t smem = dedisp_smem_bytes(false, p.g, p.wmax);
    const int tb = DD_WARPS * p.tpw;
    dim3 grid((p.nrows + tb - 1) / tb, p.ntiles);
    if (p.tpw == 2 && p.dd_off && !pgb_ablation_env("PGB_F32_RING0")) {  // the f32 ring (table built)
        int g = 8;
        while (g > 1 && fring_smem_bytes(g, p.wmax) > 227 * 1024) g >>= 1;
        const size_t rsm = fring_smem_bytes(g, p.wmax);
        if (rsm <= 227 * 1024) {
#define PGB_FRING(G_)                                                                             \
    if (g == G_) {                                                                                \
        PGB_CUDA(cudaFuncSetAttribute(dedisp_f32_ring_kernel<G_>,                                 \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm));    \
        dedisp_f32_ring_kernel<G_><<<grid, DD_THREADS, rsm, st>>>(p, rows, out, p.blk_len);       \
        PGB_CUDA(cudaGetLastError());                                                             \
        dd_which("f32-ring", G_, 0, 0);                                                           \
        return;                                                                                   \
    }
            PGB_FRING(8) PGB_FRING(4) PGB_FRING(2) PGB_FRING(1)
#undef PGB_FRING
        }
    }
    if (p.tpw == 2) {
        PGB_CUDA(cudaFuncSetAttribute(dedisp_f32_kernel<2>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        dedisp_f32_kernel<2><<<grid, DD_THREADS, smem, st>>>(p, rows, out, p.blk_len);
    } else {
        PGB_CUDA(cudaFuncSetAttribute(dedisp_f32_kernel<1>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        dedisp_f32_kernel<1><<<grid, DD_THREADS, smem, st>>>(p, rows, out, p.blk_len);
    }
    PGB_CUDA(cudaGetLastError());
}

void launch_dedisp_direct(const DedispLaunch& p, bool u8, const void* rows, void* out,
                          const uint32_t* wide_rows, uint32_t nwide, cudaStream_t st) {
    if (!nwide || p.ntiles <= p.tile0) return;
    dim3 grid(nwide, p.ntiles - p.tile0);
    if (u8)
        dedisp_u8_direct_kernel<<<grid, 256, 0, st>>>(p, static_cast<const uint8_t*>(rows),
                                                     static_cast<int32_t*>(out), wide_rows);
    else
        dedisp_f32_direct_kernel<<<grid, 256, 0, st>>>(p, static_cast<const float*>(rows),
                                                      static_cast<float*>(out), wide_rows);
    PGB_CUDA(cudaGetLastError());
}

bool dedisp_staged_fits(bool u8, uint32_t spread) {
    const uint32_t align_el = u8 ? 16 : 4;
    const uint32_t wmax = (uint32_t)((spread + DD_NT + 2 * align_el + 16 + 15) / 16 * 16);
    return dedisp_smem_bytes(u8, 1, wmax) <= DD_SMEM_BUDGET && (!u8 || wmax / 16 <= 4u * DD_THREADS);
}

void launch_series_shift(int32_t* series, uint32_t nrows, uint64_t pitch, uint64_t shift,
                         const uint32_t* keep, cudaStream_t st) {
    if (!nrows) return;
    series_shift_kernel<<<dim3(nrows, 8), 512, 0, st>>>(series, pitch, shift, keep);
    PGB_CUDA(cudaGetLastError());
}

void launch_transpose_u8(const uint8_t* in, uint64_t length, uint32_t nchans, uint8_t* rows,
                         uint64_t pitch, cudaStream_t st) {
    static const int tt = [] {  // PGB_TRANSPOSE_TT: time-tile ablation (64 / 128 / 256)
        const char* e = pgb_ablation_env("PGB_TRANSPOSE_TT");
        const int v = e ? atoi(e) : 256;
        return v == 64 || v == 128 ? v : 256;
    }();
    dim3 grid((unsigned)((length + tt - 1) / tt), (nchans + 63) / 64);
    if (tt == 64) transpose_u8_kernel<64><<<grid, 256, 0, st>>>(in, length, nchans, rows, pitch);
    else if (tt == 128) transpose_u8_kernel<128><<<grid, 256, 0, st>>>(in, length, nchans, rows, pitch);
    else transpose_u8_kernel<256><<<grid, 256, 0, st>>>(in, length, nchans, rows, pitch);
    PGB_CUDA(cudaGetLastError());
}

void launch_transpose_f32(const float* in, uint64_t length, uint32_t nchans, float* rows,
                          uint64_t pitch, cudaStream_t st) {
    dim3 grid((unsigned)((length + 31) / 32), (nchans + 31) / 32);
    transpose_f32_kernel<<<grid, 256, 0, st>>>(in, length, nchans, rows, pitch);
    PGB_CUDA(cudaGetLastError());
}

}  // namespace pgb
