// In-order fp32 dedispersion of RFI-masked 8-bit chunks from fp16-staged codes.
//
// After local-mean RFI replacement (/root/reference/proj/src/rfi.cpp:115-139) an 8-bit
// chunk holds integer codes everywhere except the cells of the flagged sample rows, which
// carry float local means.  The reference sums each output's channels in ascending order
// in fp32 (src/dedisp.cpp:146-160, tests/oracles.hpp:16-26), so the device has to repeat
// that rounding sequence: the integer SWAR kernel does not apply, and the all-float ring
// kernel reads 4 bytes of shared memory per add (its bound: 32 adds/clk/SM).
//
// Here the codes are staged as fp16 (exact for 0..255; the cells of flagged rows are
// staged as +0) and every add is one FHADD -- PTX add.rn.f32.f16, an fp32 accumulator
// plus an fp16 operand with a single rounding, full rate on sm_100a
// (tools/pipe_probe.cu) -- so an add costs 2 bytes of shared memory (64 adds/clk/SM).
// A flagged cell's float value v is added right after its channel's regular add of +0:
// fl(s + 0) = s for s >= +0, so the pair is exactly the reference's fl(s + v).  Each
// staged channel window carries the flagged rows it covers with their values (the
// exceptions, from rfi_exceptions_u8), and a warp applies those that fall in a trial's
// 1024 outputs before it adds the next channel.
//
// Tile, ring and staging as the u8 ring kernel (dedisp.cu): 32 trials x 1024 outputs, 16
// warps, G channels per stage through a 3-slot mbarrier ring, persistent CTAs.  A
// channel window is stored twice, shifted by one half (copy 0: words (h[2k], h[2k+1]),
// copy 1: (h[2k+1], h[2k+2])), so lane l reads outputs 2(l + 32m), 2(l + 32m) + 1 of a
// trial with one aligned, conflict-free LDS.32 whatever the trial's delay parity.
#include <cstdio>
#include <cstdlib>

#include "mbarrier.cuh"
#include "pgb_internal.h"

namespace pgb {

namespace {

constexpr int H_NS = 3;    // ring slots
constexpr int H_TPW = 2;   // trials per warp
constexpr int H_TB = 32;   // trials per block
constexpr int H_FOUT = DD_NT / 32;  // outputs per lane per trial (32)

struct HExc {
    uint32_t pos;  // row - window start (halves)
    float val;
};

// exception counts [NS][G] u32, padded to 16 bytes: the 8-byte lists and mbarriers follow
__host__ __device__ constexpr int hx_count_words(int g) { return (H_NS * g + 3) & ~3; }

size_t h16_smem_bytes(int g, uint32_t wmax) {
    return (size_t)H_NS * g * 4 * wmax                 // [NS][G][2 copies][wmax halves]
           + (size_t)H_NS * g * H_TB * 4               // offsets
           + (size_t)hx_count_words(g) * 4             // exception counts
           + (size_t)H_NS * g * HX_CAP * sizeof(HExc)  // exception lists
           + 2 * H_NS * sizeof(uint64_t);
}

// fp16 bits of an 8-bit code (exact)
__device__ __forceinline__ uint32_t h16_of(uint32_t b) {
    if (b == 0) return 0;
    const uint32_t e = 31 - __clz(b);                  // 0..7
    return ((e + 15) << 10) | ((b << (10 - e)) & 0x3ffu);
}

// u8 [length][nchans] -> rows [nchans][pitch] (u8 or fp16), cells of bad channels and bad
// rows zeroed; tiles of 256 samples x 64 channels as transpose_u8_kernel.
template <bool H16>
__global__ void __launch_bounds__(256)
    transpose_masked_kernel(const uint8_t* __restrict__ in, uint64_t length, uint32_t nchans,
                            const uint8_t* __restrict__ chan_bad, const uint8_t* __restrict__ samp_bad,
                            void* __restrict__ rows, uint64_t pitch) {
    constexpr int TT = 256, R = TT / 64;
    __shared__ uint8_t tile[TT][64 + 4];
    __shared__ uint8_t rbad[TT];
    const uint64_t t0 = (uint64_t)blockIdx.x * TT;
    const uint32_t c0 = blockIdx.y * 64;
    const int tid = threadIdx.x;
    rbad[tid] = (t0 + tid < length) ? samp_bad[t0 + tid] : 1;  // 256 threads, 256 rows
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
    const int c = tid >> 2;
    if (c0 + c >= nchans) return;
    const bool cbad = chan_bad[c0 + c] != 0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const int tv = ((tid & 3) + 4 * k) * 16;
        if (t0 + tv + 16 > pitch) continue;
        uint32_t b[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) b[q] = (cbad || rbad[tv + q]) ? 0u : (uint32_t)tile[tv + q][c];
        if (H16) {
            uint32_t w[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) w[q] = h16_of(b[2 * q]) | h16_of(b[2 * q + 1]) << 16;
            uint4* dst = reinterpret_cast<uint4*>(static_cast<uint16_t*>(rows) + (uint64_t)(c0 + c) * pitch + t0 + tv);
            dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
            dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
        } else {
            uint32_t w[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                w[q] = b[4 * q] | b[4 * q + 1] << 8 | b[4 * q + 2] << 16 | b[4 * q + 3] << 24;
            *reinterpret_cast<uint4*>(static_cast<uint8_t*>(rows) + (uint64_t)(c0 + c) * pitch + t0 + tv) =
                make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
}

__device__ __forceinline__ uint32_t hwarp_min(uint32_t v) {
    for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ uint32_t hwarp_max(uint32_t v) {
    for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Staging table, one warp per (trial block, channel): window start a = min delay & ~7
// (16-byte aligned in halves), 16-byte vectors per copy covering every trial's 1024
// outputs plus the copy-1 half, and per trial the byte offset (o & 1) * 2 wmax + (o >> 1) * 4
// of o = d - a in the channel's two-copy slot (low 16 bits; o itself in the high 16 bits,
// for the exception rows; wmax < 2^14 keeps both in range).
__global__ void ddh_table_kernel(const DedispLaunch p, uint2* __restrict__ win, uint32_t* __restrict__ off) {
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t blk = gw / p.nchans_pad, c = gw % p.nchans_pad;
    const uint32_t nblocks = (p.nrows + 31) / 32;
    if (blk >= nblocks) return;
    const uint32_t row0 = blk * 32, nrows_blk = min(32u, p.nrows - row0);
    const uint32_t row = row0 + min((uint32_t)lane, nrows_blk - 1);
    const uint32_t d = c < p.nchans ? (uint32_t)__ldg(p.delays_ct + (size_t)c * p.ntrials_plan + p.active[row]) : 0;
    const uint32_t dmin = hwarp_min(d), dmax = hwarp_max(d);
    const uint32_t a = dmin & ~7u;
    const uint32_t o = d - a;
    off[(size_t)gw * 32 + lane] = ((o & 1) * 2 * p.wmax + (o >> 1) * 4) | o << 16;  // byte offset | o << 16
    if (lane == 0) win[gw] = make_uint2(a, (dmax - a + DD_NT + 1 + 7) / 8);
}

__device__ __forceinline__ void fhadd(float& acc, uint32_t w, int hi) {
    const uint16_t h = hi ? (uint16_t)(w >> 16) : (uint16_t)(w & 0xffffu);
    asm("add.rn.f32.f16 %0, %1, %0;" : "+f"(acc) : "h"(h));
}

// acc[idx] = fl(acc[idx] + v) on the selected lane; idx is warp-uniform (jump table)
__device__ __forceinline__ void add_at(float (&acc)[H_FOUT], uint32_t idx, bool sel, float v) {
    switch (idx) {
#define PGB_HX_CASE(k)                                  \
    case k:                                             \
        if (sel) acc[k] = __fadd_rn(acc[k], v);         \
        break;
        PGB_HX_CASE(0) PGB_HX_CASE(1) PGB_HX_CASE(2) PGB_HX_CASE(3) PGB_HX_CASE(4) PGB_HX_CASE(5)
        PGB_HX_CASE(6) PGB_HX_CASE(7) PGB_HX_CASE(8) PGB_HX_CASE(9) PGB_HX_CASE(10) PGB_HX_CASE(11)
        PGB_HX_CASE(12) PGB_HX_CASE(13) PGB_HX_CASE(14) PGB_HX_CASE(15) PGB_HX_CASE(16) PGB_HX_CASE(17)
        PGB_HX_CASE(18) PGB_HX_CASE(19) PGB_HX_CASE(20) PGB_HX_CASE(21) PGB_HX_CASE(22) PGB_HX_CASE(23)
        PGB_HX_CASE(24) PGB_HX_CASE(25) PGB_HX_CASE(26) PGB_HX_CASE(27) PGB_HX_CASE(28) PGB_HX_CASE(29)
        PGB_HX_CASE(30) PGB_HX_CASE(31)
#undef PGB_HX_CASE
        default:
            break;
    }
}

// One (trial block, time tile) through the ring; the whole CTA calls it.
template <int G, int VPT, int UNR>
__device__ __forceinline__ void h16_tile(const DedispLaunch& p, const uint16_t* __restrict__ rows,
                                         float* __restrict__ out, const uint32_t blk, const uint32_t tile) {
    constexpr int NW = DD_WARPS, NS = H_NS, TB = H_TB, TPW = H_TPW;
    constexpr uint32_t D = NS - 1;
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t W = p.wmax;             // halves per copy
    const uint32_t CH = 4 * W;             // bytes per channel slot (two copies)
    uint8_t* buf = smem;                                                            // [NS][G][CH]
    uint32_t* offs = reinterpret_cast<uint32_t*>(smem + (size_t)NS * G * CH);      // [NS][G][TB]
    uint32_t* xcnt = offs + NS * G * TB;                                            // [NS][G]
    HExc* xl = reinterpret_cast<HExc*>(xcnt + hx_count_words(G));                   // [NS][G][HX_CAP]
    uint64_t* full = reinterpret_cast<uint64_t*>(xl + NS * G * HX_CAP);             // [NS]
    uint64_t* empty = full + NS;                                                    // [NS]

    const uint32_t row0 = blk * TB;
    const uint32_t nrows_blk = min((uint32_t)TB, p.nrows - row0);
    const uint64_t i0 = (uint64_t)tile * DD_NT;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t nstages = p.nchans_pad / G;
    constexpr int wpc = NW / G;
    const int my_cs = warp / wpc;
    const uint32_t my_t = (uint32_t)((warp % wpc) * 32 + lane);
    constexpr uint32_t vstride = (uint32_t)wpc * 32;
    const bool xthread = my_t < (uint32_t)HX_CAP;  // loads one exception of its channel
    const bool offs_thread = (int)threadIdx.x < G * TB / 4;
    const uint32_t* offtab = p.dd_off + (size_t)blk * p.nchans_pad * TB;
    const uint2* wintab = p.dd_win + (size_t)blk * p.nchans_pad;
    const uint16_t* rows_i0 = rows + i0;

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

    // bad rows before the window's first row and its end (one stage ahead of the loads)
    auto pref = [&](uint2 wv) {
        uint2 pk = make_uint2(0, 0);
        if (xthread) {
            const uint64_t s = i0 + wv.x, e = s + 8ull * wv.y + 2;
            pk.x = __ldg(p.xP + min(s, p.xlen));
            pk.y = __ldg(p.xP + min(e, p.xlen));
        }
        return pk;
    };
    auto load_stage = [&](uint32_t gi, uint2 wv, uint2 pk) {
        const uint32_t c = gi * G + my_cs;
        const uint16_t* src = rows_i0 + (size_t)c * p.rows_pitch + wv.x;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            const uint32_t vi = my_t + k * vstride;
            if (vi < wv.y) {
                v0[k] = __ldg(reinterpret_cast<const uint4*>(src + 8 * vi));
                v1[k] = __ldg(reinterpret_cast<const uint32_t*>(src + 8 * vi + 8));
            }
        }
        if (offs_thread) ov = __ldg(reinterpret_cast<const uint4*>(offtab + (size_t)gi * G * TB) + threadIdx.x);
        if (xthread) {
            xn = c < p.nchans ? min(pk.y - pk.x, (uint32_t)HX_CAP) : 0u;
            if (my_t < xn) {
                const uint32_t k = pk.x + my_t;
                xr = (uint32_t)(__ldg(p.xR + k) - (i0 + wv.x));
                xv = __ldg(p.xF + (size_t)k * p.nchans + c);
            }
        }
    };
    auto store_stage = [&](int slot, uint2 wv) {
        uint8_t* base = buf + (size_t)(slot * G + my_cs) * CH;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            const uint32_t vi = my_t + k * vstride;
            if (vi < wv.y) {
                *reinterpret_cast<uint4*>(base + 16 * vi) = v0[k];
                uint4 sh;
                sh.x = __byte_perm(v0[k].x, v0[k].y, 0x5432);
                sh.y = __byte_perm(v0[k].y, v0[k].z, 0x5432);
                sh.z = __byte_perm(v0[k].z, v0[k].w, 0x5432);
                sh.w = __byte_perm(v0[k].w, v1[k], 0x5432);
                *reinterpret_cast<uint4*>(base + 2 * W + 16 * vi) = sh;
            }
        }
        if (offs_thread) reinterpret_cast<uint4*>(offs + slot * G * TB)[threadIdx.x] = ov;
        if (xthread) {
            if (my_t < xn) xl[(slot * G + my_cs) * HX_CAP + my_t] = HExc{xr, xv};
            if (my_t == 0) xcnt[slot * G + my_cs] = xn;
        }
        __syncwarp();
        if (lane == 0) ring_arrive(full + slot);
    };

    float acc[TPW][H_FOUT];
#pragma unroll
    for (int u = 0; u < TPW; ++u)
#pragma unroll
        for (int m = 0; m < H_FOUT; ++m) acc[u][m] = 0.0f;  // the reference starts from +0.0f

    // prologue: stages 0 .. D-1 into slots 0 .. D-1
    for (uint32_t s = 0; s < D && s < nstages; ++s) {
        const uint2 w = __ldg(wintab + s * G + my_cs);
        load_stage(s, w, pref(w));
        store_stage((int)s, w);
    }
    uint2 wnext = nstages > D ? __ldg(wintab + (size_t)D * G + my_cs) : make_uint2(0, 0);
    uint2 pknext = pref(wnext);
    int slot = 0, slot2 = (int)D;
    uint32_t ph = 0, ph_prev = 0;

    for (uint32_t gi = 0; gi < nstages; ++gi) {
        const bool pre = gi + D < nstages;
        const uint2 wstage = wnext;
        if (pre) {
            load_stage(gi + D, wstage, pknext);
            if (gi + D + 1 < nstages) wnext = __ldg(wintab + (size_t)(gi + D + 1) * G + my_cs);
        }
        ring_wait(full + slot, ph);
        const uint32_t* offb = offs + slot * G * TB + warp * TPW;
        const uint8_t* bufb = buf + (size_t)slot * G * CH + 4 * lane;
        const uint32_t* xc = xcnt + slot * G;
        uint32_t xmask = 0;
#pragma unroll
        for (int cs = 0; cs < G; ++cs) xmask |= (xc[cs] != 0 ? 1u : 0u) << cs;
        // channels as a runtime loop: the exception branch inside would otherwise be
        // unrolled G x TPW times (code size), and the compiler then rematerialises addresses
#pragma unroll(UNR)
        for (int cs = 0; cs < G; ++cs) {
            const uint2 o2 = *reinterpret_cast<const uint2*>(offb + cs * TB);  // this warp's two trials
            const uint8_t* cb = bufb + (size_t)cs * CH;
#pragma unroll
            for (int u = 0; u < TPW; ++u) {
                const uint8_t* src = cb + ((u ? o2.y : o2.x) & 0xffffu);
                uint32_t w[H_FOUT / 2];
#pragma unroll
                for (int m = 0; m < H_FOUT / 2; ++m) w[m] = *reinterpret_cast<const uint32_t*>(src + 128 * m);
#pragma unroll
                for (int m = 0; m < H_FOUT / 2; ++m) {
                    fhadd(acc[u][2 * m], w[m], 0);
                    fhadd(acc[u][2 * m + 1], w[m], 1);
                }
            }
            if (xmask & (1u << cs)) {  // flagged rows in this channel's window
                const uint32_t n = xc[cs];
                const HExc* xe = xl + (slot * G + cs) * HX_CAP;
#pragma unroll
                for (int u = 0; u < TPW; ++u) {
                    const uint32_t o = (u ? o2.y : o2.x) >> 16;  // delay - window start
                    for (uint32_t e = 0; e < n; ++e) {
                        const HExc x = xe[e];
                        const uint32_t j = x.pos - o;  // output index in the tile
                        if (j < (uint32_t)DD_NT)
                            add_at(acc[u], ((j >> 6) << 1) | (j & 1), lane == (int)((j >> 1) & 31), x.val);
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) ring_arrive(empty + slot);
        if (pre) {
            if (gi + D + 1 < nstages) pknext = pref(wnext);
            if (gi >= 1) ring_wait(empty + slot2, ph_prev);  // slot2 last held stage gi-1
            store_stage(slot2, wstage);
        }
        ph_prev = ph;
        if (++slot == NS) { slot = 0; ph ^= 1; }
        if (++slot2 == NS) slot2 = 0;
    }
#pragma unroll
    for (int u = 0; u < TPW; ++u) {
        const uint32_t r = warp * TPW + u;
        if (r < nrows_blk) {
            float* dst = out + (size_t)(row0 + r) * p.out_pitch + i0;
#pragma unroll
            for (int m = 0; m < H_FOUT / 2; ++m)
                *reinterpret_cast<float2*>(dst + 2 * (lane + 32 * m)) = make_float2(acc[u][2 * m], acc[u][2 * m + 1]);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            ring_inval(full + s);
            ring_inval(empty + s);
        }
    }
}

#ifdef PGB_ABLATIONS  // the fp16 kernel ships in the ablation library only (slower than fp32 on E)
// Persistent: one CTA per SM takes (block, tile) items from a counter (blocks fastest).
template <int G, int VPT, int UNR = 2>
__global__ void __launch_bounds__(DD_THREADS, 1)
    dedisp_h16_ring_kernel(const DedispLaunch p, const uint16_t* __restrict__ rows, float* __restrict__ out,
                           const uint32_t* __restrict__ blk_len) {
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
        if ((uint64_t)tile * DD_NT >= blk_len[blk]) continue;
        h16_tile<G, VPT, UNR>(p, rows, out, blk, tile);
    }
}

int num_sms_h16() {
    static const int n = [] {
        int dev = 0, v = 0;
        PGB_CUDA(cudaGetDevice(&dev));
        PGB_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
        return v;
    }();
    return n;
}

#endif  // PGB_ABLATIONS

constexpr size_t H_SMEM_MAX = 227 * 1024;
constexpr int H_VPT_MAX = 4;

}  // namespace

int dedisp_h16_stage_width(uint32_t wmax) {
    if (wmax >= (1u << 14)) return 0;  // offsets table packs byte offset and o in 16 bits each
    for (int g = 8; g >= 1; g >>= 1) {
        const uint32_t vstride = 32u * (DD_WARPS / g);
        if (h16_smem_bytes(g, wmax) <= H_SMEM_MAX && (wmax / 8 + vstride - 1) / vstride <= (uint32_t)H_VPT_MAX)
            return g;
    }
    return 0;
}

void launch_transpose_masked(const uint8_t* in, uint64_t length, uint32_t nchans, const uint8_t* chan_bad,
                             const uint8_t* samp_bad, void* rows, uint64_t pitch, bool h16, cudaStream_t st) {
    dim3 grid((unsigned)((length + 255) / 256), (nchans + 63) / 64);
    if (h16) transpose_masked_kernel<true><<<grid, 256, 0, st>>>(in, length, nchans, chan_bad, samp_bad, rows, pitch);
    else transpose_masked_kernel<false><<<grid, 256, 0, st>>>(in, length, nchans, chan_bad, samp_bad, rows, pitch);
    PGB_CUDA(cudaGetLastError());
}

void launch_ddh_table(const DedispLaunch& p, uint2* win, uint32_t* off, cudaStream_t st) {
#ifndef PGB_ABLATIONS
    (void)p, (void)win, (void)off, (void)st;
    raise(PGB_ERR_CONFIG, "the fp16 dedispersion kernel is in the ablation library only");
#else
    const uint64_t warps = (uint64_t)((p.nrows + 31) / 32) * p.nchans_pad;
    ddh_table_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(p, win, off);
    PGB_CUDA(cudaGetLastError());
#endif
}

void launch_dedisp_h16(const DedispLaunch& p, const uint16_t* rows, float* out, cudaStream_t st) {
#ifndef PGB_ABLATIONS
    (void)p, (void)rows, (void)out, (void)st;
    raise(PGB_ERR_CONFIG, "the fp16 dedispersion kernel is in the ablation library only");
#else
    if (p.tpw != 2 || !p.dd_off || !p.work_ctr || !p.xP)
        raise(PGB_ERR_CONFIG, "fp16 dedispersion launch without its tables");
    int g = dedisp_h16_stage_width(p.wmax);
    if (const char* e = pgb_ablation_env("PGB_H16_G"))  // stage-width cap (ablation library)
        while (g > 1 && g > atoi(e)) g >>= 1;
    if (g == 0 || (p.nchans_pad % g) != 0) raise(PGB_ERR_CONFIG, "no fp16 dedispersion kernel for this window");
    const size_t smem = h16_smem_bytes(g, p.wmax);
    const uint32_t vstride = 32u * (DD_WARPS / g);
    const int vpt = (int)((p.wmax / 8 + vstride - 1) / vstride);
    static const bool which = getenv("PGB_DD_WHICH") != nullptr;  // kernel-choice log (tests)
    int unr = 2;
    if (const char* e = pgb_ablation_env("PGB_H16_UNROLL")) unr = atoi(e);
#define PGB_H16U(G_, V_, U_)                                                                       \
    if (g == G_ && vpt <= V_ && unr == U_) {                                                       \
        PGB_CUDA(cudaFuncSetAttribute(dedisp_h16_ring_kernel<G_, V_, U_>,                          \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));    \
        dedisp_h16_ring_kernel<G_, V_, U_><<<num_sms_h16(), DD_THREADS, smem, st>>>(p, rows, out, p.blk_len); \
        PGB_CUDA(cudaGetLastError());                                                              \
        if (which) fprintf(stderr, "pgb dedisp: h16-ring G=%d VPT=%d mode=%d\n", G_, V_, U_);     \
        return;                                                                                    \
    }
#define PGB_H16(G_, V_) PGB_H16U(G_, V_, 2)
    PGB_H16(8, 1) PGB_H16(8, 2) PGB_H16(8, 4)
    PGB_H16(4, 1) PGB_H16(4, 2) PGB_H16(4, 4)
    PGB_H16(2, 1) PGB_H16(2, 2) PGB_H16(2, 4)
    PGB_H16(1, 1) PGB_H16(1, 2) PGB_H16(1, 4)
#ifdef PGB_ABLATIONS  // channel-loop unroll (PGB_H16_UNROLL=1 / 8)
    PGB_H16U(8, 4, 1) PGB_H16U(8, 4, 8) PGB_H16U(4, 2, 1) PGB_H16U(4, 2, 4)
#endif
#undef PGB_H16
    raise(PGB_ERR_CONFIG, "no fp16 dedispersion kernel for this staging geometry");
#endif
}

}  // namespace pgb
