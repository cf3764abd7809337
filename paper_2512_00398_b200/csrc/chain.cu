// The per-DM-trial detection chain for sm_100a, batched over all trials of a
// chunk: baseline removal -> robust RMS -> boxcar ladder -> threshold runs.
//
// Bit-exactness against the reference build (GCC -O3 -march=native, default
// -ffp-contract=fast) is by construction; this TU is compiled with -fmad=false and
// uses explicit IEEE intrinsics:
//   * baseline (src/detect.cpp:8-55): out = float(fma(-S, 1/cnt, x)) (the reference's
//     `x - sum*inv` is contracted into one vfnmadd).  For integer series the running
//     double window sum is an exact integer, so an exact int64 running sum gives the
//     same S; for general float series the reference's sequential recurrence is
//     replayed per trial.
//   * robust RMS (src/detect.cpp:67-108, 193-214): the 4 interleaved double chains
//     plus tail are order dependent, so each (trial, chain) is one sequential thread.
//   * boxcar ladder (src/detect.cpp:216-221): s_w[i] = s_{w/2}[i] + s_{w/2}[i+w/2],
//     elementwise and exact, done level by level in shared memory.
//   * peaks (src/detect.cpp:223-296): runs of s_w[i] * (1/sqrt(w)) > thresh, first
//     maximum of each run, edge-run and valid-range filters.  Runs fully inside one
//     thread strip are emitted directly; runs touching a strip edge become fragments
//     that a second kernel stitches after a device sort.
#include <cuda_pipeline.h>

#include <algorithm>

#include <cmath>
#include <utility>

#include <cooperative_groups.h>

#include <climits>
#include <cstdio>
#include <cstdlib>

#include "pgb_internal.h"

namespace cg = cooperative_groups;

namespace pgb {

namespace {

// ---- baseline: integer series (exact int64 running window sum) -----------------

constexpr int BL_THREADS = 1024;
constexpr int BL_PER = 4;
constexpr int BL_TILE = BL_THREADS * BL_PER;

__device__ __forceinline__ long long block_sum_ll(long long v, long long* red) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    return t;
}

__global__ void __launch_bounds__(BL_THREADS)
    baseline_int_kernel(const int32_t* __restrict__ x_all, float* __restrict__ out_all,
                        const uint32_t* __restrict__ row_len, uint64_t pitch, uint64_t window) {
    __shared__ long long red[32];
    __shared__ long long wsum[32];
    const uint32_t row = blockIdx.x;
    const int64_t n = row_len[row];
    const int32_t* x = x_all + (size_t)row * pitch;
    float* out = out_all + (size_t)row * pitch;
    if (n == 0) return;
    const int64_t h = (int64_t)(window / 2);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    if (h >= n - 1) {  // global-mean path, src/detect.cpp:16-32
        long long s = 0;
        for (int64_t i = tid; i < n; i += BL_THREADS) s += x[i];
        const long long total = block_sum_ll(s, red);
        const float mean = __double2float_rn(__ddiv_rn((double)total, (double)n));
        for (int64_t i = tid; i < n; i += BL_THREADS) out[i] = __fsub_rn((float)x[i], mean);
        return;
    }
    const double inv_full = __ddiv_rn(1.0, (double)(2 * h + 1));
    // S_0 = sum x[0..h]
    long long s0 = 0;
    for (int64_t i = tid; i <= h; i += BL_THREADS) s0 += x[i];
    long long carry = block_sum_ll(s0, red);  // S_{-1} + d_0 == S_0 with d_0 := S_0 below

    for (int64_t base = 0; base < n; base += BL_TILE) {
        long long d[BL_PER];
        int32_t xv[BL_PER];
        long long local = 0;
#pragma unroll
        for (int k = 0; k < BL_PER; ++k) {
            const int64_t i = base + tid * BL_PER + k;
            long long di = 0;
            int32_t xi = 0;
            if (i < n) {
                xi = x[i];
                if (i > 0) {
                    if (i + h < n) di += x[i + h];
                    if (i - 1 - h >= 0) di -= x[i - 1 - h];
                }
            }
            d[k] = di;
            xv[k] = xi;
            local += di;
        }
        // exclusive block scan of per-thread totals
        long long incl = local;
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        __syncthreads();
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            long long w = lane < (BL_THREADS >> 5) ? wsum[lane] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                const long long y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            wsum[lane] = w;  // inclusive over warps
        }
        __syncthreads();
        long long run = carry + (warp ? wsum[warp - 1] : 0) + (incl - local);
#pragma unroll
        for (int k = 0; k < BL_PER; ++k) {
            const int64_t i = base + tid * BL_PER + k;
            run += d[k];
            if (i < n) {
                const int64_t lo = i - h > 0 ? i - h : 0;
                const int64_t hi = i + h < n - 1 ? i + h : n - 1;
                const int64_t cnt = hi - lo + 1;
                // interior windows share one reciprocal; only the 2h edge samples divide
                const double inv = cnt == 2 * h + 1 ? inv_full : __ddiv_rn(1.0, (double)cnt);
                out[i] = __double2float_rn(__fma_rn(-(double)run, inv, (double)xv[k]));
            }
        }
        carry += wsum[(BL_THREADS >> 5) - 1];
    }
}

// ---- baseline, warp segments (default) -------------------------------------------
// The row-serial kernel above walks each row's ~60 tiles in order (3 CTA barriers and a
// global-load round trip per tile) and is latency-bound at ~18 % of HBM bandwidth.  Here
// every warp owns a 4096-sample segment of a row: its starting window sum comes from
// 256-sample block sums (<= 2 x 255 edge samples + <= 123 block sums), then it scans its
// segment 128 samples at a time with warp shuffles only.  All sums are exact int64, so
// the output is the same bit for bit.
constexpr int BW_BLK = 256;   // block-sum granule (samples)
constexpr int BW_SEG = 4096;  // samples per warp segment

__device__ __forceinline__ long long warp_sum_ll(long long v) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void __launch_bounds__(256)
    block256_sums_kernel(const int32_t* __restrict__ x_all, const uint32_t* __restrict__ row_len,
                         uint64_t pitch, uint32_t nrows, uint32_t nb, long long* __restrict__ bs) {
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= (uint64_t)nrows * nb) return;
    const uint32_t row = (uint32_t)(gw / nb), b = (uint32_t)(gw % nb);
    const int64_t n = row_len[row];
    const int64_t lo = (int64_t)b * BW_BLK;
    long long s = 0;
    if (lo < n) {
        const int32_t* x = x_all + (size_t)row * pitch;
        const int64_t hi = lo + BW_BLK < n ? lo + BW_BLK : n;
        for (int64_t i = lo + lane; i < hi; i += 32) s += x[i];
    }
    s = warp_sum_ll(s);
    if (lane == 0) bs[(size_t)row * nb + b] = s;
}

// An interior warp segment of baseline_warp_kernel: 32-bit indices and differences
// (|d| < 2^21, 128-sample prefix < 2^28), the window sum itself stays int64.  A lane owns 4
// consecutive samples i4 .. i4+3 (i4 16-byte aligned) and needs x[i + h] and x[i - 1 - h]:
// each set is 4 consecutive ints starting R = h mod 4 (resp. 3 - R) past an aligned
// address, taken from two aligned 16-byte loads (the second mostly an L1 hit of the
// neighbour lane's first) instead of eight 4-byte loads.
template <int R>
__device__ __forceinline__ void baseline_interior(const int32_t* __restrict__ x, float* __restrict__ out,
                                                  int64_t s0, int64_t s1, uint32_t hh, long long carry,
                                                  double inv_full, int lane) {
    constexpr int RB = (3 - R) & 3;  // (-1 - h) mod 4
    // the next 128 samples' loads are issued before this block's scan (the carry chain
    // serialises the blocks, the loads do not depend on it)
    auto fetch = [&](uint32_t base, int4& xq, int4& a0, int4& a1, int4& b0, int4& b1) {
        const uint32_t i4 = base + 4 * lane;
        xq = *reinterpret_cast<const int4*>(x + i4);  // 16-byte aligned (pitch, base)
        const int4* pa = reinterpret_cast<const int4*>(x + i4 + hh - R);
        const int4* pb = reinterpret_cast<const int4*>(x + i4 - 1 - hh - RB);
        a0 = pa[0];
        a1 = pa[1];
        b0 = pb[0];
        b1 = pb[1];
    };
    int4 xq, a0, a1, b0, b1;
    fetch((uint32_t)s0, xq, a0, a1, b0, b1);
    for (uint32_t base = (uint32_t)s0; base < (uint32_t)s1; base += 128) {
        const int32_t av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const int32_t bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
        const int32_t xv[4] = {xq.x, xq.y, xq.z, xq.w};
        if (base + 128 < (uint32_t)s1) fetch(base + 128, xq, a0, a1, b0, b1);
        const uint32_t i4 = base + 4 * lane;
        int32_t d[4];
        int32_t local = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t i = i4 + k;
            d[k] = (i > (uint32_t)s0 && i < (uint32_t)s1) ? av[R + k] - bv[RB + k] : 0;
            local += d[k];
        }
        int32_t incl = local;
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        long long run = carry + (long long)(incl - local);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            run += d[k];
            if (i4 + k < (uint32_t)s1)
                out[i4 + k] = __double2float_rn(__fma_rn(-(double)run, inv_full, (double)xv[k]));  // :45
        }
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
}

__global__ void __launch_bounds__(256, 4)  // 32 warps per SM: latency-bound on its loads
    baseline_warp_kernel(const int32_t* __restrict__ x_all, float* __restrict__ out_all,
                         const uint32_t* __restrict__ row_len, uint64_t pitch, uint64_t window,
                         uint32_t nrows, uint32_t nseg, uint32_t nb, const long long* __restrict__ bsum) {
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= (uint64_t)nrows * nseg) return;
    const uint32_t row = (uint32_t)(gw / nseg), seg = (uint32_t)(gw % nseg);
    const int64_t n = row_len[row];
    const int64_t s0 = (int64_t)seg * BW_SEG;
    if (s0 >= n) return;
    const int64_t s1 = s0 + BW_SEG < n ? s0 + BW_SEG : n;
    const int32_t* x = x_all + (size_t)row * pitch;
    float* out = out_all + (size_t)row * pitch;
    const long long* bs = bsum + (size_t)row * nb;
    const int64_t h = (int64_t)(window / 2);
    if (h >= n - 1) {  // global-mean path, src/detect.cpp:16-32 (row total from its blocks)
        long long t = 0;
        for (int64_t b = lane; b * BW_BLK < n; b += 32) t += bs[b];
        const long long total = warp_sum_ll(t);
        const float mean = __double2float_rn(__ddiv_rn((double)total, (double)n));
        for (int64_t i = s0 + lane; i < s1; i += 32) out[i] = __fsub_rn((float)x[i], mean);
        return;
    }
    const double inv_full = __ddiv_rn(1.0, (double)(2 * h + 1));
    // window sum at s0 over [lo, hi]: whole 256-sample blocks plus the two partial ends
    const int64_t lo = s0 - h > 0 ? s0 - h : 0, hi = s0 + h < n - 1 ? s0 + h : n - 1;
    const int64_t blo = (lo + BW_BLK - 1) / BW_BLK, bhi = (hi + 1) / BW_BLK - 1;
    long long part = 0;
    if (blo <= bhi) {
        for (int64_t b = blo + lane; b <= bhi; b += 32) part += bs[b];
        for (int64_t i = lo + lane; i < blo * BW_BLK; i += 32) part += x[i];
        for (int64_t i = (bhi + 1) * BW_BLK + lane; i <= hi; i += 32) part += x[i];
    } else {
        for (int64_t i = lo + lane; i <= hi; i += 32) part += x[i];
    }
    long long carry = warp_sum_ll(part);  // S_{s0}; d_{s0} := 0 below
    if (s0 >= h + 4 && s1 - 1 + h <= n - 1 && (uint64_t)(s1 + h + 4) <= pitch) {
        // interior segment: every window is whole (one reciprocal), every x[i +- h] exists,
        // and the aligned 16-byte loads around them stay inside the row
        switch (h & 3) {  // the partners' misalignment (warp-uniform): aligned 16-byte loads
            case 0: baseline_interior<0>(x, out, s0, s1, (uint32_t)h, carry, inv_full, lane); break;
            case 1: baseline_interior<1>(x, out, s0, s1, (uint32_t)h, carry, inv_full, lane); break;
            case 2: baseline_interior<2>(x, out, s0, s1, (uint32_t)h, carry, inv_full, lane); break;
            default: baseline_interior<3>(x, out, s0, s1, (uint32_t)h, carry, inv_full, lane); break;
        }
        return;
    }
    for (int64_t base = s0; base < s1; base += 128) {
        long long d[4];
        int32_t xv[4];
        long long local = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t i = base + 4 * lane + k;
            long long di = 0;
            int32_t xi = 0;
            if (i < s1) {
                xi = x[i];
                if (i > s0) {
                    if (i + h < n) di += x[i + h];
                    if (i - 1 - h >= 0) di -= x[i - 1 - h];
                }
            }
            d[k] = di;
            xv[k] = xi;
            local += di;
        }
        long long incl = local;
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        long long run = carry + (incl - local);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t i = base + 4 * lane + k;
            run += d[k];
            if (i < s1) {
                const int64_t wlo = i - h > 0 ? i - h : 0;
                const int64_t whi = i + h < n - 1 ? i + h : n - 1;
                const int64_t cnt = whi - wlo + 1;
                // interior windows share one reciprocal; only the 2h edge samples divide
                const double inv = cnt == 2 * h + 1 ? inv_full : __ddiv_rn(1.0, (double)cnt);
                out[i] = __double2float_rn(__fma_rn(-(double)run, inv, (double)xv[k]));  // :45
            }
        }
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
}

// ---- baseline, float series: exact fixed point when provably exact -----------------
// The reference's running double window sum (src/detect.cpp:34-54) is order dependent in
// general, so a float series is replayed sequentially per trial (below).  But if every
// value is a multiple of 2^L and (2h+2) max|x| < 2^(53+L), every partial sum the reference
// forms is exactly representable, so its running sum equals the exact window sum -- which
// int64 fixed point (x * 2^-L) computes in any order.  f32_row_range_kernel measures L and
// the largest exponent per row; rows that pass run the parallel warp-segment algorithm,
// the rest (if any) the sequential replay.  Config E's masked float chunks all pass
// (sequential replay: 167 ms per 2^19-sample chunk, one uncoalesced thread per trial).
constexpr int FR_NOT_EXACT = -100000;

__global__ void __launch_bounds__(256)
    f32_row_range_kernel(const float* __restrict__ x_all, const uint32_t* __restrict__ row_len,
                         uint64_t pitch, uint64_t window, int* __restrict__ lmin_out) {
    __shared__ int s_lo[8], s_hi[8], s_bad[8];
    const uint32_t row = blockIdx.x;
    const int64_t n = row_len[row];
    const float* x = x_all + (size_t)row * pitch;
    int lo = 1 << 20, hi = -(1 << 20), bad = 0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t mag = __float_as_uint(x[i]) & 0x7fffffffu;
        if (mag == 0) continue;
        if (mag >= 0x7f800000u) { bad = 1; continue; }
        const int e = (int)(mag >> 23);
        const uint32_t m = e ? ((mag & 0x7fffffu) | 0x800000u) : (mag & 0x7fffffu);
        const int E = e ? e - 127 : -126;
        lo = min(lo, E - 23 + (__ffs((int)m) - 1));  // exponent of the lowest set bit
        hi = max(hi, E);                              // |x| < 2^(E+1)
    }
    for (int o = 16; o; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
        s_lo[threadIdx.x >> 5] = lo;
        s_hi[threadIdx.x >> 5] = hi;
        s_bad[threadIdx.x >> 5] = bad;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            lo = min(lo, s_lo[w]);
            hi = max(hi, s_hi[w]);
            bad |= s_bad[w];
        }
        int res;
        if (bad) {
            res = FR_NOT_EXACT;
        } else if (hi < lo) {  // all zero: L = 0 works
            res = 0;
        } else {
            // any partial sum is a sum of <= 2h+2 values of magnitude < 2^(hi+1)
            const uint64_t terms = 2 * (window / 2) + 2;
            int lg = 0;
            while ((1ull << lg) < terms) ++lg;
            res = (hi + 1 + lg <= 52 + lo) ? lo : FR_NOT_EXACT;
        }
        lmin_out[row] = res;
    }
}

__device__ __forceinline__ double pow2d(int k) {  // 2^k for |k| < 1000, exact
    return __longlong_as_double((long long)(1023 + k) << 52);
}

__device__ __forceinline__ long long f32_fixed(float v, double sc) {  // v * 2^-L, exact by the row check
    return __double2ll_rn(__dmul_rn((double)v, sc));
}

__global__ void __launch_bounds__(256)
    block256_sums_f32_kernel(const float* __restrict__ x_all, const uint32_t* __restrict__ row_len,
                             uint64_t pitch, uint32_t nrows, uint32_t nb, const int* __restrict__ lmin,
                             long long* __restrict__ bs) {
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= (uint64_t)nrows * nb) return;
    const uint32_t row = (uint32_t)(gw / nb), b = (uint32_t)(gw % nb);
    const int L = lmin[row];
    if (L == FR_NOT_EXACT) return;
    const double sc = pow2d(-L);
    const int64_t n = row_len[row];
    const int64_t lo = (int64_t)b * BW_BLK;
    long long s = 0;
    if (lo < n) {
        const float* x = x_all + (size_t)row * pitch;
        const int64_t hi = lo + BW_BLK < n ? lo + BW_BLK : n;
        for (int64_t i = lo + lane; i < hi; i += 32) s += f32_fixed(x[i], sc);
    }
    s = warp_sum_ll(s);
    if (lane == 0) bs[(size_t)row * nb + b] = s;
}

__global__ void __launch_bounds__(256)
    baseline_warp_f32_kernel(const float* __restrict__ x_all, float* __restrict__ out_all,
                             const uint32_t* __restrict__ row_len, uint64_t pitch, uint64_t window,
                             uint32_t nrows, uint32_t nseg, uint32_t nb, const long long* __restrict__ bsum,
                             const int* __restrict__ lmin) {
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= (uint64_t)nrows * nseg) return;
    const uint32_t row = (uint32_t)(gw / nseg), seg = (uint32_t)(gw % nseg);
    const int L = lmin[row];
    if (L == FR_NOT_EXACT) return;  // replayed sequentially by baseline_f32_kernel
    const double sc = pow2d(-L), usc = pow2d(L);
    const int64_t n = row_len[row];
    const int64_t s0 = (int64_t)seg * BW_SEG;
    if (s0 >= n) return;
    const int64_t s1 = s0 + BW_SEG < n ? s0 + BW_SEG : n;
    const float* x = x_all + (size_t)row * pitch;
    float* out = out_all + (size_t)row * pitch;
    const long long* bs = bsum + (size_t)row * nb;
    const int64_t h = (int64_t)(window / 2);
    if (h >= n - 1) {  // global-mean path: the 4-chain double sum is exact here too
        long long t = 0;
        for (int64_t b = lane; b * BW_BLK < n; b += 32) t += bs[b];
        const long long total = warp_sum_ll(t);
        const double tot = __dmul_rn((double)total, usc);
        const float mean = __double2float_rn(__ddiv_rn(tot, (double)n));
        for (int64_t i = s0 + lane; i < s1; i += 32) out[i] = __fsub_rn(x[i], mean);
        return;
    }
    const double inv_full = __ddiv_rn(1.0, (double)(2 * h + 1));
    const int64_t lo = s0 - h > 0 ? s0 - h : 0, hi = s0 + h < n - 1 ? s0 + h : n - 1;
    const int64_t blo = (lo + BW_BLK - 1) / BW_BLK, bhi = (hi + 1) / BW_BLK - 1;
    long long part = 0;
    if (blo <= bhi) {
        for (int64_t b = blo + lane; b <= bhi; b += 32) part += bs[b];
        for (int64_t i = lo + lane; i < blo * BW_BLK; i += 32) part += f32_fixed(x[i], sc);
        for (int64_t i = (bhi + 1) * BW_BLK + lane; i <= hi; i += 32) part += f32_fixed(x[i], sc);
    } else {
        for (int64_t i = lo + lane; i <= hi; i += 32) part += f32_fixed(x[i], sc);
    }
    long long carry = warp_sum_ll(part);  // S_{s0} in units of 2^L
    for (int64_t base = s0; base < s1; base += 128) {
        long long d[4];
        float xv[4];
        long long local = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t i = base + 4 * lane + k;
            long long di = 0;
            float xi = 0.0f;
            if (i < s1) {
                xi = x[i];
                if (i > s0) {
                    if (i + h < n) di += f32_fixed(x[i + h], sc);
                    if (i - 1 - h >= 0) di -= f32_fixed(x[i - 1 - h], sc);
                }
            }
            d[k] = di;
            xv[k] = xi;
            local += di;
        }
        long long incl = local;
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        long long run = carry + (incl - local);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t i = base + 4 * lane + k;
            run += d[k];
            if (i < s1) {
                const int64_t wlo = i - h > 0 ? i - h : 0;
                const int64_t whi = i + h < n - 1 ? i + h : n - 1;
                const int64_t cnt = whi - wlo + 1;
                const double inv = cnt == 2 * h + 1 ? inv_full : __ddiv_rn(1.0, (double)cnt);
                const double sum = __dmul_rn((double)run, usc);  // exact: |run| < 2^53
                out[i] = __double2float_rn(__fma_rn(-sum, inv, (double)xv[k]));  // :45
            }
        }
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
}

// ---- baseline: general float series (sequential replay, one thread per trial) ---

__global__ void baseline_f32_kernel(const float* __restrict__ x_all, float* __restrict__ out_all,
                                    const uint32_t* __restrict__ row_len, uint32_t nrows,
                                    uint64_t pitch, uint64_t window, const int* __restrict__ lmin) {
    const uint32_t row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= nrows) return;
    if (lmin && lmin[row] != FR_NOT_EXACT) return;  // done by the fixed-point kernels
    const uint64_t n = row_len[row];
    const float* x = x_all + (size_t)row * pitch;
    float* out = out_all + (size_t)row * pitch;
    if (n == 0) return;
    const uint64_t h = window / 2;
    if (h >= n - 1) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        uint64_t i = 0;
        for (; i + 4 <= n; i += 4) {
            a0 = __dadd_rn(a0, (double)x[i]);
            a1 = __dadd_rn(a1, (double)x[i + 1]);
            a2 = __dadd_rn(a2, (double)x[i + 2]);
            a3 = __dadd_rn(a3, (double)x[i + 3]);
        }
        for (; i < n; ++i) a0 = __dadd_rn(a0, (double)x[i]);
        const float mean =
            __double2float_rn(__ddiv_rn(__dadd_rn(__dadd_rn(a0, a1), __dadd_rn(a2, a3)), (double)n));
        for (uint64_t j = 0; j < n; ++j) out[j] = __fsub_rn(x[j], mean);
        return;
    }
    double sum = 0.0;
    uint64_t count = h + 1;
    for (uint64_t j = 0; j < count; ++j) sum = __dadd_rn(sum, (double)x[j]);
    for (uint64_t i = 0; i < n; ++i) {
        const double inv = __ddiv_rn(1.0, (double)count);
        out[i] = __double2float_rn(__fma_rn(-sum, inv, (double)x[i]));
        if (i + 1 + h < n) {
            sum = __dadd_rn(sum, (double)x[i + 1 + h]);
            ++count;
        }
        if (i >= h) {
            sum = __dsub_rn(sum, (double)x[i - h]);
            --count;
        }
    }
}

// ---- robust RMS: 4 sequential chains per trial ----------------------------------

template <int KIND>
__device__ __forceinline__ float load_x(const void* base, size_t idx) {
    if (KIND == 1) return (float)static_cast<const int32_t*>(base)[idx];
    return static_cast<const float*>(base)[idx];
}

// One warp = 8 trials x 4 chains.  The chains are strictly sequential (the
// reference's rounding order), so the kernel's job is to keep each chain's DADD
// dependency fed: the 8 rows stream through a 3-stage cp.async ring in shared
// memory (rows padded by 4 floats so the 32 lanes hit 32 banks), and each lane
// reads 16 values ahead of its add chain.  Both passes (sum of squares, then the
// 3-sigma-clipped sum) run in the same kernel.
constexpr int RMS_TR = 8;          // trials per warp
// Warps per block is a launch choice: the chains are latency-bound, so when the kernel
// runs beside the next chunk's dedispersion it packs up to 16 warps per block (~8
// blocks) onto few SMs with short stages (RT = 128 samples per trial); when it is on
// the critical path it spreads one warp per block with long stages (RT = 512).
constexpr int RMS_WARPS = 16;
#ifndef RMS_U
#define RMS_U 16  // values loaded and converted ahead of the add chain
#endif

template <int RT, int NST>
constexpr size_t rms_warp_smem() { return (size_t)NST * RMS_TR * (RT + 4) * sizeof(float); }

// NST: cp.async ring stages per warp (a lone warp on an SM needs a deep ring to keep
// enough bytes in flight for its 8 trials)
template <int KIND, int RT, int NST>
__global__ void __launch_bounds__(32 * RMS_WARPS)
    rms_kernel(const void* __restrict__ x_all, const uint32_t* __restrict__ row_len, uint32_t nrows,
               uint64_t pitch, float* __restrict__ frms, uint8_t* __restrict__ status) {
    constexpr int LD = RT + 4;      // padded row length (floats): the 32 lanes hit 32 banks
    constexpr int Q = RT / 128;     // float4 copies per lane per row and stage
    extern __shared__ __align__(16) float rsm_all[];  // [warps][NST][RMS_TR][LD]
    const int lane = threadIdx.x & 31, tr = lane >> 2, k = lane & 3;
    const uint32_t wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    float* rsm = rsm_all + (size_t)(threadIdx.x >> 5) * NST * RMS_TR * LD;
    const uint32_t row0 = wg * RMS_TR;
    if (row0 >= nrows) return;  // whole warp idle (warp-level code only below)
    const uint32_t row = row0 + tr;
    const bool live = row < nrows;
    const uint64_t n = live ? row_len[row] : 0;
    const uint64_t nq4 = n & ~3ull;  // elements covered by the 4-chain loop
    uint64_t nmax = n;
    for (int o = 16; o; o >>= 1) nmax = max(nmax, (uint64_t)__shfl_xor_sync(0xffffffffu, nmax, o));
    const uint64_t nstages = (nmax + RT - 1) / RT;
    // source rows of this warp's 8 trials (rows past nrows repeat the last one)
    const float* rowp[RMS_TR];
#pragma unroll
    for (int r = 0; r < RMS_TR; ++r)
        rowp[r] = static_cast<const float*>(x_all) + (size_t)min(row0 + r, nrows - 1) * pitch + 4 * lane;

    auto issue = [&](uint64_t st) {
        if (st < nstages) {
            float* dst = rsm + (st % NST) * RMS_TR * LD + 4 * lane;
#pragma unroll
            for (int r = 0; r < RMS_TR; ++r)
#pragma unroll
                for (int q = 0; q < Q; ++q)
                    __pipeline_memcpy_async(dst + r * LD + 128 * q, rowp[r] + st * RT + 128 * q, 16);
        }
        __pipeline_commit();
    };

    double a = 0.0, b = 0.0;
    uint32_t kept = 0;  // samples kept by one chain (< 2^32: series lengths are 32-bit)
    float cut = 0.0f;
    double rms0 = 0.0;
    for (int pass = 0; pass < 2; ++pass) {
        for (int st = 0; st < NST - 1; ++st) issue(st);
        for (uint64_t st = 0; st < nstages; ++st) {
            issue(st + NST - 1);
            __pipeline_wait_prior(NST - 1);
            __syncwarp();
            const float* t = rsm + (st % NST) * RMS_TR * LD + tr * LD;
            const uint64_t i0 = st * RT;
            const int jmax = nq4 > i0 ? (int)min((uint64_t)RT, nq4 - i0) : 0;
            int j = k;
            for (; j + 4 * (RMS_U - 1) < jmax; j += 4 * RMS_U) {  // RMS_U values ahead of the chain
                float v[RMS_U];
#pragma unroll
                for (int u = 0; u < RMS_U; ++u) {
                    const float f = t[j + 4 * u];
                    v[u] = KIND == 1 ? (float)__float_as_int(f) : f;
                }
                // double(v)*double(v) is exact (24+24 significant bits), so the
                // reference's a += v*v (one rounding) is one DFMA, or an exact DMUL off
                // the chain plus one DADD on it.  Pass 2 skips clipped samples with a
                // predicated DADD: b is a sum of squares (never -0), so skipping equals the
                // reference's adding nothing.
#pragma unroll
                for (int u = 0; u < RMS_U; ++u) {
                    const double dv = (double)v[u];
                    if (pass == 0) {
                        a = __fma_rn(dv, dv, a);
                    } else if (fabsf(v[u]) <= cut) {  // b + 0.0 == b: skipping the add is the same
                        b = __dadd_rn(b, __dmul_rn(dv, dv));
                        ++kept;
                    }
                }
            }
            for (; j < jmax; j += 4) {
                const float f = t[j];
                const float vv = KIND == 1 ? (float)__float_as_int(f) : f;
                const double sq = __dmul_rn((double)vv, (double)vv);
                if (pass == 0) {
                    a = __dadd_rn(a, sq);
                } else if (fabsf(vv) <= cut) {
                    b = __dadd_rn(b, sq);
                    ++kept;
                }
            }
            __syncwarp();
        }
        __pipeline_wait_prior(0);
        // tail (< 4 elements) into chain 0, src/detect.cpp:76 / :100-105
        if (k == 0 && live)
            for (uint64_t i = nq4; i < n; ++i) {
                const size_t idx = (size_t)row * pitch + i;
                const float vv = KIND == 1 ? (float)static_cast<const int32_t*>(x_all)[idx]
                                           : static_cast<const float*>(x_all)[idx];
                const double sq = __dmul_rn((double)vv, (double)vv);
                if (pass == 0) {
                    a = __dadd_rn(a, sq);
                } else if (fabsf(vv) <= cut) {
                    b = __dadd_rn(b, sq);
                    ++kept;
                }
            }
        const double x = pass == 0 ? a : b;
        const double x1 = __shfl_down_sync(0xffffffffu, x, 1, 4);
        const double x2 = __shfl_down_sync(0xffffffffu, x, 2, 4);
        const double x3 = __shfl_down_sync(0xffffffffu, x, 3, 4);
        double tot = __dadd_rn(__dadd_rn(x, x1), __dadd_rn(x2, x3));  // (a0+a1)+(a2+a3)
        tot = __shfl_sync(0xffffffffu, tot, lane & ~3);
        if (pass == 0) {
            rms0 = __dsqrt_rn(__ddiv_rn(tot, (double)n));
            cut = __double2float_rn(__dmul_rn(3.0, rms0));
        } else {
            unsigned long long kt = kept;
            kt += (unsigned long long)__shfl_down_sync(0xffffffffu, kept, 1, 4);
            kt += (unsigned long long)__shfl_down_sync(0xffffffffu, kept, 2, 4);
            kt += (unsigned long long)__shfl_down_sync(0xffffffffu, kept, 3, 4);
            if (live && k == 0) {
                uint8_t stt = 0;
                double rms = rms0;
                if (n < 2 || rms0 == 0.0) {
                    stt = 1;
                } else {
                    if (kt) rms = __dsqrt_rn(__ddiv_rn(tot, (double)kt));
                    if (rms == 0.0) stt = 1;
                }
                status[row] = stt;
                frms[row] = __double2float_rn(rms);
            }
        }
    }
}

// ---- boxcar ladder + threshold runs -----------------------------------------------

struct PeakCtx {
    const uint32_t* active;
    const double* dms;
    ChainParams cp;
    pgb_candidate* cands;
    unsigned long long* n_cands;
    uint64_t cand_cap;
    Fragment* frags;
    unsigned long long* n_frags;
    uint64_t frag_cap;
};

// Warp-aggregated append: the lanes emitting together take consecutive slots with one
// atomicAdd by the first of them (the buffer is sorted by a unique key afterwards, so the
// slot order does not matter).
__device__ __forceinline__ unsigned long long warp_slot(unsigned long long* counter) {
    const cg::coalesced_group g = cg::coalesced_threads();
    unsigned long long base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(counter, (unsigned long long)g.size());
    return g.shfl(base, 0) + g.thread_rank();
}

__device__ void emit_candidate(const PeakCtx& c, uint32_t row, uint32_t level, uint64_t m,
                               uint64_t b, uint64_t e, uint64_t pk, double pv) {
    const ChainParams& cp = c.cp;
    if (cp.drop_left && b == 0) return;           // src/detect.cpp:235
    if (cp.drop_right && e == m - 1) return;      // :236
    const uint64_t abs_peak = cp.start_sample + pk;
    if (abs_peak < cp.valid_begin || abs_peak >= cp.valid_end) return;  // :237-238
    const unsigned long long slot = warp_slot(c.n_cands);
    if (slot >= c.cand_cap) return;
    pgb_candidate out;
    out.snr = __double2float_rn(pv);
    out._pad0 = 0;
    out.peak_sample = abs_peak;
    out.time_s = __dmul_rn((double)abs_peak, cp.tsamp);
    out.width_index = level;
    out._pad1 = 0;
    out.width_samples = 1ull << level;
    const uint32_t trial = c.active[row];
    out.dm_trial = trial;
    out._pad2 = 0;
    out.dm = c.dms[trial];
    out.begin_sample = cp.start_sample + b;
    out.end_sample = cp.start_sample + e;
    c.cands[slot] = out;
}

__device__ void emit_fragment(const PeakCtx& c, uint32_t row, uint32_t level, uint64_t b,
                              uint64_t e, uint64_t pk, double pv) {
    const unsigned long long slot = warp_slot(c.n_frags);
    if (slot >= c.frag_cap) return;
    Fragment f;
    f.key = (uint64_t)row << 40 | (uint64_t)level << 35 | b;
    f.row = row;
    f.level = level;
    f.begin = b;
    f.end = e;
    f.peak = pk;
    f.peak_v = pv;
    c.frags[slot] = f;
}

// One ladder level whose partner element is H registers further in the same thread
// (k ascending: r[k + H] is read before it is updated).  Partners past the tile add 0;
// they only feed outputs beyond the tile's T valid ones.
template <int S, int H>
__device__ __forceinline__ void ladder_regs(double (&r)[S]) {
#pragma unroll
    for (int k = 0; k < S; ++k) r[k] = __dadd_rn(r[k], k + H < S ? r[k + H] : 0.0);  // :219
}

template <int KIND, int S>
__device__ __forceinline__ void boxcar_tile(const void* __restrict__ x_all, const uint32_t* __restrict__ row_len,
                                            const float* __restrict__ frms_all, const uint8_t* __restrict__ status,
                                            uint64_t pitch, uint64_t bmax, const double* __restrict__ scale,
                                            const PeakCtx& ctx, double* __restrict__ lvl_out, const uint32_t row,
                                            const uint32_t tile) {
    constexpr int N = BX_THREADS * S;
    // S == 16 (boxcar_max <= 4096): each buffer carries a zero pad of N/4 >= max half so
    // the shifted read needs no bounds test; S == 24 (8192) tests instead (smem limit).
    constexpr bool kPad = S == 16;
    constexpr uint32_t LD = kPad ? N + N / 4 : N;
    extern __shared__ double sbuf[];  // ping-pong [2][LD]
    if (status[row]) return;
    const uint64_t n = row_len[row];
    const uint32_t T = N - (uint32_t)bmax;
    const uint64_t i0 = (uint64_t)tile * T;
    if (i0 >= n) return;
    const float frms = frms_all[row];
    const int tid = threadIdx.x;
    const double thr = ctx.cp.threshold;
    double* cur = sbuf;
    double* nxt = sbuf + LD;
    // valid input samples of this tile (32-bit from here on)
    const uint32_t nin = (uint32_t)(n - i0 < (uint64_t)N ? n - i0 : (uint64_t)N);
    const size_t base = (size_t)row * pitch + i0;

    // all S loads in flight before the first division (the division's slow-path call
    // would otherwise serialise one global latency per element)
    float xin[S];
#pragma unroll
    for (int k = 0; k < S; ++k) {
        const uint32_t j = tid + BX_THREADS * k;
        xin[k] = j < nin ? load_x<KIND>(x_all, base + j) : 0.0f;
    }
    double r[S];
#pragma unroll
    for (int k = 0; k < S; ++k) {
        const uint32_t j = tid + BX_THREADS * k;
        const double v = j < nin ? (double)__fdiv_rn(xin[k], frms) : 0.0;  // :211
        r[k] = v;
        cur[j] = v;
    }
    if (kPad)
        for (uint32_t j = N + tid; j < LD; j += BX_THREADS) cur[j] = nxt[j] = 0.0;

    // One barrier per level: level l reads `cur` (written at l-1, published by
    // l-1's __syncthreads_or) and writes `nxt`, which nobody reads until l's barrier.
    uint32_t level = 0;
    for (uint64_t w = 1; w <= bmax && w <= n; w <<= 1, ++level) {
        const uint64_t m = n - w + 1;
        const uint32_t half = (uint32_t)(w >> 1);
        // half >= BX_THREADS: element j + half = tid + BX_THREADS (k + half / BX_THREADS)
        // is this thread's own register; the level needs no shared memory (cur is only
        // refreshed when a scan needs it)
        const bool in_regs = half >= (uint32_t)BX_THREADS;
        if (in_regs) {
            switch (half / BX_THREADS) {
                case 1: ladder_regs<S, 1>(r); break;
                case 2: ladder_regs<S, 2>(r); break;
                case 4: ladder_regs<S, 4>(r); break;
                case 8: ladder_regs<S, 8>(r); break;
                default: ladder_regs<S, S>(r); break;  // beyond the tile: adds zeros
            }
        } else if (w > 1) {
            // cur and nxt are distinct buffers: read a batch of shifted values before
            // storing any of them, so the LDS latencies overlap instead of serialising
            // behind the stores the compiler cannot prove independent
            const double* __restrict__ src = cur;
            double* __restrict__ dst = nxt;
            constexpr int HB = 8;
#pragma unroll
            for (int k0 = 0; k0 < S; k0 += HB) {
                double sh[HB];
#pragma unroll
                for (int q = 0; q < HB; ++q) {
                    const uint32_t j = tid + BX_THREADS * (k0 + q);
                    sh[q] = (kPad || j + half < N) ? src[j + half] : 0.0;
                }
#pragma unroll
                for (int q = 0; q < HB; ++q) {
                    const uint32_t j = tid + BX_THREADS * (k0 + q);
                    r[k0 + q] = __dadd_rn(r[k0 + q], sh[q]);  // :219
                    dst[j] = r[k0 + q];
                }
            }
            double* t = cur;
            cur = nxt;
            nxt = t;
        }
        const double sc = scale[level];
        const uint32_t lim2 = m > i0 ? (uint32_t)(m - i0 < (uint64_t)T ? m - i0 : (uint64_t)T) : 0;  // valid local outputs
        int any = 0;
#pragma unroll
        for (int k = 0; k < S; ++k) {
            const uint32_t j = tid + BX_THREADS * k;
            any |= (j < lim2) & (__dmul_rn(r[k], sc) > thr);
        }
        if (__syncthreads_or(any)) {
            if (in_regs) {  // publish the register level for the strip scan
#pragma unroll
                for (int k = 0; k < S; ++k) cur[tid + BX_THREADS * k] = r[k];
                __syncthreads();
            }
            // contiguous strip scan: thread owns [tid*S, tid*S + S) of the tile
            const uint32_t lo = (uint32_t)tid * S;
            const uint32_t hi = min(lo + S, lim2);
            bool in_run = false;
            uint32_t rb = 0, pk = 0;
            double pv = 0.0;
            for (uint32_t j = lo; j < hi; ++j) {
                const double v = __dmul_rn(cur[j], sc);
                if (v > thr) {
                    if (!in_run) {
                        in_run = true;
                        rb = j;
                        pk = j;
                        pv = v;
                    } else if (v > pv) {
                        pk = j;
                        pv = v;
                    }
                } else if (in_run) {
                    in_run = false;
                    const bool left_open = rb == lo && i0 + lo > 0;
                    if (left_open)
                        emit_fragment(ctx, row, level, i0 + rb, i0 + j - 1, i0 + pk, pv);
                    else
                        emit_candidate(ctx, row, level, m, i0 + rb, i0 + j - 1, i0 + pk, pv);
                }
            }
            if (in_run) {
                const bool left_open = rb == lo && i0 + lo > 0;
                const bool right_open = i0 + hi < m;
                if (left_open || right_open)
                    emit_fragment(ctx, row, level, i0 + rb, i0 + hi - 1, i0 + pk, pv);
                else
                    emit_candidate(ctx, row, level, m, i0 + rb, i0 + hi - 1, i0 + pk, pv);
            }
        }
    }
    // boxcar_max beyond the tile ladder: hand the top level (w = bmax, valid for the
    // tile's first T outputs) to boxcar_level_kernel through global memory
    if (lvl_out && n >= bmax) {
        const uint64_t m = n - bmax + 1;
        const uint32_t lim2 = m > i0 ? (uint32_t)(m - i0 < (uint64_t)T ? m - i0 : (uint64_t)T) : 0;
        double* dst = lvl_out + base;
#pragma unroll
        for (int k = 0; k < S; ++k) {
            const uint32_t j = tid + BX_THREADS * k;
            if (j < lim2) dst[j] = r[k];
        }
    }
}

// The reference's doubling tree level by level in shared memory (src/detect.cpp:216-221),
// for every (row, tile) of the grid, or -- list mode -- for the tiles the prefix kernel
// could not prove exact.
template <int KIND, int S>
__global__ void __launch_bounds__(BX_THREADS)
    boxcar_peaks_kernel(const void* __restrict__ x_all, const uint32_t* __restrict__ row_len,
                        const float* __restrict__ frms_all, const uint8_t* __restrict__ status,
                        uint64_t pitch, uint64_t bmax, const double* __restrict__ scale,
                        PeakCtx ctx, double* __restrict__ lvl_out, const uint2* __restrict__ list,
                        const unsigned* __restrict__ nlist) {
    if (!list) {
        boxcar_tile<KIND, S>(x_all, row_len, frms_all, status, pitch, bmax, scale, ctx, lvl_out, blockIdx.x,
                             blockIdx.y);  // rows on x: more than 65535 trials are legal
        return;
    }
    const unsigned cnt = *nlist;
    for (unsigned i = blockIdx.x; i < cnt; i += gridDim.x) {
        const uint2 t = list[i];
        boxcar_tile<KIND, S>(x_all, row_len, frms_all, status, pitch, bmax, scale, ctx, lvl_out, t.x, t.y);
        __syncthreads();  // the next tile reuses the shared buffers
    }
}

// ---- prefix-sum boxcar ------------------------------------------------------------
// The tree sums of a level are sums of contiguous ranges of s = double(x / rms).  If every
// s of a tile is a multiple of 2^L and every prefix sum of the tile is below 2^51 * 2^L in
// magnitude, each partial sum the tree forms (a range sum, |.| < 2^52 * 2^L) is exactly
// representable, so every level value IS the exact range sum P[j + w] - P[j] of the
// tile's prefix sums -- which are then exact in double as well.  The kernel checks that per
// tile (the values are floats, so it holds unless a tile mixes magnitudes ~2^24 apart;
// a rounded prefix sum would show up as |P| >= 2^51 * 2^L), then tests each level as one DADD +
// DSETP against an exact cut (fl(d * sc) > thr <=> d > cut_w, d a multiple of 2^L): no
// level-to-level dependency, no barrier or shared-memory write per level.  Levels w >= 8
// first bound a whole strip -- max P over its partners' strips minus min P over its own
// outputs -- and compute the strip only when the bound reaches the cut (rare for noise).
// Runs are scanned per thread strip, as in the tree kernel, only for the levels some
// element exceeds; tiles that fail the check go to boxcar_peaks_kernel (list mode).
__device__ __forceinline__ uint32_t XP(uint32_t j) { return j + (j >> 5); }

template <int KIND, int S>
__global__ void __launch_bounds__(BX_THREADS)
    boxcar_prefix_kernel(const void* __restrict__ x_all, const uint32_t* __restrict__ row_len,
                         const float* __restrict__ frms_all, const uint8_t* __restrict__ status,
                         uint64_t pitch, uint64_t bmax, const double* __restrict__ scale, PeakCtx ctx,
                         double* __restrict__ lvl_out, uint2* __restrict__ fb_list, unsigned* __restrict__ fb_n) {
    constexpr int N = BX_THREADS * S;
    constexpr int NW = BX_THREADS / 32;
    extern __shared__ __align__(16) uint8_t bsm[];
    // shared arrays padded by one element per 32 (XP): the strip accesses of a warp (stride
    // S elements) spread over the banks instead of hitting 2-8 of them
    double* P = reinterpret_cast<double*>(bsm);                     // [XP(N) + 1]: P[XP(j)] = sum s[0..j)
    float* xs = reinterpret_cast<float*>(P + XP(N) + 2);            // [XP(N)] the tile's inputs
    __shared__ double s_tot[NW], s_amax[NW], s_cut[32];
    __shared__ double s_smax[BX_THREADS + 2], s_smin[BX_THREADS + 2];  // per strip extremes of P
    __shared__ float s_fmax[NW], s_fmin[NW];
    __shared__ unsigned s_mask;
    const uint32_t row = blockIdx.x, tile = blockIdx.y;
    if (status[row]) return;
    const uint32_t n = row_len[row];  // series lengths and tile starts are 32-bit (row_len)
    const uint32_t T = N - (uint32_t)bmax;
    const uint32_t i0 = tile * T;
    if (i0 >= n) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float frms = frms_all[row];
    const uint32_t nin = min(n - i0, (uint32_t)N);
    const size_t base = (size_t)row * pitch + i0;
    // coalesced loads, staged so each thread can take a contiguous strip
    const uint32_t xp0 = XP(tid);  // XP(tid + 512 k) = XP(tid) + 528 k
#pragma unroll
    for (int k = 0; k < S; ++k) {
        const uint32_t j = tid + BX_THREADS * k;
        xs[xp0 + (BX_THREADS + BX_THREADS / 32) * k] = j < nin ? load_x<KIND>(x_all, base + j) : 0.0f;
    }
    if (tid == 0) s_mask = 0;
    __syncthreads();
    // strip [S*tid, S*tid + S): the reference's float quotients (:211), strip prefix in double
    const uint32_t j0 = (uint32_t)S * tid;
    double ps[S + 1];  // ps[k] = P[j0 + k]
    ps[0] = 0.0;
    float fhi = 0.0f, flo = INFINITY;  // largest |s| and smallest nonzero |s|
#pragma unroll
    for (int k = 0; k < S; ++k) {
        const float f = j0 + k < nin ? __fdiv_rn(xs[XP(j0 + k)], frms) : 0.0f;
        const float af = fabsf(f);  // (no -0 reaches here: series sums start at +0.0f, the
        // baseline's exact zeros are +0, so all-(-0) tree ranges cannot occur)
        fhi = fmaxf(fhi, af);
        flo = fminf(flo, af > 0.0f ? af : INFINITY);
        ps[k + 1] = __dadd_rn(ps[k], (double)f);
    }
    // block exclusive scan of the strip totals (exact when the tile passes the check)
    double tot = ps[S];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double v = __shfl_up_sync(0xffffffffu, tot, o);
        if (lane >= o) tot = __dadd_rn(tot, v);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        fhi = fmaxf(fhi, __shfl_xor_sync(0xffffffffu, fhi, o));
        flo = fminf(flo, __shfl_xor_sync(0xffffffffu, flo, o));
    }
    if (lane == 31) s_tot[warp] = tot;
    if (lane == 0) {
        s_fmax[warp] = fhi;
        s_fmin[warp] = flo;
    }
    __syncthreads();
    double off = __dsub_rn(tot, ps[S]);  // exclusive within the warp
    for (int w = 0; w < warp; ++w) off = __dadd_rn(off, s_tot[w]);
    fhi = s_fmax[0];
    flo = s_fmin[0];
#pragma unroll
    for (int w = 1; w < NW; ++w) {
        fhi = fmaxf(fhi, s_fmax[w]);
        flo = fminf(flo, s_fmin[w]);
    }
    // L: the lsb exponent of the smallest nonzero |s| bounds every value's lsb from below
    // (a float's lsb is 2^(e - 23), e its exponent, subnormals 2^-149)
    int L = 0;
    bool exact = !(fhi > 3.0e38f);  // inf / NaN: never exact
    if (flo < INFINITY) {
        const uint32_t be = __float_as_uint(flo) >> 23;
        L = (be ? (int)be - 127 : -126) - 23;
    }
    ps[0] = off;
    double smx = off, smn = off;
#pragma unroll
    for (int k = 1; k <= S; ++k) {
        ps[k] = __dadd_rn(ps[k], off);
        if (k < S) {
            smx = ps[k] > smx ? ps[k] : smx;
            smn = ps[k] < smn ? ps[k] : smn;
        }
    }
#pragma unroll
    for (int k = 0; k < S; ++k) P[XP(j0 + k)] = ps[k];
    double amax = fmax(fmax(fabs(smx), fabs(smn)), fabs(ps[S]));
    if (tid == BX_THREADS - 1) {  // P[N], then pseudo-strips past the tile
        P[XP(N)] = ps[S];
        s_smax[BX_THREADS] = s_smin[BX_THREADS] = ps[S];
        s_smax[BX_THREADS + 1] = -INFINITY;
        s_smin[BX_THREADS + 1] = INFINITY;
    }
    s_smax[tid] = smx;
    s_smin[tid] = smn;
#pragma unroll
    for (int o = 16; o; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if (lane == 0) s_amax[warp] = amax;
    // exact per-level cuts: cut_w = C 2^L with C the largest integer such that
    // fl(C 2^L sc_w) <= thr (monotone), so a multiple d of 2^L passes iff d > cut_w
    const uint32_t nlev = 32 - __clz((uint32_t)min(bmax, (uint64_t)n));
    const double thr = ctx.cp.threshold;
    const double p2l = ldexp(1.0, max(L, -1074)), p2nl = ldexp(1.0, min(-L, 1023));
    if (warp == 0 && (uint32_t)lane < nlev) {
        const double sc = scale[lane];
        const double lim = 9007199254740992.0;  // 2^53
        const double c0 = floor(__dmul_rn(thr / sc, p2nl));
        double c;
        if (!(c0 < lim)) c = lim;              // no level value reaches it
        else if (!(c0 > -lim)) c = -lim - 1.0;  // every level value passes
        else {
            c = c0;
            while (c + 1.0 < lim && !(__dmul_rn(__dmul_rn(c + 1.0, p2l), sc) > thr)) c += 1.0;
            while (c > -lim && __dmul_rn(__dmul_rn(c, p2l), sc) > thr) c -= 1.0;
        }
        s_cut[lane] = __dmul_rn(c, p2l);
    }
    __syncthreads();
    amax = s_amax[0];
#pragma unroll
    for (int w = 1; w < NW; ++w) amax = fmax(amax, s_amax[w]);
    // every value a multiple of 2^L (normal range), every prefix sum below 2^51 * 2^L: every
    // range sum (tree partial sums, the scan's partial totals) is then below 2^52 * 2^L, i.e.
    // representable, and a rounded one could not have hidden below the bound
    exact = exact && L >= -1000 && L <= 1000 && amax < ldexp(1.0, 51 + L);
    if (!exact) {  // block-uniform: the tree kernel takes this tile
        if (tid == 0) fb_list[atomicAdd(fb_n, 1u)] = make_uint2(row, tile);
        return;
    }
    // levels w <= 4: every output of the strip, d = P[j + w] - P[j] from the strip's registers
    // (partners past the strip from shared memory)
    uint32_t level = 0;
#pragma unroll
    for (int l = 0; l < 3; ++l) {
        const uint32_t w = 1u << l;
        if (w > bmax || w > n) continue;  // (levels stop at the first such w)
        const uint32_t m = n - (uint32_t)w + 1;
        const uint32_t lim2 = m > i0 ? min(m - i0, T) : 0;
        const double cut = s_cut[l];
        int any = 0;
#pragma unroll
        for (int k = 0; k < S; ++k) {
            const double hi = k + (int)w <= S ? ps[k + (int)w <= S ? k + w : 0] : P[XP(min(j0 + k + w, (uint32_t)N))];
            any |= (j0 + k < lim2) & (__dsub_rn(hi, ps[k]) > cut);
        }
        if (__any_sync(0xffffffffu, any) && lane == 0) atomicOr(&s_mask, 1u << l);
        level = l + 1;
    }
    // levels w >= 8: a strip can hold an output above the cut only if max P over the strips
    // covering its partners [j0 + w, j0 + w + S) minus min P over its own outputs exceeds it
    for (uint32_t w = 8; w <= (uint32_t)bmax && w <= n && level < 32; w <<= 1, ++level) {
        const uint32_t m = n - (uint32_t)w + 1;
        const uint32_t lim2 = m > i0 ? min(m - i0, T) : 0;
        const double cut = s_cut[level];
        const uint32_t q = w / S;
        const uint32_t a = min((uint32_t)tid + q, (uint32_t)BX_THREADS + 1);
        const uint32_t b = min((uint32_t)tid + q + 1, (uint32_t)BX_THREADS + 1);
        int any = 0;
        if (j0 < lim2 && __dsub_rn(fmax(s_smax[a], s_smax[b]), s_smin[tid]) > cut) {
#pragma unroll
            for (int k = 0; k < S; ++k)
                any |= (j0 + k < lim2) & (__dsub_rn(P[XP(min(j0 + k + (uint32_t)w, (uint32_t)N))], ps[k]) > cut);
        }
        if (__any_sync(0xffffffffu, any) && lane == 0) atomicOr(&s_mask, 1u << level);
    }
    __syncthreads();
    // threshold runs of the flagged levels on contiguous strips, as the tree kernel (the
    // mask's set bits only: most tiles flag none)
    for (unsigned mask = s_mask; mask; mask &= mask - 1) {
        level = __ffs(mask) - 1;
        const uint32_t w = 1u << level;
        const uint32_t m = n - w + 1;
        const uint32_t lim2 = m > i0 ? min(m - i0, T) : 0;
        {
            const double sc = scale[level];
            const uint32_t lo = j0;
            const uint32_t hi = min(lo + S, lim2);
            bool in_run = false;
            uint32_t rb = 0, pk = 0;
            double pv = 0.0;
            for (uint32_t j = lo; j < hi; ++j) {
                // the exact level sum times 1/sqrt(w) (:219)
                const double v = __dmul_rn(__dsub_rn(P[XP(j + (uint32_t)w)], P[XP(j)]), sc);
                if (v > thr) {
                    if (!in_run) {
                        in_run = true;
                        rb = j;
                        pk = j;
                        pv = v;
                    } else if (v > pv) {
                        pk = j;
                        pv = v;
                    }
                } else if (in_run) {
                    in_run = false;
                    const bool left_open = rb == lo && i0 + lo > 0;
                    if (left_open)
                        emit_fragment(ctx, row, level, i0 + rb, i0 + j - 1, i0 + pk, pv);
                    else
                        emit_candidate(ctx, row, level, m, i0 + rb, i0 + j - 1, i0 + pk, pv);
                }
            }
            if (in_run) {
                const bool left_open = rb == lo && i0 + lo > 0;
                const bool right_open = i0 + hi < m;
                if (left_open || right_open)
                    emit_fragment(ctx, row, level, i0 + rb, i0 + hi - 1, i0 + pk, pv);
                else
                    emit_candidate(ctx, row, level, m, i0 + rb, i0 + hi - 1, i0 + pk, pv);
            }
        }
    }
    // boxcar_max beyond the tile ladder: the top level's exact values for the level kernel
    if (lvl_out && n >= bmax) {
        const uint32_t m = n - (uint32_t)bmax + 1;
        const uint32_t lim2 = m > i0 ? min(m - i0, T) : 0;
        double* dst = lvl_out + base;
#pragma unroll
        for (int k = 0; k < S; ++k) {
            const uint32_t j = tid + BX_THREADS * k;
            if (j < lim2) dst[j] = __dsub_rn(P[XP(j + (uint32_t)bmax)], P[XP(j)]);
        }
    }
}

// One ladder level above the tile kernel's (boxcar_max > 8192): out[i] = in[i] +
// in[i + half] for i < m_w = n - w + 1 (the reference's in-place ascending update,
// src/detect.cpp:216-221, reads the previous level at i + half, so out-of-place is the
// same), then the threshold runs of the level as in the tile kernel: a thread scans a
// strip of BXL_S consecutive outputs; runs inside it become candidates, runs touching a
// strip edge fragments for stitch_kernel.  HBM-bound: 16 B read + 8 B written per output.
constexpr int BXL_S = 16;
__global__ void __launch_bounds__(256)
    boxcar_level_kernel(const double* __restrict__ in, double* __restrict__ out,
                        const uint32_t* __restrict__ row_len, const uint8_t* __restrict__ status,
                        uint64_t pitch, uint32_t level, double sc, PeakCtx ctx) {
    const uint32_t row = blockIdx.x;
    if (status[row]) return;
    const uint64_t n = row_len[row];
    const uint64_t w = 1ull << level, half = w >> 1;
    if (n < w) return;
    const uint64_t m = n - w + 1;
    const uint64_t lo = ((uint64_t)blockIdx.y * blockDim.x + threadIdx.x) * BXL_S;
    if (lo >= m) return;
    const uint64_t hi = lo + BXL_S < m ? lo + BXL_S : m;
    const double* a = in + (size_t)row * pitch;
    double* o = out + (size_t)row * pitch;
    const double thr = ctx.cp.threshold;
    bool in_run = false;
    uint64_t rb = 0, pk = 0;
    double pv = 0.0;
    for (uint64_t j = lo; j < hi; ++j) {
        const double s = __dadd_rn(a[j], a[j + half]);  // :219
        o[j] = s;
        const double v = __dmul_rn(s, sc);
        if (v > thr) {
            if (!in_run) {
                in_run = true;
                rb = pk = j;
                pv = v;
            } else if (v > pv) {
                pk = j;
                pv = v;
            }
        } else if (in_run) {
            in_run = false;
            if (rb == lo && lo > 0) emit_fragment(ctx, row, level, rb, j - 1, pk, pv);
            else emit_candidate(ctx, row, level, m, rb, j - 1, pk, pv);
        }
    }
    if (in_run) {
        if ((rb == lo && lo > 0) || hi < m) emit_fragment(ctx, row, level, rb, hi - 1, pk, pv);
        else emit_candidate(ctx, row, level, m, rb, hi - 1, pk, pv);
    }
}

__global__ void stitch_kernel(const Fragment* __restrict__ f, uint64_t nf,
                              const uint32_t* __restrict__ row_len, PeakCtx ctx,
                              const unsigned long long* __restrict__ d_nf) {
    if (d_nf) nf = *d_nf < nf ? *d_nf : nf;  // device count, capped at the buffer (nf = cap)
    const uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= nf) return;
    const Fragment a = f[idx];
    if (idx > 0) {
        const Fragment& p = f[idx - 1];
        if (p.row == a.row && p.level == a.level && p.end + 1 == a.begin) return;  // not a head
    }
    uint64_t e = a.end, pk = a.peak;
    double pv = a.peak_v;
    for (uint64_t g = idx + 1; g < nf; ++g) {
        const Fragment& q = f[g];
        if (q.row != a.row || q.level != a.level || q.begin != e + 1) break;
        if (q.peak_v > pv) {  // strict: the earliest maximum wins (src/detect.cpp:286)
            pv = q.peak_v;
            pk = q.peak;
        }
        e = q.end;
    }
    const uint64_t n = row_len[a.row];
    const uint64_t m = n - (1ull << a.level) + 1;
    emit_candidate(ctx, a.row, a.level, m, a.begin, e, pk, pv);
}

}  // namespace

void launch_baseline_int(const int32_t* x, float* out, const uint32_t* row_len, uint32_t nrows,
                         uint64_t pitch, uint64_t window, long long* block_sums, cudaStream_t st) {
    if (!nrows) return;
    if (!block_sums) {  // row-serial kernel (ablation: PGB_BASELINE_SERIAL=1)
        baseline_int_kernel<<<nrows, BL_THREADS, 0, st>>>(x, out, row_len, pitch, window);
    } else {
        const uint32_t nb = (uint32_t)((pitch + BW_BLK - 1) / BW_BLK);
        const uint32_t nseg = (uint32_t)((pitch + BW_SEG - 1) / BW_SEG);  // pitch >= every row length
        const uint64_t w1 = (uint64_t)nrows * nb, w2 = (uint64_t)nrows * nseg;
        block256_sums_kernel<<<(unsigned)((w1 * 32 + 255) / 256), 256, 0, st>>>(x, row_len, pitch, nrows, nb,
                                                                                 block_sums);
        baseline_warp_kernel<<<(unsigned)((w2 * 32 + 255) / 256), 256, 0, st>>>(x, out, row_len, pitch, window,
                                                                                nrows, nseg, nb, block_sums);
    }
    PGB_CUDA(cudaGetLastError());
}

size_t baseline_block_sums_bytes(uint32_t nrows, uint64_t pitch) {
    return (size_t)nrows * ((pitch + BW_BLK - 1) / BW_BLK) * sizeof(long long);
}

void launch_baseline_f32(const float* x, float* out, const uint32_t* row_len, uint32_t nrows,
                         uint64_t pitch, uint64_t window, long long* block_sums, int* row_lmin,
                         cudaStream_t st) {
    if (!nrows) return;
    if (block_sums && row_lmin) {  // exact rows in fixed point, the rest replayed below
        const uint32_t nb = (uint32_t)((pitch + BW_BLK - 1) / BW_BLK);
        const uint32_t nseg = (uint32_t)((pitch + BW_SEG - 1) / BW_SEG);
        const uint64_t w1 = (uint64_t)nrows * nb, w2 = (uint64_t)nrows * nseg;
        f32_row_range_kernel<<<nrows, 256, 0, st>>>(x, row_len, pitch, window, row_lmin);
        block256_sums_f32_kernel<<<(unsigned)((w1 * 32 + 255) / 256), 256, 0, st>>>(x, row_len, pitch, nrows, nb,
                                                                                     row_lmin, block_sums);
        baseline_warp_f32_kernel<<<(unsigned)((w2 * 32 + 255) / 256), 256, 0, st>>>(
            x, out, row_len, pitch, window, nrows, nseg, nb, block_sums, row_lmin);
    }
    baseline_f32_kernel<<<(nrows + 63) / 64, 64, 0, st>>>(x, out, row_len, nrows, pitch, window,
                                                          block_sums && row_lmin ? row_lmin : nullptr);
    PGB_CUDA(cudaGetLastError());
}

void launch_rms(const void* x, int kind, const uint32_t* row_len, uint32_t nrows, uint64_t pitch,
                float* frms, uint8_t* status, bool packed, cudaStream_t st) {
    if (!nrows) return;
    // packed: about 8 blocks (1001 trials: 16 warps each; a 125-trial shard: 2 each), so the
    // chains stay on few SMs without stacking so many warps per SM that they slow down
    const uint32_t nwarps = (nrows + RMS_TR - 1) / RMS_TR;
    const int nw = packed ? (int)std::min<uint32_t>(RMS_WARPS, std::max<uint32_t>(1, nwarps / 8)) : 1;
    const unsigned blocks = (nrows + RMS_TR * nw - 1) / (RMS_TR * nw);
#define PGB_RMS(K, RT, NS)                                                                         \
    do {                                                                                           \
        const size_t smem = (size_t)nw * rms_warp_smem<RT, NS>();                                  \
        PGB_CUDA(cudaFuncSetAttribute(rms_kernel<K, RT, NS>,                                       \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));    \
        rms_kernel<K, RT, NS><<<blocks, 32 * nw, smem, st>>>(x, row_len, nrows, pitch, frms, status); \
    } while (0)
    // a warp's ring: 99 KB at RT 512 x 6 stages (one warp per block), 12.4 KB at 128 x 3
    if (nw == 1) {
        if (kind == 1) PGB_RMS(1, 512, 6);
        else PGB_RMS(0, 512, 6);
    } else {
        if (kind == 1) PGB_RMS(1, 128, 3);
        else PGB_RMS(0, 128, 3);
    }
#undef PGB_RMS
    PGB_CUDA(cudaGetLastError());
}

void launch_boxcar_peaks(const void* x, int kind, const uint32_t* row_len, const float* frms,
                         const uint8_t* status, uint32_t nrows, uint64_t pitch, uint64_t max_len,
                         const ChainParams& cp, const uint32_t* active, const double* dms,
                         const double* scale, pgb_candidate* cands, unsigned long long* n_cands,
                         uint64_t cand_cap, Fragment* frags, unsigned long long* n_frags,
                         uint64_t frag_cap, double* levels, void* scratch, cudaStream_t st) {
    if (!nrows || !max_len) return;
    PeakCtx ctx{active, dms, cp, cands, n_cands, cand_cap, frags, n_frags, frag_cap};
    // boxcar_max > BX_TILE_MAX: the tile kernel runs the ladder to w = BX_TILE_LADDER and
    // stores that level; boxcar_level_kernel then doubles in global memory (ping-pong
    // `levels`, 2 x nrows x pitch doubles) up to boxcar_max
    const bool ext = cp.boxcar_max > BX_TILE_MAX;
    const uint64_t bmax = ext ? BX_TILE_LADDER : cp.boxcar_max;
    double* lvl_out = ext ? levels : nullptr;
    // 2 x N doubles must fit in 227 KB.  A tile yields N - bmax outputs, so for the
    // long ladders S = 24 (N = 12288, 1.5x halo overhead instead of 2x at bmax 4096)
    const int S = bmax <= 2048 ? 16 : 24;
    const uint64_t N = (uint64_t)BX_THREADS * S;
    const uint64_t LD = S == 16 ? N + N / 4 : N;
    const uint64_t T = N - bmax;
    const unsigned tiles = (unsigned)((max_len + T - 1) / T);
    const size_t smem = 2 * LD * sizeof(double);
    dim3 grid(nrows, tiles);
    // default: the prefix-sum kernel, then the tree kernel for the tiles it could not prove
    // exact (list mode, a device-side count); PGB_BOXCAR_TREE=1: the tree kernel everywhere
    const bool tree = pgb_ablation_env("PGB_BOXCAR_TREE") != nullptr;
    uint2* fb_list = reinterpret_cast<uint2*>(static_cast<char*>(scratch) + 16);
    unsigned* fb_n = static_cast<unsigned*>(scratch);
    if (!tree) {
        PGB_CUDA(cudaMemsetAsync(fb_n, 0, sizeof(unsigned), st));
        const size_t psm = (N + N / 32 + 2) * sizeof(double) + (N + N / 32) * sizeof(float);
#define PGB_BXP(K, SS)                                                                        \
    do {                                                                                      \
        PGB_CUDA(cudaFuncSetAttribute(boxcar_prefix_kernel<K, SS>,                            \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm)); \
        boxcar_prefix_kernel<K, SS><<<grid, BX_THREADS, psm, st>>>(x, row_len, frms, status, pitch, bmax, \
                                                                   scale, ctx, lvl_out, fb_list, fb_n); \
    } while (0)
        if (S == 16) {
            if (kind == 1) PGB_BXP(1, 16);
            else PGB_BXP(0, 16);
        } else {
            if (kind == 1) PGB_BXP(1, 24);
            else PGB_BXP(0, 24);
        }
#undef PGB_BXP
        PGB_CUDA(cudaGetLastError());
    }
    static const bool which = getenv("PGB_DD_WHICH") != nullptr;  // kernel-choice log (tests)
    if (which && !tree) {
        unsigned nfb = 0;
        PGB_CUDA(cudaMemcpyAsync(&nfb, fb_n, sizeof nfb, cudaMemcpyDeviceToHost, st));
        PGB_CUDA(cudaStreamSynchronize(st));
        fprintf(stderr, "pgb boxcar: prefix kernel, %u of %llu tiles to the tree kernel\n", nfb,
                (unsigned long long)nrows * tiles);
    }
    const dim3 tgrid = tree ? grid : dim3(148);  // list mode: one wave, looping over the list
    const uint2* lst = tree ? nullptr : fb_list;
#define PGB_BX(K, SS)                                                                        \
    do {                                                                                     \
        PGB_CUDA(cudaFuncSetAttribute(boxcar_peaks_kernel<K, SS>,                            \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        boxcar_peaks_kernel<K, SS><<<tgrid, BX_THREADS, smem, st>>>(x, row_len, frms, status, \
                                                                    pitch, bmax, scale, ctx, lvl_out, lst, fb_n); \
    } while (0)
    if (S == 16) {
        if (kind == 1) PGB_BX(1, 16);
        else PGB_BX(0, 16);
    } else {
        if (kind == 1) PGB_BX(1, 24);
        else PGB_BX(0, 24);
    }
#undef PGB_BX
    PGB_CUDA(cudaGetLastError());
    if (ext) {
        double* in = levels;
        double* out = levels + (size_t)nrows * pitch;
        uint32_t level = 0;
        while ((1ull << level) < bmax) ++level;
        for (uint64_t w = bmax << 1; w <= cp.boxcar_max && w <= max_len; w <<= 1) {
            ++level;
            const double sc = 1.0 / std::sqrt((double)(1ull << level));  // as the host table (src/engine.cpp:207)
            const uint64_t per = 256ull * BXL_S;
            dim3 g2(nrows, (unsigned)((max_len + per - 1) / per));
            boxcar_level_kernel<<<g2, 256, 0, st>>>(in, out, row_len, status, pitch, level, sc, ctx);
            PGB_CUDA(cudaGetLastError());
            std::swap(in, out);
        }
    }
}

size_t boxcar_scratch_bytes(uint32_t nrows, uint64_t max_len, uint64_t boxcar_max) {
    const uint64_t bmax = boxcar_max > BX_TILE_MAX ? BX_TILE_LADDER : boxcar_max;
    const uint64_t T = (uint64_t)BX_THREADS * (bmax <= 2048 ? 16 : 24) - bmax;
    return 16 + (size_t)nrows * ((max_len + T - 1) / T) * sizeof(uint2);
}

size_t boxcar_levels_bytes(uint64_t boxcar_max, uint32_t nrows, uint64_t pitch) {
    return boxcar_max > BX_TILE_MAX ? 2 * (size_t)nrows * pitch * sizeof(double) : 0;
}

void launch_stitch(const Fragment* frags_sorted, uint64_t nfrags, const uint32_t* row_len,
                   const ChainParams& cp, const uint32_t* active, const double* dms,
                   pgb_candidate* cands, unsigned long long* n_cands, uint64_t cand_cap,
                   cudaStream_t st) {
    if (!nfrags) return;
    PeakCtx ctx{active, dms, cp, cands, n_cands, cand_cap, nullptr, nullptr, 0};
    stitch_kernel<<<(unsigned)((nfrags + 255) / 256), 256, 0, st>>>(frags_sorted, nfrags, row_len,
                                                                   ctx, nullptr);
    PGB_CUDA(cudaGetLastError());
}

void launch_stitch_dev(const Fragment* frags_sorted, uint64_t frag_cap, const unsigned long long* d_nf,
                       const uint32_t* row_len, const ChainParams& cp, const uint32_t* active,
                       const double* dms, pgb_candidate* cands, unsigned long long* n_cands,
                       uint64_t cand_cap, cudaStream_t st) {
    if (!frag_cap) return;
    PeakCtx ctx{active, dms, cp, cands, n_cands, cand_cap, nullptr, nullptr, 0};
    stitch_kernel<<<(unsigned)((frag_cap + 255) / 256), 256, 0, st>>>(frags_sorted, frag_cap, row_len,
                                                                     ctx, d_nf);
    PGB_CUDA(cudaGetLastError());
}

}  // namespace pgb
