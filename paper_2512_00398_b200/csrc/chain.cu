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
#include "pgb_internal.h"

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
                const double inv = __ddiv_rn(1.0, (double)(hi - lo + 1));
                out[i] = __double2float_rn(__fma_rn(-(double)run, inv, (double)xv[k]));
            }
        }
        carry += wsum[(BL_THREADS >> 5) - 1];
    }
}

// ---- baseline: general float series (sequential replay, one thread per trial) ---

__global__ void baseline_f32_kernel(const float* __restrict__ x_all, float* __restrict__ out_all,
                                    const uint32_t* __restrict__ row_len, uint32_t nrows,
                                    uint64_t pitch, uint64_t window) {
    const uint32_t row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= nrows) return;
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

template <int KIND>
__global__ void rms_kernel(const void* __restrict__ x_all, const uint32_t* __restrict__ row_len,
                           uint32_t nrows, uint64_t pitch, float* __restrict__ frms,
                           uint8_t* __restrict__ status) {
    const uint32_t gt = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t row = gt >> 2;
    const int k = gt & 3;
    const bool live = row < nrows;
    const uint64_t n = live ? row_len[row] : 0;
    const size_t base = (size_t)(live ? row : 0) * pitch;
    const uint64_t nq = n / 4;  // full groups of 4

    // pass 1: a_k = sum over i = 4j + k of x^2, tail into chain 0
    double a = 0.0;
    {
        uint64_t j = 0;
        for (; j + 8 <= nq; j += 8) {
            float v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = load_x<KIND>(x_all, base + 4 * (j + u) + k);
#pragma unroll
            for (int u = 0; u < 8; ++u) a = __dadd_rn(a, __dmul_rn((double)v[u], (double)v[u]));
        }
        for (; j < nq; ++j) {
            const float v = load_x<KIND>(x_all, base + 4 * j + k);
            a = __dadd_rn(a, __dmul_rn((double)v, (double)v));
        }
        if (k == 0)
            for (uint64_t i = 4 * nq; i < n; ++i) {
                const float v = load_x<KIND>(x_all, base + i);
                a = __dadd_rn(a, __dmul_rn((double)v, (double)v));
            }
    }
    const unsigned mask = 0xffffffffu;
    const double a1 = __shfl_down_sync(mask, a, 1, 4);
    const double a2 = __shfl_down_sync(mask, a, 2, 4);
    const double a3 = __shfl_down_sync(mask, a, 3, 4);
    double sumsq = __dadd_rn(__dadd_rn(a, a1), __dadd_rn(a2, a3));  // valid on k == 0
    sumsq = __shfl_sync(mask, sumsq, 0, 4);
    const double rms0 = __dsqrt_rn(__ddiv_rn(sumsq, (double)n));
    const float cut = __double2float_rn(__dmul_rn(3.0, rms0));

    // pass 2: |x| <= cut
    double b = 0.0;
    unsigned long long kept = 0;
    {
        uint64_t j = 0;
        for (; j + 8 <= nq; j += 8) {
            float v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = load_x<KIND>(x_all, base + 4 * (j + u) + k);
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (fabsf(v[u]) <= cut) {
                    b = __dadd_rn(b, __dmul_rn((double)v[u], (double)v[u]));
                    ++kept;
                }
        }
        for (; j < nq; ++j) {
            const float v = load_x<KIND>(x_all, base + 4 * j + k);
            if (fabsf(v) <= cut) {
                b = __dadd_rn(b, __dmul_rn((double)v, (double)v));
                ++kept;
            }
        }
        if (k == 0)
            for (uint64_t i = 4 * nq; i < n; ++i) {
                const float v = load_x<KIND>(x_all, base + i);
                if (fabsf(v) <= cut) {
                    b = __dadd_rn(b, __dmul_rn((double)v, (double)v));
                    ++kept;
                }
            }
    }
    const double b1 = __shfl_down_sync(mask, b, 1, 4);
    const double b2 = __shfl_down_sync(mask, b, 2, 4);
    const double b3 = __shfl_down_sync(mask, b, 3, 4);
    unsigned long long kt = kept;
    kt += __shfl_down_sync(mask, kept, 1, 4);
    kt += __shfl_down_sync(mask, kept, 2, 4);
    kt += __shfl_down_sync(mask, kept, 3, 4);
    if (live && k == 0) {
        const double kept_sumsq = __dadd_rn(__dadd_rn(b, b1), __dadd_rn(b2, b3));
        uint8_t st = 0;
        double rms = rms0;
        if (n < 2 || rms0 == 0.0) {
            st = 1;
        } else {
            if (kt) rms = __dsqrt_rn(__ddiv_rn(kept_sumsq, (double)kt));
            if (rms == 0.0) st = 1;
        }
        status[row] = st;
        frms[row] = __double2float_rn(rms);
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

__device__ void emit_candidate(const PeakCtx& c, uint32_t row, uint32_t level, uint64_t m,
                               uint64_t b, uint64_t e, uint64_t pk, double pv) {
    const ChainParams& cp = c.cp;
    if (cp.drop_left && b == 0) return;           // src/detect.cpp:235
    if (cp.drop_right && e == m - 1) return;      // :236
    const uint64_t abs_peak = cp.start_sample + pk;
    if (abs_peak < cp.valid_begin || abs_peak >= cp.valid_end) return;  // :237-238
    const unsigned long long slot = atomicAdd(c.n_cands, 1ull);
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
    const unsigned long long slot = atomicAdd(c.n_frags, 1ull);
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

template <int KIND, int S>
__global__ void __launch_bounds__(BX_THREADS)
    boxcar_peaks_kernel(const void* __restrict__ x_all, const uint32_t* __restrict__ row_len,
                        const float* __restrict__ frms_all, const uint8_t* __restrict__ status,
                        uint64_t pitch, uint64_t bmax, const double* __restrict__ scale,
                        PeakCtx ctx) {
    constexpr int N = BX_THREADS * S;
    extern __shared__ double sbuf[];  // [N]
    const uint32_t row = blockIdx.y;
    if (status[row]) return;
    const uint64_t n = row_len[row];
    const uint64_t T = N - bmax;
    const uint64_t i0 = (uint64_t)blockIdx.x * T;
    if (i0 >= n) return;
    const float frms = frms_all[row];
    const size_t base = (size_t)row * pitch;
    const int tid = threadIdx.x;
    const double thr = ctx.cp.threshold;

    double r[S];
#pragma unroll
    for (int k = 0; k < S; ++k) {
        const uint64_t j = tid + (uint64_t)BX_THREADS * k;
        const uint64_t i = i0 + j;
        double v = 0.0;
        if (i < n) v = (double)__fdiv_rn(load_x<KIND>(x_all, base + i), frms);  // :211
        r[k] = v;
        sbuf[j] = v;
    }

    uint32_t level = 0;
    for (uint64_t w = 1; w <= bmax && w <= n; w <<= 1, ++level) {
        const uint64_t m = n - w + 1;
        if (w > 1) {
            const uint64_t half = w >> 1;
            double sh[S];
            __syncthreads();
#pragma unroll
            for (int k = 0; k < S; ++k) {
                const uint64_t j = tid + (uint64_t)BX_THREADS * k + half;
                sh[k] = j < N ? sbuf[j] : 0.0;
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < S; ++k) {
                r[k] = __dadd_rn(r[k], sh[k]);  // :219
                sbuf[tid + BX_THREADS * k] = r[k];
            }
        }
        const double sc = scale[level];
        const uint64_t lim2 = m > i0 ? (m - i0 < T ? m - i0 : T) : 0;  // valid local outputs
        int any = 0;
#pragma unroll
        for (int k = 0; k < S; ++k) {
            const uint64_t j = tid + (uint64_t)BX_THREADS * k;
            any |= (j < lim2) && (__dmul_rn(r[k], sc) > thr);
        }
        if (__syncthreads_or(any)) {
            // contiguous strip scan: thread owns [tid*S, tid*S + S) of the tile
            const uint64_t lo = (uint64_t)tid * S;
            const uint64_t hi = min(lo + S, lim2);
            bool in_run = false;
            uint64_t rb = 0, pk = 0;
            double pv = 0.0;
            for (uint64_t j = lo; j < hi; ++j) {
                const double v = __dmul_rn(sbuf[j], sc);
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
}

__global__ void stitch_kernel(const Fragment* __restrict__ f, uint64_t nf,
                              const uint32_t* __restrict__ row_len, PeakCtx ctx) {
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
                         uint64_t pitch, uint64_t window, cudaStream_t st) {
    if (!nrows) return;
    baseline_int_kernel<<<nrows, BL_THREADS, 0, st>>>(x, out, row_len, pitch, window);
    PGB_CUDA(cudaGetLastError());
}

void launch_baseline_f32(const float* x, float* out, const uint32_t* row_len, uint32_t nrows,
                         uint64_t pitch, uint64_t window, cudaStream_t st) {
    if (!nrows) return;
    baseline_f32_kernel<<<(nrows + 63) / 64, 64, 0, st>>>(x, out, row_len, nrows, pitch, window);
    PGB_CUDA(cudaGetLastError());
}

void launch_rms(const void* x, int kind, const uint32_t* row_len, uint32_t nrows, uint64_t pitch,
                float* frms, uint8_t* status, cudaStream_t st) {
    if (!nrows) return;
    const unsigned threads = 128;
    const unsigned blocks = (unsigned)((4ull * nrows + threads - 1) / threads);
    if (kind == 1)
        rms_kernel<1><<<blocks, threads, 0, st>>>(x, row_len, nrows, pitch, frms, status);
    else
        rms_kernel<0><<<blocks, threads, 0, st>>>(x, row_len, nrows, pitch, frms, status);
    PGB_CUDA(cudaGetLastError());
}

void launch_boxcar_peaks(const void* x, int kind, const uint32_t* row_len, const float* frms,
                         const uint8_t* status, uint32_t nrows, uint64_t pitch, uint64_t max_len,
                         const ChainParams& cp, const uint32_t* active, const double* dms,
                         const double* scale, pgb_candidate* cands, unsigned long long* n_cands,
                         uint64_t cand_cap, Fragment* frags, unsigned long long* n_frags,
                         uint64_t frag_cap, cudaStream_t st) {
    if (!nrows || !max_len) return;
    PeakCtx ctx{active, dms, cp, cands, n_cands, cand_cap, frags, n_frags, frag_cap};
    const uint64_t bmax = cp.boxcar_max;
    const int S = bmax <= 4096 ? 16 : 32;
    const uint64_t N = (uint64_t)BX_THREADS * S;
    const uint64_t T = N - bmax;
    const unsigned tiles = (unsigned)((max_len + T - 1) / T);
    const size_t smem = N * sizeof(double);
    dim3 grid(tiles, nrows);
#define PGB_BX(K, SS)                                                                        \
    do {                                                                                     \
        PGB_CUDA(cudaFuncSetAttribute(boxcar_peaks_kernel<K, SS>,                            \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        boxcar_peaks_kernel<K, SS><<<grid, BX_THREADS, smem, st>>>(x, row_len, frms, status, \
                                                                   pitch, bmax, scale, ctx); \
    } while (0)
    if (S == 16) {
        if (kind == 1) PGB_BX(1, 16);
        else PGB_BX(0, 16);
    } else {
        if (kind == 1) PGB_BX(1, 32);
        else PGB_BX(0, 32);
    }
#undef PGB_BX
    PGB_CUDA(cudaGetLastError());
}

void launch_stitch(const Fragment* frags_sorted, uint64_t nfrags, const uint32_t* row_len,
                   const ChainParams& cp, const uint32_t* active, const double* dms,
                   pgb_candidate* cands, unsigned long long* n_cands, uint64_t cand_cap,
                   cudaStream_t st) {
    if (!nfrags) return;
    PeakCtx ctx{active, dms, cp, cands, n_cands, cand_cap, nullptr, nullptr, 0};
    stitch_kernel<<<(unsigned)((nfrags + 255) / 256), 256, 0, st>>>(frags_sorted, nfrags, row_len,
                                                                   ctx);
    PGB_CUDA(cudaGetLastError());
}

}  // namespace pgb
