// Device RFI excision, bit-identical to the reference's
// flag_narrowband / flag_broadband / apply_mask (/root/reference/proj/src/rfi.cpp).
//
//   * channel statistics (:42-54): mean[c] = sum_i x (double, time order), then
//     var[c] += d*d with d = x - mean -- the reference build contracts this into a
//     fused multiply-add (vfmadd213pd), so each channel is one sequential thread with
//     __fma_rn.  Loads are coalesced across channels.
//   * zero-DM series (:74-80): per sample, sum over channels in ascending order in
//     double; samples are tiled through shared memory so each thread's sequential
//     sum reads conflict-free.
//   * medians and MADs (:10-28): exact order statistics from a device radix sort
//     (nth_element picks order statistics, so any exact selection agrees).
//   * apply_mask (:93-139): zero or local-mean replacement computed from the
//     original values, written into a separate float chunk.
#include <cuda_pipeline.h>
#include <cub/device/device_radix_sort.cuh>
#include <cstdlib>
#include <type_traits>

#include "pgb_internal.h"

namespace pgb {

namespace {

template <typename T>
__device__ __forceinline__ double cell(const T* x, size_t i) {
    return (double)(float)x[i];
}

template <typename T>
__global__ void chan_stats_kernel(const T* __restrict__ x, uint64_t n, uint32_t nch,
                                  double* __restrict__ mean, double* __restrict__ var) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nch) return;
    double s = 0.0;
    uint64_t i = 0;
    for (; i + 8 <= n; i += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = cell(x, (i + u) * nch + c);
#pragma unroll
        for (int u = 0; u < 8; ++u) s = __dadd_rn(s, v[u]);
    }
    for (; i < n; ++i) s = __dadd_rn(s, cell(x, i * nch + c));
    const double m = __ddiv_rn(s, (double)n);
    double a = 0.0;
    for (i = 0; i + 8 <= n; i += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __dsub_rn(cell(x, (i + u) * nch + c), m);
#pragma unroll
        for (int u = 0; u < 8; ++u) a = __fma_rn(v[u], v[u], a);  // contracted, src/rfi.cpp:51
    }
    for (; i < n; ++i) {
        const double d = __dsub_rn(cell(x, i * nch + c), m);
        a = __fma_rn(d, d, a);
    }
    mean[c] = m;
    var[c] = __ddiv_rn(a, (double)n);
}

// zero-DM: 128 samples per block; channel tiles of 32 staged transposed in smem.
template <typename T>
__global__ void zero_dm_kernel(const T* __restrict__ x, uint64_t n, uint32_t nch,
                               double* __restrict__ zdm) {
    __shared__ float tile[32][129];
    const uint64_t i0 = (uint64_t)blockIdx.x * 128;
    const int tid = threadIdx.x;  // 128 threads
    double s = 0.0;
    for (uint32_t c0 = 0; c0 < nch; c0 += 32) {
        __syncthreads();
        for (int k = tid; k < 128 * 32; k += 128) {
            const int r = k >> 5, cc = k & 31;
            const uint64_t i = i0 + r;
            tile[cc][r] = (i < n && c0 + cc < nch) ? (float)x[i * nch + c0 + cc] : 0.0f;
        }
        __syncthreads();
        const uint32_t lim = min(32u, nch - c0);
        for (uint32_t cc = 0; cc < lim; ++cc) s = __dadd_rn(s, (double)tile[cc][tid]);
    }
    if (i0 + tid < n) zdm[i0 + tid] = s;
}

// ---- 8-bit chunks: integer sums are exact in any order -------------------------------
// The reference's channel sums and zero-DM sums add doubles of 8-bit codes: every partial
// sum is an integer < 2^53, so the result is the exact integer sum however it is formed.
// Those two passes run HBM-parallel in integers; only the variance pass (an FMA chain whose
// rounding depends on order) stays one sequential chain per channel, fed from shared
// memory.  Fast paths need nch % 16 == 0 (16-byte rows); other shapes use the kernels above.
__global__ void chan_sum_u8_kernel(const uint8_t* __restrict__ x, uint64_t n, uint32_t nch,
                                   uint64_t rows_per, unsigned long long* __restrict__ sums) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;  // channel quad
    if (4 * q >= nch) return;
    const uint64_t r0 = (uint64_t)blockIdx.y * rows_per;
    const uint64_t r1 = r0 + rows_per < n ? r0 + rows_per : n;
    uint32_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;  // rows_per <= 2^24
    const uint32_t* src = reinterpret_cast<const uint32_t*>(x) + q;
    const uint32_t pitch = nch / 4;
#pragma unroll 8
    for (uint64_t r = r0; r < r1; ++r) {
        const uint32_t w = __ldg(src + r * pitch);
        a0 += w & 0xffu;
        a1 += (w >> 8) & 0xffu;
        a2 += (w >> 16) & 0xffu;
        a3 += w >> 24;
    }
    atomicAdd(sums + 4 * q + 0, (unsigned long long)a0);
    atomicAdd(sums + 4 * q + 1, (unsigned long long)a1);
    atomicAdd(sums + 4 * q + 2, (unsigned long long)a2);
    atomicAdd(sums + 4 * q + 3, (unsigned long long)a3);
}

// one warp per sample row: zdm[i] = exact sum of the row's codes
__global__ void zero_dm_u8_kernel(const uint8_t* __restrict__ x, uint64_t n, uint32_t nch,
                                  double* __restrict__ zdm) {
    const uint64_t row = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    const uint4* src = reinterpret_cast<const uint4*>(x + row * nch);
    uint32_t s = 0;
    for (uint32_t v = lane; v < nch / 16; v += 32) {
        const uint4 w = __ldg(src + v);
        s = __dp4a(w.x, 0x01010101u, s);
        s = __dp4a(w.y, 0x01010101u, s);
        s = __dp4a(w.z, 0x01010101u, s);
        s = __dp4a(w.w, 0x01010101u, s);
    }
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) zdm[row] = (double)s;
}

// var[c] = sum_i fma chain of (x - mean)^2 in time order (src/rfi.cpp:48-52), one thread
// per channel, 128 channels per CTA; rows staged 256 at a time through a 4-slot cp.async ring.
constexpr int CV_CH = 128, CV_ROWS = 256, CV_NS = 4;

__global__ void __launch_bounds__(CV_CH)
    chan_var_u8_kernel(const uint8_t* __restrict__ x, uint64_t n, uint32_t nch,
                       const unsigned long long* __restrict__ sums, double* __restrict__ mean,
                       double* __restrict__ var) {
    extern __shared__ __align__(16) uint8_t tile[];  // [CV_NS][CV_ROWS][CV_CH]
    const uint32_t c0 = blockIdx.x * CV_CH;
    const uint32_t cw = min((uint32_t)CV_CH, nch - c0);  // multiple of 16
    const uint32_t parts = cw / 16;
    const int tid = threadIdx.x;
    const uint32_t c = c0 + tid;
    const bool live = tid < (int)cw;
    const double m = live ? __ddiv_rn((double)sums[c], (double)n) : 0.0;
    const uint64_t nst = (n + CV_ROWS - 1) / CV_ROWS;
    auto issue = [&](uint64_t k) {
        if (k < nst) {
            const uint64_t r0 = k * CV_ROWS;
            const uint32_t rows = (uint32_t)min((uint64_t)CV_ROWS, n - r0);
            uint8_t* dst = tile + (size_t)(k % CV_NS) * CV_ROWS * CV_CH;
            for (uint32_t j = tid; j < rows * parts; j += CV_CH) {
                const uint32_t r = j / parts, pp = j % parts;
                __pipeline_memcpy_async(dst + r * CV_CH + 16 * pp, x + (r0 + r) * nch + c0 + 16 * pp, 16);
            }
        }
        __pipeline_commit();
    };
    for (int k = 0; k < CV_NS - 1; ++k) issue(k);
    double a = 0.0;
    for (uint64_t k = 0; k < nst; ++k) {
        __pipeline_wait_prior(CV_NS - 2);
        __syncthreads();
        issue(k + CV_NS - 1);  // into the slot stage k-1 used; everyone is past it
        const uint8_t* t = tile + (size_t)(k % CV_NS) * CV_ROWS * CV_CH + tid;
        const uint32_t rows = (uint32_t)min((uint64_t)CV_ROWS, n - k * CV_ROWS);
        if (live) {
            if (rows == CV_ROWS) {
#pragma unroll 16
                for (int r = 0; r < CV_ROWS; ++r) {
                    const double d = __dsub_rn((double)t[r * CV_CH], m);
                    a = __fma_rn(d, d, a);
                }
            } else {
                for (uint32_t r = 0; r < rows; ++r) {
                    const double d = __dsub_rn((double)t[r * CV_CH], m);
                    a = __fma_rn(d, d, a);
                }
            }
        }
    }
    if (live) {
        mean[c] = m;
        var[c] = __ddiv_rn(a, (double)n);
    }
}

// widen to float with bad channels already zeroed (apply_mask's column rule), 4 cells a thread
template <typename T>
__global__ void widen_rows_kernel(const T* __restrict__ x, uint64_t n, uint32_t nch,
                                  const uint8_t* __restrict__ chan_bad, float* __restrict__ out) {
    const uint32_t q4 = nch / 4;
    for (uint64_t r = blockIdx.x; r < n; r += gridDim.x) {
        for (uint32_t q = threadIdx.x; q < q4; q += blockDim.x) {
            const uint32_t bad = reinterpret_cast<const uint32_t*>(chan_bad)[q];
            float4 v;
            if constexpr (sizeof(T) == 1) {
                const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(x + r * nch) + q);
                v = make_float4((float)(w & 0xffu), (float)((w >> 8) & 0xffu), (float)((w >> 16) & 0xffu),
                                (float)(w >> 24));
            } else {
                v = __ldg(reinterpret_cast<const float4*>(x + r * nch) + q);
            }
            if (bad) {
                if (bad & 0xffu) v.x = 0.0f;
                if (bad & 0xff00u) v.y = 0.0f;
                if (bad & 0xff0000u) v.z = 0.0f;
                if (bad & 0xff000000u) v.w = 0.0f;
            }
            reinterpret_cast<float4*>(out + r * nch)[q] = v;
        }
    }
}

__global__ void absdev_kernel(const double* __restrict__ v, uint64_t n,
                              const double* __restrict__ center, double* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = fabs(__dsub_rn(v[i], *center));
}

// median of a sorted array (src/rfi.cpp:10-19): odd -> x[mid]; even -> 0.5*(x[mid]+x[mid-1])
__global__ void median_kernel(const double* __restrict__ sorted, uint64_t n, double scale,
                              double* __restrict__ out) {
    const uint64_t mid = n / 2;
    double m = sorted[mid];
    if (n % 2 == 0) m = __dmul_rn(0.5, __dadd_rn(m, sorted[mid - 1]));
    *out = scale == 1.0 ? m : __dmul_rn(m, scale);
}

__global__ void chan_flags_kernel(const double* __restrict__ mean, const double* __restrict__ var,
                                  uint32_t nch, const double* __restrict__ st, double k_mad,
                                  uint8_t* __restrict__ bad) {
    // st: [med_mean, sig_mean, med_var, sig_var]
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nch) return;
    const bool bm = fabs(__dsub_rn(mean[c], st[0])) > __dmul_rn(k_mad, st[1]);
    const bool bv = fabs(__dsub_rn(var[c], st[2])) > __dmul_rn(k_mad, st[3]);
    bad[c] = (bm || bv) ? 1 : 0;
}

__global__ void samp_flags_kernel(const double* __restrict__ zdm, uint64_t n,
                                  const double* __restrict__ st, double k_sigma,
                                  uint8_t* __restrict__ bad) {
    // st: [center, sigma]; sigma == 0 -> no flags (src/rfi.cpp:84)
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double sigma = st[1];
    bad[i] = (sigma != 0.0 && fabs(__dsub_rn(zdm[i], st[0])) > __dmul_rn(k_sigma, sigma)) ? 1 : 0;
}

template <typename T>
__global__ void widen_kernel(const T* __restrict__ x, size_t cells, float* __restrict__ out) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < cells;
         i += (size_t)gridDim.x * blockDim.x)
        out[i] = (float)x[i];
}

// apply_mask's replacement of cell (i, c) of a bad row (src/rfi.cpp:115-136): the local
// mean of the channel's unflagged cells within +-32 rows (double sum in row order), 0 for a
// bad channel or under the zero policy
template <typename T>
__device__ __forceinline__ float mask_value(const T* __restrict__ x, uint64_t n, uint32_t nch,
                                            const uint8_t* __restrict__ chan_bad,
                                            const uint8_t* __restrict__ samp_bad, uint64_t i, uint32_t c,
                                            int local_mean) {
    if (!local_mean || chan_bad[c]) return 0.0f;
    const uint64_t lo = i > 32 ? i - 32 : 0;
    const uint64_t hi = min(n, i + 33);
    double sum = 0.0;
    uint64_t count = 0;
    for (uint64_t j = lo; j < hi; ++j) {
        if (samp_bad[j]) continue;
        sum = __dadd_rn(sum, (double)(float)x[j * nch + c]);
        ++count;
    }
    return count ? __double2float_rn(__ddiv_rn(sum, (double)count)) : 0.0f;
}

// masked cells of bad samples (rows) and bad channels (columns)
template <typename T>
__global__ void mask_kernel(const T* __restrict__ x, uint64_t n, uint32_t nch,
                            const uint8_t* __restrict__ chan_bad, const uint8_t* __restrict__ samp_bad,
                            const uint64_t* __restrict__ bad_rows, uint64_t nbad_rows, int local_mean,
                            float* __restrict__ out) {
    // one block per bad row (blockIdx.x < nbad_rows) or per column sweep
    const uint64_t k = blockIdx.x;
    if (k < nbad_rows) {
        const uint64_t i = bad_rows[k];
        for (uint32_t c = threadIdx.x; c < nch; c += blockDim.x)
            out[i * nch + c] = mask_value(x, n, nch, chan_bad, samp_bad, i, c, local_mean);
    }
}

// exceptions of the fp16 dedispersion path: value of every cell of the k-th bad row (rows
// in ascending order), F[k][c]
__global__ void mask_values_kernel(const uint8_t* __restrict__ x, uint64_t n, uint32_t nch,
                                   const uint8_t* __restrict__ chan_bad, const uint8_t* __restrict__ samp_bad,
                                   const uint32_t* __restrict__ rows, int local_mean, float* __restrict__ F) {
    const uint64_t k = blockIdx.x;
    const uint64_t i = rows[k];
    for (uint32_t c = threadIdx.x; c < nch; c += blockDim.x)
        F[k * nch + c] = mask_value(x, n, nch, chan_bad, samp_bad, i, c, local_mean);
}

// P[r] = number of bad rows < r (r <= n) and the ascending bad-row list R[P[r]] = r, in
// blocks of 1024 rows: counts, one-CTA scan of the counts, per-block ballot scan
constexpr int XR_ROWS = 1024;

__global__ void __launch_bounds__(XR_ROWS) flag_counts_kernel(const uint8_t* __restrict__ bad, uint64_t n,
                                                              uint32_t* __restrict__ cnt) {
    const uint64_t r = (uint64_t)blockIdx.x * XR_ROWS + threadIdx.x;
    const int f = r < n && bad[r];
    const int c = __syncthreads_count(f);
    if (threadIdx.x == 0) cnt[blockIdx.x] = (uint32_t)c;
}

__global__ void __launch_bounds__(1024) flag_scan_kernel(uint32_t* __restrict__ cnt, uint32_t nb) {
    __shared__ uint32_t part[1024];
    const uint32_t per = (nb + 1023) / 1024;
    const uint32_t b0 = threadIdx.x * per, b1 = min(nb, b0 + per);
    uint32_t s = 0;
    for (uint32_t b = b0; b < b1; ++b) s += cnt[b];
    part[threadIdx.x] = s;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {  // inclusive Hillis-Steele scan of the thread sums
        const uint32_t v = threadIdx.x >= (unsigned)o ? part[threadIdx.x - o] : 0u;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    uint32_t run = part[threadIdx.x] - s;  // exclusive
    for (uint32_t b = b0; b < b1; ++b) {
        const uint32_t v = cnt[b];
        cnt[b] = run;
        run += v;
    }
}

__global__ void __launch_bounds__(XR_ROWS) flag_rows_kernel(const uint8_t* __restrict__ bad, uint64_t n,
                                                            const uint32_t* __restrict__ base,
                                                            uint32_t* __restrict__ P, uint32_t* __restrict__ R) {
    __shared__ uint32_t wsum[XR_ROWS / 32];
    const uint64_t r = (uint64_t)blockIdx.x * XR_ROWS + threadIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool f = r < n && bad[r];
    const uint32_t m = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wsum[warp] = __popc(m);
    __syncthreads();
    uint32_t before = 0;
    for (int w = 0; w < warp; ++w) before += wsum[w];
    const uint32_t p = base[blockIdx.x] + before + __popc(m & ((1u << lane) - 1u));
    if (r <= n) P[r] = p;
    if (f) R[p] = (uint32_t)r;
}

__global__ void zero_channels_kernel(uint64_t n, uint32_t nch, const uint8_t* __restrict__ chan_bad,
                                     float* __restrict__ out) {
    const uint32_t c = blockIdx.y * blockDim.x + threadIdx.x;
    if (c >= nch || !chan_bad[c]) return;
    for (uint64_t i = blockIdx.x; i < n; i += gridDim.x) out[i * nch + c] = 0.0f;
}

__global__ void compact_rows_kernel(const uint8_t* __restrict__ samp_bad, uint64_t n,
                                    uint64_t* __restrict__ rows, unsigned long long* __restrict__ cnt) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && samp_bad[i]) rows[atomicAdd(cnt, 1ull)] = i;
}

unsigned nblk(uint64_t n, unsigned t = 256) { return (unsigned)((n + t - 1) / t); }

void sorted_median(const double* v, uint64_t n, double scale, double* out, DevBuf& tmp,
                   double* sorted, cudaStream_t st) {
    size_t bytes = 0;
    PGB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, v, sorted, (int)n, 0, 64, st));
    tmp.reserve(bytes);
    PGB_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, bytes, v, sorted, (int)n, 0, 64, st));
    median_kernel<<<1, 1, 0, st>>>(sorted, n, scale, out);
}

// median + 1.4826 * MAD of v[n] into st[0], st[1]
void median_mad(const double* v, uint64_t n, double* st2, DevBuf& tmp, double* scratch_a,
                double* scratch_b, cudaStream_t st) {
    sorted_median(v, n, 1.0, st2, tmp, scratch_a, st);
    absdev_kernel<<<nblk(n), 256, 0, st>>>(v, n, st2, scratch_b);
    sorted_median(scratch_b, n, 1.4826, st2 + 1, tmp, scratch_a, st);
}

}  // namespace

template <typename T>
void rfi_flags_impl(const T* x, uint64_t n, uint32_t nch, const RfiParams& rp, RfiWork& w, cudaStream_t st,
                    uint64_t* n_bad_ch, uint64_t* n_bad_s) {
    w.chan_bad.reserve(nch);
    w.samp_bad.reserve(n);
    PGB_CUDA(cudaMemsetAsync(w.chan_bad.p, 0, nch, st));
    PGB_CUDA(cudaMemsetAsync(w.samp_bad.p, 0, n, st));
    const uint64_t big = std::max<uint64_t>(n, nch);
    w.dbl.reserve(sizeof(double) * (4 * big + 8));
    double* d = w.dbl.as<double>();
    double* stats = d;            // [8]
    double* a = d + 8;            // [big]
    double* b = a + big;          // [big]
    double* s1 = b + big;         // [big]
    double* s2 = s1 + big;        // [big]
    if (rp.narrowband) {          // src/rfi.cpp:32-68
        if (nch < 4) raise(PGB_ERR_INSUFFICIENT, "narrowband flagging needs at least 4 channels");
        if (n == 0) raise(PGB_ERR_INSUFFICIENT, "empty chunk");
        if (std::is_same<T, uint8_t>::value && nch % 16 == 0 && !pgb_ablation_env("PGB_RFI_SERIAL")) {
            auto* sums = reinterpret_cast<unsigned long long*>(s1);  // scratch until median_mad
            PGB_CUDA(cudaMemsetAsync(sums, 0, sizeof(unsigned long long) * nch, st));
            const uint32_t gx = (nch / 4 + 255) / 256;
            uint64_t gy = std::max<uint64_t>(1, (148 * 16) / gx);
            gy = std::max<uint64_t>(gy, (n + (1u << 24) - 1) >> 24);
            gy = std::min<uint64_t>(gy, std::max<uint64_t>(1, n / 64));
            const uint64_t rows_per = (n + gy - 1) / gy;
            gy = (n + rows_per - 1) / rows_per;
            chan_sum_u8_kernel<<<dim3(gx, (unsigned)gy), 256, 0, st>>>(
                reinterpret_cast<const uint8_t*>(x), n, nch, rows_per, sums);
            const size_t sm = (size_t)CV_NS * CV_ROWS * CV_CH;
            // per call: the attribute is per device, and contexts may live on different GPUs
            PGB_CUDA(cudaFuncSetAttribute(chan_var_u8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            chan_var_u8_kernel<<<(nch + CV_CH - 1) / CV_CH, CV_CH, sm, st>>>(reinterpret_cast<const uint8_t*>(x),
                                                                           n, nch, sums, a, b);
        } else {
            chan_stats_kernel<T><<<nblk(nch, 128), 128, 0, st>>>(x, n, nch, a, b);
        }
        median_mad(a, nch, stats, w.tmp, s1, s2, st);
        median_mad(b, nch, stats + 2, w.tmp, s1, s2, st);
        chan_flags_kernel<<<nblk(nch), 256, 0, st>>>(a, b, nch, stats, rp.k_mad, w.chan_bad.as<uint8_t>());
    }
    if (rp.broadband && n > 0) {  // src/rfi.cpp:70-91
        if (std::is_same<T, uint8_t>::value && nch % 16 == 0 && !pgb_ablation_env("PGB_RFI_SERIAL"))
            zero_dm_u8_kernel<<<(unsigned)((n * 32 + 255) / 256), 256, 0, st>>>(reinterpret_cast<const uint8_t*>(x),
                                                                                n, nch, a);
        else
            zero_dm_kernel<T><<<nblk(n, 128), 128, 0, st>>>(x, n, nch, a);
        median_mad(a, n, stats + 4, w.tmp, s1, s2, st);
        samp_flags_kernel<<<nblk(n), 256, 0, st>>>(a, n, stats + 4, rp.k_sigma, w.samp_bad.as<uint8_t>());
    }
    // counts (and the bad-row list) decide whether apply_mask runs at all (pipeline.cpp:86)
    w.rows.reserve(sizeof(uint64_t) * (n + 1) + 16);
    auto* cnt = reinterpret_cast<unsigned long long*>(w.rows.as<uint64_t>() + n);
    PGB_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st));
    compact_rows_kernel<<<nblk(n), 256, 0, st>>>(w.samp_bad.as<uint8_t>(), n, w.rows.as<uint64_t>(), cnt);
    std::vector<uint8_t> cb(nch);
    unsigned long long nrows_bad = 0;
    PGB_CUDA(cudaMemcpyAsync(&nrows_bad, cnt, sizeof nrows_bad, cudaMemcpyDeviceToHost, st));
    PGB_CUDA(cudaMemcpyAsync(cb.data(), w.chan_bad.p, nch, cudaMemcpyDeviceToHost, st));
    PGB_CUDA(cudaStreamSynchronize(st));
    uint64_t nbc = 0;
    for (auto v : cb) nbc += v;
    *n_bad_ch = nbc;
    *n_bad_s = nrows_bad;
}

template <typename T>
void rfi_mask_impl(const T* x, uint64_t n, uint32_t nch, const RfiParams& rp, RfiWork& w, float* out,
                   cudaStream_t st, uint64_t nbc, uint64_t nrows_bad) {
    const size_t cells = (size_t)n * nch;
    const bool rows4 = nch % 4 == 0 && !pgb_ablation_env("PGB_RFI_SERIAL");
    if (rows4)  // bad channels zeroed while widening
        widen_rows_kernel<T><<<148 * 16, 256, 0, st>>>(x, n, nch, w.chan_bad.as<uint8_t>(), out);
    else
        widen_kernel<T><<<148 * 8, 256, 0, st>>>(x, cells, out);
    if (nbc == 0 && nrows_bad == 0) return;
    if (nrows_bad) {
        // the row list from atomics is unordered; each row is independent, so order is moot
        mask_kernel<T><<<(unsigned)nrows_bad, 256, 0, st>>>(x, n, nch, w.chan_bad.as<uint8_t>(),
                                                            w.samp_bad.as<uint8_t>(), w.rows.as<uint64_t>(),
                                                            nrows_bad, rp.local_mean, out);
    }
    if (nbc && !rows4) {
        dim3 g((unsigned)std::min<uint64_t>(n, 4096), (nch + 255) / 256);
        zero_channels_kernel<<<g, 256, 0, st>>>(n, nch, w.chan_bad.as<uint8_t>(), out);
    }
    PGB_CUDA(cudaGetLastError());
}

template <typename T>
void rfi_clean_impl(const T* x, uint64_t n, uint32_t nch, const RfiParams& rp, RfiWork& w,
                    float* out, cudaStream_t st, uint64_t* n_bad_ch, uint64_t* n_bad_s) {
    rfi_flags_impl(x, n, nch, rp, w, st, n_bad_ch, n_bad_s);
    rfi_mask_impl(x, n, nch, rp, w, out, st, *n_bad_ch, *n_bad_s);
}

void rfi_exceptions_u8(const uint8_t* x, uint64_t n, uint32_t nch, const RfiParams& rp, RfiWork& w,
                       uint64_t nbad, cudaStream_t st, std::vector<uint32_t>* rows_host) {
    if (n >= (1ull << 32)) raise(PGB_ERR_CONFIG, "chunk longer than 2^32 samples");
    const uint32_t nb = (uint32_t)((n + 1 + XR_ROWS - 1) / XR_ROWS);  // rows 0 .. n (P[n] = total)
    w.xcnt.reserve(sizeof(uint32_t) * nb);
    w.xP.reserve(sizeof(uint32_t) * (n + 1));
    w.xR.reserve(sizeof(uint32_t) * std::max<uint64_t>(nbad, 1));
    w.xF.reserve(sizeof(float) * std::max<uint64_t>(nbad, 1) * nch);
    const uint8_t* bad = w.samp_bad.as<uint8_t>();
    flag_counts_kernel<<<nb, XR_ROWS, 0, st>>>(bad, n, w.xcnt.as<uint32_t>());
    flag_scan_kernel<<<1, 1024, 0, st>>>(w.xcnt.as<uint32_t>(), nb);
    flag_rows_kernel<<<nb, XR_ROWS, 0, st>>>(bad, n, w.xcnt.as<uint32_t>(), w.xP.as<uint32_t>(),
                                             w.xR.as<uint32_t>());
    if (nbad)
        mask_values_kernel<<<(unsigned)nbad, 256, 0, st>>>(x, n, nch, w.chan_bad.as<uint8_t>(), bad,
                                                           w.xR.as<uint32_t>(), rp.local_mean, w.xF.as<float>());
    PGB_CUDA(cudaGetLastError());
    if (rows_host) {
        rows_host->resize(nbad);
        if (nbad)
            PGB_CUDA(cudaMemcpyAsync(rows_host->data(), w.xR.p, nbad * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        PGB_CUDA(cudaStreamSynchronize(st));
    }
}

template void rfi_clean_impl<uint8_t>(const uint8_t*, uint64_t, uint32_t, const RfiParams&, RfiWork&,
                                      float*, cudaStream_t, uint64_t*, uint64_t*);
template void rfi_clean_impl<float>(const float*, uint64_t, uint32_t, const RfiParams&, RfiWork&, float*,
                                    cudaStream_t, uint64_t*, uint64_t*);
template void rfi_flags_impl<uint8_t>(const uint8_t*, uint64_t, uint32_t, const RfiParams&, RfiWork&,
                                      cudaStream_t, uint64_t*, uint64_t*);
template void rfi_mask_impl<uint8_t>(const uint8_t*, uint64_t, uint32_t, const RfiParams&, RfiWork&, float*,
                                     cudaStream_t, uint64_t, uint64_t);

}  // namespace pgb
