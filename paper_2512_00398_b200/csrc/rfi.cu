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
#include <cub/device/device_radix_sort.cuh>

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
        for (uint32_t c = threadIdx.x; c < nch; c += blockDim.x) {
            float rep = 0.0f;
            if (local_mean && !chan_bad[c]) {  // src/rfi.cpp:122-136
                const uint64_t lo = i > 32 ? i - 32 : 0;
                const uint64_t hi = min(n, i + 33);
                double sum = 0.0;
                uint64_t count = 0;
                for (uint64_t j = lo; j < hi; ++j) {
                    if (samp_bad[j]) continue;
                    sum = __dadd_rn(sum, (double)(float)x[j * nch + c]);
                    ++count;
                }
                rep = count ? __double2float_rn(__ddiv_rn(sum, (double)count)) : 0.0f;
            }
            out[i * nch + c] = rep;
        }
    }
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
void rfi_clean_impl(const T* x, uint64_t n, uint32_t nch, const RfiParams& rp, RfiWork& w,
                    float* out, cudaStream_t st, uint64_t* n_bad_ch, uint64_t* n_bad_s) {
    const size_t cells = (size_t)n * nch;
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
        chan_stats_kernel<T><<<nblk(nch, 128), 128, 0, st>>>(x, n, nch, a, b);
        median_mad(a, nch, stats, w.tmp, s1, s2, st);
        median_mad(b, nch, stats + 2, w.tmp, s1, s2, st);
        chan_flags_kernel<<<nblk(nch), 256, 0, st>>>(a, b, nch, stats, rp.k_mad, w.chan_bad.as<uint8_t>());
    }
    if (rp.broadband && n > 0) {  // src/rfi.cpp:70-91
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
    widen_kernel<T><<<148 * 8, 256, 0, st>>>(x, cells, out);
    if (nbc == 0 && nrows_bad == 0) return;
    if (nrows_bad) {
        // the row list from atomics is unordered; each row is independent, so order is moot
        mask_kernel<T><<<(unsigned)nrows_bad, 256, 0, st>>>(x, n, nch, w.chan_bad.as<uint8_t>(),
                                                            w.samp_bad.as<uint8_t>(), w.rows.as<uint64_t>(),
                                                            nrows_bad, rp.local_mean, out);
    }
    if (nbc) {
        dim3 g((unsigned)std::min<uint64_t>(n, 4096), (nch + 255) / 256);
        zero_channels_kernel<<<g, 256, 0, st>>>(n, nch, w.chan_bad.as<uint8_t>(), out);
    }
    PGB_CUDA(cudaGetLastError());
}

template void rfi_clean_impl<uint8_t>(const uint8_t*, uint64_t, uint32_t, const RfiParams&, RfiWork&,
                                      float*, cudaStream_t, uint64_t*, uint64_t*);
template void rfi_clean_impl<float>(const float*, uint64_t, uint32_t, const RfiParams&, RfiWork&,
                                    float*, cudaStream_t, uint64_t*, uint64_t*);

}  // namespace pgb
