// Device ordering of candidates and run fragments (CUB radix sort on packed keys).
//
// Candidate order is the reference's (peak_sample, dm_trial, width_index)
// (src/engine.cpp:257-262, src/pipeline.cpp:100-105); the packed key is unique per
// candidate, so the result never depends on atomic emission order.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>

#include "pgb_internal.h"

namespace pgb {

namespace {

__global__ void frag_keys_kernel(const Fragment* __restrict__ f, uint64_t n, uint64_t* keys,
                                 uint32_t* idx) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        keys[i] = f[i].key;
        idx[i] = (uint32_t)i;
    }
}

template <typename T>
__global__ void gather_kernel(const T* __restrict__ in, const uint32_t* __restrict__ idx,
                              uint64_t n, T* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[idx[i]];
}

// peak_sample < 2^39, dm_trial < 2^20, width_index < 2^5
__global__ void cand_keys_kernel(const pgb_candidate* __restrict__ c, uint64_t n, uint64_t* keys,
                                 uint32_t* idx) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        keys[i] = c[i].peak_sample << 25 | (uint64_t)c[i].dm_trial << 5 | c[i].width_index;
        idx[i] = (uint32_t)i;
    }
}

unsigned nblk(uint64_t n) { return (unsigned)((n + 255) / 256); }

// ---- device-count variants (file search: no host round trip per chunk) -------------
// The item count lives on the device (an emission counter, possibly above the buffer's
// capacity when it overflowed); `cap` items are sorted, the ones past the count carry
// the largest key so they sort last and are never gathered.
__device__ __forceinline__ uint64_t dev_count(const unsigned long long* d_n, uint64_t cap) {
    const uint64_t n = *d_n;
    return n < cap ? n : cap;
}

__global__ void frag_keys_dev_kernel(const Fragment* __restrict__ f, uint64_t cap,
                                     const unsigned long long* d_n, uint64_t* keys, uint32_t* idx) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < cap) {
        keys[i] = i < dev_count(d_n, cap) ? f[i].key : ~0ull;
        idx[i] = (uint32_t)i;
    }
}

__global__ void cand_keys_dev_kernel(const pgb_candidate* __restrict__ c, uint64_t cap,
                                     const unsigned long long* d_n, uint64_t* keys, uint32_t* idx) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < cap) {
        keys[i] = i < dev_count(d_n, cap)
                      ? c[i].peak_sample << 25 | (uint64_t)c[i].dm_trial << 5 | c[i].width_index
                      : ~0ull;
        idx[i] = (uint32_t)i;
    }
}

template <typename T>
__global__ void gather_dev_kernel(const T* __restrict__ in, const uint32_t* __restrict__ idx,
                                  uint64_t cap, const unsigned long long* d_n, T* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < dev_count(d_n, cap)) out[i] = in[idx[i]];
}

// dst[total + i] = src[i] for i < count (file-level candidate list); total is bumped by
// a separate one-thread kernel so every thread of this one reads the same base
__global__ void append_dev_kernel(const pgb_candidate* __restrict__ src, uint64_t cap,
                                  const unsigned long long* d_n, pgb_candidate* __restrict__ dst,
                                  const unsigned long long* d_total, uint64_t dst_cap) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t base = *d_total;
    if (i < dev_count(d_n, cap) && base + i < dst_cap) dst[base + i] = src[i];
}

// total += count; high-water marks of the emission counters (overflow detection)
__global__ void bump_dev_kernel(const unsigned long long* d_counts, unsigned long long* d_total,
                                unsigned long long* d_hiwater, uint64_t cap) {
    const unsigned long long nc = d_counts[0], nf = d_counts[1];
    d_hiwater[0] = max(d_hiwater[0], nc);
    d_hiwater[1] = max(d_hiwater[1], nf);
    *d_total += nc < cap ? nc : cap;
}

__global__ void copy_words_kernel(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

}  // namespace

void launch_copy_from_host(void* dst, const void* pinned_src, size_t bytes, cudaStream_t st) {
    // whole 32-bit words (every staged array is 4- or 8-byte typed)
    const size_t n = (bytes + 3) / 4;
    const unsigned blocks = (unsigned)std::min<size_t>(64, (n + 255) / 256);
    copy_words_kernel<<<blocks, 256, 0, st>>>(static_cast<uint32_t*>(dst),
                                              static_cast<const uint32_t*>(pinned_src), n);
    PGB_CUDA(cudaGetLastError());
}

void sort_fragments_dev(Fragment* frags, Fragment* out, uint64_t cap, const unsigned long long* d_n,
                        void* temp, size_t temp_bytes, uint64_t* keys_a, uint64_t* keys_b,
                        uint32_t* idx_a, uint32_t* idx_b, cudaStream_t st) {
    if (!cap) return;
    frag_keys_dev_kernel<<<nblk(cap), 256, 0, st>>>(frags, cap, d_n, keys_a, idx_a);
    cub::DoubleBuffer<uint64_t> k(keys_a, keys_b);
    cub::DoubleBuffer<uint32_t> v(idx_a, idx_b);
    PGB_CUDA(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k, v, (int)cap, 0, 64, st));
    gather_dev_kernel<Fragment><<<nblk(cap), 256, 0, st>>>(frags, v.Current(), cap, d_n, out);
    PGB_CUDA(cudaGetLastError());
}

void sort_candidates_dev(const pgb_candidate* in, pgb_candidate* out, uint64_t cap,
                         const unsigned long long* d_n, void* temp, size_t temp_bytes,
                         uint64_t* keys_a, uint64_t* keys_b, uint32_t* idx_a, uint32_t* idx_b,
                         cudaStream_t st) {
    if (!cap) return;
    cand_keys_dev_kernel<<<nblk(cap), 256, 0, st>>>(in, cap, d_n, keys_a, idx_a);
    cub::DoubleBuffer<uint64_t> k(keys_a, keys_b);
    cub::DoubleBuffer<uint32_t> v(idx_a, idx_b);
    PGB_CUDA(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k, v, (int)cap, 0, 64, st));
    gather_dev_kernel<pgb_candidate><<<nblk(cap), 256, 0, st>>>(in, v.Current(), cap, d_n, out);
    PGB_CUDA(cudaGetLastError());
}

void append_candidates_dev(const pgb_candidate* sorted, uint64_t cap, const unsigned long long* d_counts,
                           pgb_candidate* file_cands, unsigned long long* d_total, uint64_t file_cap,
                           unsigned long long* d_hiwater, cudaStream_t st) {
    if (cap) append_dev_kernel<<<nblk(cap), 256, 0, st>>>(sorted, cap, d_counts, file_cands, d_total, file_cap);
    bump_dev_kernel<<<1, 1, 0, st>>>(d_counts, d_total, d_hiwater, cap);
    PGB_CUDA(cudaGetLastError());
}

size_t sort_fragments_temp_bytes(uint64_t n) {
    size_t bytes = 0;
    cub::DoubleBuffer<uint64_t> k(nullptr, nullptr);
    cub::DoubleBuffer<uint32_t> v(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, k, v, (int)n);
    return bytes;
}

void sort_fragments(Fragment* frags, Fragment* tmp, uint64_t n, void* temp, size_t temp_bytes,
                    uint64_t* keys_a, uint64_t* keys_b, uint32_t* idx_a, uint32_t* idx_b,
                    cudaStream_t st) {
    if (n < 2) {
        if (n == 1) PGB_CUDA(cudaMemcpyAsync(tmp, frags, sizeof(Fragment), cudaMemcpyDeviceToDevice, st));
        return;
    }
    frag_keys_kernel<<<nblk(n), 256, 0, st>>>(frags, n, keys_a, idx_a);
    cub::DoubleBuffer<uint64_t> k(keys_a, keys_b);
    cub::DoubleBuffer<uint32_t> v(idx_a, idx_b);
    PGB_CUDA(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k, v, (int)n, 0, 64, st));
    gather_kernel<Fragment><<<nblk(n), 256, 0, st>>>(frags, v.Current(), n, tmp);
    PGB_CUDA(cudaGetLastError());
}

size_t sort_candidates_temp_bytes(uint64_t n) { return sort_fragments_temp_bytes(n); }

void sort_candidates(const pgb_candidate* in, pgb_candidate* out, uint64_t n, void* temp,
                     size_t temp_bytes, uint64_t* keys_a, uint64_t* keys_b, uint32_t* idx_a,
                     uint32_t* idx_b, cudaStream_t st) {
    if (n < 2) {
        if (n == 1)
            PGB_CUDA(cudaMemcpyAsync(out, in, sizeof(pgb_candidate), cudaMemcpyDeviceToDevice, st));
        return;
    }
    cand_keys_kernel<<<nblk(n), 256, 0, st>>>(in, n, keys_a, idx_a);
    cub::DoubleBuffer<uint64_t> k(keys_a, keys_b);
    cub::DoubleBuffer<uint32_t> v(idx_a, idx_b);
    PGB_CUDA(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k, v, (int)n, 0, 64, st));
    gather_kernel<pgb_candidate><<<nblk(n), 256, 0, st>>>(in, v.Current(), n, out);
    PGB_CUDA(cudaGetLastError());
}

}  // namespace pgb
