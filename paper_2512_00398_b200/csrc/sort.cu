// Device ordering of candidates and run fragments (CUB radix sort on packed keys).
//
// Candidate order is the reference's (peak_sample, dm_trial, width_index)
// (src/engine.cpp:257-262, src/pipeline.cpp:100-105); the packed key is unique per
// candidate, so the result never depends on atomic emission order.
#include <cub/device/device_radix_sort.cuh>

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

}  // namespace

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
