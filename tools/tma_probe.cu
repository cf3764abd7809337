// Standalone probe: does a 2D u8 TMA load with 256-byte boxes work on this box,
// with and without an explicit 1x1x1 cluster launch?  nvcc -arch=sm_100a tma_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void probe(const __grid_constant__ CUtensorMap map, uint8_t* out, int x0, int y0) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(256) : "memory");
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(su32(sm)), "l"(reinterpret_cast<uint64_t>(&map)), "r"(x0), "r"(y0), "r"(su32(&bar)) : "memory");
    }
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }"
                     : "=r"(done) : "r"(su32(&bar)) : "memory");
    for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = sm[i];
}

int main() {
    const size_t pitch = 4096, rows = 8;
    uint8_t *d, *o;
    cudaMalloc(&d, pitch * rows);
    cudaMalloc(&o, 256);
    uint8_t h[pitch * rows];
    for (size_t i = 0; i < pitch * rows; ++i) h[i] = (uint8_t)(i * 7 + i / pitch);
    cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    CUtensorMap map;
    cuuint64_t dims[2] = {pitch, rows};
    cuuint64_t str[1] = {pitch};
    cuuint32_t box[2] = {256, 1}, es[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d q %d\n", (int)r, (int)q);
    for (int variant = 0; variant < 3; ++variant) {
        int x0 = variant == 2 ? 13 : 0, y0 = 3;
        cudaMemset(o, 0, 256);
        if (variant == 1) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = 1; cfg.blockDim = 128; cfg.dynamicSmemBytes = 2048;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.attrs = at; cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, probe, map, o, x0, y0);
        } else {
            probe<<<1, 128, 2048>>>(map, o, x0, y0);
        }
        cudaError_t e = cudaDeviceSynchronize();
        uint8_t ho[256];
        cudaMemcpy(ho, o, 256, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int i = 0; i < 256; ++i) bad += ho[i] != h[y0 * pitch + x0 + i];
        printf("variant %d: %s, mismatches %d\n", variant, cudaGetErrorString(e), bad);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
