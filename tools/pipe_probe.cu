// Pipe-throughput probe for the fp32 dedispersion redesign (round 2): FADD, FHADD (f32 + f16
// operand, PTX add.rn.f32.f16), FADD2 (add.rn.f32x2), PRMT, HADD2, and two inner-loop
// shapes (half staging + FHADD; u8 staging + PRMT magic + FADD2).  Prints per-SM
// operations per clock.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o
// tools/pipe_probe tools/pipe_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;
constexpr int CH = 8;  // independent chains per thread

__global__ void k_fadd(float* out, float x) {
    float a[CH];
    for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(x));
    float s = 0;
    for (int i = 0; i < CH; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_fhadd(float* out, unsigned short h) {
    float a[CH];
    for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) asm volatile("add.rn.f32.f16 %0, %1, %0;" : "+f"(a[i]) : "h"(h));
    float s = 0;
    for (int i = 0; i < CH; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_fadd2(float* out, unsigned long long x) {
    unsigned long long a[CH];
    for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(x));
    float s = 0;
    for (int i = 0; i < CH; ++i) s += __int_as_float((int)a[i]) + __int_as_float((int)(a[i] >> 32));
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_prmt(float* out, unsigned x) {
    unsigned a[CH];
    for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) asm volatile("prmt.b32 %0, %0, %1, 0x5140;" : "+r"(a[i]) : "r"(x));
    unsigned s = 0;
    for (int i = 0; i < CH; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_hadd2(float* out, unsigned x) {
    unsigned a[CH];
    for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) asm volatile("add.rn.f16x2 %0, %0, %1;" : "+r"(a[i]) : "r"(x));
    unsigned s = 0;
    for (int i = 0; i < CH; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_i2f(float* out, unsigned x) {
    float a[CH];
    for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * i;
    unsigned w = x ^ threadIdx.x;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            float f;
            asm volatile("cvt.rn.f32.u8 %0, %1;" : "=f"(f) : "h"((unsigned short)((w >> (8 * (i & 3))) & 0xff)));
            a[i] += f;
            w += 0x01010101u;
        }
    float s = 0;
    for (int i = 0; i < CH; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// mixed FHADD + FADD2 in the same loop (do they share a pipe?)
__global__ void k_fhadd_fadd2(float* out, unsigned short h, unsigned long long x) {
    float a[CH];
    unsigned long long b[CH];
    for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * i, b[i] = i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            asm volatile("add.rn.f32.f16 %0, %1, %0;" : "+f"(a[i]) : "h"(h));
            asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(b[i]) : "l"(x));
        }
    float s = 0;
    for (int i = 0; i < CH; ++i) s += a[i] + __int_as_float((int)b[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// loop shape A: halves staged in smem, LDS.64 (4 halves) + 4 FHADD per word, 8 words per thread
__global__ void k_shapeA(float* out, int shift) {
    __shared__ uint2 sm[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = make_uint2(0x3c003c00u * (i & 1), 0x3c00u);
    __syncthreads();
    float a[8][4];
    for (int m = 0; m < 8; ++m) for (int j = 0; j < 4; ++j) a[m][j] = 0;
    int lane = threadIdx.x & 31;
    for (int it = 0; it < ITERS / 8; ++it) {
        int base = ((it * shift) & 1023) + lane;
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            uint2 w = sm[(base + 32 * m) & 4095];
            unsigned short h0 = w.x & 0xffff, h1 = w.x >> 16, h2 = w.y & 0xffff, h3 = w.y >> 16;
            asm volatile("add.rn.f32.f16 %0, %1, %0;" : "+f"(a[m][0]) : "h"(h0));
            asm volatile("add.rn.f32.f16 %0, %1, %0;" : "+f"(a[m][1]) : "h"(h1));
            asm volatile("add.rn.f32.f16 %0, %1, %0;" : "+f"(a[m][2]) : "h"(h2));
            asm volatile("add.rn.f32.f16 %0, %1, %0;" : "+f"(a[m][3]) : "h"(h3));
        }
    }
    float s = 0;
    for (int m = 0; m < 8; ++m) for (int j = 0; j < 4; ++j) s += a[m][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// loop shape B: u8 staged, LDS.32 + 4 PRMT (2^23 magic) + 2 FADD2 (unbias) + 2 FADD2 (acc)
__global__ void k_shapeB(float* out, int shift) {
    __shared__ unsigned sm[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i * 0x01010101u;
    __syncthreads();
    unsigned long long a[8][2];
    for (int m = 0; m < 8; ++m) a[m][0] = a[m][1] = 0;
    const unsigned long long bias = 0xCB000000CB000000ull;  // -2^23, -2^23
    int lane = threadIdx.x & 31;
    for (int it = 0; it < ITERS / 8; ++it) {
        int base = ((it * shift) & 1023) + lane;
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            unsigned w = sm[(base + 32 * m) & 8191];
            unsigned f0 = __byte_perm(w, 0x4b000000u, 0x7440), f1 = __byte_perm(w, 0x4b000000u, 0x7441);
            unsigned f2 = __byte_perm(w, 0x4b000000u, 0x7442), f3 = __byte_perm(w, 0x4b000000u, 0x7443);
            unsigned long long p0 = (unsigned long long)f1 << 32 | f0, p1 = (unsigned long long)f3 << 32 | f2;
            asm("add.rn.f32x2 %0, %0, %1;" : "+l"(p0) : "l"(bias));
            asm("add.rn.f32x2 %0, %0, %1;" : "+l"(p1) : "l"(bias));
            asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[m][0]) : "l"(p0));
            asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[m][1]) : "l"(p1));
        }
    }
    float s = 0;
    for (int m = 0; m < 8; ++m) s += __int_as_float((int)a[m][0]) + __int_as_float((int)a[m][1]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// loop shape C: the current fp32 design, floats staged in smem (LDS.128 = 4 floats) + 4 FADD
__global__ void k_shapeC(float* out, int shift) {
    __shared__ float4 sm[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_float4(1, 2, 3, i);
    __syncthreads();
    float a[8][4];
    for (int m = 0; m < 8; ++m) for (int j = 0; j < 4; ++j) a[m][j] = 0;
    int lane = threadIdx.x & 31;
    for (int it = 0; it < ITERS / 8; ++it) {
        int base = ((it * shift) & 1023) + lane;
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            float4 w = sm[(base + 32 * m) & 2047];
            asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[m][0]) : "f"(w.x));
            asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[m][1]) : "f"(w.y));
            asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[m][2]) : "f"(w.z));
            asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[m][3]) : "f"(w.w));
        }
    }
    float s = 0;
    for (int m = 0; m < 8; ++m) for (int j = 0; j < 4; ++j) s += a[m][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
void run(const char* name, F launch, double ops_per_thread, int threads) {
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    launch();
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    const double ops = ops_per_thread * threads * sms;
    const double per_clk_sm = ops / (best * 1e-3) / sms / (clk * 1e3);
    printf("%-14s %8.3f ms  %7.1f ops/clk/SM (at max clock %d MHz)  %.2f T/s\n", name, best, per_clk_sm,
           clk / 1000, ops / (best * 1e-3) / 1e12);
    if (cudaGetLastError() != cudaSuccess) printf("error\n");
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    const int T = 512, B = sms * 2;
    cudaMalloc(&out, sizeof(float) * T * B * 2);
    const double n = (double)ITERS * CH * 2;  // 2 CTAs per SM
    run("FADD", [&] { k_fadd<<<B, T>>>(out, 1.0f); }, n, T);
    run("FHADD", [&] { k_fhadd<<<B, T>>>(out, (unsigned short)0x3c00); }, n, T);
    run("FADD2(lanes)", [&] { k_fadd2<<<B, T>>>(out, 0x3f8000003f800000ull); }, 2 * n, T);
    run("PRMT", [&] { k_prmt<<<B, T>>>(out, 0x12345678u); }, n, T);
    run("I2F.U8+FADD", [&] { k_i2f<<<B, T>>>(out, 0x12345678u); }, n, T);
    run("HADD2(lanes)", [&] { k_hadd2<<<B, T>>>(out, 0x3c003c00u); }, 2 * n, T);
    run("FHADD+FADD2", [&] { k_fhadd_fadd2<<<B, T>>>(out, (unsigned short)0x3c00, 0x3f8000003f800000ull); }, 3 * n, T);
    const double adds = (double)(ITERS / 8) * 8 * 4 * 2;
    run("shapeA adds", [&] { k_shapeA<<<B, T>>>(out, 37); }, adds, T);
    run("shapeB adds", [&] { k_shapeB<<<B, T>>>(out, 37); }, adds, T);
    run("shapeC adds", [&] { k_shapeC<<<B, T>>>(out, 37); }, adds, T);
    return 0;
}
