#include <cstdio>
#include <cstdint>
__global__ void k(double* out, long long* cyc, int n, double x) {
    double a = x, b = x * 0.5, c = 1.0000001;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { a = __fma_rn(c, c, a); }
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) { b = __dadd_rn(b, c); }
    long long t2 = clock64();
    float f = (float)x, g = 1.0001f;
    for (int i = 0; i < n; ++i) { f = __fmaf_rn(g, g, f); }
    long long t3 = clock64();
    // float -> double convert + dfma chain with the converted value off-chain
    double d = x; float v = (float)x;
    for (int i = 0; i < n; ++i) { v = v * 1.0000001f; double dv = (double)v; d = __fma_rn(dv, dv, d); }
    long long t4 = clock64();
    out[threadIdx.x] = a + b + f + d;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMallocManaged(&c, 64);
    int n = 1 << 16;
    k<<<1, 32>>>(o, c, n, 1.0); cudaDeviceSynchronize();
    k<<<1, 32>>>(o, c, n, 1.0); cudaDeviceSynchronize();
    printf("cycles/op: DFMA chain %.2f  DADD chain %.2f  FFMA chain %.2f  F2F+DFMA %.2f\n",
           (double)c[0] / n, (double)c[1] / n, (double)c[2] / n, (double)c[3] / n);
}
