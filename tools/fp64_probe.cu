// Microbenchmark: FP64 / conversion pipe throughput on B200 (sm_100a).
// Used to size the FP64 budget of the quantize kernels.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe tools/fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096
#define CHAINS 8

__global__ void k_dadd(double* out, double a) {
    double x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; c++) x[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < ITERS; i++) {
#pragma unroll
        for (int c = 0; c < CHAINS; c++) x[c] = __dadd_rn(x[c], a);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; c++) s += x[c];
    if (s == 12345.0) out[0] = s;
}
__global__ void k_dmul(double* out, double a) {
    double x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; c++) x[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < ITERS; i++) {
#pragma unroll
        for (int c = 0; c < CHAINS; c++) x[c] = __dmul_rn(x[c], a);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; c++) s += x[c];
    if (s == 12345.0) out[0] = s;
}
__global__ void k_ddiv(double* out, double a) {
    double x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; c++) x[c] = threadIdx.x * 1e-3 + c + 1;
    for (int i = 0; i < ITERS / 16; i++) {
#pragma unroll
        for (int c = 0; c < CHAINS; c++) x[c] = __ddiv_rn(x[c], a);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; c++) s += x[c];
    if (s == 12345.0) out[0] = s;
}
// f32 -> f64 -> f32 round trips (F2F both directions)
__global__ void k_f2f(double* out, float a) {
    float x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; c++) x[c] = threadIdx.x * 1e-3f + c;
    for (int i = 0; i < ITERS; i++) {
#pragma unroll
        for (int c = 0; c < CHAINS; c++) {
            double d = (double)x[c];
            x[c] = __double2float_rn(__dadd_rn(d, (double)a));
        }
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; c++) s += x[c];
    if (s == 12345.0f) out[0] = s;
}
// double -> int floor and back
__global__ void k_f2i(double* out, double a) {
    double x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; c++) x[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < ITERS; i++) {
#pragma unroll
        for (int c = 0; c < CHAINS; c++) {
            int q = __double2int_rd(x[c]);
            x[c] = __dadd_rn((double)q, a);
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; c++) s += x[c];
    if (s == 12345.0) out[0] = s;
}
__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    size_t st = (size_t)gridDim.x * blockDim.x;
    for (; i < n; i += st) b[i] = a[i];
}

template <typename F>
float timeit(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < 5; r++) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
}

int main() {
    double* out; cudaMalloc(&out, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    int blocks = sms * 8, threads = 256;
    double ops = (double)blocks * threads * ITERS * CHAINS;
    float t;
    t = timeit([&] { k_dadd<<<blocks, threads>>>(out, 1.0000001); });
    printf("DADD   %.3f ms  %.2f Tops/s  %.1f warp-ops/clk/SM(@%d MHz)\n", t, ops / t / 1e9, ops / 32 / (t * 1e-3) / sms / (clk * 1e3), clk / 1000);
    t = timeit([&] { k_dmul<<<blocks, threads>>>(out, 1.0000001); });
    printf("DMUL   %.3f ms  %.2f Tops/s  %.2f warp-ops/clk/SM\n", t, ops / t / 1e9, ops / 32 / (t * 1e-3) / sms / (clk * 1e3));
    t = timeit([&] { k_ddiv<<<blocks, threads>>>(out, 1.0000001); });
    printf("DDIV   %.3f ms  %.3f Tops/s\n", t, ops / 16 / t / 1e9);
    t = timeit([&] { k_f2f<<<blocks, threads>>>(out, 1.0f); });
    printf("F2F+DADD+F2F %.3f ms  %.2f Giters/s\n", t, ops / t / 1e9 / 1e3 * 1e3);
    t = timeit([&] { k_f2i<<<blocks, threads>>>(out, 0.5); });
    printf("F2I+I2F+DADD %.3f ms  %.2f Giters/s\n", t, ops / t / 1e9);
    size_t n = (size_t)1 << 28;  // 1 GiB of float4? 2^28 float4 = 4 GiB
    n = (size_t)1 << 26;         // 1 GiB
    float4 *a, *b;
    cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
    cudaMemset(a, 0, n * 16);
    t = timeit([&] { k_copy<<<sms * 16, 512>>>(a, b, n); });
    printf("COPY   %.3f ms  %.1f GB/s (read+write)\n", t, 2.0 * n * 16 / t / 1e6);
    cudaError_t e = cudaGetLastError();
    printf("err=%s\n", cudaGetErrorString(e));
    return 0;
}
