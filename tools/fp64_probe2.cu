// Does F2F.F64.F32 / F2F.F32.F64 share the issue budget of DADD?  (B200 pipe probe)
#include <cstdio>
#include <cuda_runtime.h>
#define IT 2048
__global__ void k_dadd8(double* o, double a) {   // 8 DADD per iter
    double x[8];
    for (int c = 0; c < 8; c++) x[c] = threadIdx.x + c;
    for (int i = 0; i < IT; i++)
#pragma unroll
        for (int c = 0; c < 8; c++) x[c] = __dadd_rn(x[c], a);
    double s = 0; for (int c = 0; c < 8; c++) s += x[c]; if (s == 1.2345) o[0] = s;
}
__global__ void k_dadd8_f2f2(double* o, double a) {  // 8 DADD + 2 F2F.F64.F32 per iter
    double x[8]; float f[2];
    for (int c = 0; c < 8; c++) x[c] = threadIdx.x + c;
    f[0] = threadIdx.x; f[1] = threadIdx.x + 1;
    for (int i = 0; i < IT; i++) {
#pragma unroll
        for (int c = 0; c < 8; c++) x[c] = __dadd_rn(x[c], a);
        double d0 = (double)f[0], d1 = (double)f[1];
        f[0] = __int_as_float(__double2hiint(d0) ^ 1); f[1] = __int_as_float(__double2hiint(d1) ^ 1);
    }
    double s = f[0] + f[1]; for (int c = 0; c < 8; c++) s += x[c]; if (s == 1.2345) o[0] = s;
}
__global__ void k_f2f2(double* o, double a) {  // 2 F2F.F64.F32 per iter only
    float f[2];
    f[0] = threadIdx.x; f[1] = threadIdx.x + 1;
    for (int i = 0; i < IT; i++) {
        double d0 = (double)f[0], d1 = (double)f[1];
        f[0] = __int_as_float(__double2hiint(d0) ^ 1); f[1] = __int_as_float(__double2hiint(d1) ^ 1);
    }
    double s = f[0] + f[1]; if (s == 1.2345) o[0] = s;
}
__global__ void k_dadd8_d2f2(double* o, double a) {  // 8 DADD + 2 F2F.F32.F64 per iter
    double x[8]; double y[2];
    for (int c = 0; c < 8; c++) x[c] = threadIdx.x + c;
    y[0] = threadIdx.x; y[1] = threadIdx.x + 1;
    for (int i = 0; i < IT; i++) {
#pragma unroll
        for (int c = 0; c < 8; c++) x[c] = __dadd_rn(x[c], a);
        float f0 = __double2float_rn(y[0]), f1 = __double2float_rn(y[1]);
        y[0] = __hiloint2double(__float_as_int(f0), 7); y[1] = __hiloint2double(__float_as_int(f1), 9);
    }
    double s = y[0] + y[1]; for (int c = 0; c < 8; c++) s += x[c]; if (s == 1.2345) o[0] = s;
}
template <typename F> float tm(F f) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    f(); cudaDeviceSynchronize(); cudaEventRecord(a); for (int r = 0; r < 5; r++) f(); cudaEventRecord(b);
    cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); return ms / 5;
}
int main() {
    double* o; cudaMalloc(&o, 8);
    int B = 148 * 8, T = 256;
    printf("8 DADD            %.3f ms\n", tm([&] { k_dadd8<<<B, T>>>(o, 1.0000001); }));
    printf("8 DADD + 2 F2F.64 %.3f ms\n", tm([&] { k_dadd8_f2f2<<<B, T>>>(o, 1.0000001); }));
    printf("2 F2F.64 only     %.3f ms\n", tm([&] { k_f2f2<<<B, T>>>(o, 1.0000001); }));
    printf("8 DADD + 2 F2F.32 %.3f ms\n", tm([&] { k_dadd8_d2f2<<<B, T>>>(o, 1.0000001); }));
    return 0;
}
