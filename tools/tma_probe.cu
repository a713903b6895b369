// TMA probe: per-warp 3-D box loads (in-bounds / out-of-bounds) with per-warp mbarriers.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/bin/tma_probe tools/tma_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>

typedef unsigned long long u64;
typedef uint32_t u32;
__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap tmap, float* out, int nwarps_active, int c0, int c1, int c2,
                      int box_elems, int mode) {
    extern __shared__ __align__(128) unsigned char smem[];
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float* tile = (float*)(smem + warp * 8192);
    u64* bar = (u64*)(smem + 8 * 8192 + warp * 16);
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp >= nwarps_active) return;
    if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(box_elems * 4) : "memory");
        if (mode == 0)
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                    smem_u32(tile)),
                "l"((u64)&tmap), "r"(c0), "r"(c1 + warp), "r"(c2), "r"(smem_u32(bar))
                : "memory");
        else
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                    smem_u32(tile)),
                "l"((u64)&tmap), "r"(c0), "r"(c1 + warp), "r"(c2), "r"(smem_u32(bar))
                : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(smem_u32(bar)),
        "r"(0)
        : "memory");
    __syncwarp();
    for (int t = lane; t < box_elems; t += 32) out[warp * 2048 + t] = tile[t];
}

int main(int argc, char** argv) {
    int nx = 16, ny = 16, nz = 16;
    std::vector<float> h(nx * ny * nz);
    for (size_t i = 0; i < h.size(); i++) h[i] = (float)i;
    float *d, *o;
    cudaMalloc(&d, h.size() * 4);
    cudaMalloc(&o, 32 * 2048 * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 8192 + 256);
    struct T { int nw, c0, c1, c2, mode; const char* what; };
    T tests[] = {{1, 0, 0, 0, 0, "in-bounds"},       {1, 4, 0, 0, 0, "c0=4 fits"},
                 {1, 8, 0, 0, 0, "c0=8 oob16B"},      {1, 10, 0, 0, 0, "c0=10 oob"},
                 {1, 0, 10, 0, 0, "y oob"},           {1, 0, 0, 10, 0, "x oob"},
                 {1, 2, 0, 0, 0, "c0=2 fits"},        {1, 10, 0, 0, 1, "c0=10 oob cta"}};
    int which = argc > 1 ? atoi(argv[1]) : 0;
    for (int ti = which; ti <= which; ti++) {
        T& t = tests[ti];
        CUtensorMap m;
        cuuint64_t dims[3] = {(cuuint64_t)nz, (cuuint64_t)ny, (cuuint64_t)nx};
        cuuint64_t strides[2] = {(cuuint64_t)nz * 4, (cuuint64_t)nz * ny * 4};
        cuuint32_t box[3] = {12, 10, 10};
        cuuint32_t es[3] = {1, 1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        probe<<<1, 32 * 8, 8 * 8192 + 256>>>(m, o, t.nw, t.c0, t.c1, t.c2, 1200, t.mode);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> ho(2048);
        cudaMemcpy(ho.data(), o, 2048 * 4, cudaMemcpyDeviceToHost);
        printf("%-22s enc=%d -> %s  first %g %g last %g\n", t.what, (int)r, cudaGetErrorString(e), ho[0], ho[1], ho[1199]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
