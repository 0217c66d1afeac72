// Standalone TMA probe: 3-D fp32 box copies of various shapes into shared memory.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__device__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap m, int bx, int by, int bz, int x, int y, float* out) {
    extern __shared__ __align__(1024) float sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(bx * by * bz * 4) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(su(sm)), "l"(reinterpret_cast<uint64_t>(&m)), "r"(x), "r"(y), "r"(0), "r"(su(&bar)) : "memory");
    }
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" ::"r"(su(&bar)) : "memory");
    __syncthreads();
    for (int i = threadIdx.x; i < bx * by * bz; i += blockDim.x) out[i] = sm[i];
}
int main() {
    void* p; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    EncodeTiledFn enc = (EncodeTiledFn)p;
    const int W = 64, H = 64, Z = 6;
    float* g; cudaMalloc(&g, W * H * Z * 4);
    float* h = (float*)malloc(W * H * Z * 4); for (int i = 0; i < W * H * Z; ++i) h[i] = i;
    cudaMemcpy(g, h, W * H * Z * 4, cudaMemcpyHostToDevice);
    float* out; cudaMalloc(&out, 256 * 256 * 4 * 4);
    int shapes[][5] = {{64, 72, 1, 0, 0}, {64, 72, 3, 0, 0}, {64, 72, 1, -12, -12}, {64, 72, 3, -12, -12}, {32, 32, 1, 0, 0}};
    for (auto& s : shapes) {
        CUtensorMap m;
        cuuint64_t dims[3] = {W, H, Z}, str[2] = {W * 4, W * H * 4};
        cuuint32_t box[3] = {(cuuint32_t)s[0], (cuuint32_t)s[1], (cuuint32_t)s[2]}, es[3] = {1, 1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        size_t smem = (size_t)s[0] * s[1] * s[2] * 4;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
        k<<<1, 128, smem>>>(m, s[0], s[1], s[2], s[3], s[4], out);
        cudaError_t e = cudaDeviceSynchronize();
        printf("box %dx%dx%d at (%d,%d): encode=%d launch=%s\n", s[0], s[1], s[2], s[3], s[4], (int)r, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
