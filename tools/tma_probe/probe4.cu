#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__device__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
struct Args { CUtensorMap m0, m1; int x, y; float* out; };
__device__ void body(const CUtensorMap* m, int x, int y, float* out) {
    extern __shared__ __align__(1024) float sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(64 * 72 * 3 * 4) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(su(sm)), "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(0), "r"(su(&bar)) : "memory");
    }
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" ::"r"(su(&bar)) : "memory");
    __syncthreads();
    if (threadIdx.x == 0) out[0] = sm[100];
}
__global__ void kA(const __grid_constant__ CUtensorMap m, int x, int y, float* out) { body(&m, x, y, out); }
__global__ void kB(const __grid_constant__ Args a) { body(&a.m0, a.x, a.y, a.out); }
__global__ void kC(const __grid_constant__ Args a) { body(&a.m1, a.x, a.y, a.out); }
int main() {
    void* p; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    EncodeTiledFn enc = (EncodeTiledFn)p;
    const int W = 64, H = 64;
    float *E, *out; cudaMalloc(&E, W * H * 6 * 4); cudaMalloc(&out, 64);
    CUtensorMap m;
    cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, 6}, str[2] = {W * 4ull, W * H * 4ull};
    cuuint32_t box[3] = {64, 72, 3}, es[3] = {1, 1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, E, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    Args a; a.m0 = m; a.m1 = m; a.x = -6; a.y = -6; a.out = out;
    for (auto f : {(const void*)kA, (const void*)kB, (const void*)kC})
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    struct { const char* n; int which; size_t smem; int thr; } v[] = {
        {"A small", 0, 55296, 128}, {"A big smem", 0, 196672, 128}, {"A 384thr", 0, 55296, 384},
        {"B struct m0", 1, 55296, 128}, {"C struct m1", 2, 55296, 128}, {"B big", 1, 196672, 384}};
    for (auto& t : v) {
        if (t.which == 0) kA<<<1, t.thr, t.smem>>>(m, -6, -6, out);
        else if (t.which == 1) kB<<<1, t.thr, t.smem>>>(a);
        else kC<<<1, t.thr, t.smem>>>(a);
        cudaError_t e = cudaDeviceSynchronize();
        printf("%-12s: %s\n", t.n, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
