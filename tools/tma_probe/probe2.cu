// TMA probe 2: struct parameter with three tensor maps, large dynamic smem, barriers at the end.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__device__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
struct Args { CUtensorMap tmE, tmY, tmD; int tma; const float* x; float* out; int mode; };
constexpr int P = 64 * 72;
__global__ void __launch_bounds__(384, 1) k(const __grid_constant__ Args a) {
    extern __shared__ __align__(1024) float4 smem4[];
    float* sm = reinterpret_cast<float*>(smem4);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 8 * P + 12288);
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int i = 0; i < 3; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bars[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        const CUtensorMap* maps[4] = {&a.tmE, &a.tmE, &a.tmY, &a.tmD};
        float* dst[4] = {sm, sm + 3 * P, sm + 6 * P, sm + 7 * P};
        int z[4] = {0, 3, 0, 0};
        unsigned by[4] = {3u * P * 4, 3u * P * 4, P * 4u, P * 4u};
        int bi[4] = {0, 1, 2, 2};
        for (int i = 0; i < 4; ++i) {
            if (!(a.mode & (1 << i))) continue;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bars[bi[i]])), "r"(by[i]) : "memory");
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(su(dst[i])), "l"(reinterpret_cast<uint64_t>(maps[i])), "r"(-6), "r"(-6), "r"(z[i]), "r"(su(&bars[bi[i]])) : "memory");
        }
    }
    for (int i = 0; i < 3; ++i) {
        int need = (i == 0 && (a.mode & 1)) || (i == 1 && (a.mode & 2)) || (i == 2 && (a.mode & 12));
        if (need) asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" ::"r"(su(&bars[i])) : "memory");
    }
    __syncthreads();
    if (tid == 0) a.out[0] = sm[6 * 64 + 6];
}
int main() {
    void* p; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    EncodeTiledFn enc = (EncodeTiledFn)p;
    const int W = 64, H = 64;
    float *E, *Y, *D, *out; cudaMalloc(&E, W * H * 6 * 4); cudaMalloc(&Y, W * H * 4); cudaMalloc(&D, W * H * 4); cudaMalloc(&out, 64);
    Args a;
    auto mk = [&](CUtensorMap* m, float* g, int z, int bz) {
        cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)z}, str[2] = {W * 4ull, W * H * 4ull};
        cuuint32_t box[3] = {64, 72, (cuuint32_t)bz}, es[3] = {1, 1, 1};
        return (int)enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    printf("encode %d %d %d\n", mk(&a.tmE, E, 6, 3), mk(&a.tmY, Y, 1, 1), mk(&a.tmD, D, 1, 1));
    a.out = out;
    const size_t smem = (8 * P + 12288) * 4 + 64;
    printf("set attr: %s\n", cudaGetErrorString(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)));
    for (int mode : {1, 2, 4, 8, 15}) {
        a.mode = mode;
        k<<<1, 384, smem>>>(a);
        cudaError_t e = cudaDeviceSynchronize();
        printf("mode %d: %s\n", mode, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
