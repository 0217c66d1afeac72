// sf_map.cu -- Spherepix input mapping (DESIGN reading 31):
// a pinhole camera's brightness and z-depth resampled onto the grid, one thread per grid pixel,
// in the float32 operation order of the oracle's or_map_inputs.
#include <math.h>
#include <string.h>

#include "sf_internal.cuh"

namespace {

__global__ void k_map_inputs(const float4* __restrict__ G0, const float* __restrict__ Ycam,
                             const float* __restrict__ Zcam, float* Y, float* D, MapParams m, size_t HW, int B) {
    const size_t n = HW * B;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const size_t p = i % HW, b = i / HW;
        const float4 s = __ldg(G0 + p);
        const size_t cam = b * (size_t)m.Hc * m.Wc;
        map_cell(m, s.x, s.y, s.z, Ycam + cam, Zcam + cam, Y[i], D[i]);
    }
}

}  // namespace

static sf_status make_map_params(int32_t cam_height, int32_t cam_width, const float* K, const float* Rcg,
                                 MapParams* m) {
    if (!K) return SF_E_DATA;
    if (cam_height < 1 || cam_width < 1 || (long long)cam_height * cam_width > (1LL << 31)) return SF_E_CONFIG;
    if (!(K[0] != 0.0f) || !(K[1] != 0.0f) || !isfinite(K[0]) || !isfinite(K[1]) || !isfinite(K[2]) ||
        !isfinite(K[3]))
        return SF_E_CONFIG;
    if (Rcg) {
        memcpy(m->R, Rcg, sizeof(m->R));
    } else {
        const float I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
        memcpy(m->R, I, sizeof(m->R));
    }
    m->fx = K[0];
    m->fy = K[1];
    m->cx = K[2];
    m->cy = K[3];
    m->Hc = cam_height;
    m->Wc = cam_width;
    return SF_OK;
}

extern "C" sf_status sf_map_inputs(sf_ctx* c, const float* Ycam, const float* Zcam, int32_t cam_height,
                                   int32_t cam_width, const float* K, const float* Rcg, float* Y, float* D) {
    SF_NVTX("sf_map_inputs");
    if (!c || !Ycam || !Zcam || !K || !Y || !D) return SF_E_DATA;
    SF_DEVICE_GUARD(c);
    MapParams m;
    sf_status st = make_map_params(cam_height, cam_width, K, Rcg, &m);
    if (st != SF_OK) return st;
    const FrameParams& f = c->fp;
    const size_t HW = (size_t)f.H * f.W, n = HW * f.B;
    const unsigned blocks = (unsigned)((n + 255) / 256 < 8 * 148 ? (n + 255) / 256 : 8 * 148);
    k_map_inputs<<<blocks, 256, 0, c->stream>>>(c->G0, Ycam, Zcam, Y, D, m, HW, f.B);
    SF_TRY(cudaGetLastError());
    return SF_OK;
}

// One frame straight from camera images: k_map_inputs into context buffers, then sf_step.  (Doing
// the mapping inside the fused kernel's staging was measured slower -- 38.2 vs 37.2 us at 512^2:
// the per-cell gathers lengthen the one-wave kernel's prologue.)
extern "C" sf_status sf_step_camera(sf_ctx* c, const float* Ycam, const float* Zcam, int32_t cam_height,
                                    int32_t cam_width, const float* K, const float* Rcg) {
    SF_NVTX("sf_step_camera");
    if (!c || !Ycam || !Zcam || !K) return SF_E_DATA;
    SF_DEVICE_GUARD(c);
    MapParams m;
    sf_status st = make_map_params(cam_height, cam_width, K, Rcg, &m);
    if (st != SF_OK) return st;
    const size_t n = (size_t)c->fp.B * c->fp.H * c->fp.W;
    if (!c->mY) {  // committed only when both allocations succeed
        float *y = nullptr, *d = nullptr;
        if (cudaMalloc(&y, n * sizeof(float)) != cudaSuccess || cudaMalloc(&d, n * sizeof(float)) != cudaSuccess) {
            if (y) cudaFree(y);
            return SF_E_CUDA;
        }
        c->mY = y;
        c->mD = d;
    }
    st = sf_map_inputs(c, Ycam, Zcam, cam_height, cam_width, K, Rcg, c->mY, c->mD);
    if (st != SF_OK) return st;
    return sf_step(c, c->mY, c->mD);
}
