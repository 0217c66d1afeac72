// sf_map.cu -- Spherepix input mapping (DESIGN reading 31):
// a pinhole camera's brightness and z-depth resampled onto the grid, one thread per grid pixel,
// in the float32 operation order of the oracle's or_map_inputs.
#include <math.h>
#include <string.h>

#include "sf_internal.cuh"

namespace {

struct MapParams {
    float R[9];  // grid -> camera rotation, row-major
    float fx, fy, cx, cy;
    int Hc, Wc;
};

__global__ void k_map_inputs(const float4* __restrict__ G0, const float* __restrict__ Ycam,
                             const float* __restrict__ Zcam, float* Y, float* D, MapParams m, size_t HW, int B) {
    const size_t n = HW * B;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const size_t p = i % HW, b = i / HW;
        const float4 s = __ldg(G0 + p);
        float t[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) t[r] = xfma(m.R[3 * r + 2], s.z, xfma(m.R[3 * r + 1], s.y, xmul(m.R[3 * r], s.x)));
        const bool front = t[2] > 0.0f;
        float u = 0.0f, v = 0.0f;
        if (front) {
            u = xfma(m.fx, __fdiv_rn(t[0], t[2]), m.cx);
            v = xfma(m.fy, __fdiv_rn(t[1], t[2]), m.cy);
        }
        const bool inside =
            front && u >= -0.5f && u <= (float)m.Wc - 0.5f && v >= -0.5f && v <= (float)m.Hc - 0.5f;
        const float uc = fminf(fmaxf(u, 0.0f), (float)(m.Wc - 1)), vc = fminf(fmaxf(v, 0.0f), (float)(m.Hc - 1));
        const int j0 = (int)floorf(uc), i0 = (int)floorf(vc);
        const int j1 = min(j0 + 1, m.Wc - 1), i1 = min(i0 + 1, m.Hc - 1);
        const float bw = xsub(uc, (float)j0), aw = xsub(vc, (float)i0);
        const size_t base = b * (size_t)m.Hc * m.Wc;
        const size_t q00 = base + (size_t)i0 * m.Wc + j0, q01 = base + (size_t)i0 * m.Wc + j1;
        const size_t q10 = base + (size_t)i1 * m.Wc + j0, q11 = base + (size_t)i1 * m.Wc + j1;
        {
            const float y00 = __ldg(Ycam + q00), y01 = __ldg(Ycam + q01), y10 = __ldg(Ycam + q10),
                        y11 = __ldg(Ycam + q11);
            const float r0 = xfma(bw, xsub(y01, y00), y00), r1 = xfma(bw, xsub(y11, y10), y10);
            Y[i] = xfma(aw, xsub(r1, r0), r0);
        }
        const float z00 = __ldg(Zcam + q00), z01 = __ldg(Zcam + q01), z10 = __ldg(Zcam + q10), z11 = __ldg(Zcam + q11);
        const bool zok = isfinite(z00) && z00 > 0.0f && isfinite(z01) && z01 > 0.0f && isfinite(z10) &&
                         z10 > 0.0f && isfinite(z11) && z11 > 0.0f;
        if (inside && zok) {
            const float r0 = xfma(bw, xsub(z01, z00), z00), r1 = xfma(bw, xsub(z11, z10), z10);
            D[i] = __fdiv_rn(xfma(aw, xsub(r1, r0), r0), t[2]);
        } else {
            D[i] = __int_as_float(0x7fc00000);
        }
    }
}

}  // namespace

extern "C" sf_status sf_map_inputs(sf_ctx* c, const float* Ycam, const float* Zcam, int32_t cam_height,
                                   int32_t cam_width, const float* K, const float* Rcg, float* Y, float* D) {
    if (!c || !Ycam || !Zcam || !K || !Y || !D) return SF_E_DATA;
    if (cam_height < 1 || cam_width < 1 || (long long)cam_height * cam_width > (1LL << 31)) return SF_E_CONFIG;
    if (!(K[0] != 0.0f) || !(K[1] != 0.0f) || !isfinite(K[0]) || !isfinite(K[1]) || !isfinite(K[2]) ||
        !isfinite(K[3]))
        return SF_E_CONFIG;
    MapParams m;
    if (Rcg) {
        memcpy(m.R, Rcg, sizeof(m.R));
    } else {
        const float I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
        memcpy(m.R, I, sizeof(m.R));
    }
    m.fx = K[0];
    m.fy = K[1];
    m.cx = K[2];
    m.cy = K[3];
    m.Hc = cam_height;
    m.Wc = cam_width;
    const FrameParams& f = c->fp;
    const size_t HW = (size_t)f.H * f.W, n = HW * f.B;
    const unsigned blocks = (unsigned)((n + 255) / 256 < 8 * 148 ? (n + 255) / 256 : 8 * 148);
    k_map_inputs<<<blocks, 256, 0, c->stream>>>(c->G0, Ycam, Zcam, Y, D, m, HW, f.B);
    SF_TRY(cudaGetLastError());
    return SF_OK;
}
