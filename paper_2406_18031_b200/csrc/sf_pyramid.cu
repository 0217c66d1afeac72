// sf_pyramid.cu -- H = 2 pyramid plumbing (DESIGN readings 24-30):
// 2x2-mean down-sampling of the measurements for the top level, bilinear up-sampling of the top
// flow with the reconstruction w = up(w^2) + dw (eq:hflow_reconstruction), and the unpacking of the
// bottom-level state.  The transport / update kernels of the bottom level live in sf_passes.cu;
// the top level is an ordinary H = 1 context (sf_api.cu).
#include "sf_internal.cuh"

namespace {

// reading 24: Y2 = ((Y00 + Y01) + (Y10 + Y11)) * 0.25; depth likewise when all four samples are
// valid, else NaN (invalid)
__global__ void k_down2(const float* __restrict__ Y, const float* __restrict__ D, float* Y2, float* D2, int H, int W,
                        int B, int is_inv) {
    const int Hc = H / 2, Wc = W / 2;
    const size_t n = (size_t)B * Hc * Wc;
    for (size_t o = blockIdx.x * (size_t)blockDim.x + threadIdx.x; o < n; o += (size_t)gridDim.x * blockDim.x) {
        const int J = (int)(o % Wc), I = (int)((o / Wc) % Hc), b = (int)(o / ((size_t)Wc * Hc));
        const size_t a = ((size_t)b * H + 2 * I) * W + 2 * J, c = a + W;
        Y2[o] = xmul(xadd(xadd(Y[a], Y[a + 1]), xadd(Y[c], Y[c + 1])), 0.25f);
        const float d0 = D[a], d1 = D[a + 1], d2 = D[c], d3 = D[c + 1];
        const bool ok = depth_valid(d0, is_inv) && depth_valid(d1, is_inv) && depth_valid(d2, is_inv) &&
                        depth_valid(d3, is_inv);
        D2[o] = ok ? xmul(xadd(xadd(d0, d1), xadd(d2, d3)), 0.25f) : __int_as_float(0x7fc00000);
    }
}

// reading 25: bilinear at the fine pixel centres, weights (3/4, 1/4), replicate border;
// h_r = fma(wc1, X[r][c1], X[r][c0] wc0), up = fma(wr1, h_r1, h_r0 wr0); out = (up + dw, Yhat)
__global__ void k_up2_add(const float4* __restrict__ w2, const float4* __restrict__ dwr, const float* __restrict__ yh,
                          float4* out, int H, int W, int B) {
    const int Hc = H / 2, Wc = W / 2;
    const size_t n = (size_t)B * H * W;
    for (size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x; p < n; p += (size_t)gridDim.x * blockDim.x) {
        const int j = (int)(p % W), i = (int)((p / W) % H), b = (int)(p / ((size_t)W * H));
        out[p] = up2_add_at(w2 + (size_t)b * (H / 2) * (W / 2), i, j, H, W, dwr[p], yh[p]);
    }
}

__global__ void k_unpack_pyr(const float4* __restrict__ Wf, const float4* __restrict__ A, float* w, float* rho,
                             float* yhat, size_t n) {
    for (size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x; p < n; p += (size_t)gridDim.x * blockDim.x) {
        const float4 v = Wf[p];
        if (w) {
            w[3 * p] = v.x;
            w[3 * p + 1] = v.y;
            w[3 * p + 2] = v.z;
        }
        if (yhat) yhat[p] = v.w;
        if (rho) rho[p] = A[p].w;
    }
}

inline unsigned blocks_for(size_t n) {
    const size_t b = (n + 255) / 256;
    return (unsigned)(b < 8 * 148 ? b : 8 * 148);
}

}  // namespace

cudaError_t sf_launch_down2(sf_ctx* c, const float* Y, const float* D) {
    const FrameParams& f = c->fp;
    const size_t n = (size_t)f.B * (f.H / 2) * (f.W / 2);
    k_down2<<<blocks_for(n), 256, 0, c->stream>>>(Y, D, c->Y2, c->D2, f.H, f.W, f.B, f.is_inv);
    return cudaGetLastError();
}

cudaError_t sf_launch_up2_add(sf_ctx* c, const float4* w2, const float4* dwr, const float* yh, float4* out) {
    const FrameParams& f = c->fp;
    const size_t n = (size_t)f.B * f.H * f.W;
    k_up2_add<<<blocks_for(n), 256, 0, c->stream>>>(w2, dwr, yh, out, f.H, f.W, f.B);
    return cudaGetLastError();
}

cudaError_t sf_launch_unpack_pyr(sf_ctx* c, float* w, float* rho, float* yhat) {
    const FrameParams& f = c->fp;
    const size_t n = (size_t)f.B * f.H * f.W;
    k_unpack_pyr<<<blocks_for(n), 256, 0, c->stream>>>(c->Wf[c->cur], c->state[c->cur], w, rho, yhat, n);
    return cudaGetLastError();
}
