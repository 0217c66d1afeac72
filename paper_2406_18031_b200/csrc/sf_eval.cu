// sf_eval.cu -- evaluation outputs: tangent / normal flow in pixels
// (eq:tangent_flow, eq:normal_flow) and RMSE / AAE against a ground truth
// (eq:RMSE_vel and the AAE of P:L726-734), per pixel, with per-batch-member means.
// Arithmetic order as DESIGN.md section 4 / readings 22-23 (the float32 oracle's or_flow_px /
// or_eval follow the same order): float32 for the flows and the RMSE, double for the AAE.
#include "sf_internal.cuh"

namespace {

constexpr int EB = 256;  // threads per block

__device__ __forceinline__ double ddot3(double a0, double a1, double a2, double x0, double x1, double x2) {
    return __fma_rn(a2, x2, __fma_rn(a1, x1, __dmul_rn(a0, x0)));
}

// tangent = (e1 . t, e2 . t), t = P(s) w = w - s <s,w>;  normal = <s,w> / ds
__global__ void k_flow_px(const float4* __restrict__ st, const float4* __restrict__ G0, const float4* __restrict__ G1,
                          const float4* __restrict__ G2, float2* tangent, float* normal, size_t HW, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const size_t p = i % HW;
        const float4 w = st[i], s = __ldg(G0 + p), e1 = __ldg(G1 + p), e2 = __ldg(G2 + p);
        const float sw = xdot3(s, w);
        const float4 t = make_float4(xfma(-s.x, sw, w.x), xfma(-s.y, sw, w.y), xfma(-s.z, sw, w.z), 0.0f);
        if (tangent) tangent[i] = make_float2(xdot3(e1, t), xdot3(e2, t));
        if (normal) normal[i] = __fdiv_rn(sw, e1.w);
    }
}

// Per-pixel RMSE (float) and AAE (double, degrees) on rows [r0, r1) of each batch member;
// block partial sums in a fixed tree order (deterministic).
__global__ void __launch_bounds__(EB) k_eval(const float4* __restrict__ st, const float* __restrict__ wgt,
                                             const float4* __restrict__ G1, float* rmse, double* aae, int W,
                                             size_t HW, int r0, int r1, double* part) {
    __shared__ double red[2][EB];
    const int b = blockIdx.y;
    const size_t lo = (size_t)r0 * W, hi = (size_t)r1 * W;
    double s0 = 0.0, s1 = 0.0;
    for (size_t p = lo + blockIdx.x * (size_t)EB + threadIdx.x; p < hi; p += (size_t)gridDim.x * EB) {
        const size_t i = (size_t)b * HW + p;
        const float4 w = st[i];
        const float g0 = wgt[3 * i], g1 = wgt[3 * i + 1], g2 = wgt[3 * i + 2];
        const float ds = __ldg(&G1[p].w);
        const float4 d = make_float4(__fdiv_rn(xsub(g0, w.x), ds), __fdiv_rn(xsub(g1, w.y), ds),
                                     __fdiv_rn(xsub(g2, w.z), ds), 0.0f);
        const float e = __fsqrt_rn(xdot3(d, d));
        const double dd = (double)ds;
        const double a0 = __ddiv_rn(g0, dd), a1 = __ddiv_rn(g1, dd), a2 = __ddiv_rn(g2, dd);
        const double b0 = __ddiv_rn(w.x, dd), b1 = __ddiv_rn(w.y, dd), b2 = __ddiv_rn(w.z, dd);
        double c = __ddiv_rn(__dadd_rn(1.0, ddot3(a0, a1, a2, b0, b1, b2)),
                             __dmul_rn(__dsqrt_rn(__dadd_rn(1.0, ddot3(a0, a1, a2, a0, a1, a2))),
                                       __dsqrt_rn(__dadd_rn(1.0, ddot3(b0, b1, b2, b0, b1, b2)))));
        c = fmin(fmax(c, -1.0), 1.0);
        const double ang = __dmul_rn(acos(c), 180.0 / 3.14159265358979323846);
        if (rmse) rmse[i] = e;
        if (aae) aae[i] = ang;
        s0 += (double)e;
        s1 += ang;
    }
    red[0][threadIdx.x] = s0;
    red[1][threadIdx.x] = s1;
    __syncthreads();
    for (int k = EB / 2; k > 0; k >>= 1) {
        if (threadIdx.x < k) {
            red[0][threadIdx.x] += red[0][threadIdx.x + k];
            red[1][threadIdx.x] += red[1][threadIdx.x + k];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[2 * ((size_t)b * gridDim.x + blockIdx.x)] = red[0][0];
        part[2 * ((size_t)b * gridDim.x + blockIdx.x) + 1] = red[1][0];
    }
}

constexpr int SF_EVAL_BLOCKS = 296;  // 2 x 148 SMs

}  // namespace

extern "C" sf_status sf_flow_px(sf_ctx* c, float* tangent, float* normal) {
    SF_NVTX("sf_flow_px");
    if (!c) return SF_E_DATA;
    SF_DEVICE_GUARD(c);
    if (!c->initialized) return SF_E_STATE;
    const FrameParams& f = c->fp;
    const size_t HW = (size_t)f.H * f.W, n = HW * f.B;
    if (!tangent && !normal) return SF_OK;
    const int blocks = (int)((n + 255) / 256 < 4 * 148 ? (n + 255) / 256 : 4 * 148);
    k_flow_px<<<blocks, 256, 0, c->stream>>>(sf_flow_plane(c), c->G0, c->G1, c->G2,
                                             reinterpret_cast<float2*>(tangent), normal, HW, n);
    SF_TRY(cudaGetLastError());
    return SF_OK;
}

extern "C" sf_status sf_eval(sf_ctx* c, const float* w_gt, float* rmse, double* aae_deg, double* mean_rmse,
                             double* mean_aae) {
    SF_NVTX("sf_eval");
    if (!c || !w_gt) return SF_E_DATA;
    SF_DEVICE_GUARD(c);
    if (!c->initialized) return SF_E_STATE;
    const FrameParams& f = c->fp;
    const size_t HW = (size_t)f.H * f.W;
    const size_t np = (size_t)f.B * SF_EVAL_BLOCKS * 2;
    if (!c->eval_part) SF_TRY(cudaMalloc(&c->eval_part, np * sizeof(double)));
    // means over the owned rows (the whole grid unless banded)
    const int r0 = c->own_begin - c->ext_begin, r1 = c->own_end - c->ext_begin;
    k_eval<<<dim3(SF_EVAL_BLOCKS, f.B), EB, 0, c->stream>>>(sf_flow_plane(c), w_gt, c->G1, rmse, aae_deg, f.W, HW,
                                                          r0, r1, c->eval_part);
    SF_TRY(cudaGetLastError());
    if (mean_rmse || mean_aae) {
        double* h = (double*)malloc(np * sizeof(double));
        if (!h) return SF_E_CUDA;
        cudaError_t e = cudaMemcpyAsync(h, c->eval_part, np * sizeof(double), cudaMemcpyDeviceToHost, c->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
        if (e != cudaSuccess) {
            free(h);
            return SF_E_CUDA;
        }
        const double cnt = (double)(r1 - r0) * f.W;
        for (int b = 0; b < f.B; ++b) {
            double s0 = 0.0, s1 = 0.0;
            for (int k = 0; k < SF_EVAL_BLOCKS; ++k) {
                s0 += h[2 * ((size_t)b * SF_EVAL_BLOCKS + k)];
                s1 += h[2 * ((size_t)b * SF_EVAL_BLOCKS + k) + 1];
            }
            if (mean_rmse) mean_rmse[b] = s0 / cnt;
            if (mean_aae) mean_aae[b] = s1 / cnt;
        }
        free(h);
    }
    return SF_OK;
}
