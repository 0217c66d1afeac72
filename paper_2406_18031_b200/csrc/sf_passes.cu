// sf_passes.cu -- the per-pass kernels of the structure-flow filter (one launch per
// transport pass / update stage).  This is the simple reference GPU path and the one
// the banded multi-GPU mode uses between halo exchanges; sf_fused.cu computes the same
// bits in one launch per frame.  Arithmetic order: DESIGN.md section 4.
#include "sf_internal.cuh"

namespace {

constexpr int BX = 32, BY = 8;

inline dim3 grid_for(const FrameParams& f) { return dim3((f.W + BX - 1) / BX, (f.H + BY - 1) / BY, f.B); }

// ------------------------------------------------------------------ geometry
// e_k = b_k / ds (IEEE division), d2 = ds * ds (reading 5).
__global__ void k_geometry(const float* __restrict__ g10, float4* G0, float4* G1, float4* G2, int n) {
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const float* g = g10 + 10 * (size_t)p;
    const float ds = g[9];
    G0[p] = make_float4(g[0], g[1], g[2], xmul(ds, ds));
    const float4 e1 = make_float4(__fdiv_rn(g[3], ds), __fdiv_rn(g[4], ds), __fdiv_rn(g[5], ds), ds);
    const float4 e2 = make_float4(__fdiv_rn(g[6], ds), __fdiv_rn(g[7], ds), __fdiv_rn(g[8], ds), 0.0f);
    G1[p] = e1;
    G2[p] = e2;
}

// The padded e planes (sf_internal.cuh SF_EPAD): cell (i, j) of [H + 2 EPAD][W + 2 EPAD] holds e of
// the clamped grid cell (i - EPAD, j - EPAD).
__global__ void k_epad(const float4* __restrict__ G1, const float4* __restrict__ G2, float* E, int H, int W) {
    const int EW = sf_ew(W), EH = sf_eh(H);
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= EW * EH) return;
    const int i = iclamp(q / EW - SF_EPAD, 0, H - 1), j = iclamp(q % EW - SF_EPAD, 0, W - 1);
    const size_t pe = (size_t)EW * EH, p = (size_t)i * W + j;
    const float4 e1 = G1[p], e2 = G2[p];
    E[q] = e1.x;
    E[pe + q] = e1.y;
    E[2 * pe + q] = e1.z;
    E[3 * pe + q] = e2.x;
    E[4 * pe + q] = e2.y;
    E[5 * pe + q] = e2.z;
}

// ------------------------------------------------------------------ transport pass (P1-P4)
// AXIS 0: column pass (beta_1, neighbours (i, j+-1), e1).
// AXIS 1: row pass    (beta_2, neighbours (i+-1, j), e2), P:L674-683 (reading 3).
// Rows [r0, r1) of the grid (the banded substep exchange updates the rows next to a band's cut
// edges after the others, sf_band.cu); the whole grid otherwise.
template <int AXIS>
__global__ void __launch_bounds__(BX* BY) k_pass(const float4* __restrict__ in, float4* __restrict__ out,
                                                const float4* __restrict__ G0, const float4* __restrict__ Ge,
                                                FrameParams f, unsigned* flags, int r0, int r1) {
    const int j = blockIdx.x * BX + threadIdx.x, i = r0 + blockIdx.y * BY + threadIdx.y, b = blockIdx.z;
    const bool live = (i < r1) && (j < f.W);
    const int ii = live ? i : 0, jj = live ? j : 0;
    int im = ii, ip = ii, jm = jj, jp = jj;
    if (AXIS == 0) {
        jm = max(jj - 1, 0);
        jp = min(jj + 1, f.W - 1);
    } else {
        im = max(ii - 1, 0);
        ip = min(ii + 1, f.H - 1);
    }
    const size_t base = (size_t)b * f.H * f.W;
    const int g = ii * f.W + jj, gm = im * f.W + jm, gp = ip * f.W + jp;
    const float4 c = in[base + g], cm = in[base + gm], cp = in[base + gp];
    const float um = xdot3(Ge[gm], cm), up = xdot3(Ge[gp], cp);  // u at p-, p+ (eq:oflow_numeric)
    float uh = dominant(um, up, f.rule);
    bool clamped = false, cfl = false;
    if (f.clamp) {
        clamped = fabsf(uh) > f.U;
        uh = fminf(fmaxf(uh, -f.U), f.U);
    } else {
        cfl = xmul(f.dt, fabsf(uh)) > 1.0f;
    }
    const float q = xmul(f.sigma, xdot3(G0[g], c));  // sigma <s, w> at p
    const bool fwd = uh > 0.0f;
    float4 o;
    // f* = fma(-dt, fma(u_hat, D, f q), f), D = upwind difference
    o.x = xfma(-f.dt, xfma(uh, fwd ? xsub(c.x, cm.x) : xsub(cp.x, c.x), xmul(c.x, q)), c.x);
    o.y = xfma(-f.dt, xfma(uh, fwd ? xsub(c.y, cm.y) : xsub(cp.y, c.y), xmul(c.y, q)), c.y);
    o.z = xfma(-f.dt, xfma(uh, fwd ? xsub(c.z, cm.z) : xsub(cp.z, c.z), xmul(c.z, q)), c.z);
    o.w = xfma(-f.dt, xfma(uh, fwd ? xsub(c.w, cm.w) : xsub(cp.w, c.w), xmul(c.w, q)), c.w);
    const bool own = live && i >= f.fr0 && i < f.fr1;  // banded mode: owned rows only
    raise_flag(flags, own && clamped, SF_FLAG_CLAMPED);
    raise_flag(flags, own && cfl, SF_FLAG_CFL);
    if (AXIS == 1 && f.imu) {  // inertial stage after the row pass (reading 32)
        const float4 sg = G0[g];
        imu_stage(f, sg.x, sg.y, sg.z, o.x, o.y, o.z, o.w);
    }
    if (live) out[base + g] = o;
}

// ------------------------------------------------------------------ pyramid bottom level (NEXT #1)
// One transport pass of the 8 bottom-level fields (reading 26-27): A = (dw, rho) and
// Wf = (w, Yhat), all advected by the dominant flow of the reconstructed w; w, dw and rho carry
// the dilation term sigma <s, w>, Yhat none (eq:img_propagation_low):
//   f* = fma(-dt, fma(u_hat, D, f q), f)   and   Yhat* = fma(-dt, u_hat D, Yhat).
template <int AXIS>
__global__ void __launch_bounds__(BX* BY) k_pass_low(const float4* __restrict__ inA, const float4* __restrict__ inW,
                                                    float4* __restrict__ outA, float4* __restrict__ outW,
                                                    const float4* __restrict__ G0, const float4* __restrict__ Ge,
                                                    FrameParams f, unsigned* flags) {
    const int j = blockIdx.x * BX + threadIdx.x, i = blockIdx.y * BY + threadIdx.y, b = blockIdx.z;
    const bool live = (i < f.H) && (j < f.W);
    const int ii = live ? i : 0, jj = live ? j : 0;
    int im = ii, ip = ii, jm = jj, jp = jj;
    if (AXIS == 0) {
        jm = max(jj - 1, 0);
        jp = min(jj + 1, f.W - 1);
    } else {
        im = max(ii - 1, 0);
        ip = min(ii + 1, f.H - 1);
    }
    const size_t base = (size_t)b * f.H * f.W;
    const int g = ii * f.W + jj, gm = im * f.W + jm, gp = ip * f.W + jp;
    const float4 w = inW[base + g], wm = inW[base + gm], wp = inW[base + gp];
    const float4 a = inA[base + g], am = inA[base + gm], ap = inA[base + gp];
    const float um = xdot3(Ge[gm], wm), up = xdot3(Ge[gp], wp);
    float uh = dominant(um, up, f.rule);
    bool clamped = false, cfl = false;
    if (f.clamp) {
        clamped = fabsf(uh) > f.U;
        uh = fminf(fmaxf(uh, -f.U), f.U);
    } else {
        cfl = xmul(f.dt, fabsf(uh)) > 1.0f;
    }
    const float q = xmul(f.sigma, xdot3(G0[g], w));
    const bool fwd = uh > 0.0f;
    auto tr = [&](float c, float cm, float cp) {
        return xfma(-f.dt, xfma(uh, fwd ? xsub(c, cm) : xsub(cp, c), xmul(c, q)), c);
    };
    float4 oA, oW;
    oA.x = tr(a.x, am.x, ap.x);
    oA.y = tr(a.y, am.y, ap.y);
    oA.z = tr(a.z, am.z, ap.z);
    oA.w = tr(a.w, am.w, ap.w);
    oW.x = tr(w.x, wm.x, wp.x);
    oW.y = tr(w.y, wm.y, wp.y);
    oW.z = tr(w.z, wm.z, wp.z);
    oW.w = xfma(-f.dt, xmul(uh, fwd ? xsub(w.w, wm.w) : xsub(wp.w, w.w)), w.w);
    raise_flag(flags, live && clamped, SF_FLAG_CLAMPED);
    raise_flag(flags, live && cfl, SF_FLAG_CFL);
    if (live) {
        outA[base + g] = oA;
        outW[base + g] = oW;
    }
}

// ------------------------------------------------------------------ update kernels (U1-U6)
// Horizontal taps of the brightness model: HG = hz(g, Y), HH = hz(h, Y).
__global__ void __launch_bounds__(BX* BY) k_hconv(const float* __restrict__ Y, float* HG, float* HH, FrameParams f,
                                                 unsigned* flags) {
    const int j = blockIdx.x * BX + threadIdx.x, i = blockIdx.y * BY + threadIdx.y, b = blockIdx.z;
    const bool live = (i < f.H) && (j < f.W);
    bool bad = false;
    if (live) {
        const float* row = Y + ((size_t)b * f.H + i) * f.W;
        const float x0 = row[max(j - 2, 0)], x1 = row[max(j - 1, 0)], x2 = row[j], x3 = row[min(j + 1, f.W - 1)],
                    x4 = row[min(j + 2, f.W - 1)];
        const size_t p = ((size_t)b * f.H + i) * f.W + j;
        HG[p] = tap_g(x0, x1, x2, x3, x4);
        HH[p] = tap_h(x0, x1, x2, x3, x4);
        bad = !isfinite(x2) && i >= f.fr0 && i < f.fr1;
    }
    raise_flag(flags, bad, SF_FLAG_NONFINITE);
}

struct Models {
    float yh, b1, b2;     // Yhat^{k+1}, beta_hat
    float rh, br1, br2;   // rhohat, beta_rho
    bool valid;
};

__device__ __forceinline__ Models eval_models(const float* __restrict__ HG, const float* __restrict__ HH,
                                              const float* __restrict__ D, int b, int i, int j, const FrameParams& f) {
    Models M;
    const size_t pl = (size_t)b * f.H * f.W;
    float g[5], h[5];
#pragma unroll
    for (int t = 0; t < 5; ++t) {
        const size_t r = pl + (size_t)iclamp(i + t - 2, 0, f.H - 1) * f.W + j;
        g[t] = HG[r];
        h[t] = HH[r];
    }
    M.yh = tap_g(g[0], g[1], g[2], g[3], g[4]);
    M.b1 = tap_g(h[0], h[1], h[2], h[3], h[4]);
    M.b2 = tap_h(g[0], g[1], g[2], g[3], g[4]);
    const float* Dp = D + pl;
    const float dc = Dp[(size_t)i * f.W + j];
    const float dl = Dp[(size_t)i * f.W + max(j - 1, 0)], dr = Dp[(size_t)i * f.W + min(j + 1, f.W - 1)];
    const float du = Dp[(size_t)max(i - 1, 0) * f.W + j], dd = Dp[(size_t)min(i + 1, f.H - 1) * f.W + j];
    const bool vc = depth_valid(dc, f.is_inv), vl = depth_valid(dl, f.is_inv), vr = depth_valid(dr, f.is_inv),
               vu = depth_valid(du, f.is_inv), vd = depth_valid(dd, f.is_inv);
    M.rh = rho_hat(dc, f.is_inv);
    M.br1 = pick_side(M.rh, vc, rho_hat(dl, f.is_inv), vl, rho_hat(dr, f.is_inv), vr);
    M.br2 = pick_side(M.rh, vc, rho_hat(du, f.is_inv), vu, rho_hat(dd, f.is_inv), vd);
    M.valid = vc;
    return M;
}

// First frame: w = 0, rho = rhohat, Yhat = brightness model.
__global__ void __launch_bounds__(BX* BY) k_init(const float* __restrict__ HG, const float* __restrict__ HH,
                                                const float* __restrict__ D, float4* state, float* yhat, FrameParams f) {
    const int j = blockIdx.x * BX + threadIdx.x, i = blockIdx.y * BY + threadIdx.y, b = blockIdx.z;
    if (i >= f.H || j >= f.W) return;
    const Models M = eval_models(HG, HH, D, b, i, j, f);
    const size_t p = ((size_t)b * f.H + i) * f.W + j;
    state[p] = make_float4(0.0f, 0.0f, 0.0f, M.rh);
    yhat[p] = M.yh;
}

// Models + per-pixel LS + fusion (U1-U3, U5) in one launch (reads w^{k+}, rho^{k+} from pred,
// rho^k from st, Yhat^k from yin[i * ys]; writes (w_LS, rho^{k+1}) to out, Yhat^{k+1} to yout): the block stages its (BY + 4) x (BX + 4) brightness window
// (replicate border) in shared memory, forms the horizontal g- and h-taps of its BY + 4 rows,
// then every pixel takes the vertical taps, the inverse-depth model, the LS solve and the
// fusion (operation order: DESIGN.md section 4).
__global__ void __launch_bounds__(BX* BY) k_update(const float* __restrict__ Y, const float* __restrict__ D,
                                                  const float4* __restrict__ pred, const float4* __restrict__ st,
                                                  const float* __restrict__ yin, int ys, float* __restrict__ yout,
                                                  float4* out, const float4* __restrict__ G0,
                                                  const float4* __restrict__ G1, const float4* __restrict__ G2,
                                                  FrameParams f, unsigned* flags) {
    __shared__ float yw[BY + 4][BX + 4];
    __shared__ float hgs[BY + 4][BX], hhs[BY + 4][BX];
    const int tx = threadIdx.x, ty = threadIdx.y, b = blockIdx.z;
    const int j0 = blockIdx.x * BX, i0 = blockIdx.y * BY;
    const float* Yp = Y + (size_t)b * f.H * f.W;
    for (int t = ty * BX + tx; t < (BY + 4) * (BX + 4); t += BX * BY) {
        const int r = t / (BX + 4), c = t % (BX + 4);
        yw[r][c] = Yp[(size_t)iclamp(i0 + r - 2, 0, f.H - 1) * f.W + iclamp(j0 + c - 2, 0, f.W - 1)];
    }
    __syncthreads();
    for (int r = ty; r < BY + 4; r += BY) {
        const float x0 = yw[r][tx], x1 = yw[r][tx + 1], x2 = yw[r][tx + 2], x3 = yw[r][tx + 3], x4 = yw[r][tx + 4];
        hgs[r][tx] = tap_g(x0, x1, x2, x3, x4);
        hhs[r][tx] = tap_h(x0, x1, x2, x3, x4);
    }
    __syncthreads();
    const int j = j0 + tx, i = i0 + ty;
    const bool live = (i < f.H) && (j < f.W);
    bool bad = false;
    if (live) {
        bad = !isfinite(yw[ty + 2][tx + 2]) && i >= f.fr0 && i < f.fr1;  // as k_hconv
        Models M;
        M.yh = tap_g(hgs[ty][tx], hgs[ty + 1][tx], hgs[ty + 2][tx], hgs[ty + 3][tx], hgs[ty + 4][tx]);
        M.b1 = tap_g(hhs[ty][tx], hhs[ty + 1][tx], hhs[ty + 2][tx], hhs[ty + 3][tx], hhs[ty + 4][tx]);
        M.b2 = tap_h(hgs[ty][tx], hgs[ty + 1][tx], hgs[ty + 2][tx], hgs[ty + 3][tx], hgs[ty + 4][tx]);
        const float* Dp = D + (size_t)b * f.H * f.W;
        const float dc = Dp[(size_t)i * f.W + j];
        const float dl = Dp[(size_t)i * f.W + max(j - 1, 0)], dr = Dp[(size_t)i * f.W + min(j + 1, f.W - 1)];
        const float du = Dp[(size_t)max(i - 1, 0) * f.W + j], dd = Dp[(size_t)min(i + 1, f.H - 1) * f.W + j];
        const bool vc = depth_valid(dc, f.is_inv), vl = depth_valid(dl, f.is_inv), vr = depth_valid(dr, f.is_inv),
                   vu = depth_valid(du, f.is_inv), vd = depth_valid(dd, f.is_inv);
        M.rh = rho_hat(dc, f.is_inv);
        M.br1 = pick_side(M.rh, vc, rho_hat(dl, f.is_inv), vl, rho_hat(dr, f.is_inv), vr);
        M.br2 = pick_side(M.rh, vc, rho_hat(du, f.is_inv), vu, rho_hat(dd, f.is_inv), vd);
        M.valid = vc;
        const int gi = i * f.W + j;
        const size_t p = (size_t)b * f.H * f.W + gi;
        const float4 s = G0[gi], e1 = G1[gi], e2 = G2[gi];
        const float d2 = s.w;
        const float e1a[3] = {e1.x, e1.y, e1.z}, e2a[3] = {e2.x, e2.y, e2.z}, sa[3] = {s.x, s.y, s.z};
        float gh[3], m[3];
        const float d2r = xmul(d2, M.rh);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            gh[a] = xmul(d2, xfma(e2a[a], M.b2, xmul(e1a[a], M.b1)));
            const float drr = xmul(d2, xfma(e2a[a], M.br2, xmul(e1a[a], M.br1)));
            m[a] = xfma(d2r, sa[a], drr);
        }
        const float4 wp = pred[p];
        const float4 sk = st[p];
        const float cY = xmul(d2, xsub(M.yh, yin[p * ys]));
        const float cr = xmul(d2, xsub(M.rh, sk.w));
        const float wpa[3] = {wp.x, wp.y, wp.z};
        float x[3];
        ls_solve3(gh, m, cY, cr, wpa, f.g1, M.valid ? f.g2 : 0.0f, f.g3, x);
        const float kap = M.valid ? f.kappa : 0.0f;
        const float rn = xfma(kap, xsub(M.rh, wp.w), wp.w);
        out[p] = make_float4(x[0], x[1], x[2], rn);
        yout[p] = M.yh;
        bad = bad || (!(isfinite(x[0]) && isfinite(x[1]) && isfinite(x[2]) && isfinite(rn)) && i >= f.fr0 && i < f.fr1);
    }
    raise_flag(flags, bad, SF_FLAG_NONFINITE);
}

// 5x5 box smoothing (reading 13); .w (rho^{k+1}) rides along unchanged.
// One whole box iteration (horizontal 5-sums, then vertical 5-sums / 25; the order of k_box_h +
// k_box_v) per launch: the block stages its (BY + 4) x (BX + 4) window (replicate border) in
// shared memory, forms the horizontal sums of its BY + 4 rows, then the vertical sums.
// w2 (optional, pyramid bottom level): the last box pass also writes the reconstruction
// wf = (up(w2) + dw, Yhat) of its cells (the k_up2_add of the frame, reading 25).
__global__ void __launch_bounds__(BX* BY) k_box(const float4* __restrict__ in, float4* __restrict__ out,
                                               FrameParams f, const float4* __restrict__ w2 = nullptr,
                                               const float* __restrict__ yh = nullptr, float4* wf = nullptr) {
    __shared__ float3 win[BY + 4][BX + 4];
    __shared__ float3 hs[BY + 4][BX];
    const int tx = threadIdx.x, ty = threadIdx.y, b = blockIdx.z;
    const int j0 = blockIdx.x * BX, i0 = blockIdx.y * BY;
    const float4* pl = in + (size_t)b * f.H * f.W;
    for (int t = ty * BX + tx; t < (BY + 4) * (BX + 4); t += BX * BY) {
        const int r = t / (BX + 4), c = t % (BX + 4);
        const float4 v = pl[(size_t)iclamp(i0 + r - 2, 0, f.H - 1) * f.W + iclamp(j0 + c - 2, 0, f.W - 1)];
        win[r][c] = make_float3(v.x, v.y, v.z);
    }
    __syncthreads();
    for (int r = ty; r < BY + 4; r += BY) {
        float3 a = win[r][tx];
#pragma unroll
        for (int k = 1; k < 5; ++k) {
            const float3 v = win[r][tx + k];
            a.x = xadd(a.x, v.x);
            a.y = xadd(a.y, v.y);
            a.z = xadd(a.z, v.z);
        }
        hs[r][tx] = a;
    }
    __syncthreads();
    const int i = i0 + ty, j = j0 + tx;
    if (i >= f.H || j >= f.W) return;
    float3 a = hs[ty][tx];
#pragma unroll
    for (int k = 1; k < 5; ++k) {
        const float3 v = hs[ty + k][tx];
        a.x = xadd(a.x, v.x);
        a.y = xadd(a.y, v.y);
        a.z = xadd(a.z, v.z);
    }
    const size_t p = ((size_t)b * f.H + i) * f.W + j;
    const float4 o = make_float4(div25(a.x), div25(a.y), div25(a.z), in[p].w);
    out[p] = o;
    if (w2) wf[p] = up2_add_at(w2 + (size_t)b * (f.H / 2) * (f.W / 2), i, j, f.H, f.W, o, yh[p]);
}

__global__ void k_unpack(const float4* __restrict__ src, float* w, float* rho, size_t n) {
    size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const float4 v = src[p];
    if (w) {
        w[3 * p] = v.x;
        w[3 * p + 1] = v.y;
        w[3 * p + 2] = v.z;
    }
    if (rho) rho[p] = v.w;
}

__global__ void k_pack(const float* __restrict__ w, const float* __restrict__ rho, float4* dst, size_t n) {
    size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    dst[p] = make_float4(w[3 * p], w[3 * p + 1], w[3 * p + 2], rho[p]);
}

}  // namespace

cudaError_t sf_launch_geometry(sf_ctx* c, const float* g10) {
    const int n = c->fp.H * c->fp.W;
    k_geometry<<<(n + 255) / 256, 256, 0, c->stream>>>(g10, c->G0, c->G1, c->G2, n);
    const int ne = sf_ew(c->fp.W) * sf_eh(c->fp.H);
    k_epad<<<(ne + 255) / 256, 256, 0, c->stream>>>(c->G1, c->G2, c->E, c->fp.H, c->fp.W);
    return cudaGetLastError();
}

// Prediction: N x (column pass, row pass); state[cur] -> pred, state[cur] kept (reading 9).
cudaError_t sf_launch_predict_passes(sf_ctx* c) {
    const FrameParams& f = c->fp;
    const dim3 g = grid_for(f), blk(BX, BY);
    const float4* src = c->state[c->cur];
    for (int n = 0; n < f.N; ++n) {
        k_pass<0><<<g, blk, 0, c->stream>>>(src, c->tmp, c->G0, c->G1, f, c->flags, 0, f.H);
        k_pass<1><<<g, blk, 0, c->stream>>>(c->tmp, c->pred, c->G0, c->G2, f, c->flags, 0, f.H);
        src = c->pred;
    }
    return cudaGetLastError();
}

// Update: on init, fill state[cur]; otherwise state[cur] (k) + pred (k+) -> state[1-cur] (k+1).
cudaError_t sf_launch_update_passes(sf_ctx* c, const float* Y, const float* D, bool init) {
    const FrameParams& f = c->fp;
    const dim3 g = grid_for(f), blk(BX, BY);
    if (init) {
        k_hconv<<<g, blk, 0, c->stream>>>(Y, c->HG, c->HH, f, c->flags);
        k_init<<<g, blk, 0, c->stream>>>(c->HG, c->HH, D, c->state[c->cur], c->yhat[c->cur], f);
        return cudaGetLastError();
    }
    float4* nxt = c->state[1 - c->cur];
    float4* solved = f.S > 0 ? c->tmp : nxt;
    k_update<<<g, blk, 0, c->stream>>>(Y, D, c->pred, c->state[c->cur], c->yhat[c->cur], 1, c->yhat[1 - c->cur],
                                       solved, c->G0, c->G1, c->G2, f, c->flags);
    for (int s = 0; s < f.S; ++s) {  // ping-pong tmp <-> tmp2, the last pass into nxt
        const float4* src = (s & 1) ? c->tmp2 : c->tmp;
        float4* dst = s == f.S - 1 ? nxt : ((s & 1) ? c->tmp : c->tmp2);
        k_box<<<g, blk, 0, c->stream>>>(src, dst, f);
    }
    return cudaGetLastError();
}

// Busy-wait ~ns nanoseconds on the device (sf_step_timed queues the timed kernels behind it, so that
// the CUDA events around them measure device time, not host launch latency).
__global__ void k_spin(long long ns) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while ((long long)(t - t0) < ns);
}
cudaError_t sf_launch_spin(sf_ctx* c, long long ns) {
    k_spin<<<1, 1, 0, c->stream>>>(ns);
    return cudaGetLastError();
}

// ---- building blocks of the banded substep-exchange step (sf_band.cu)
cudaError_t sf_launch_pass(sf_ctx* c, int axis, const float4* in, float4* out, int r0, int r1, cudaStream_t s) {
    const FrameParams& f = c->fp;
    if (r1 <= r0) return cudaSuccess;
    const dim3 g((f.W + BX - 1) / BX, (r1 - r0 + BY - 1) / BY, f.B), blk(BX, BY);
    if (axis == 0)
        k_pass<0><<<g, blk, 0, s>>>(in, out, c->G0, c->G1, f, c->flags, r0, r1);
    else
        k_pass<1><<<g, blk, 0, s>>>(in, out, c->G0, c->G2, f, c->flags, r0, r1);
    return cudaGetLastError();
}
cudaError_t sf_launch_update_solve(sf_ctx* c, const float* Y, const float* D, float4* out) {
    const FrameParams& f = c->fp;
    k_update<<<grid_for(f), dim3(BX, BY), 0, c->stream>>>(Y, D, c->pred, c->state[c->cur], c->yhat[c->cur], 1,
                                                          c->yhat[1 - c->cur], out, c->G0, c->G1, c->G2, f, c->flags);
    return cudaGetLastError();
}
cudaError_t sf_launch_box(sf_ctx* c, const float4* in, float4* out) {
    k_box<<<grid_for(c->fp), dim3(BX, BY), 0, c->stream>>>(in, out, c->fp);
    return cudaGetLastError();
}

cudaError_t sf_launch_unpack(sf_ctx* c, const float4* src, float* w, float* rho) {
    const size_t n = (size_t)c->fp.B * c->fp.H * c->fp.W;
    k_unpack<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(src, w, rho, n);
    return cudaGetLastError();
}

cudaError_t sf_launch_pack(sf_ctx* c, const float* w, const float* rho, float4* dst) {
    const size_t n = (size_t)c->fp.B * c->fp.H * c->fp.W;
    k_pack<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(w, rho, dst, n);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ pyramid bottom level launchers
// Prediction [P_[]]: N x (column, row) passes of (A, Wf) = ((dw, rho), (w, Yhat)) -> (pred, Wpred).
cudaError_t sf_launch_predict_low(sf_ctx* c) {
    const FrameParams& f = c->fp;
    const dim3 g = grid_for(f), blk(BX, BY);
    const float4* sA = c->state[c->cur];
    const float4* sW = c->Wf[c->cur];
    for (int n = 0; n < f.N; ++n) {
        k_pass_low<0><<<g, blk, 0, c->stream>>>(sA, sW, c->tmp, c->Wtmp, c->G0, c->G1, f, c->flags);
        k_pass_low<1><<<g, blk, 0, c->stream>>>(c->tmp, c->Wtmp, c->pred, c->Wpred, c->G0, c->G2, f, c->flags);
        sA = c->pred;
        sW = c->Wpred;
    }
    return cudaGetLastError();
}

// Update [dU] (reading 28): the H = 1 solve with prior dw^{k+}, references Yhat^{k+}
// (Wpred.w) and rho^{k+} (pred.w), S box passes on dw, fusion -> state[1 - cur]; Yhat^{k+1} ->
// yhat[0] (consumed by the reconstruction).  init: dw = 0, rho = rhohat, Yhat = Yhat(Y).
// The bottom-level update's last box pass can carry the reconstruction (sf_launch_box_up2) when
// the update runs on the per-pass kernels with S >= 1.
bool sf_update_low_defers(const sf_ctx* c) { return c->upd_fused || c->fp.S > 0; }

// The deferred end of the bottom-level update with the reconstruction: the tiled k_upd launch
// (upd_fused: the whole update) or the per-pass path's last box pass.
cudaError_t sf_launch_update_low_last(sf_ctx* c, const float* Y, const float* D, const float4* w2, float4* wf) {
    const FrameParams& f = c->fp;
    float4* nxt = c->state[1 - c->cur];
    if (c->upd_fused)
        return sf_launch_update_fused(c, Y, D, c->pred, reinterpret_cast<const float*>(c->pred) + 3, 4,
                                      reinterpret_cast<const float*>(c->Wpred) + 3, 4, nxt, c->yhat[0], w2, wf);
    const int s = f.S - 1;
    const float4* src = (s & 1) ? c->tmp2 : c->tmp;
    k_box<<<grid_for(f), dim3(BX, BY), 0, c->stream>>>(src, nxt, f, w2, c->yhat[0], wf);
    return cudaGetLastError();
}

// defer_last (sf_update_low_defers): the end of the update (the last box pass, or all of the
// tiled update) is left to sf_launch_update_low_last.
cudaError_t sf_launch_update_low(sf_ctx* c, const float* Y, const float* D, bool init, bool defer_last) {
    const FrameParams& f = c->fp;
    const dim3 g = grid_for(f), blk(BX, BY);
    if (init) {
        k_hconv<<<g, blk, 0, c->stream>>>(Y, c->HG, c->HH, f, c->flags);
        k_init<<<g, blk, 0, c->stream>>>(c->HG, c->HH, D, c->state[c->cur], c->yhat[0], f);
        return cudaGetLastError();
    }
    float4* nxt = c->state[1 - c->cur];
    if (c->upd_fused && defer_last) return cudaSuccess;  // (all of it in sf_launch_update_low_last)
    if (c->upd_fused)  // one tiled launch (sf_update.cu): references rho^{k+} = pred.w, Yhat^{k+} = Wpred.w
        return sf_launch_update_fused(c, Y, D, c->pred, reinterpret_cast<const float*>(c->pred) + 3, 4,
                                      reinterpret_cast<const float*>(c->Wpred) + 3, 4, nxt, c->yhat[0]);
    float4* solved = f.S > 0 ? c->tmp : nxt;
    k_update<<<g, blk, 0, c->stream>>>(Y, D, c->pred, c->pred, reinterpret_cast<const float*>(c->Wpred) + 3, 4,
                                       c->yhat[0], solved, c->G0, c->G1, c->G2, f, c->flags);
    for (int s = 0; s < f.S - (defer_last ? 1 : 0); ++s) {  // ping-pong tmp <-> tmp2, the last pass into nxt
        const float4* src = (s & 1) ? c->tmp2 : c->tmp;
        float4* dst = s == f.S - 1 ? nxt : ((s & 1) ? c->tmp : c->tmp2);
        k_box<<<g, blk, 0, c->stream>>>(src, dst, f);
    }
    return cudaGetLastError();
}
