// sf_fused.cu -- temporally blocked, fused predict + update: one launch per frame for
// N <= 8 (ceil(N/8) launches beyond).  Same bits as sf_passes.cu.
//
// Layout.  A CTA owns an output tile TH x TW and computes on a
// region RH x RW = (TH + 2R) x (TW + 2R), R = max(M, 2) + 2S (M substeps in this launch,
// S box passes).  Thread (warp w, lane l) owns a vertical run of K cells of region column
// c = 32*(w % NWX) + l, rows K*(w / NWX) ... + K-1:
//   * its fields (w.x, w.y, w.z, rho) and its direction s stay in REGISTERS for the whole
//     frame; e1/e2 live in shared-memory planes;
//   * column pass (j +- 1): neighbours are lanes +- 1 -> warp shuffles (the upwind value
//     with a per-lane source lane); warp-edge lanes swap through shared memory;
//   * row pass (i +- 1): neighbours are in the thread's own run (registers); only the run
//     ends swap through shared memory;
//   * one __syncthreads per pass; the valid (exact) region shrinks by one cell per pass at
//     cut edges and stays exact at grid edges (replicate boundary, reading 10);
//   * update: Y and rhohat planes are loaded with the grid clamp baked in (replicated
//     borders), separable brightness taps + occlusion-aware rho differences + the 3x3
//     LDL^T solve per cell, then S box passes, rho fusion, one coalesced store per tile.
// The transport update of the 4 fields uses paired f32x2 ops (FADD2/FMUL2/FFMA2).
#include "sf_internal.cuh"

namespace {

constexpr unsigned FULL = 0xffffffffu;

// ---- paired float32 ops (sm_100a f32x2; each lane op is the IEEE float32 op)
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
        : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
        : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}"
        : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}

// f* = fma(-dt, fma(|u_hat|, f - f_up, f q), f)  -- equal (up to the sign of a zero) to
// the literal fma(-dt, fma(u_hat, D, f q), f) with D the upwind difference,
// because |u_hat| (f - f_up) and u_hat D are the same exact product.
__device__ __forceinline__ float4 transport(float4 v, float4 fu, float a, float q, float ndt) {
    const float2 A = make_float2(a, a), Q = make_float2(q, q), T = make_float2(ndt, ndt);
    const float2 v01 = make_float2(v.x, v.y), v23 = make_float2(v.z, v.w);
    const float2 d01 = sub2(v01, make_float2(fu.x, fu.y)), d23 = sub2(v23, make_float2(fu.z, fu.w));
    const float2 t01 = fma2(A, d01, mul2(v01, Q)), t23 = fma2(A, d23, mul2(v23, Q));
    const float2 o01 = fma2(T, t01, v01), o23 = fma2(T, t23, v23);
    return make_float4(o01.x, o01.y, o23.x, o23.y);
}

__device__ __forceinline__ float dot3s(float ax, float ay, float az, float4 x) {
    return xfma(az, x.z, xfma(ay, x.y, xmul(ax, x.x)));
}

struct FusedArgs {
    const float4* fin;  // fields at launch start (state k or a partial prediction)
    const float4* sk;   // state k (rho^k for the update)
    float4* fout;       // state k+1 (upd) or partial prediction
    const float* yin;   // Yhat^k
    float* yout;        // Yhat^{k+1}
    const float* Y;
    const float* D;
    const float4* G0;   // (s, d2)
    const float* E;     // [6][H*W]
    unsigned* flags;
    FrameParams f;
    int M;    // substeps in this launch
    int upd;  // 1: run the update after the substeps
    int R;    // halo
    int TH, TW;
};

template <int K, int NWX, int NWY>
struct Cfg {
    static constexpr int RW = 32 * NWX, RH = K * NWY, P = RW * RH, NT = 32 * NWX * NWY;
    static constexpr int NXC = ((NWY * NWX * 2 * K) + 3) & ~3;  // column-exchange slots (padded)
    static constexpr int NXR = NWY * 2 * RW;                    // row-exchange slots
    static constexpr int XFLOATS = 5 * NXC + 5 * NXR;
    static constexpr int UFLOATS = 4 * P > XFLOATS ? 4 * P : XFLOATS;
    static constexpr size_t SMEM = sizeof(float) * (6 * (size_t)P + UFLOATS);
};

template <int K, int NWX, int NWY>
__global__ void __launch_bounds__(32 * NWX * NWY, 1) k_fused(const FusedArgs a) {
    using C = Cfg<K, NWX, NWY>;
    constexpr int RW = C::RW, RH = C::RH, P = C::P, NT = C::NT;
    extern __shared__ float4 smem4[];
    float* const Es = reinterpret_cast<float*>(smem4);
    float* const Ub = Es + 6 * P;
    float4* const XCf = reinterpret_cast<float4*>(Ub);
    float* const XCu = reinterpret_cast<float*>(XCf + C::NXC);
    float4* const XRf = reinterpret_cast<float4*>(XCu + C::NXC);
    float* const XRv = reinterpret_cast<float*>(XRf + C::NXR);

    const FrameParams& f = a.f;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wx = warp % NWX, wy = warp / NWX;
    const int c = 32 * wx + lane, r0 = K * wy;
    const int b = blockIdx.z;
    const int R = a.R;
    const int gi0 = blockIdx.y * a.TH - R, gj0 = blockIdx.x * a.TW - R;
    // in-grid cells of the region: rows [rmin, rmax], cols [cmin, cmax] (also the clamp bounds)
    const int cmin = max(0, -gj0), cmax = min(RW - 1, f.W - 1 - gj0);
    const int rmin = max(0, -gi0), rmax = min(RH - 1, f.H - 1 - gi0);
    const size_t HW = (size_t)f.H * f.W, plane = (size_t)b * HW;
    const int gj = iclamp(gj0 + c, 0, f.W - 1);
    const bool incol = c >= cmin && c <= cmax;

    // ---- load e1/e2 planes (replicated clamp) and this thread's cells
    for (int idx = tid; idx < P; idx += NT) {
        const int rr = idx / RW, cc = idx % RW;
        const size_t g = (size_t)iclamp(gi0 + rr, 0, f.H - 1) * f.W + iclamp(gj0 + cc, 0, f.W - 1);
#pragma unroll
        for (int p = 0; p < 6; ++p) Es[p * P + idx] = __ldg(a.E + p * HW + g);
    }
    float4 fv[K];
    float sx[K], sy[K], sz[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const size_t g = (size_t)iclamp(gi0 + r0 + k, 0, f.H - 1) * f.W + gj;
        fv[k] = a.fin[plane + g];
        const float4 s4 = __ldg(a.G0 + g);
        sx[k] = s4.x;
        sy[k] = s4.y;
        sz[k] = s4.z;
    }
    __syncthreads();

    // exactness bookkeeping: a cut edge (region edge inside the grid) loses one exact cell per pass
    const int cutL = gj0 > 0, cutR = gj0 + RW - 1 < f.W - 1, cutT = gi0 > 0, cutB = gi0 + RH - 1 < f.H - 1;
    int eL = 0, eR = RW - 1, eT = 0, eB = RH - 1;
    const float ndt = -f.dt;
    unsigned fl = 0;

    for (int n = 0; n < a.M; ++n) {
        // ================= column pass (beta_1)
        {
            float u[K];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int idx = (r0 + k) * RW + c;
                u[k] = dot3s(Es[idx], Es[P + idx], Es[2 * P + idx], fv[k]);
            }
            if (lane == 0 || lane == 31) {
                const int base = ((wy * NWX + wx) * 2 + (lane == 31)) * K;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    XCf[base + k] = fv[k];
                    XCu[base + k] = u[k];
                }
            }
            __syncthreads();
            const int nL = eL + cutL, nR = eR - cutR;
            const bool cex = incol && c >= nL && c <= nR;
            const int lbase = ((wy * NWX + wx - 1) * 2 + 1) * K, rbase = ((wy * NWX + wx + 1) * 2 + 0) * K;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                float um = __shfl_up_sync(FULL, u[k], 1), up = __shfl_down_sync(FULL, u[k], 1);
                if (lane == 0 && wx > 0) um = XCu[lbase + k];
                if (lane == 31 && wx < NWX - 1) up = XCu[rbase + k];
                if (c <= cmin) um = u[k];
                if (c >= cmax) up = u[k];
                float uh = dominant(um, up, f.rule);
                const int r = r0 + k;
                const bool ex = cex && r >= eT && r <= eB && r >= rmin && r <= rmax;
                if (f.clamp) {
                    if (ex && fabsf(uh) > f.U) fl |= SF_FLAG_CLAMPED;
                    uh = fminf(fmaxf(uh, -f.U), f.U);
                } else if (ex && xmul(f.dt, fabsf(uh)) > 1.0f) {
                    fl |= SF_FLAG_CFL;
                }
                const bool fwd = uh > 0.0f;
                const int src = (fwd ? lane - 1 : lane + 1) & 31;
                float4 fu;
                fu.x = __shfl_sync(FULL, fv[k].x, src);
                fu.y = __shfl_sync(FULL, fv[k].y, src);
                fu.z = __shfl_sync(FULL, fv[k].z, src);
                fu.w = __shfl_sync(FULL, fv[k].w, src);
                if (fwd) {
                    if (c <= cmin) fu = fv[k];
                    else if (lane == 0) fu = XCf[lbase + k];
                } else {
                    if (c >= cmax) fu = fv[k];
                    else if (lane == 31) fu = XCf[rbase + k];
                }
                const float q = xmul(f.sigma, dot3s(sx[k], sy[k], sz[k], fv[k]));
                fv[k] = transport(fv[k], fu, fabsf(uh), q, ndt);
            }
            eL = nL;
            eR = nR;
        }
        // ================= row pass (beta_2, reading 3)
        {
            float v[K];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int idx = (r0 + k) * RW + c;
                v[k] = dot3s(Es[3 * P + idx], Es[4 * P + idx], Es[5 * P + idx], fv[k]);
            }
            XRf[(wy * 2 + 0) * RW + c] = fv[0];
            XRv[(wy * 2 + 0) * RW + c] = v[0];
            XRf[(wy * 2 + 1) * RW + c] = fv[K - 1];
            XRv[(wy * 2 + 1) * RW + c] = v[K - 1];
            __syncthreads();
            float4 ftop = fv[0], fbot = fv[K - 1];
            float vtop = v[0], vbot = v[K - 1];
            if (wy > 0) {
                ftop = XRf[((wy - 1) * 2 + 1) * RW + c];
                vtop = XRv[((wy - 1) * 2 + 1) * RW + c];
            }
            if (wy < NWY - 1) {
                fbot = XRf[((wy + 1) * 2 + 0) * RW + c];
                vbot = XRv[((wy + 1) * 2 + 0) * RW + c];
            }
            const int nT = eT + cutT, nB = eB - cutB;
            const bool cex = incol && c >= eL && c <= eR;
            float4 prev = ftop;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int r = r0 + k;
                float vm = (k > 0) ? v[k - 1] : vtop;
                float vp = (k < K - 1) ? v[k + 1] : vbot;
                float4 fm = prev;
                float4 fp = (k < K - 1) ? fv[k + 1] : fbot;
                if (r <= rmin) {
                    vm = v[k];
                    fm = fv[k];
                }
                if (r >= rmax) {
                    vp = v[k];
                    fp = fv[k];
                }
                float vh = dominant(vm, vp, f.rule);
                const bool ex = cex && r >= nT && r <= nB && r >= rmin && r <= rmax;
                if (f.clamp) {
                    if (ex && fabsf(vh) > f.U) fl |= SF_FLAG_CLAMPED;
                    vh = fminf(fmaxf(vh, -f.U), f.U);
                } else if (ex && xmul(f.dt, fabsf(vh)) > 1.0f) {
                    fl |= SF_FLAG_CFL;
                }
                const float4 fu = (vh > 0.0f) ? fm : fp;
                prev = fv[k];
                const float q = xmul(f.sigma, dot3s(sx[k], sy[k], sz[k], fv[k]));
                fv[k] = transport(fv[k], fu, fabsf(vh), q, ndt);
            }
            eT = nT;
            eB = nB;
        }
    }

    const int TH = a.TH, TW = a.TW;
    if (a.upd) {
        const int S = f.S;
        __syncthreads();  // exchange buffers are reused below
        float* const Ys = Ub;
        float* const Rs = Ub + P;
        float* const HGs = Ub + 2 * P;
        float* const HHs = Ub + 3 * P;
        const float qnan = __int_as_float(0x7fffffff);
        for (int idx = tid; idx < P; idx += NT) {
            const int rr = idx / RW, cc = idx % RW;
            const size_t g = (size_t)iclamp(gi0 + rr, 0, f.H - 1) * f.W + iclamp(gj0 + cc, 0, f.W - 1);
            const float y = a.Y[plane + g];
            const float d = a.D[plane + g];
            Ys[idx] = y;
            Rs[idx] = depth_valid(d, f.is_inv) ? rho_hat(d, f.is_inv) : qnan;  // NaN = no measurement
            const bool tile = rr >= R && rr < R + TH && cc >= R && cc < R + TW && rr >= rmin && rr <= rmax &&
                              cc >= cmin && cc <= cmax;
            if (tile && !isfinite(y)) fl |= SF_FLAG_NONFINITE;
        }
        __syncthreads();
        for (int idx = tid; idx < P; idx += NT) {  // horizontal brightness taps
            const int cc = idx % RW;
            if (cc >= 2 && cc <= RW - 3) {
                const float x0 = Ys[idx - 2], x1 = Ys[idx - 1], x2 = Ys[idx], x3 = Ys[idx + 1], x4 = Ys[idx + 2];
                HGs[idx] = tap_g(x0, x1, x2, x3, x4);
                HHs[idx] = tap_h(x0, x1, x2, x3, x4);
            }
        }
        __syncthreads();
        const int slo = R - 2 * S;  // solve region: tile + 2S
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int r = r0 + k;
            const bool solve = r >= slo && r < R + TH + 2 * S && c >= slo && c < R + TW + 2 * S && r >= rmin &&
                               r <= rmax && incol;
            if (solve) {
                const int idx = r * RW + c;
                const float g0 = HGs[idx - 2 * RW], g1 = HGs[idx - RW], g2 = HGs[idx], g3 = HGs[idx + RW],
                            g4 = HGs[idx + 2 * RW];
                const float h0 = HHs[idx - 2 * RW], h1 = HHs[idx - RW], h2 = HHs[idx], h3 = HHs[idx + RW],
                            h4 = HHs[idx + 2 * RW];
                const float yh = tap_g(g0, g1, g2, g3, g4);  // Yhat^{k+1}
                const float be1 = tap_g(h0, h1, h2, h3, h4);
                const float be2 = tap_h(g0, g1, g2, g3, g4);
                const float rc = Rs[idx], rl = Rs[idx - 1], rr = Rs[idx + 1], ru = Rs[idx - RW], rd = Rs[idx + RW];
                const bool vc = !isnan(rc), vl = !isnan(rl), vr = !isnan(rr), vu = !isnan(ru), vd = !isnan(rd);
                const float rh = vc ? rc : 0.0f;
                const float br1 = pick_side(rh, vc, rl, vl, rr, vr);
                const float br2 = pick_side(rh, vc, ru, vu, rd, vd);
                const size_t g = (size_t)(gi0 + r) * f.W + (gj0 + c);
                const float d2 = __ldg(&a.G0[g].w);
                const float e1a[3] = {Es[idx], Es[P + idx], Es[2 * P + idx]};
                const float e2a[3] = {Es[3 * P + idx], Es[4 * P + idx], Es[5 * P + idx]};
                const float sa[3] = {sx[k], sy[k], sz[k]};
                float gh[3], m[3];
                const float d2r = xmul(d2, rh);
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    gh[q] = xmul(d2, xfma(e2a[q], be2, xmul(e1a[q], be1)));
                    const float dr = xmul(d2, xfma(e2a[q], br2, xmul(e1a[q], br1)));
                    m[q] = xfma(d2r, sa[q], dr);
                }
                const float cY = xmul(d2, xsub(yh, a.yin[plane + g]));
                const float cr = xmul(d2, xsub(rh, a.sk[plane + g].w));
                const float wp[3] = {fv[k].x, fv[k].y, fv[k].z};
                float x[3];
                ls_solve3(gh, m, cY, cr, wp, f.g1, vc ? f.g2 : 0.0f, f.g3, x);
                const float kap = vc ? f.kappa : 0.0f;
                const float rn = xfma(kap, xsub(rh, fv[k].w), fv[k].w);
                fv[k] = make_float4(x[0], x[1], x[2], rn);
                if (!(isfinite(x[0]) && isfinite(x[1]) && isfinite(x[2]) && isfinite(rn))) fl |= SF_FLAG_NONFINITE;
                if (r >= R && r < R + TH && c >= R && c < R + TW) a.yout[plane + g] = yh;
            } else {
                fv[k] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            }
        }
        // ---- S x 5x5 box: horizontal 5-sum, vertical 5-sum, / 25; replicate border
        float* const Wx = Ub;
        float* const Wy = Ub + P;
        float* const Wz = Ub + 2 * P;
        for (int it = 0; it < S; ++it) {
            __syncthreads();
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int idx = (r0 + k) * RW + c;
                Wx[idx] = fv[k].x;
                Wy[idx] = fv[k].y;
                Wz[idx] = fv[k].z;
            }
            __syncthreads();
            const int c0 = iclamp(c - 2, cmin, cmax), c1 = iclamp(c - 1, cmin, cmax), c3 = iclamp(c + 1, cmin, cmax),
                      c4 = iclamp(c + 2, cmin, cmax);
            float hx[K], hy[K], hz[K];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int rb = (r0 + k) * RW;
                hx[k] = xadd(xadd(xadd(xadd(Wx[rb + c0], Wx[rb + c1]), Wx[rb + c]), Wx[rb + c3]), Wx[rb + c4]);
                hy[k] = xadd(xadd(xadd(xadd(Wy[rb + c0], Wy[rb + c1]), Wy[rb + c]), Wy[rb + c3]), Wy[rb + c4]);
                hz[k] = xadd(xadd(xadd(xadd(Wz[rb + c0], Wz[rb + c1]), Wz[rb + c]), Wz[rb + c3]), Wz[rb + c4]);
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int idx = (r0 + k) * RW + c;
                Wx[idx] = hx[k];
                Wy[idx] = hy[k];
                Wz[idx] = hz[k];
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int r = r0 + k;
                const int i0 = iclamp(r - 2, rmin, rmax) * RW, i1 = iclamp(r - 1, rmin, rmax) * RW,
                          i2 = r * RW, i3 = iclamp(r + 1, rmin, rmax) * RW, i4 = iclamp(r + 2, rmin, rmax) * RW;
                const float vx = xadd(xadd(xadd(xadd(Wx[i0 + c], Wx[i1 + c]), Wx[i2 + c]), Wx[i3 + c]), Wx[i4 + c]);
                const float vy = xadd(xadd(xadd(xadd(Wy[i0 + c], Wy[i1 + c]), Wy[i2 + c]), Wy[i3 + c]), Wy[i4 + c]);
                const float vz = xadd(xadd(xadd(xadd(Wz[i0 + c], Wz[i1 + c]), Wz[i2 + c]), Wz[i3 + c]), Wz[i4 + c]);
                fv[k].x = __fdiv_rn(vx, 25.0f);
                fv[k].y = __fdiv_rn(vy, 25.0f);
                fv[k].z = __fdiv_rn(vz, 25.0f);
            }
        }
    }
    // ---- store the tile
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int r = r0 + k;
        if (r >= R && r < R + TH && c >= R && c < R + TW && r >= rmin && r <= rmax && incol)
            a.fout[plane + (size_t)(gi0 + r) * f.W + (gj0 + c)] = fv[k];
    }
    const unsigned any = __reduce_or_sync(FULL, fl);
    if (lane == 0 && any) atomicOr(a.flags, any);
}

// The one configuration used today: RW = 64, RH = 72, 384 threads, 1 CTA / SM.
constexpr int FK = 12, FNWX = 2, FNWY = 6;
using FC = Cfg<FK, FNWX, FNWY>;
constexpr int MMAX = 8;  // substeps per launch

struct Plan {
    int launches;
    int M[8];
    int R[8];
};

Plan make_plan(const FrameParams& f) {
    Plan p{};
    p.launches = (f.N + MMAX - 1) / MMAX;
    for (int l = 0; l < p.launches; ++l) {
        p.M[l] = (l < p.launches - 1) ? MMAX : f.N - MMAX * (p.launches - 1);
        const bool upd = l == p.launches - 1;
        p.R[l] = upd ? (p.M[l] > 2 ? p.M[l] : 2) + 2 * f.S : p.M[l];
    }
    return p;
}

}  // namespace

bool sf_fused_supported(const sf_ctx* c) {
    const Plan p = make_plan(c->fp);
    if (p.launches > 8) return false;
    for (int l = 0; l < p.launches; ++l)
        if (FC::RW - 2 * p.R[l] < 8 || FC::RH - 2 * p.R[l] < 8) return false;
    // opt in to the large dynamic shared-memory carve-out (one CTA per SM)
    return cudaFuncSetAttribute(k_fused<FK, FNWX, FNWY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)FC::SMEM) == cudaSuccess;
}

int sf_fused_launches(const sf_ctx* c) { return make_plan(c->fp).launches; }

cudaError_t sf_launch_fused_step(sf_ctx* c, const float* Y, const float* D) {
    const FrameParams& f = c->fp;
    const Plan p = make_plan(f);
    const float4* src = c->state[c->cur];
    float4* bufs[2] = {c->pred, c->tmp};
    for (int l = 0; l < p.launches; ++l) {
        const bool upd = l == p.launches - 1;
        FusedArgs a;
        a.fin = src;
        a.sk = c->state[c->cur];
        a.fout = upd ? c->state[1 - c->cur] : bufs[l & 1];
        a.yin = c->yhat[c->cur];
        a.yout = c->yhat[1 - c->cur];
        a.Y = Y;
        a.D = D;
        a.G0 = c->G0;
        a.E = c->E;
        a.flags = c->flags;
        a.f = f;
        a.M = p.M[l];
        a.upd = upd ? 1 : 0;
        a.R = p.R[l];
        a.TW = FC::RW - 2 * a.R;
        a.TH = FC::RH - 2 * a.R;
        const dim3 grid((f.W + a.TW - 1) / a.TW, (f.H + a.TH - 1) / a.TH, f.B);
        k_fused<FK, FNWX, FNWY><<<grid, FC::NT, FC::SMEM, c->stream>>>(a);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        src = a.fout;
    }
    return cudaSuccess;
}
