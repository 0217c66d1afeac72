// sf_update.cu -- the update step U1-U5 as ONE tiled kernel per frame: brightness
// model (eq:img_model), inverse-depth model (eq:dominant_b1/b2), the per-
// pixel 3x3 LS (eq:LS_update), S passes of the 5x5 box (reading 13) and the
// inverse-depth fusion (eq:cost_invdepth).  Same bits as sf_passes.cu's k_update +
// S x k_box.
//
// Layout.  A CTA owns an output tile TH x TW and works on shared planes
// of PH x PW cells: the tile plus a margin of MR = h + 2 rows and MG >= h + 3 columns (h = 2S,
// MG a multiple of 4 so the box's 16-byte accesses stay aligned).  The box passes need w_LS on the
// tile +- h, so the LS is solved there (the solve region, SR); the models need Y on SR +- 2 and the
// depth on SR +- 1.  Y and depth are loaded with replicate-clamped indices (reading 10), so the
// models need no edge logic; the box's out-of-grid window cells are filled with their clamped
// in-grid cell (edge CTAs only).
//   stage 0: Y, depth -> planes (two TMA tensor copies of the whole plane, issued before the wait
//            on the transport kernel: they are the caller's inputs, and the transport kernel has
//            prefetched them into L2; edge CTAs, whose plane reaches outside the grid, and builds
//            without TMA: cp.async with replicate-clamped indices); the first solve item's global
//            inputs fetched (the first two items);
//   stage 1: rhohat plane (NaN = invalid) + horizontal taps HG = hz(g, Y), HH = hz(h, Y);
//   stage 2: per SR pair of cells: vertical taps -> Yhat', beta_1, beta_2; rho one-sided
//            differences; ghat, m; c_Y, c_rho; LDL^T solve -> w_LS planes; Yhat^{k+1} of tile cells
//            stored; the next item's global inputs (w^{k+}, s, e1, e2, references) fetched one
//            item ahead;
//   stage 3: S box passes, each a register-tiled separable stencil (one item = one component
//            of a 4-column x 6-row output block: 10 horizontal 5-sums, sliding vertical 5-sums);
//   stage 4: rho fusion and the coalesced store of (w^{k+1}, rho^{k+1}) for the tile.
// The top level (H = 1) and the pyramid's bottom level [dU] (reading 28: references Yhat^{k+},
// rho^{k+} instead of Yhat^k, rho^k) run the same kernel with different reference pointers.
#include <stdint.h>
#include <stdlib.h>

#include "sf_pair.cuh"

namespace {

using namespace sfp;

struct UpdArgs {
    CUtensorMap tmY;           // [B][H][W] brightness, box PW x PH x 1 (valid when tma)
    CUtensorMap tmD;           // [B][H][W] depth, box PW x PH x 1
    int tma;
    const float4* pred;        // [B][H][W] (w^{k+}, rho^{k+})
    const float* rref;         // rho reference of c_rho, element p at rref[p * rs]
    const float* yref;         // Yhat reference of c_Y, element p at yref[p * ys]
    int rs, ys;
    const float* Y;            // [B][H][W] brightness
    const float* D;            // [B][H][W] depth (or inverse depth)
    const float4* G0;          // (s, d2)
    const float* E;            // padded e planes [6][EH][EW] (e1.xyz, e2.xyz; cell (i, j) at (i + EPAD, j + EPAD))
    int EW;                    // padded row length
    size_t EP;                 // plane stride
    int e8;                    // 1: EW even and E 8-byte aligned (a pair's e components by one 8-byte load)
    float4* out;               // (w^{k+1}, rho^{k+1})
    const float4* w2;          // pyramid bottom level (optional): the new top-level state [B][H/2][W/2] ...
    float4* wf;                // ... and the reconstruction (up(w2) + dw, Yhat^{k+1}) written with out
    float* yout;               // Yhat^{k+1}
    unsigned* flags;
    FrameParams f;
    int TH, TW, h, MR, MG, PH, PW, P;  // P: plane stride of Y, rhohat, HG, HH (a multiple of 32 floats)
    int PF;                            // plane stride of the 6 box planes (= 12 mod 32: bank-spread)
    int dbg;                           // SF_DEBUG_SKIP (debug builds only): 8192 = phase profile, 16384 = CTA trace
    int dslot;                         // trace slot (frame & 3)
};

// 14 warps, one CTA per SM (<= 128 registers: 4 warps on the busiest scheduler x 32 x 128 = its 16K
// registers); the 48 x 40 tile's 1344 solve pairs are exactly 3 per thread
constexpr int UPD_NT = 448;

// Replicate fill (reading 10) of the out-of-grid cells of [ra, rb] x [ca, cb] (clipped to the
// plane) in NP planes (p, p + P, ...) of row stride PW: each takes the value of its clamped
// in-grid cell.  The four out-of-grid bands (top and bottom rows with the corners, left and right
// columns) are enumerated as one flat index range, so that every thread copies at most a cell or
// two in one step (a few hundred cells in an edge CTA).
template <int NP>
__device__ __forceinline__ void fill_planes(float* p, int P, int PW, int PH, int ra, int rb, int ca, int cb, int rmin,
                                            int rmax, int cmin, int cmax, int tid) {
    ra = max(ra, 0);
    rb = min(rb, PH - 1);
    ca = max(ca, 0);
    cb = min(cb, PW - 1);
    const int mr0 = max(ra, rmin), mr1 = min(rb, rmax);  // the in-grid rows of the rectangle
    // bands (first row, rows, first column, columns); empty bands count 0 cells
    const int b0r = ra, b0n = max(0, min(rb, rmin - 1) - ra + 1);
    const int b1r = max(ra, rmax + 1), b1n = max(0, rb - b1r + 1);
    const int wc = max(0, cb - ca + 1), lc = max(0, min(cb, cmin - 1) - ca + 1);
    const int rc0 = max(ca, cmax + 1), rcn = max(0, cb - rc0 + 1), mn = max(0, mr1 - mr0 + 1);
    const int n0 = b0n * wc, n1 = n0 + b1n * wc, n2 = n1 + mn * lc, n3 = n2 + mn * rcn;
#pragma unroll 1
    for (int t = tid; t < n3; t += UPD_NT) {
        int r, c;
        if (t < n1) {  // top / bottom rows
            const int u = t < n0 ? t : t - n0, q = u / wc;
            r = (t < n0 ? b0r : b1r) + q;
            c = ca + u - q * wc;
        } else if (t < n2) {  // left columns
            const int u = t - n1, q = u / lc;
            r = mr0 + q;
            c = ca + u - q * lc;
        } else {  // right columns
            const int u = t - n2, q = u / rcn;
            r = mr0 + q;
            c = rc0 + u - q * rcn;
        }
        const int from = iclamp(r, rmin, rmax) * PW + iclamp(c, cmin, cmax), to = r * PW + c;
        SF_DASSERT(r >= 0 && r < PH && c >= 0 && c < PW && (r < rmin || r > rmax || c < cmin || c > cmax));
#pragma unroll
        for (int k = 0; k < NP; ++k) p[k * P + to] = p[k * P + from];
    }
}

// The global inputs of one solve item (a horizontal pair of SR cells).  The directions e1, e2 come
// from the padded planar E array (24 bytes per cell, a pair's component in one 8-byte load) rather
// than the float4 G1 / G2 records (32 bytes per cell): the solve's loads are L2-throughput bound.
struct SolveIn {
    float4 wa, wb;   // pred: (w^{k+}, rho^{k+})
    float4 sa, sb;   // G0: (s, d2)
    float2 e[6];     // e1.x, e1.y, e1.z, e2.x, e2.y, e2.z of the pair
    float2 y, rk;    // Yhat and rho references
};

SF_TRACE_ARRAY(g_trace_upd);

__global__ void __launch_bounds__(UPD_NT, 1) k_upd(const __grid_constant__ UpdArgs a) {
    extern __shared__ __align__(1024) float sm[];  // TMA destinations: 128-byte aligned planes
    const FrameParams& f = a.f;
    const int tid = threadIdx.x;
    const int PH = a.PH, PW = a.PW, P = a.P, PF = a.PF, h = a.h, MR = a.MR, MG = a.MG, TH = a.TH, TW = a.TW;
    float* const Ys = sm;          // Y; after the models: rho^{k+} of the SR cells (RP)
    float* const RHs = sm + P;     // depth -> rhohat (NaN = invalid), read by the fusion
    float* const HG = sm + 2 * P;  // horizontal g-taps of Y
    float* const HH = sm + 3 * P;  // horizontal h-taps of Y
    float* const F0 = sm + 4 * P;           // 3 planes (stride PF): w_LS, then the box ping
    float* const F1 = sm + 4 * P + 3 * PF;  // 3 planes: the box pong
    float* const RP = Ys;
    uint64_t* const bar = reinterpret_cast<uint64_t*>(sm + 4 * P + 6 * PF);
    const int b = blockIdx.z;
    int tx, ty;
    edge_first_tile(true, tx, ty);  // (edge CTAs carry the replicate fills)
    const int i0 = ty * TH, j0 = tx * TW;
    const int oi = i0 - MR, oj = j0 - MG;  // global cell of plane cell (0, 0)
    // in-grid part of the plane (also the replicate-clamp bounds), plane coordinates
    const int rmin = max(0, -oi), rmax = min(PH - 1, f.H - 1 - oi);
    const int cmin = max(0, -oj), cmax = min(PW - 1, f.W - 1 - oj);
    const size_t HW = (size_t)f.H * f.W, pl = (size_t)b * HW;
    const int lc0 = MG - h - 2, ncl = TW + 2 * h + 4;  // columns of Y used: SR +- 2 (depth: SR +- 1)
    SF_PROF_DECL(a.dbg & 8192);
    SF_TRACE_BEGIN(a.dbg & 16384);
#ifdef SF_DEBUG_KNOBS
    if (a.dbg & 32) return;  // launch-overhead experiment
#endif
    SF_PROF();

    // ---------------- stage 0: Y and depth (caller inputs, prefetched into L2 by the transport
    // kernel): the whole plane by TMA, or the used columns by cp.async with clamped indices
    // edge CTAs (the plane reaches outside the grid) take the clamped cp.async path: no zero-filled
    // cells to replace afterwards
    const bool ydtma = a.tma && !(rmin > 0 || rmax < PH - 1 || cmin > 0 || cmax < PW - 1);
    if (ydtma) {
        if (tid == 0) {
            mbar_init(bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
            mbar_expect_tx(bar, 2u * PH * PW * 4u);
            tma_load_3d(Ys, &a.tmY, oj, oi, b, bar);
            tma_load_3d(RHs, &a.tmD, oj, oi, b, bar);
        }
        __syncthreads();  // the barrier's initialisation is visible to every waiting thread
    } else {
        SF_FOR_RECT(r, c, 0, PH - 1, lc0, lc0 + ncl - 1, UPD_NT, tid) {
            const size_t g = pl + (size_t)iclamp(oi + r, 0, f.H - 1) * f.W + iclamp(oj + c, 0, f.W - 1);
            cp_async4(Ys + r * PW + c, a.Y + g);
            cp_async4(RHs + r * PW + c, a.D + g);
        }
        cp_async_commit();
    }

    // solve region (in-grid), its pair grid, and the first item's global inputs (geometry now,
    // the transported fields once the transport kernel has completed).  Fetches are branch-free
    // (a thread past the region re-fetches the region's last row) so that no in-flight load is
    // copied between registers before its first use.
    const int srl = max(MR - h, rmin), srh = min(MR + TH + h - 1, rmax);
    const int scl = max(MG - h, cmin), sch = min(MG + TW + h - 1, cmax);  // scl even (MG - h even, or the grid's column 0)
    const int np = (sch - scl + 2) >> 1;
    const int pdr = UPD_NT / np, pdc = UPD_NT % np;
    int rn = srl + tid / np, pn = tid % np;
    SolveIn nx;
    auto fetch_geo = [&](int r, int pc, SolveIn& q) {
        r = min(r, srh);
        const int c = scl + 2 * pc;
        const size_t cell = (size_t)(oi + r) * f.W + (oj + c), d = c + 1 <= sch ? 1 : 0;  // ragged: the first cell again
        q.sa = __ldg(a.G0 + cell);
        q.sb = __ldg(a.G0 + cell + d);
        const float* ep = a.E + (size_t)(oi + r + SF_EPAD) * a.EW + (oj + c + SF_EPAD);
        SF_DASSERT(oi + r >= 0 && oi + r < f.H && oj + c >= 0 && oj + c < f.W && oj + c + SF_EPAD + 1 < a.EW);
        if (a.e8) {  // (a ragged pair's second cell reads the padding: in bounds, unused)
#pragma unroll
            for (int p = 0; p < 6; ++p) q.e[p] = __ldg(reinterpret_cast<const float2*>(ep + p * a.EP));
        } else {
#pragma unroll
            for (int p = 0; p < 6; ++p) q.e[p] = make_float2(__ldg(ep + p * a.EP), __ldg(ep + p * a.EP + d));
        }
    };
    auto fetch_fld = [&](int r, int pc, SolveIn& q) {
        r = min(r, srh);
        const int c = scl + 2 * pc;
        const size_t ga = pl + (size_t)(oi + r) * f.W + (oj + c), gb = ga + (c + 1 <= sch ? 1 : 0);
        SF_DASSERT(oi + r >= 0 && oi + r < f.H && oj + c >= 0 && oj + c + (c + 1 <= sch ? 1 : 0) < f.W);
        q.wa = a.pred[ga];
        q.wb = a.pred[gb];
        q.y = make_float2(a.yref[ga * a.ys], a.yref[gb * a.ys]);
        q.rk = make_float2(a.rref[ga * a.rs], a.rref[gb * a.rs]);
    };
    auto advance = [&](int& r, int& pc) {
        r += pdr + ((pc + pdc >= np) ? 1 : 0);
        pc = (pc + pdc >= np) ? pc + pdc - np : pc + pdc;
    };
    // the first two items' inputs are requested before the models run (the solve's loads are
    // L2-throughput bound, the models are not): item 1 in nx, item 2 in ny
    SolveIn ny;
    int rm = rn, pm = pn;  // the item after (rn, pn)
    advance(rm, pm);
    fetch_geo(rn, pn, nx);
    fetch_geo(rm, pm, ny);
    griddep_wait();  // w^{k+} and the references come from the preceding kernels
    SF_PROF();  // 0: stage-0 issue + griddep
    fetch_fld(rn, pn, nx);
    fetch_fld(rm, pm, ny);
    if (ydtma) {
        mbar_wait(bar, 0);
    } else {
        cp_async_wait<0>();
    }
    __syncthreads();
    SF_PROF();  // 1: Y / depth landed (+ edge fill)

    // ---------------- stage 1: rhohat + horizontal brightness taps, pairs of cells
    const float qnan = __int_as_float(0x7fffffff);
    unsigned fl = 0;
    bool okall = true;  // every reciprocal took rcp_fast's exact range
    const int tr0 = max(MR, rmin), tr1 = min(MR + TH - 1, rmax);  // tile rows / columns in the grid
    const int tc0 = max(MG, cmin), tc1 = min(MG + TW - 1, cmax);
    {
        auto ld2 = [&](const float* p, int i) { return *reinterpret_cast<const float2*>(p + i); };
#pragma unroll 1
        SF_FOR_RECT(r, pc, 0, PH - 1, 0, (ncl >> 1) - 1, UPD_NT, tid) {
            const int c = lc0 + 2 * pc, idx = r * PW + c;
            const float2 d = ld2(RHs, idx);
            bool ok0 = true, ok1 = true;
            const float rh0 = f.is_inv ? d.x : rcp_fast(d.x, ok0), rh1 = f.is_inv ? d.y : rcp_fast(d.y, ok1);
            const bool v0 = depth_valid(d.x, f.is_inv), v1 = depth_valid(d.y, f.is_inv);
            *reinterpret_cast<float2*>(RHs + idx) = make_float2(v0 ? rh0 : qnan, v1 ? rh1 : qnan);
            okall = okall && (ok0 || !v0) && (ok1 || !v1);
            if (c >= MG - h && c < MG + TW + h) {  // HG / HH on the SR columns
                const float2 ya = ld2(Ys, idx - 2), yb = ld2(Ys, idx), yc = ld2(Ys, idx + 2);
                const float2 x1 = make_float2(ya.y, yb.x), x3 = make_float2(yb.y, yc.x);
                *reinterpret_cast<float2*>(HG + idx) = tap2_g(ya, x1, yb, x3, yc);
                *reinterpret_cast<float2*>(HH + idx) = tap2_h(ya, x1, yb, x3, yc);
                if (r >= tr0 && r <= tr1 && oi + r >= f.fr0 && oi + r < f.fr1) {  // Y of tile cells finite
                    if (c >= tc0 && c <= tc1 && !isfinite(yb.x)) fl |= SF_FLAG_NONFINITE;
                    if (c + 1 >= tc0 && c + 1 <= tc1 && !isfinite(yb.y)) fl |= SF_FLAG_NONFINITE;
                }
            }
        }
    }
    if (__syncthreads_or(!okall)) {  // (never for depths in [2^-126, 2^126)): exact reciprocals
#pragma unroll 1
        SF_FOR_RECT(r, c, 0, PH - 1, lc0, lc0 + ncl - 1, UPD_NT, tid) {
            // the depth itself is gone: recompute from the global input (replicate-clamped)
            const size_t g = pl + (size_t)iclamp(oi + r, 0, f.H - 1) * f.W + iclamp(oj + c, 0, f.W - 1);
            const float d = a.D[g];
            RHs[r * PW + c] = depth_valid(d, f.is_inv) ? rho_hat(d, f.is_inv) : qnan;
        }
        __syncthreads();
    }

    SF_PROF();  // 2: models
    // ---------------- stage 2: per-pixel LS on SR, a horizontal pair of cells per item
    // The loop is unrolled twice with two input buffers (nx, ny): each item's inputs are fetched
    // one item ahead straight into the buffer the item will be solved from (no register copies of
    // in-flight loads).
    {
        auto ld2 = [&](const float* p, int i) { return *reinterpret_cast<const float2*>(p + i); };
        auto solve_item = [&](int r, int pn_, const SolveIn& cu) {
            const int c = scl + 2 * pn_;
            const bool full = c + 1 <= sch;
            const int idx = r * PW + c;  // even: 8-byte aligned pairs (a ragged pair's second cell is unused)
            const float2 g0 = ld2(HG, idx - 2 * PW), g1 = ld2(HG, idx - PW), g2 = ld2(HG, idx), g3 = ld2(HG, idx + PW),
                         g4 = ld2(HG, idx + 2 * PW);
            const float2 h0 = ld2(HH, idx - 2 * PW), h1 = ld2(HH, idx - PW), h2 = ld2(HH, idx), h3 = ld2(HH, idx + PW),
                         h4 = ld2(HH, idx + 2 * PW);
            const float2 yh = tap2_g(g0, g1, g2, g3, g4);  // Yhat^{k+1}
            const float2 be1 = tap2_g(h0, h1, h2, h3, h4);
            const float2 be2 = tap2_h(g0, g1, g2, g3, g4);
            const float2 rc = ld2(RHs, idx), ru = ld2(RHs, idx - PW), rd = ld2(RHs, idx + PW);
            const float rl = RHs[idx - 1], rr = RHs[idx + 2];
            const bool vc0 = !isnan(rc.x), vc1 = !isnan(rc.y);
            const float2 rh = make_float2(vc0 ? rc.x : 0.0f, vc1 ? rc.y : 0.0f);
            // eq:dominant_b1 / b2 per cell (the pair's cells are each other's row neighbour)
            const float2 br1 = make_float2(pick_side(rh.x, vc0, rl, !isnan(rl), rc.y, vc1),
                                           pick_side(rh.y, vc1, rc.x, vc0, rr, !isnan(rr)));
            const float2 br2 = make_float2(pick_side(rh.x, vc0, ru.x, !isnan(ru.x), rd.x, !isnan(rd.x)),
                                           pick_side(rh.y, vc1, ru.y, !isnan(ru.y), rd.y, !isnan(rd.y)));
            const float2 d2 = make_float2(cu.sa.w, cu.sb.w);
            const float2 e1a[3] = {cu.e[0], cu.e[1], cu.e[2]};
            const float2 e2a[3] = {cu.e[3], cu.e[4], cu.e[5]};
            const float2 sp[3] = {make_float2(cu.sa.x, cu.sb.x), make_float2(cu.sa.y, cu.sb.y),
                                  make_float2(cu.sa.z, cu.sb.z)};
            float2 gh[3], m[3];
            const float2 d2r = mul2(d2, rh);
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                gh[q] = mul2(d2, fma2(e2a[q], be2, mul2(e1a[q], be1)));
                const float2 drq = mul2(d2, fma2(e2a[q], br2, mul2(e1a[q], br1)));
                m[q] = fma2(d2r, sp[q], drq);
            }
            const float2 cY = mul2(d2, sub2(yh, cu.y));   // eq:img_cost_top
            const float2 cr = mul2(d2, sub2(rh, cu.rk));  // eq:invdepth_cost_top
            const float2 wp[3] = {make_float2(cu.wa.x, cu.wb.x), make_float2(cu.wa.y, cu.wb.y),
                                  make_float2(cu.wa.z, cu.wb.z)};
            float2 x[3];
#ifdef SF_DEBUG_KNOBS
            if (a.dbg & 1024) {  // timing experiment: no LDL^T solve (wrong results)
                x[0] = fma2(gh[0], cY, wp[0]);
                x[1] = fma2(m[1], cr, wp[1]);
                x[2] = wp[2];
            } else
#endif
            ls_solve3x2(gh, m, cY, cr, wp, f.g1, make_float2(vc0 ? f.g2 : 0.0f, vc1 ? f.g2 : 0.0f), f.g3, x);
            *reinterpret_cast<float2*>(F0 + idx) = x[0];  // (a ragged pair's second cell: out of the grid, unused)
            *reinterpret_cast<float2*>(F0 + PF + idx) = x[1];
            *reinterpret_cast<float2*>(F0 + 2 * PF + idx) = x[2];
            *reinterpret_cast<float2*>(RP + idx) = make_float2(cu.wa.w, cu.wb.w);
            if (r >= tr0 && r <= tr1) {  // tile cells: Yhat^{k+1}, non-finite solve flag
                const size_t g = pl + (size_t)(oi + r) * f.W + (oj + c);
                const bool in0 = c >= tc0 && c <= tc1, in1 = full && c + 1 >= tc0 && c + 1 <= tc1;
                if (in0) a.yout[g] = yh.x;
                if (in1) a.yout[g + 1] = yh.y;
                const bool bad = (in0 && !(isfinite(x[0].x) && isfinite(x[1].x) && isfinite(x[2].x))) ||
                                 (in1 && !(isfinite(x[0].y) && isfinite(x[1].y) && isfinite(x[2].y)));
                if (bad && oi + r >= f.fr0 && oi + r < f.fr1) fl |= SF_FLAG_NONFINITE;
            }
        };
        bool first = true;  // (ny already holds item 2)
#pragma unroll 1
        while (rn <= srh) {
#ifdef SF_DEBUG_KNOBS
            if (!(a.dbg & 16))  // timing experiment: 16 = no global fetches in the loop (wrong results)
#endif
            if (!first) {
                fetch_geo(rm, pm, ny);
                fetch_fld(rm, pm, ny);
            }
            first = false;
            solve_item(rn, pn, nx);
            if (rm > srh) break;
            rn = rm;
            pn = pm;
            advance(rn, pn);
#ifdef SF_DEBUG_KNOBS
            if (!(a.dbg & 16))  // timing experiment: 16 = no global fetches in the loop (wrong results)
#endif
            {
                fetch_geo(rn, pn, nx);
                fetch_fld(rn, pn, nx);
            }
            solve_item(rm, pm, ny);
            rm = rn;
            pm = pn;
            advance(rm, pm);
        }
    }

    // the next kernel's CTAs may launch once the solve's L2-bound loads are done (triggering at the
    // start instead: 25.52 vs 25.38 us/frame -- its prologue's loads then compete with the solve's)
    griddep_launch_dependents();
    SF_PROF();  // 3: solve
    // ---------------- stage 3: S x 5x5 box (reading 13) as a register-tiled separable
    // stencil: one item = one component's 4-column quad over 6 output rows, read as a window of 10
    // rows x 8 columns (8- and 16-byte shared loads) -> horizontal 5-sums left to right of the 10
    // rows -> vertical 5-sums top to bottom -> / 25 (div25: the IEEE quotient).  The passes
    // ping-pong between F0 and F1.  Window rows below a pass's last output row (the planes carry
    // 8 spare rows) and columns outside its window feed only unstored outputs.
    const bool edge = i0 - h < 0 || i0 + TH + h > f.H || j0 - h < 0 || j0 + TW + h > f.W;  // SR leaves the grid
    const int S = f.S;
    const float2 y25 = make_float2(0.04f, 0.04f), m25 = make_float2(-25.0f, -25.0f);
    float* src = F0;
    float* dst = F1;
#pragma unroll 1
    for (int it = 0; it < S; ++it) {
        const int mo = 2 * (S - 1 - it);  // this pass's output: tile +- mo, in the grid
        const int or0 = max(MR - mo, rmin), or1 = min(MR + TH + mo - 1, rmax);
        const int oc0 = max(MG - mo, cmin), oc1 = min(MG + TW + mo - 1, cmax);
        const int bc0 = oc0 & ~3, nbc = (oc1 - bc0) / 4 + 1;  // 16-byte aligned quads over [oc0, oc1]
        __syncthreads();
        if (edge) {
            fill_planes<3>(src, PF, PW, PH, or0 - 2, or1 + 2, oc0 - 2, oc1 + 2, rmin, rmax, cmin, cmax, tid);
            __syncthreads();
        }
#pragma unroll 1
        SF_FOR_RECT(sg, bq, 0, (or1 - or0) / 6, 0, 3 * nbc - 1, UPD_NT, tid) {
            // bq = 3 quad + component: with PF = 12 (mod 32) the 8 lanes of a quarter warp hit 8
            // distinct 16-byte bank groups (bank group of lane l steps by 3 mod 8)
            const int quad = (bq * 43691) >> 17, q = bq - 3 * quad;  // bq / 3 (exact for bq < 2^15)
            const int c = bc0 + 4 * quad, r = or0 + 6 * sg;
            const float* row = src + q * PF + (r - 2) * PW + c - 2;
            float2 hs[10][2];  // horizontal 5-sums of rows r-2 .. r+7, column pairs (c, c+1) (c+2, c+3)
#pragma unroll
            for (int i = 0; i < 10; ++i, row += PW) {
                const float2 xa = *reinterpret_cast<const float2*>(row);
                const float4 xb = *reinterpret_cast<const float4*>(row + 2);
                const float2 xc = *reinterpret_cast<const float2*>(row + 6);
                const float2 xab = make_float2(xa.y, xb.x), xbb = make_float2(xb.y, xb.z), xbc = make_float2(xb.w, xc.x);
                const float2 xlo = make_float2(xb.x, xb.y), xhi = make_float2(xb.z, xb.w);
                // sums of columns (c + j - 2 .. c + j + 2), j = 0..3, paired: ((((x0 + x1) + x2) + x3) + x4)
                hs[i][0] = add2(add2(add2(add2(xa, xab), xlo), xbb), xhi);
                hs[i][1] = add2(add2(add2(add2(xlo, xbb), xhi), xbc), xc);
            }
            float* out = dst + q * PF + r * PW + c;
#pragma unroll
            for (int i = 0; i < 6; ++i, out += PW) {
                float o[4];
#pragma unroll
                for (int jp = 0; jp < 2; ++jp) {
                    const float2 v = add2(add2(add2(add2(hs[i][jp], hs[i + 1][jp]), hs[i + 2][jp]), hs[i + 3][jp]),
                                          hs[i + 4][jp]);
                    const float2 qq = mul2(v, y25);
                    const float2 q1 = fma2(fma2(qq, m25, v), y25, qq);
                    o[2 * jp] = isfinite(v.x) ? q1.x : qq.x;
                    o[2 * jp + 1] = isfinite(v.y) ? q1.y : qq.y;
                }
                if (r + i <= or1) *reinterpret_cast<float4*>(out) = make_float4(o[0], o[1], o[2], o[3]);
            }
        }
        float* tmp = src;
        src = dst;
        dst = tmp;
    }
    __syncthreads();
    SF_PROF();  // 4: box

    // ---------------- stage 4: rho fusion and the store of the tile
    const float kap = f.kappa;
#pragma unroll 1
    SF_FOR_RECT(r, c, tr0, tr1, tc0, tc1, UPD_NT, tid) {
        const int idx = r * PW + c;
        const float rh = RHs[idx], rp = RP[idx];
        const bool v = !isnan(rh);
        const float rn1 = xfma(v ? kap : 0.0f, xsub(v ? rh : 0.0f, rp), rp);
        if (!isfinite(rn1) && oi + r >= f.fr0 && oi + r < f.fr1) fl |= SF_FLAG_NONFINITE;
        const size_t g = pl + (size_t)(oi + r) * f.W + (oj + c);
        const float4 o = make_float4(src[idx], src[PF + idx], src[2 * PF + idx], rn1);
        a.out[g] = o;
        if (a.w2)  // (Yhat^{k+1} of the tile cell: stored by this CTA's solve, visible after its barriers)
            a.wf[g] = up2_add_at(a.w2 + (size_t)b * (f.H / 2) * (f.W / 2), oi + r, oj + c, f.H, f.W, o, a.yout[g]);
    }
    SF_PROF();  // 5: fusion + store
    SF_PROF_PRINT("upd");
    const unsigned any = __reduce_or_sync(FULL, fl);
    if ((tid & 31) == 0 && any) atomicOr(a.flags, any);
    SF_TRACE_END(g_trace_upd, a.dslot);
}

// Tile shapes tried by the launcher (TW a multiple of 4).
struct TileOpt {
    int TW, TH;
};
constexpr TileOpt kTiles[] = {{64, 48}, {48, 40}, {32, 32}, {32, 16}, {16, 16}};

bool plan_tiles(const FrameParams& f, int h, UpdArgs& a, size_t& smem) {
    int sms = 148;
    {
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int MR = h + 2, MG = (h + 6) & ~3;  // MG >= h + 3, a multiple of 4
    long long best = -1;
    for (const TileOpt& t : kTiles) {
        // planes of PH rows + 8 spare rows (read by the box's last row segment): Y, rhohat, HG, HH
        // 128-byte aligned (TMA destinations), the 6 box planes at a stride of 12 (mod 32) floats
        const int PW = t.TW + 2 * MG, PH = t.TH + 2 * MR, P = (PW * (PH + 8) + 31) & ~31;
        const int PF = P + 12;
        const size_t bytes = sizeof(float) * (4 * (size_t)P + 6 * (size_t)PF) + 64;
        if (bytes > 227 * 1024) continue;
        const long long tiles = (long long)((f.W + t.TW - 1) / t.TW) * ((f.H + t.TH - 1) / t.TH) * f.B;
        const long long waves = (tiles + sms - 1) / sms;
        const long long cost = waves * (long long)(t.TW + 2 * h + 4) * (t.TH + 2 * h + 4);  // plane work per SM
        if (best < 0 || cost < best) {
            best = cost;
            a.TW = t.TW;
            a.TH = t.TH;
            a.MR = MR;
            a.MG = MG;
            a.PW = PW;
            a.PH = PH;
            a.P = P;
            a.PF = PF;
            smem = bytes;
        }
    }
    return best >= 0;
}

}  // namespace

// Supported when the box halo fits the planes (S <= 8).
bool sf_update_fused_supported(const sf_ctx* c) {
    if (c->fp.S > 8) return false;
    UpdArgs a;
    size_t smem = 0;
    if (!plan_tiles(c->fp, 2 * c->fp.S, a, smem)) return false;
    return cudaFuncSetAttribute(k_upd, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) == cudaSuccess;
}

// One update: pred (w^{k+}, rho^{k+}) + references + (Y, depth) -> out (state k+1), yout.
cudaError_t sf_launch_update_fused(sf_ctx* c, const float* Y, const float* D, const float4* pred, const float* rref,
                                   int rs, const float* yref, int ys, float4* out, float* yout, const float4* w2,
                                   float4* wf) {
    const FrameParams& f = c->fp;
    UpdArgs a;
    size_t smem = 0;
    a.h = 2 * f.S;
    if (!plan_tiles(f, a.h, a, smem)) return cudaErrorInvalidConfiguration;
    a.tma = sf_tma_encode3d(&a.tmY, Y, f.W, f.H, f.B, a.PW, a.PH, 1) &&
            sf_tma_encode3d(&a.tmD, D, f.W, f.H, f.B, a.PW, a.PH, 1);
    a.pred = pred;
    a.rref = rref;
    a.rs = rs;
    a.yref = yref;
    a.ys = ys;
    a.Y = Y;
    a.D = D;
    a.G0 = c->G0;
    a.E = c->E;
    a.EW = sf_ew(f.W);
    a.EP = (size_t)a.EW * sf_eh(f.H);
    a.e8 = (a.EW % 2 == 0 && (reinterpret_cast<uintptr_t>(c->E) & 7) == 0) ? 1 : 0;
    a.out = out;
    a.yout = yout;
    a.w2 = w2;
    a.wf = wf;
    a.flags = c->flags;
    a.f = f;
    {
        static const int dbg_env = [] {
            const char* e = getenv("SF_DEBUG_SKIP");
            return e ? atoi(e) : 0;
        }();
        a.dbg = dbg_env;
    }
    a.dslot = c->dbg_frame;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((f.W + a.TW - 1) / a.TW, (f.H + a.TH - 1) / a.TH, f.B);
    lc.blockDim = dim3(UPD_NT);
    lc.dynamicSmemBytes = smem;
    lc.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL behind the transport kernel
    at[0].val.programmaticStreamSerializationAllowed = sf_pdl_enabled() ? 1 : 0;
    lc.attrs = at;
    lc.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&lc, k_upd, a);
    if (e == cudaSuccess) e = cudaGetLastError();
    return e;
}

#ifdef SF_DEBUG_KNOBS
// Debug builds: the k_upd per-CTA timeline of trace slot `slot` (as sf_debug_trace_trans).
extern "C" int sf_debug_trace_upd(int slot, unsigned long long* out, int n) {
    return cudaMemcpyFromSymbol(out, g_trace_upd, sizeof(unsigned long long) * 3 * n,
                                sizeof(unsigned long long) * 3 * 4096 * (slot & 3)) == cudaSuccess ? 0 : -1;
}
#endif
