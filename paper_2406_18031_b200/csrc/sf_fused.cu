// sf_fused.cu -- temporally blocked, fused predict + update: one launch per frame for
// N <= 8 (ceil(N/8) launches beyond).  Same bits as sf_passes.cu.
//
// Layout.  A CTA owns an output tile TH x TW and computes on a
// region RH x RW = (TH + 2R) x (TW + 2R), RW = 64 = one warp of lanes owning 2 adjacent
// columns each, RH = K * NWY (NWY warps stacked vertically, K rows per thread).
// R = max(M, 2) + 2S (M substeps in this launch, S box passes), rounded up to even.
//   * each thread owns a 2 x K micro-tile; its fields (w.x, w.y, w.z, rho) and directions s
//     stay in REGISTERS for the whole frame; e1/e2 live in shared-memory planes;
//   * column pass (j +- 1): the partner column is in registers, the other neighbour is one
//     lane away -> warp shuffles only; no shared memory, no barrier;
//   * row pass (i +- 1): neighbours are in the thread's own rows except the run ends, which
//     are swapped through a double-buffered shared row buffer: one __syncthreads per pass;
//   * CTAs whose region touches the grid border take the EDGE instantiation (replicate
//     boundary, reading 10); interior CTAs carry no boundary logic at all;
//   * cut region edges produce inexact ("garbage") cells that never reach the tile: the
//     halo R covers the dependency radius (M per axis for the transport, 2S + 2 for the
//     update); flags are taken only from tile cells, which are exact at every pass;
//   * e planes, Y and depth are staged by TMA bulk tensor copies issued at kernel start (Y and
//     depth land while the transport runs; cp.async fallback when W % 4 != 0), and
//     while the transport runs; the update computes the brightness / inverse-depth models,
//     the 3x3 LDL^T solve and S box passes on shared planes, then fuses rho and stores.
// The per-cell arithmetic of the transport runs on cell pairs as f32x2 ops (FADD2/FMUL2/FFMA2).
#include <cuda.h>
#include <stdio.h>
#include <stdlib.h>

#include <string.h>

#include <mutex>

#include "sf_pair.cuh"

namespace {

using namespace sfp;



// Replicate-border fill (reading 10) of the out-of-grid cells of the rectangle [ra, rb] x [ca, cb]
// of NP shared planes: each takes the value of its clamped in-grid cell.  Only the out-of-grid
// bands are visited (top and bottom rows with corners, then left and right columns).
template <int NP, int RW, int RH, int NT>
__device__ __forceinline__ void edge_fill(float* p0, float* p1, float* p2, int ra, int rb, int ca, int cb, int rmin,
                                          int rmax, int cmin, int cmax, int tid) {
    ra = max(ra, 0);
    rb = min(rb, RH - 1);
    ca = max(ca, 0);
    cb = min(cb, RW - 1);
    auto cp = [&](int r, int c) {
        const int from = iclamp(r, rmin, rmax) * RW + iclamp(c, cmin, cmax), to = r * RW + c;
        p0[to] = p0[from];
        p1[to] = p1[from];
        if (NP > 2) p2[to] = p2[from];
    };
    // one band: empty bands are skipped before any index arithmetic (block-uniform test)
    auto band = [&](int r0, int r1, int c0, int c1) {
        const int nc = c1 - c0 + 1, nr = r1 - r0 + 1;
        if (nc <= 0 || nr <= 0) return;
#pragma unroll 1
        for (int t = tid; t < nc * nr; t += NT) {
            const int q = t / nc;
            cp(r0 + q, c0 + t - q * nc);
        }
    };
    band(ra, min(rb, rmin - 1), ca, cb);
    band(max(ra, rmax + 1), rb, ca, cb);
    band(max(ra, rmin), min(rb, rmax), ca, min(cb, cmin - 1));
    band(max(ra, rmin), min(rb, rmax), max(ca, cmax + 1), cb);
}

struct FusedArgs {
    CUtensorMap tmE;    // [6][H][W] e planes, box 64 x 72 x 3   (valid when tma)
    CUtensorMap tmY;    // [B][H][W] brightness, box 64 x 72 x 1
    CUtensorMap tmD;    // [B][H][W] depth, box 64 x 72 x 1
    int tma;            // 1: stage e / Y / depth with TMA (needs W % 4 == 0, 16-byte aligned bases)
    int flush;          // k_trans: regions flush with the grid border where the grid is large enough
    int onebody;        // k_trans A/B: interior CTAs on the COLFIX instantiation
    int y16;            // 1: Y and depth bases 16-byte aligned (the cp.async fallback may copy 16 bytes)
    int dbg_skip;       // timing experiments only (SF_DEBUG_SKIP): 1 = skip transport, 2 = skip update,
                        // 4 = no e TMA, 8 = no Y/depth TMA, 16 = no field / s loads, 32 = exit at entry,
                        // 64 = no column passes, 128 = no row passes, 256 = print phase clocks of CTA (6,5),
                        // 512 = no box passes, 1024 = no solve, 2048 = print per-CTA globaltimer stamps,
                        // 4096 = every CTA takes the edge instantiation of the transport
    const float4* fin;  // fields at launch start (state k or a partial prediction)
    const float4* sk;   // state k (rho^k for the update)
    float4* fout;       // state k+1 (upd) or partial prediction
    const float* yin;   // Yhat^k
    float* yout;        // Yhat^{k+1}
    const float* Y;
    const float* D;
    const float4* G0;   // (s, d2)
    const float4* G1;   // e1
    const float4* G2;   // e2
    const float* E;     // [6][H*W] (e1.xyz, e2.xyz planes)
    unsigned* flags;
    int dslot;          // debug builds: trace slot (frame & 3)
    float* rk;          // k_trans, first launch of a frame: rho^k of the tile cells -> [B][H][W] (k_upd's c_rho
                        // reference, read there 4 bytes per cell); null otherwise
    FrameParams f;
    int M;    // substeps in this launch
    int upd;  // 1: run the update after the substeps
    int R;    // halo (even)
    int TH, TW;
};

template <int K, int NWY>
struct Cfg {
    static constexpr int RW = 64, RH = K * NWY, P = RW * RH, NT = 32 * NWY;
    static constexpr int XR = NWY * 2 * RW;  // float4 slots of one row-exchange buffer
    // smem floats: E planes 6P | Ys P | Ds/Rs P | XR buffers 2 x 4 XR (>= 2P for HG/HH, and
    // Ys..end >= 3P for the box planes)
    static constexpr int XRF = 2 * 4 * XR > 4 * P ? 2 * 4 * XR : 4 * P;  // row buffers | HG HH Fy Fz
    static constexpr size_t SMEM = sizeof(float) * (8 * (size_t)P + XRF) + 64;  // + mbarriers
};


// The transport: M substeps of a column pass then a row pass on the thread's
// 2 x K cells, held cell-paired: W[0..2][k] = w (x, y, z), W[3][k] = rho, each a float2 over the
// thread's two columns.  Grid borders (replicate clamp, reading 10) are handled by REPLICA cells:
// the out-of-grid cell next to a grid edge is kept equal to the edge cell (loaded that way, and
// refreshed after each pass that changed the edge), so the neighbour read of the edge cell
// returns its own value and the pass bodies carry no boundary logic.  A grid edge on the
// region border itself needs no replica: it lies R cells from the tile, outside the tile's
// dependency cone, like any cut edge.
// EDGE = false (interior CTAs, no grid edge in the region) and IMU = false compile the edge
// replicas and the inertial stage out, so the substep loop is straight-line code between barriers.
// EREG: the lane's e1 / e2 (ER[0..2] = e1.xyz, ER[3..5] = e2.xyz, cell-paired) are held in
// registers instead of being read from the shared e planes each pass, and the run-end rows' v is
// exchanged through the row buffer (as a fifth component) instead of being recomputed from e2.
// COLFIX: the region's first / last column is the grid's first / last column (fixL / fixR): the
// replicate border is applied in the column pass itself -- lane 0's cell 0 and lane 31's cell 1 take
// their own u and their own value as the outside neighbour's -- instead of through replica cells.
template <int K, int NWY, int RULE, bool CLAMP, int NF = 4, bool EDGE = true, bool IMU = true, bool EREG = false,
          bool COLFIX = false>
__device__ __forceinline__ void transport_passes(const FrameParams& f, int M, float2 (&W)[NF][K], const float2 (&SX)[K],
                                                 const float2 (&SY)[K], const float2 (&SZ)[K], float (&mx)[K],
                                                 const float* Es, float2* XB0, int lane, int wy, int cmin, int cmax,
                                                 int rmin, int rmax, int dbg, const float* Ss = nullptr,
                                                 const float2 (*ER)[K] = nullptr, bool fixL = false,
                                                 bool fixR = false) {
    using C = Cfg<K, NWY>;
    constexpr int RW = C::RW, P = C::P, RH = C::RH;
    // NF = 4: (w, rho), all dilated.  NF = 8 (pyramid bottom level): (w, dw, rho, Yhat), the last
    // one without dilation (eq:img_propagation_low)
    constexpr int ND = NF == 8 ? 7 : NF;
    constexpr int NX = EREG ? NF + 1 : NF;  // row-buffer components (+ v with EREG)
    constexpr int XBS = NX * NWY * 2 * 32;  // float2 slots of one row-exchange buffer
    const int c0_ = 2 * lane, r0_ = K * wy;
    auto e1v = [&](int k, int q) -> float2 {  // component q of (e1, e2) at the lane's row k
        if (EREG) return ER[q][k];
        return *reinterpret_cast<const float2*>(Es + q * P + (r0_ + k) * RW + c0_);
    };
    // NF = 4: two buffers (substep parity); NF = 8: one buffer (shared memory is short) and a
    // second barrier per substep after the neighbour rows are read
    constexpr int NXB = NF == 8 ? 1 : 2;
    const int c0 = 2 * lane, r0 = K * wy;
    const float U = f.U;
    // s of the lane's cells: registers (NF = 4), or shared planes Ss[3][P] (NF = 8: registers
    // are taken by the 8 fields)
    auto sdot = [&](int k) -> float2 {
        if (NF == 8) {
            const int ib = (r0 + k) * RW + c0;
            return dot2(*reinterpret_cast<const float2*>(Ss + ib), *reinterpret_cast<const float2*>(Ss + P + ib),
                        *reinterpret_cast<const float2*>(Ss + 2 * P + ib), W[0][k], W[1][k], W[2][k]);
        }
        return dot2(SX[k], SY[k], SZ[k], W[0][k], W[1][k], W[2][k]);
    };
    const float2 T2 = make_float2(-f.dt, -f.dt), SG = make_float2(f.sigma, f.sigma);
    const int srcL = lane - 1, srcR = lane + 1;
    const bool eL = COLFIX && fixL && lane == 0, eR = COLFIX && fixR && lane == 31;
    // replica bookkeeping (block-uniform except for the lane / k tests)
    const bool repL = EDGE && cmin > 0, repR = EDGE && cmax < RW - 1, repT = EDGE && rmin > 0,
               repB = EDGE && rmax < RH - 1;
    const int laneL = cmin / 2 - 1;                            // owns replica column cmin-1 as its cell 1
    const int laneR = (cmax & 1) ? (cmax + 1) / 2 : cmax / 2;  // owns replica column cmax+1
    const bool rOdd = (cmax & 1) != 0;                         // replica is cell 0 of laneR (else its cell 1)
#ifdef SF_EXP_NO_IN1
    const bool in1 = true;
#else
    const bool in1 = !EDGE || c0 + 1 <= cmax;                  // cell 1 inside the grid (for the flag max)
#endif
    const int keT = rmin - r0, keB = rmax - r0;                // edge rows in this thread's run
    // warp-uniform (a vote result) so the refresh branches below need no reconvergence regions
    const bool doT = __all_sync(FULL, repT && keT >= 1 && keT <= K - 1);
    const bool doB = __all_sync(FULL, repB && keB >= 0 && keB <= K - 2);

    // dominant flow of both cells -> flag max, clamp, (|u_hat0|, |u_hat1|)
    // (the clamp keeps the sign since U > 0, and |clamp(u, -U, U)| = min(|u|, U) -- also for a
    //  NaN u_hat, which the clamp turns into -U: upwind side "not > 0", weight U)
    auto flow = [&](int k, float uh0, float uh1, bool& p0, bool& p1) -> float2 {
        p0 = uh0 > 0.0f;
        p1 = uh1 > 0.0f;
        const float a0 = fabsf(uh0), a1 = fabsf(uh1);
        mx[k] = fmaxf(mx[k], fmaxf(a0, in1 ? a1 : 0.0f));
        if (CLAMP) return make_float2(fminf(a0, U), fminf(a1, U));
        return make_float2(a0, a1);
    };

    for (int n = 0; n < M; ++n) {
        // ================= column pass (beta_1): registers + shuffles only
        if (!(dbg & 64))
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const float2 u = dot2(e1v(k, 0), e1v(k, 1), e1v(k, 2), W[0][k], W[1][k], W[2][k]);
            float uL = __shfl_up_sync(FULL, u.y, 1);    // lane-1's cell 1 = left of cell 0
            float uR = __shfl_down_sync(FULL, u.x, 1);  // lane+1's cell 0 = right of cell 1
            if (COLFIX) {  // grid edge at the region edge: the outside neighbour is the cell itself
                uL = eL ? u.x : uL;
                uR = eR ? u.y : uR;
            }
            bool p0, p1;
            const float2 A = flow(k, dominant(uL, u.y, RULE), dominant(u.x, uR, RULE), p0, p1);
            // upwind value by per-lane source: cell 0 takes lane-1's cell 1 (u_hat > 0) or its own
            // cell 1; cell 1 takes its own cell 0 (u_hat > 0) or lane+1's cell 0
            const int s0 = p0 ? srcL : lane, s1 = p1 ? lane : srcR;
            const bool own0 = COLFIX && eL && p0, own1 = COLFIX && eR && !p1;
            const float2 q = mul2(SG, sdot(k));
#pragma unroll
            for (int c = 0; c < NF; ++c) {
                float2 fu = make_float2(__shfl_sync(FULL, W[c][k].y, s0), __shfl_sync(FULL, W[c][k].x, s1));
                if (COLFIX) fu = make_float2(own0 ? W[c][k].x : fu.x, own1 ? W[c][k].y : fu.y);
                W[c][k] = c < ND ? tr2(W[c][k], fu, A, q, T2) : fma2(T2, mul2(A, sub2(W[c][k], fu)), W[c][k]);
            }
        }
        // column replicas <- their edge cells
#ifndef SF_EXP_NO_COLREP  // (SF_EXP_*: timing experiments, tools/gpu_gtexp.sh; wrong results)
        if (repL) {
            const bool me = lane == laneL;
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
                for (int c = 0; c < NF; ++c) {
                    const float e = __shfl_down_sync(FULL, W[c][k].x, 1);
                    W[c][k].y = me ? e : W[c][k].y;
                }
        }
        if (repR) {
            const bool me = lane == laneR;
            if (rOdd) {
#pragma unroll
                for (int k = 0; k < K; ++k)
#pragma unroll
                    for (int c = 0; c < NF; ++c) {
                        const float e = __shfl_up_sync(FULL, W[c][k].y, 1);
                        W[c][k].x = me ? e : W[c][k].x;
                    }
            } else {
#pragma unroll
                for (int k = 0; k < K; ++k)
#pragma unroll
                    for (int c = 0; c < NF; ++c) W[c][k].y = me ? W[c][k].x : W[c][k].y;
            }
        }
#endif
        // row replicas inside this thread's run <- their edge rows (before the row pass reads)
#ifndef SF_EXP_NO_ROWREP
        if (doT) {
#pragma unroll
            for (int k = 0; k < K - 1; ++k) {
                const bool p = (keT - 1 - k) == 0;
#pragma unroll
                for (int c = 0; c < NF; ++c) W[c][k] = sel2(p, p, W[c][k + 1], W[c][k]);
            }
        }
        if (doB) {
#pragma unroll
            for (int k = K - 1; k >= 1; --k) {
                const bool p = (keB + 1 - k) == 0;
#pragma unroll
                for (int c = 0; c < NF; ++c) W[c][k] = sel2(p, p, W[c][k - 1], W[c][k]);
            }
        }
#endif
        // ================= row pass (beta_2, reading 3)
        if (!(dbg & 128)) {
            // run-end rows to the exchange buffer: [comp][warp][end][lane] float2
            float2* const XB = XB0 + (NXB == 2 ? (n & 1) * XBS : 0);
#pragma unroll
            for (int c = 0; c < NF; ++c) {
                XB[((c * NWY + wy) * 2 + 0) * 32 + lane] = W[c][0];
                XB[((c * NWY + wy) * 2 + 1) * 32 + lane] = W[c][K - 1];
            }
            float2 v[K];
#pragma unroll
            for (int k = 0; k < K; ++k) v[k] = dot2(e1v(k, 3), e1v(k, 4), e1v(k, 5), W[0][k], W[1][k], W[2][k]);
            if (EREG) {  // the run ends' v for the neighbour warps
                XB[((NF * NWY + wy) * 2 + 0) * 32 + lane] = v[0];
                XB[((NF * NWY + wy) * 2 + 1) * 32 + lane] = v[K - 1];
            }
            // row k in place from its upwind values fu (selected from the pre-pass rows k-1 / k+1)
            auto row_update = [&](int k, float2 vm, float2 vp, const float2 (&fm)[NF], const float2 (&fp)[NF]) {
                bool p0, p1;
                const float2 A = flow(k, dominant(vm.x, vp.x, RULE), dominant(vm.y, vp.y, RULE), p0, p1);
                const float2 q = mul2(SG, sdot(k));
#pragma unroll
                for (int c = 0; c < NF; ++c) {
                    const float2 fu = sel2(p0, p1, fm[c], fp[c]);
                    W[c][k] = c < ND ? tr2(W[c][k], fu, A, q, T2) : fma2(T2, mul2(A, sub2(W[c][k], fu)), W[c][k]);
                }
            };
            // pre-pass rows 1 and K-2 are kept for the run ends; the interior rows 1..K-2 need no
            // exchanged value and are updated before the barrier, in place, in increasing k: row
            // k's neighbours are the pre-pass row k-1 (kept one step) and row k+1 (not yet updated)
            float2 o1[NF], oK[NF], prev[NF];
#pragma unroll
            for (int c = 0; c < NF; ++c) {
                o1[c] = W[c][1];
                oK[c] = W[c][K - 2];
                prev[c] = W[c][0];
            }
#pragma unroll
            for (int k = 1; k <= K - 2; ++k) {
                float2 cur[NF], nxt[NF];
#pragma unroll
                for (int c = 0; c < NF; ++c) {
                    cur[c] = W[c][k];
                    nxt[c] = W[c][k + 1];
                }
                row_update(k, v[k - 1], v[k + 1], prev, nxt);
#pragma unroll
                for (int c = 0; c < NF; ++c) prev[c] = cur[c];
            }
            __syncthreads();
            float2 t[NF], bb[NF];
            float2 vt = v[0], vb = v[K - 1];
#pragma unroll
            for (int c = 0; c < NF; ++c) {
                t[c] = W[c][0];
                bb[c] = W[c][K - 1];
            }
            // neighbour run ends; at an edge row on a run boundary the replica is the row itself.
            // Select form: the neighbour warp's entry and the e planes one row outside the run are
            // always read (warp index and row clamped to the region).
            {
                const bool useT = wy > 0 && !(repT && keT == 0), useB = wy < NWY - 1 && !(repB && keB == K - 1);
                const int wt = wy > 0 ? wy - 1 : 0, wb = wy < NWY - 1 ? wy + 1 : NWY - 1;
                float2 tn[NF], bn[NF];
#pragma unroll
                for (int c = 0; c < NF; ++c) {
                    tn[c] = XB[((c * NWY + wt) * 2 + 1) * 32 + lane];
                    bn[c] = XB[((c * NWY + wb) * 2 + 0) * 32 + lane];
                }
                // (rows clamped to the region: the first / last warp's unused read stays off Y's plane,
                //  which the Y / depth loads may still be writing)
                float2 vtn, vbn;
                if (EREG) {  // the neighbours' own v of those rows (the same bits as recomputing it)
                    vtn = XB[((NF * NWY + wt) * 2 + 1) * 32 + lane];
                    vbn = XB[((NF * NWY + wb) * 2 + 0) * 32 + lane];
                } else {
                    const int it = (wy > 0 ? r0 - 1 : r0) * RW + c0, ibb = (wy < NWY - 1 ? r0 + K : r0 + K - 1) * RW + c0;
                    vtn = dot2(*reinterpret_cast<const float2*>(Es + 3 * P + it),
                               *reinterpret_cast<const float2*>(Es + 4 * P + it),
                               *reinterpret_cast<const float2*>(Es + 5 * P + it), tn[0], tn[1], tn[2]);
                    vbn = dot2(*reinterpret_cast<const float2*>(Es + 3 * P + ibb),
                               *reinterpret_cast<const float2*>(Es + 4 * P + ibb),
                               *reinterpret_cast<const float2*>(Es + 5 * P + ibb), bn[0], bn[1], bn[2]);
                }
#pragma unroll
                for (int c = 0; c < NF; ++c) {
                    t[c] = sel2(useT, useT, tn[c], t[c]);
                    bb[c] = sel2(useB, useB, bn[c], bb[c]);
                }
                vt = sel2(useT, useT, vtn, vt);
                vb = sel2(useB, useB, vbn, vb);
            }
            row_update(0, vt, v[1], t, o1);
            row_update(K - 1, v[K - 2], vb, oK, bb);
            if (NXB == 1) __syncthreads();  // the single exchange buffer is rewritten next substep
        }
        if (NF == 4 && IMU && f.imu) {  // inertial stage after the row pass (reading 32), per cell
#pragma unroll
            for (int k = 0; k < K; ++k) {
                imu_stage(f, SX[k].x, SY[k].x, SZ[k].x, W[0][k].x, W[1][k].x, W[2][k].x, W[3][k].x);
                imu_stage(f, SX[k].y, SY[k].y, SZ[k].y, W[0][k].y, W[1][k].y, W[2][k].y, W[3][k].y);
            }
        }
        // (row passes keep column replicas valid; the next column pass keeps row replicas as
        //  they are and they are refreshed again before the next row pass)
    }
}

template <int K, int NWY, int RULE, bool CLAMP>
__global__ void __launch_bounds__(32 * NWY, 1) k_fused(const __grid_constant__ FusedArgs a) {
    using C = Cfg<K, NWY>;
    constexpr int RW = C::RW, RH = C::RH, P = C::P, NT = C::NT;
    extern __shared__ __align__(1024) float4 smem4[];  // TMA destinations need 128-byte alignment
    float* const sm = reinterpret_cast<float*>(smem4);
    float* const Es = sm;          // transport: 6 planes e1.xyz, e2.xyz
    float* const Ys = sm + 6 * P;  // Y (replicated clamp)
    float* const Ds = sm + 7 * P;  // depth -> rhohat (NaN = invalid)
    float* const Xb = sm + 8 * P;  // transport: 2 row-exchange buffers
    float2* const XB0 = reinterpret_cast<float2*>(Xb);

    const FrameParams& f = a.f;
    const int tid = threadIdx.x, lane = tid & 31, wy = tid >> 5;
    const int c0 = 2 * lane, r0 = K * wy;
    const int b = blockIdx.z, R = a.R, TH = a.TH, TW = a.TW;
    const int gi0 = blockIdx.y * TH - R, gj0 = blockIdx.x * TW - R;
    // in-grid part of the region (also the replicate-clamp bounds)
    const int cmin = max(0, -gj0), cmax = min(RW - 1, f.W - 1 - gj0);
    const int rmin = max(0, -gi0), rmax = min(RH - 1, f.H - 1 - gi0);
    const bool edgeC = cmin > 0 || cmax < RW - 1;  // block-uniform
    const bool edgeR = rmin > 0 || rmax < RH - 1;
    const size_t HW = (size_t)f.H * f.W, plane = (size_t)b * HW;

#ifdef SF_DEBUG_KNOBS
    const int dbg = a.dbg_skip;  // timing experiments (build with SF_BUILD_DEBUG=1)
#else
    constexpr int dbg = 0;       // production build: every knob folds away
#endif
    if (dbg & 32) return;
    long long T_[16];
    int nT_ = 0;
    const bool tim = (dbg & 256) && blockIdx.z == 0 &&
                     ((blockIdx.x == 6 && blockIdx.y == 5) || (blockIdx.x == 0 && blockIdx.y == 0) ||
                      (blockIdx.x == 0 && blockIdx.y == 5) || (blockIdx.x == gridDim.x - 1 && blockIdx.y == gridDim.y - 1));
#define SF_TICK() do { if (tim) { __syncthreads(); if (tid == 0) T_[nT_] = clock64(); ++nT_; } } while (0)
    SF_TICK();
    unsigned long long gt0_ = 0, gt1_ = 0, gte_ = 0, gtt_ = 0;  // dbg 2048: globaltimer at entry / griddep release /
    // e planes in / transport done / exit
    if (dbg & 2048) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt0_));
    // ---------------- staging: e1 / e2 planes (transport), Y and depth (update)
    uint64_t* const bars = reinterpret_cast<uint64_t*>(sm + 8 * P + C::XRF);
    if (a.tma) {
        // TMA: one thread issues three bulk tensor copies of the whole region (out-of-range cells
        // arrive as zeros; the replica e cells next to grid edges come from E's padding)
        if (tid == 0) {
            mbar_init(&bars[0], 1);
            mbar_init(&bars[1], 1);
            mbar_init(&bars[2], 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
        if (tid == 0 && !(dbg & 4)) {  // geometry: independent of the previous frame
            mbar_expect_tx(&bars[0], 3u * P * 4u);
            tma_load_3d(Es, &a.tmE, gj0 + SF_EPAD, gi0 + SF_EPAD, 0, &bars[0]);
            mbar_expect_tx(&bars[1], 3u * P * 4u);
            tma_load_3d(Es + 3 * P, &a.tmE, gj0 + SF_EPAD, gi0 + SF_EPAD, 3, &bars[1]);
        }
    } else {
        const bool pair = !edgeC && (f.W & 1) == 0;  // both cells contiguous and 8-byte aligned
        const int EW = sf_ew(f.W);
        const size_t EP = (size_t)EW * sf_eh(f.H);  // padded e planes: clamped cell (i, j) at (i + EPAD, j + EPAD)
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int r = r0 + k;
            const size_t gr = (size_t)(iclamp(gi0 + r, 0, f.H - 1) + SF_EPAD) * EW + SF_EPAD;
            const size_t ga = gr + iclamp(gj0 + c0, 0, f.W - 1), gb = gr + iclamp(gj0 + c0 + 1, 0, f.W - 1);
#pragma unroll
            for (int p = 0; p < 6; ++p) {
                float* dst = Es + p * P + r * RW + c0;
                if (pair) {
                    cp_async8(dst, a.E + p * EP + ga);
                } else {
                    cp_async4(dst, a.E + p * EP + ga);
                    cp_async4(dst + 1, a.E + p * EP + gb);
                }
            }
        }
        cp_async_commit();
        griddep_wait();  // inputs / state of this frame may come from the preceding kernel
        if (dbg & 2048) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt1_));
        if (a.upd) {
            if (a.y16 && !edgeC && !edgeR && (f.W & 3) == 0 && (gj0 & 3) == 0) {
                for (int idx = tid; idx < P / 4; idx += NT) {
                    const int r = idx / (RW / 4), c = (idx % (RW / 4)) * 4;
                    const size_t g = plane + (size_t)(gi0 + r) * f.W + (gj0 + c);
                    cp_async16(Ys + r * RW + c, a.Y + g);
                    cp_async16(Ds + r * RW + c, a.D + g);
                }
            } else {
                for (int idx = tid; idx < P; idx += NT) {
                    const int r = idx / RW, c = idx % RW;
                    const size_t g = plane + (size_t)iclamp(gi0 + r, 0, f.H - 1) * f.W + iclamp(gj0 + c, 0, f.W - 1);
                    cp_async4(Ys + idx, a.Y + g);
                    cp_async4(Ds + idx, a.D + g);
                }
            }
        }
        cp_async_commit();
    }

    // ---------------- own fields and directions -> registers
    float2 W[4][K];  // cell-paired fields: w.x, w.y, w.z, rho
    float2 SX[K], SY[K], SZ[K];
    float mx[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const size_t gr = (size_t)iclamp(gi0 + r0 + k, 0, f.H - 1) * f.W;
        const size_t ga = gr + iclamp(gj0 + c0, 0, f.W - 1), gb = gr + iclamp(gj0 + c0 + 1, 0, f.W - 1);
        const float4 sa = (dbg & 16) ? make_float4(0, 0, 1, 0) : __ldg(a.G0 + ga);
        const float4 sb = (dbg & 16) ? make_float4(0, 0, 1, 0) : __ldg(a.G0 + gb);
        SX[k] = make_float2(sa.x, sb.x);
        SY[k] = make_float2(sa.y, sb.y);
        SZ[k] = make_float2(sa.z, sb.z);
        mx[k] = 0.0f;
    }
    // ---- programmatic dependent launch: everything above is frame-invariant geometry; the state
    // and the frame's inputs may be written by the preceding kernel in the stream
    if (a.tma) {
        griddep_wait();
        if (dbg & 2048) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt1_));
        if (tid == 0 && a.upd && !(dbg & 8)) {
            mbar_expect_tx(&bars[2], 2u * P * 4u);
            tma_load_3d(Ys, &a.tmY, gj0, gi0, b, &bars[2]);
            tma_load_3d(Ds, &a.tmD, gj0, gi0, b, &bars[2]);
        }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const size_t gr = (size_t)iclamp(gi0 + r0 + k, 0, f.H - 1) * f.W;
        const size_t ga = gr + iclamp(gj0 + c0, 0, f.W - 1), gb = gr + iclamp(gj0 + c0 + 1, 0, f.W - 1);
        const float4 fa = (dbg & 16) ? make_float4(0, 0, 0, 0.5f) : a.fin[plane + ga];
        const float4 fb = (dbg & 16) ? make_float4(0, 0, 0, 0.5f) : a.fin[plane + gb];
        W[0][k] = make_float2(fa.x, fb.x);
        W[1][k] = make_float2(fa.y, fb.y);
        W[2][k] = make_float2(fa.z, fb.z);
        W[3][k] = make_float2(fa.w, fb.w);
    }
    griddep_launch_dependents();  // the next frame's CTAs may start their geometry loads
    SF_TICK();
    if (a.tma && !(dbg & 4)) {
        mbar_wait(&bars[0], 0);
        mbar_wait(&bars[1], 0);
        // (replica e cells next to grid edges arrive with the load: padded E, reading 10)
        if (dbg & 2048) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gte_));
    } else {
        cp_async_wait<1>();  // own e cells landed (each thread reads only what it copied until the 1st barrier)
    }

    if (!(dbg & 1))
    {
        if (edgeC || edgeR || f.imu || (dbg & 4096))
            transport_passes<K, NWY, RULE, CLAMP, 4, true, true>(f, a.M, W, SX, SY, SZ, mx, Es, XB0, lane, wy, cmin,
                                                                 cmax, rmin, rmax, dbg);
        else
            transport_passes<K, NWY, RULE, CLAMP, 4, false, false>(f, a.M, W, SX, SY, SZ, mx, Es, XB0, lane, wy,
                                                                   cmin, cmax, rmin, rmax, dbg);
    }
    if (dbg & 2048) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gtt_));
    const float U = f.U;

    // ---------------- flags from tile cells (exact at every pass); |u_hat| before the clamp
    unsigned fl = 0;
    {
        const bool tcol = c0 >= R && c0 < R + TW && c0 >= cmin && c0 <= cmax;  // R, TW even: both cells or none
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int r = r0 + k;
            if (tcol && r >= R && r < R + TH && r >= rmin && r <= rmax && gi0 + r >= f.fr0 && gi0 + r < f.fr1) {
                if (CLAMP) {
                    if (mx[k] > U) fl |= SF_FLAG_CLAMPED;
                } else if (xmul(f.dt, mx[k]) > 1.0f) {
                    fl |= SF_FLAG_CFL;
                }
            }
        }
    }

    SF_TICK();
    if (!a.upd || (dbg & 2)) {  // intermediate launch: store the partial prediction of the tile
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int r = r0 + k;
            if (r >= R && r < R + TH && r >= rmin && r <= rmax) {
                const size_t g = plane + (size_t)(gi0 + r) * f.W + (gj0 + c0);
                if (c0 >= R && c0 < R + TW && c0 >= cmin && c0 <= cmax)
                    a.fout[g] = make_float4(W[0][k].x, W[1][k].x, W[2][k].x, W[3][k].x);
                if (c0 + 1 >= R && c0 + 1 < R + TW && c0 + 1 >= cmin && c0 + 1 <= cmax)
                    a.fout[g + 1] = make_float4(W[0][k].y, W[1][k].y, W[2][k].y, W[3][k].y);
            }
        }
    } else {
        // =========================== update (U1-U5) on shared planes, compact runtime loops
        // planes: E (e1, e2) stay until the solve; HG, HH, Fy and rhohat take the row-buffer region
        // (rhohat lives to the end); Fx and Fz take Y's and depth's planes once the models are done
        float* const HG = Xb;
        float* const HH = Xb + P;
        float* const Fx = Ys;  // w^{k+} -> w_LS -> smoothed w (in place)
        float* const Fy = Xb + 2 * P;
        float* const Fz = Ds;
        float* const RHs = Xb + 3 * P;  // rhohat (NaN = invalid)
        const int S = f.S;
        // solve region = tile + 2S (clipped to the grid); models needed on it +-2 rows, +-1 cols
        const int rlo = max(R - 2 * S, rmin), rhi = min(R + TH + 2 * S - 1, rmax);
        const int clo = max(R - 2 * S, cmin), chi = min(R + TW + 2 * S - 1, cmax);
        // the solve's work distribution (pairs of the solve region over the threads) and its first
        // pair's global inputs (s, ds^2, Yhat^k, rho^k), fetched here so that their latency hides
        // behind the models; later pairs are fetched one pair ahead inside the solve loop
        const int ncol = ((dbg & 1024) ? clo - 1 : chi) - clo + 1;
        const int nc = (ncol + 1) >> 1, dr = nc > 0 ? NT / nc : 0, dc = nc > 0 ? NT % nc : 0;
        int rn = nc > 0 ? rlo + tid / nc : rhi + 1, pn = nc > 0 ? tid % nc : 0;
        auto fetch = [&](int r, int pc, float4& sa, float4& sb, float2& y, float2& sk) {
            const int c = clo + 2 * pc, c1 = min(c + 1, chi);
            const size_t ga = (size_t)(gi0 + r) * f.W + (gj0 + c), gb = (size_t)(gi0 + r) * f.W + (gj0 + c1);
            sa = __ldg(a.G0 + ga);
            sb = __ldg(a.G0 + gb);
            y = make_float2(__ldg(a.yin + plane + ga), __ldg(a.yin + plane + gb));
            sk = make_float2(__ldg(&a.sk[plane + ga].w), __ldg(&a.sk[plane + gb].w));
        };
        float4 san, sbn;
        float2 yn, skn;
        if (rn <= rhi) fetch(rn, pn, san, sbn, yn, skn);
        if (a.tma && !(dbg & 8)) {
            mbar_wait(&bars[2], 0);
            if (edgeC || edgeR) {  // out-of-grid cells of Y / depth read below take their clamped cell's value
                __syncthreads();
                edge_fill<2, RW, RH, NT>(Ys, Ds, nullptr, rlo - 2, rhi + 2, clo - 3, chi + 3, rmin, rmax, cmin, cmax, tid);
            }
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();  // Y / depth complete; row buffers dead
        const float qnan = __int_as_float(0x7fffffff);
        SF_TICK();
        bool okall = true;  // every reciprocal below took rcp_fast's exact range
        {
            // rhohat plane + horizontal brightness taps on the solve region +-2 rows, +-1 cols, two
            // horizontally adjacent cells per item (8-byte aligned pairs from an even column; the taps as
            // f32x2, each lane the scalar tap order).  A pair may add one cell on either side of the
            // range: its values are never read (inputs there are in the plane / filled bands).
            const int ca = (clo - 1) & ~1, npc = (chi + 1 - ca) / 2 + 1;
            auto ld2 = [&](const float* pl, int i) { return *reinterpret_cast<const float2*>(pl + i); };
#pragma unroll 2
            SF_FOR_RECT(r, pc, rlo - 2, rhi + 2, 0, npc - 1, NT, tid) {
                const int c = ca + 2 * pc, idx = r * RW + c;
                const float2 d = ld2(Ds, idx);
                bool ok0 = true, ok1 = true;
                const float rh0 = f.is_inv ? d.x : rcp_fast(d.x, ok0), rh1 = f.is_inv ? d.y : rcp_fast(d.y, ok1);
                const bool v0 = depth_valid(d.x, f.is_inv), v1 = depth_valid(d.y, f.is_inv);
                *reinterpret_cast<float2*>(RHs + idx) = make_float2(v0 ? rh0 : qnan, v1 ? rh1 : qnan);
                okall = okall && (ok0 || !v0) && (ok1 || !v1);
                const float2 ya = ld2(Ys, idx - 2), yb = ld2(Ys, idx), yc = ld2(Ys, idx + 2);
                const float2 x0 = ya, x1 = make_float2(ya.y, yb.x), x2 = yb, x3 = make_float2(yb.y, yc.x), x4 = yc;
                *reinterpret_cast<float2*>(HG + idx) = tap2_g(x0, x1, x2, x3, x4);
                *reinterpret_cast<float2*>(HH + idx) = tap2_h(x0, x1, x2, x3, x4);
                if (r >= R && r < R + TH && r >= rmin && r <= rmax && gi0 + r >= f.fr0 && gi0 + r < f.fr1) {
                    if (c >= R && c < R + TW && c >= cmin && c <= cmax && !isfinite(yb.x)) fl |= SF_FLAG_NONFINITE;
                    if (c + 1 >= R && c + 1 < R + TW && c + 1 >= cmin && c + 1 <= cmax && !isfinite(yb.y))
                        fl |= SF_FLAG_NONFINITE;
                }
            }
        }
        if (__syncthreads_or(!okall)) {  // (never for depths in [2^-126, 2^126)): exact reciprocals
#pragma unroll 1
            SF_FOR_RECT(r, c, rlo - 2, rhi + 2, clo - 1, chi + 1, NT, tid) {
                const int idx = r * RW + c;
                const float d = Ds[idx];
                RHs[idx] = depth_valid(d, f.is_inv) ? rho_hat(d, f.is_inv) : qnan;
            }
        }
        __syncthreads();  // Y and depth planes dead: w^{k+} goes to the F planes
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int ib = (r0 + k) * RW + c0;
            *reinterpret_cast<float2*>(Fx + ib) = W[0][k];
            *reinterpret_cast<float2*>(Fy + ib) = W[1][k];
            *reinterpret_cast<float2*>(Fz + ib) = W[2][k];
        }
        __syncthreads();
        SF_TICK();
        // per-pixel LS on the solve region, two horizontally adjacent cells per iteration (the
        // arithmetic cell-paired as f32x2; a ragged last pair computes its first cell twice and
        // stores it once).  The pair's global inputs (s, ds^2, Y, rho^k) are fetched one pair ahead.
        {
#pragma unroll 1
            while (rn <= rhi) {
                const int r = rn, c = clo + 2 * pn;
                const float4 sA = san, sB = sbn;
                const float2 ycur = yn, skcur = skn;
                rn += dr + ((pn + dc >= nc) ? 1 : 0);
                pn = (pn + dc >= nc) ? pn + dc - nc : pn + dc;
                if (rn <= rhi) fetch(rn, pn, san, sbn, yn, skn);
                const bool full = c + 1 <= chi;
                const int idx = r * RW + c;  // even: 8-byte aligned pairs (reads past chi are harmless)
                auto ld2 = [&](const float* pl, int i) { return *reinterpret_cast<const float2*>(pl + i); };
                const float2 g0 = ld2(HG, idx - 2 * RW), g1 = ld2(HG, idx - RW), g2 = ld2(HG, idx),
                             g3 = ld2(HG, idx + RW), g4 = ld2(HG, idx + 2 * RW);
                const float2 h0 = ld2(HH, idx - 2 * RW), h1 = ld2(HH, idx - RW), h2 = ld2(HH, idx),
                             h3 = ld2(HH, idx + RW), h4 = ld2(HH, idx + 2 * RW);
                const float2 yh = tap2_g(g0, g1, g2, g3, g4);  // Yhat^{k+1}
                const float2 be1 = tap2_g(h0, h1, h2, h3, h4);
                const float2 be2 = tap2_h(g0, g1, g2, g3, g4);
                const float2 rc = ld2(RHs, idx), ru = ld2(RHs, idx - RW), rd = ld2(RHs, idx + RW);
                const float rl = RHs[idx - 1], rr = RHs[idx + 2];
                const bool vc0 = !isnan(rc.x), vc1 = !isnan(rc.y);
                const float2 rh = make_float2(vc0 ? rc.x : 0.0f, vc1 ? rc.y : 0.0f);
                // eq:dominant_b1 / b2 per cell (the pair's cells are each other's row neighbour)
                const float2 br1 = make_float2(pick_side(rh.x, vc0, rl, !isnan(rl), rc.y, vc1),
                                               pick_side(rh.y, vc1, rc.x, vc0, rr, !isnan(rr)));
                const float2 br2 = make_float2(pick_side(rh.x, vc0, ru.x, !isnan(ru.x), rd.x, !isnan(rd.x)),
                                               pick_side(rh.y, vc1, ru.y, !isnan(ru.y), rd.y, !isnan(rd.y)));
                const float2 d2 = make_float2(sA.w, sB.w);
                const float2 e1a[3] = {ld2(Es, idx), ld2(Es, P + idx), ld2(Es, 2 * P + idx)};
                const float2 e2a[3] = {ld2(Es, 3 * P + idx), ld2(Es, 4 * P + idx), ld2(Es, 5 * P + idx)};
                const float2 sp[3] = {make_float2(sA.x, sB.x), make_float2(sA.y, sB.y), make_float2(sA.z, sB.z)};
                float2 gh[3], m[3];
                const float2 d2r = mul2(d2, rh);
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    gh[q] = mul2(d2, fma2(e2a[q], be2, mul2(e1a[q], be1)));
                    const float2 drq = mul2(d2, fma2(e2a[q], br2, mul2(e1a[q], br1)));
                    m[q] = fma2(d2r, sp[q], drq);
                }
                const float2 cY = mul2(d2, sub2(yh, ycur));   // eq:img_cost_top
                const float2 cr = mul2(d2, sub2(rh, skcur));  // eq:invdepth_cost_top
                const float2 wp[3] = {ld2(Fx, idx), ld2(Fy, idx), ld2(Fz, idx)};
                float2 x[3];
                ls_solve3x2(gh, m, cY, cr, wp, f.g1, make_float2(vc0 ? f.g2 : 0.0f, vc1 ? f.g2 : 0.0f), f.g3, x);
                const bool bad0 = !(isfinite(x[0].x) && isfinite(x[1].x) && isfinite(x[2].x));
                const bool bad1 = full && !(isfinite(x[0].y) && isfinite(x[1].y) && isfinite(x[2].y));
                if (full) {
                    *reinterpret_cast<float2*>(Fx + idx) = x[0];
                    *reinterpret_cast<float2*>(Fy + idx) = x[1];
                    *reinterpret_cast<float2*>(Fz + idx) = x[2];
                } else {
                    Fx[idx] = x[0].x;
                    Fy[idx] = x[1].x;
                    Fz[idx] = x[2].x;
                }
                if ((bad0 || bad1) && gi0 + r >= f.fr0 && gi0 + r < f.fr1) fl |= SF_FLAG_NONFINITE;
                if (r >= R && r < R + TH) {
                    const size_t g = plane + (size_t)(gi0 + r) * f.W + (gj0 + c);
                    if (c >= R && c < R + TW) a.yout[g] = yh.x;
                    if (full && c + 1 >= R && c + 1 < R + TW) a.yout[g + 1] = yh.y;
                }
            }
        }
        // ---- S x 5x5 box (reading 13) as a register-tiled 2-D stencil: one work item = one
        // component of a 4 x 4 output block, read as an 8 x 8 window (8-byte shared loads) ->
        // horizontal 5-sums of 8 rows -> vertical 5-sums -> / 25, both passes in registers; the
        // passes ping-pong between the F planes and the e planes (dead after the solve).  In edge
        // CTAs the out-of-grid cells of the input planes are first set to their clamped in-grid cell
        // (replicate border, reading 10).
        SF_TICK();
        const bool edge = edgeC || edgeR;
        float* src[3] = {Fx, Fy, Fz};
        float* dst[3] = {Es, Es + P, Es + 2 * P};
        for (int it = 0; it < ((dbg & 512) ? 0 : S); ++it) {
            const int m = 2 * (S - 1 - it);  // output of this pass: tile + 2(S-1-it), in the grid
            const int or0 = max(R - m, rmin), or1 = min(R + TH + m - 1, rmax);
            const int oc0 = max(R - m, cmin), oc1 = min(R + TW + m - 1, cmax);
            const int bc0 = oc0 & ~3;  // 16-byte aligned output blocks
            const int nbc = (oc1 - bc0) / 4 + 1, nbr = (or1 - or0) / 4 + 1;
            __syncthreads();
            if (edge) {
                edge_fill<3, RW, RH, NT>(src[0], src[1], src[2], or0 - 2, or1 + 2, oc0 - 2, oc1 + 2, rmin, rmax, cmin, cmax, tid);
                __syncthreads();
            }
            SF_TICK();
            const int items = 3 * nbc * nbr;
#pragma unroll 1
            for (int t = tid; t < items; t += NT) {
                // Item order (bank-conflict free 16-byte shared accesses): plane-major, then strips of
                // 8 block columns, row-major inside a strip, so the 8 lanes of a quarter warp read 8
                // distinct 16-byte bank groups.
                const int nb = nbr * nbc, q = t / nb, u = t - q * nb;
                const int nfull = nbc >> 3, ufull = nbr * 8 * nfull;
                int br, bc;
                if (u < ufull) {
                    const int s8 = u / (8 * nbr), v = u - s8 * 8 * nbr;
                    br = v >> 3;
                    bc = 8 * s8 + (v & 7);
                } else {
                    const int wl = nbc - 8 * nfull, v = u - ufull;
                    br = v / wl;
                    bc = 8 * nfull + (v - br * wl);
                }
                const int r = or0 + 4 * br, c = bc0 + 4 * bc;
                const float* in = q == 0 ? src[0] : (q == 1 ? src[1] : src[2]);
                float* out = q == 0 ? dst[0] : (q == 1 ? dst[1] : dst[2]);
                // Window columns c-2 .. c+5 stay inside the plane row (c - 2 >= bc0 - 2 >= 2) or
                // run at most one cell into the next row (harmless: it only feeds unstored columns);
                // window rows are clamped (rows outside [or0-2, or1+2] only feed unstored rows).
                float2 h[8][2];  // horizontal 5-sums, column pairs (0,1) (2,3)
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const float* row = in + iclamp(r - 2 + i, 0, RH - 1) * RW + c - 2;
                    const float2 xa = *reinterpret_cast<const float2*>(row);
                    const float4 xb = *reinterpret_cast<const float4*>(row + 2);
                    const float2 xc = *reinterpret_cast<const float2*>(row + 6);
                    const float x[8] = {xa.x, xa.y, xb.x, xb.y, xb.z, xb.w, xc.x, xc.y};
                    float hs[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        hs[j] = xadd(xadd(xadd(xadd(x[j], x[j + 1]), x[j + 2]), x[j + 3]), x[j + 4]);
                    h[i][0] = make_float2(hs[0], hs[1]);
                    h[i][1] = make_float2(hs[2], hs[3]);
                }
                // vertical 5-sums (paired columns) and x / 25 (div25, paired): q = x RN(1/25),
                // q1 = fma(fma(-q, 25, x), RN(1/25), q); non-finite sums take q (= the IEEE quotient)
                const float2 y25 = make_float2(0.04f, 0.04f), m25 = make_float2(-25.0f, -25.0f);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    float o[4];
#pragma unroll
                    for (int jp = 0; jp < 2; ++jp) {
                        const float2 v =
                            add2(add2(add2(add2(h[i][jp], h[i + 1][jp]), h[i + 2][jp]), h[i + 3][jp]), h[i + 4][jp]);
                        const float2 q = mul2(v, y25);
                        const float2 q1 = fma2(fma2(q, m25, v), y25, q);
                        o[2 * jp] = isfinite(v.x) ? q1.x : q.x;
                        o[2 * jp + 1] = isfinite(v.y) ? q1.y : q.y;
                    }
                    if (r + i <= or1)
                        *reinterpret_cast<float4*>(out + (r + i) * RW + c) = make_float4(o[0], o[1], o[2], o[3]);
                }
            }
#pragma unroll
            for (int qq = 0; qq < 3; ++qq) {  // this pass's output is the next pass's input
                float* tmp = src[qq];
                src[qq] = dst[qq];
                dst[qq] = tmp;
            }
        }
        float* const Wx = src[0];
        float* const Wy = src[1];
        float* const Wz = src[2];
        __syncthreads();
        SF_TICK();
        // ---- rho fusion by the threads that hold rho^{k+} in registers, and the store of
        // the tile (w^{k+1}, rho^{k+1}): two adjacent cells per thread per row, coalesced
        const float kap = f.kappa;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int r = r0 + k;
            if (r >= R && r < R + TH && r >= rmin && r <= rmax && c0 >= R && c0 < R + TW && c0 >= cmin &&
                c0 <= cmax) {
                const int idx = r * RW + c0;
                const float2 wx = *reinterpret_cast<const float2*>(Wx + idx);
                const float2 wy2 = *reinterpret_cast<const float2*>(Wy + idx);
                const float2 wz = *reinterpret_cast<const float2*>(Wz + idx);
                const float2 rh2 = *reinterpret_cast<const float2*>(RHs + idx);
                const bool v0 = !isnan(rh2.x), v1 = !isnan(rh2.y);
                const float rn0 = xfma(v0 ? kap : 0.0f, xsub(v0 ? rh2.x : 0.0f, W[3][k].x), W[3][k].x);
                const float rn1 = xfma(v1 ? kap : 0.0f, xsub(v1 ? rh2.y : 0.0f, W[3][k].y), W[3][k].y);
                if (!(isfinite(rn0) && isfinite(rn1)) && gi0 + r >= f.fr0 && gi0 + r < f.fr1) fl |= SF_FLAG_NONFINITE;
                const size_t g = plane + (size_t)(gi0 + r) * f.W + (gj0 + c0);
                a.fout[g] = make_float4(wx.x, wy2.x, wz.x, rn0);
                if (c0 + 1 <= cmax) a.fout[g + 1] = make_float4(wx.y, wy2.y, wz.y, rn1);
            }
        }
    }
    SF_TICK();
    if (tim && tid == 0) {
        long long d[12];
        for (int i = 0; i < 12; ++i) d[i] = (i + 1 < nT_) ? T_[i + 1] - T_[i] : 0;
        printf("SFTIME %2d,%2d: %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld tot=%lld\n", blockIdx.x,
               blockIdx.y, d[0], d[1], d[2], d[3], d[4], d[5], d[6], d[7], d[8], d[9], d[10], d[11],
               T_[nT_ - 1] - T_[0]);
    }
#undef SF_TICK
    if ((dbg & 2048) && tid == 0) {
        unsigned long long t2_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2_));
        printf("SFGT %d %d %llu %llu %llu %llu %llu\n", blockIdx.x, blockIdx.y, gt0_, gt1_, t2_, gte_, gtt_);
    }
    const unsigned any = __reduce_or_sync(FULL, fl);
    if (lane == 0 && any) atomicOr(a.flags, any);
}

// ================================================================== transport-only kernel (split step)
// The prediction P1-P5 alone: M substeps on a RW x RH region with the halo R = M (rounded up to
// 4) -- the update's 2S box halo is not carried through the transport (it is recomputed by the
// update kernel, sf_update.cu, on its own tiles).  Same arithmetic and register layout as k_fused's
// transport; writes (w*, rho*) of the tile.
template <int K, int NWY, bool EREG = false>
struct TransCfg {
    static constexpr int RW = 64, RH = K * NWY, P = RW * RH, NT = 32 * NWY;
    // floats: 2 row-exchange buffers of float2 slots, 4 components (+ v with EREG)
    static constexpr int XBF = 2 * (EREG ? 5 : 4) * NWY * 2 * 32 * 2;
    static constexpr size_t SMEM = sizeof(float) * (6 * (size_t)P + XBF) + 64;  // e planes | XB | bars
};

// EREG: e1 / e2 of the lane's cells held in registers for the whole frame (transport_passes).
SF_TRACE_ARRAY(g_trace_trans);

template <int K, int NWY, int RULE, bool CLAMP, bool EREG>
__global__ void __launch_bounds__(32 * NWY, 1) k_trans(const __grid_constant__ FusedArgs a) {
    using C = TransCfg<K, NWY, EREG>;
    constexpr int RW = C::RW, RH = C::RH, P = C::P;
    extern __shared__ __align__(1024) float4 smem4[];
    float* const sm = reinterpret_cast<float*>(smem4);
    float* const Es = sm;
    float2* const XB0 = reinterpret_cast<float2*>(sm + 6 * P);
    uint64_t* const bars = reinterpret_cast<uint64_t*>(sm + 6 * P + C::XBF);
    const FrameParams& f = a.f;
    const int tid = threadIdx.x, lane = tid & 31, wy = tid >> 5;
    const int c0 = 2 * lane, r0 = K * wy;
    const int b = blockIdx.z, R = a.R, TH = a.TH, TW = a.TW;
    // Row placement: the first and last tile rows put the region flush with the grid's top / bottom
    // row (when the grid is at least RH rows tall), so that the grid border IS the region border:
    // the row pass's run-end logic then replicates there by itself (the first / last warp uses its
    // own edge row as the neighbour), no row replica is needed, and top / bottom CTAs run the
    // interior instantiation.  The tile keeps >= R rows of halo towards the grid interior.
    // Columns likewise (the column pass then replicates at lanes 0 / 31, COLFIX) when the grid is
    // at least RW wide and the right-flush origin keeps the TMA box 16-byte aligned.
    int tx, ty;
    edge_first_tile(false, tx, ty);  // (the left / right tile columns run the slower COLFIX body)
    const int ti0 = ty * TH, tj0 = tx * TW;
    const int gi0 = a.flush && f.H >= RH ? min(max(ti0 - R, 0), f.H - RH) : ti0 - R;
    const bool colfit = a.flush && f.W >= RW && (f.W & 3) == 0;
    const int gj0 = colfit ? min(max(tj0 - R, 0), f.W - RW) : tj0 - R;
    const int Rr = ti0 - gi0, Rc = tj0 - gj0;  // tile rows / columns in the region: [Rr, Rr + TH) x [Rc, Rc + TW)
    const int cmin = max(0, -gj0), cmax = min(RW - 1, f.W - 1 - gj0);
    const int rmin = max(0, -gi0), rmax = min(RH - 1, f.H - 1 - gi0);
    const bool edge = cmin > 0 || cmax < RW - 1 || rmin > 0 || rmax < RH - 1;  // block-uniform
    const size_t HW = (size_t)f.H * f.W, plane = (size_t)b * HW;
    SF_PROF_DECL(a.dbg_skip & 8192);
    SF_TRACE_BEGIN(a.dbg_skip & 16384);
#ifdef SF_DEBUG_KNOBS
    if (a.dbg_skip & 32) return;  // launch-overhead experiment
#endif
    SF_PROF();
    // ---- the update kernel's inputs Y and depth (a.Y / a.D, 16-byte aligned; null when no update
    // follows): each CTA prefetches its share of the frame into L2, so that the update kernel's
    // loads hit L2 (a hint: L2 is the point of coherence, so it may run before the wait)
    if (a.Y && tid == 0) {
        const size_t bytes = (size_t)f.B * HW * sizeof(float) & ~(size_t)15;
        const size_t ncta = (size_t)gridDim.x * gridDim.y * gridDim.z;
        const size_t cta = blockIdx.x + (size_t)gridDim.x * (blockIdx.y + (size_t)gridDim.y * blockIdx.z);
        const size_t chunk = ((bytes + ncta - 1) / ncta + 15) & ~(size_t)15, off = cta * chunk;
        if (off < bytes) {
            const unsigned n = (unsigned)min(chunk, bytes - off);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(reinterpret_cast<const char*>(a.Y) + off), "r"(n)
                         : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(reinterpret_cast<const char*>(a.D) + off), "r"(n)
                         : "memory");
        }
    }
    // ---- e planes: TMA (geometry, independent of the previous kernel) or cp.async
    if (a.tma) {
        if (tid == 0) {
            mbar_init(&bars[0], 1);
            mbar_init(&bars[1], 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
        if (tid == 0) {
            mbar_expect_tx(&bars[0], 3u * P * 4u);
            tma_load_3d(Es, &a.tmE, gj0 + SF_EPAD, gi0 + SF_EPAD, 0, &bars[0]);
            mbar_expect_tx(&bars[1], 3u * P * 4u);
            tma_load_3d(Es + 3 * P, &a.tmE, gj0 + SF_EPAD, gi0 + SF_EPAD, 3, &bars[1]);
        }
    } else {
        const int EW = sf_ew(f.W);
        const size_t EP = (size_t)EW * sf_eh(f.H);  // padded e planes: clamped cell (i, j) at (i + EPAD, j + EPAD)
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int r = r0 + k;
            const size_t gr = (size_t)(iclamp(gi0 + r, 0, f.H - 1) + SF_EPAD) * EW + SF_EPAD;
            const size_t ga = gr + iclamp(gj0 + c0, 0, f.W - 1), gb = gr + iclamp(gj0 + c0 + 1, 0, f.W - 1);
#pragma unroll
            for (int p = 0; p < 6; ++p) {
                float* dst = Es + p * P + r * RW + c0;
                cp_async4(dst, a.E + p * EP + ga);
                cp_async4(dst + 1, a.E + p * EP + gb);
            }
        }
        cp_async_commit();
    }
    // ---- own directions s -> registers (geometry), then the fields once the previous kernel is done
    float2 W[4][K];
    float2 SX[K], SY[K], SZ[K];
    float mx[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const size_t gr = (size_t)iclamp(gi0 + r0 + k, 0, f.H - 1) * f.W;
        const size_t ga = gr + iclamp(gj0 + c0, 0, f.W - 1), gb = gr + iclamp(gj0 + c0 + 1, 0, f.W - 1);
        const float4 sa = __ldg(a.G0 + ga), sb = __ldg(a.G0 + gb);
        SX[k] = make_float2(sa.x, sb.x);
        SY[k] = make_float2(sa.y, sb.y);
        SZ[k] = make_float2(sa.z, sb.z);
        mx[k] = 0.0f;
    }
    griddep_wait();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const size_t gr = (size_t)iclamp(gi0 + r0 + k, 0, f.H - 1) * f.W;
        const size_t ga = gr + iclamp(gj0 + c0, 0, f.W - 1), gb = gr + iclamp(gj0 + c0 + 1, 0, f.W - 1);
        const float4 fa = a.fin[plane + ga], fb = a.fin[plane + gb];
        W[0][k] = make_float2(fa.x, fb.x);
        W[1][k] = make_float2(fa.y, fb.y);
        W[2][k] = make_float2(fa.z, fb.z);
        W[3][k] = make_float2(fa.w, fb.w);
    }
    griddep_launch_dependents();  // the update kernel's CTAs may start their geometry loads
    const bool t0 = c0 >= Rc && c0 < Rc + TW && c0 >= cmin && c0 <= cmax;
    const bool t1 = c0 + 1 >= Rc && c0 + 1 < Rc + TW && c0 + 1 >= cmin && c0 + 1 <= cmax;
    if (a.rk) {  // rho^k of the tile cells for the update kernel (each grid cell written by one CTA)
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int r = r0 + k;
            if (r >= Rr && r < Rr + TH && r >= rmin && r <= rmax) {
                const size_t g = plane + (size_t)(gi0 + r) * f.W + (gj0 + c0);
                SF_DASSERT(!t0 || (gi0 + r >= 0 && gi0 + r < f.H && gj0 + c0 >= 0 && gj0 + c0 < f.W));
                SF_DASSERT(!t1 || (gj0 + c0 + 1 >= 0 && gj0 + c0 + 1 < f.W));
                if (t0) a.rk[g] = W[3][k].x;
                if (t1) a.rk[g + 1] = W[3][k].y;
            }
        }
    }
    SF_PROF();  // 0: prologue (s, griddep, fields)
    if (a.tma) {
        mbar_wait(&bars[0], 0);
        mbar_wait(&bars[1], 0);
    } else {
        cp_async_wait<0>();
    }
    SF_PROF();  // 1: e planes landed
#ifdef SF_DEBUG_KNOBS
    const int kdbg = a.dbg_skip;  // timing experiments: 64 = no column passes, 128 = no row passes
#else
    constexpr int kdbg = 0;
#endif
    float2 ER[EREG ? 6 : 1][K];
    if (EREG) {
#pragma unroll
        for (int q = 0; q < (EREG ? 6 : 1); ++q)
#pragma unroll
            for (int k = 0; k < K; ++k) ER[q][k] = *reinterpret_cast<const float2*>(Es + q * P + (r0 + k) * RW + c0);
    }
    const bool fixL = gj0 == 0, fixR = gj0 + RW == f.W;  // (block-uniform)
    if (f.imu)  // (the inertial stage only where it is on: it costs registers and scheduling freedom)
        transport_passes<K, NWY, RULE, CLAMP, 4, true, true, EREG, true>(f, a.M, W, SX, SY, SZ, mx, Es, XB0, lane, wy,
                                                                         cmin, cmax, rmin, rmax, kdbg, nullptr, ER,
                                                                         fixL, fixR);
    else if (edge)  // (grids narrower than the region: replica cells; a flush side by COLFIX)
        transport_passes<K, NWY, RULE, CLAMP, 4, true, false, EREG, true>(f, a.M, W, SX, SY, SZ, mx, Es, XB0, lane, wy,
                                                                          cmin, cmax, rmin, rmax, kdbg, nullptr, ER,
                                                                          fixL, fixR);
    else if (fixL || fixR || a.onebody)  // (onebody: A/B switch, interior CTAs on the same body)
        transport_passes<K, NWY, RULE, CLAMP, 4, false, false, EREG, true>(f, a.M, W, SX, SY, SZ, mx, Es, XB0, lane, wy,
                                                                           cmin, cmax, rmin, rmax, kdbg, nullptr, ER,
                                                                           fixL, fixR);
    else
        transport_passes<K, NWY, RULE, CLAMP, 4, false, false, EREG>(f, a.M, W, SX, SY, SZ, mx, Es, XB0, lane, wy,
                                                                     cmin, cmax, rmin, rmax, kdbg, nullptr, ER);
    SF_PROF();  // 2: transport
    // ---- flags from tile cells (exact at every pass; |u_hat| before the clamp) and the tile store
    unsigned fl = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int r = r0 + k;
        if (r >= Rr && r < Rr + TH && r >= rmin && r <= rmax) {
            if (t0 && gi0 + r >= f.fr0 && gi0 + r < f.fr1) {  // (R, TW even: the pair is in or out together)
                if (CLAMP) {
                    if (mx[k] > f.U) fl |= SF_FLAG_CLAMPED;
                } else if (xmul(f.dt, mx[k]) > 1.0f) {
                    fl |= SF_FLAG_CFL;
                }
            }
            const size_t g = plane + (size_t)(gi0 + r) * f.W + (gj0 + c0);
            if (t0) a.fout[g] = make_float4(W[0][k].x, W[1][k].x, W[2][k].x, W[3][k].x);
            if (t1) a.fout[g + 1] = make_float4(W[0][k].y, W[1][k].y, W[2][k].y, W[3][k].y);
        }
    }
    SF_PROF();  // 3: store
    SF_PROF_PRINT("trans");
    const unsigned any = __reduce_or_sync(FULL, fl);
    if (lane == 0 && any) atomicOr(a.flags, any);
    SF_TRACE_END(g_trace_trans, a.dslot);
}

// ================================================================== pyramid bottom level (NEXT #1)
// Fused prediction [P_[]] of the bottom level: M substeps of the 8-field transport (w, dw, rho,
// Yhat advected by the reconstructed w; readings 26-27) for one tile, fields in registers
// (cell-paired), e planes staged by TMA, deep halo R = M (rounded up to 4).  The update runs on
// the per-pass kernels (sf_passes.cu).
struct LowArgs {
    CUtensorMap tmE;   // [6][H][W] e planes, box RW x RH x 3 (valid when tma)
    int tma;
    const float4* finA;  // (dw, rho)
    const float4* finW;  // (w, Yhat)
    float4* foutA;
    float4* foutW;
    const float4* G0;
    const float* E;
    unsigned* flags;
    FrameParams f;
    int M, R, TH, TW;
};

template <int K, int NWY>
struct LowCfg {
    static constexpr int RW = 64, RH = K * NWY, P = RW * RH, NT = 32 * NWY;
    static constexpr int XBF = 8 * NWY * 2 * 32 * 2;  // floats of the (single) row-exchange buffer
    static constexpr size_t SMEM = sizeof(float) * (9 * (size_t)P + XBF) + 64;  // e | s | XB | bars
};

template <int K, int NWY, int RULE, bool CLAMP>
__global__ void __launch_bounds__(32 * NWY, 1) k_low(const __grid_constant__ LowArgs a) {
    using C = LowCfg<K, NWY>;
    constexpr int RW = C::RW, RH = C::RH, P = C::P;
    extern __shared__ __align__(1024) float4 smem4[];
    float* const sm = reinterpret_cast<float*>(smem4);
    float* const Es = sm;
    float* const Ss = sm + 6 * P;  // s.x, s.y, s.z planes
    float2* const XB0 = reinterpret_cast<float2*>(sm + 9 * P);
    uint64_t* const bars = reinterpret_cast<uint64_t*>(sm + 9 * P + C::XBF);
    const FrameParams& f = a.f;
    const int tid = threadIdx.x, lane = tid & 31, wy = tid >> 5;
    const int c0 = 2 * lane, r0 = K * wy;
    const int b = blockIdx.z, R = a.R, TH = a.TH, TW = a.TW;
    // region placement flush with the grid border where the grid is large enough (k_trans):
    // replicate by the row pass's run ends and by COLFIX, no replica cells; edge tiles first in the
    // launch order (the COLFIX CTAs are the slow ones)
    int tx, ty;
    edge_first_tile(false, tx, ty);
    const int ti0 = ty * TH, tj0 = tx * TW;
    const int gi0 = f.H >= RH ? min(max(ti0 - R, 0), f.H - RH) : ti0 - R;
    const int gj0 = (f.W >= RW && (f.W & 3) == 0) ? min(max(tj0 - R, 0), f.W - RW) : tj0 - R;
    const int Rr = ti0 - gi0, Rc = tj0 - gj0;
    const int cmin = max(0, -gj0), cmax = min(RW - 1, f.W - 1 - gj0);
    const int rmin = max(0, -gi0), rmax = min(RH - 1, f.H - 1 - gi0);
    const size_t HW = (size_t)f.H * f.W, plane = (size_t)b * HW;
    if (a.tma) {
        if (tid == 0) {
            mbar_init(&bars[0], 1);
            mbar_init(&bars[1], 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
        if (tid == 0) {
            mbar_expect_tx(&bars[0], 3u * P * 4u);
            tma_load_3d(Es, &a.tmE, gj0 + SF_EPAD, gi0 + SF_EPAD, 0, &bars[0]);
            mbar_expect_tx(&bars[1], 3u * P * 4u);
            tma_load_3d(Es + 3 * P, &a.tmE, gj0 + SF_EPAD, gi0 + SF_EPAD, 3, &bars[1]);
        }
    } else {
        const int EW = sf_ew(f.W);
        const size_t EP = (size_t)EW * sf_eh(f.H);  // padded e planes: clamped cell (i, j) at (i + EPAD, j + EPAD)
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int r = r0 + k;
            const size_t gr = (size_t)(iclamp(gi0 + r, 0, f.H - 1) + SF_EPAD) * EW + SF_EPAD;
            const size_t ga = gr + iclamp(gj0 + c0, 0, f.W - 1), gb = gr + iclamp(gj0 + c0 + 1, 0, f.W - 1);
#pragma unroll
            for (int p = 0; p < 6; ++p) {
                float* dst = Es + p * P + r * RW + c0;
                cp_async4(dst, a.E + p * EP + ga);
                cp_async4(dst + 1, a.E + p * EP + gb);
            }
        }
        cp_async_commit();
    }
    float2 W[8][K];
    float2 SX[K], SY[K], SZ[K];
    float mx[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const size_t gr = (size_t)iclamp(gi0 + r0 + k, 0, f.H - 1) * f.W;
        const size_t ga = gr + iclamp(gj0 + c0, 0, f.W - 1), gb = gr + iclamp(gj0 + c0 + 1, 0, f.W - 1);
        const float4 sa = __ldg(a.G0 + ga), sb = __ldg(a.G0 + gb);
        const int ib = (r0 + k) * RW + c0;  // own cells only: no barrier needed before the reads
        *reinterpret_cast<float2*>(Ss + ib) = make_float2(sa.x, sb.x);
        *reinterpret_cast<float2*>(Ss + P + ib) = make_float2(sa.y, sb.y);
        *reinterpret_cast<float2*>(Ss + 2 * P + ib) = make_float2(sa.z, sb.z);
        SX[k] = SY[k] = SZ[k] = make_float2(0.0f, 0.0f);  // unused (s lives in Ss)
        mx[k] = 0.0f;
    }
    griddep_wait();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const size_t gr = (size_t)iclamp(gi0 + r0 + k, 0, f.H - 1) * f.W;
        const size_t ga = plane + gr + iclamp(gj0 + c0, 0, f.W - 1), gb = plane + gr + iclamp(gj0 + c0 + 1, 0, f.W - 1);
        const float4 wa = a.finW[ga], wb = a.finW[gb], da = a.finA[ga], db = a.finA[gb];
        W[0][k] = make_float2(wa.x, wb.x);
        W[1][k] = make_float2(wa.y, wb.y);
        W[2][k] = make_float2(wa.z, wb.z);
        W[3][k] = make_float2(da.x, db.x);
        W[4][k] = make_float2(da.y, db.y);
        W[5][k] = make_float2(da.z, db.z);
        W[6][k] = make_float2(da.w, db.w);
        W[7][k] = make_float2(wa.w, wb.w);
    }
    griddep_launch_dependents();
    if (a.tma) {
        mbar_wait(&bars[0], 0);
        mbar_wait(&bars[1], 0);
    } else {
        cp_async_wait<0>();
    }
    // (replica e cells next to grid edges arrive with the load: padded E, reading 10)
    __syncthreads();
    const bool fixL = gj0 == 0, fixR = gj0 + RW == f.W;
    if (cmin > 0 || cmax < RW - 1 || rmin > 0 || rmax < RH - 1)
        transport_passes<K, NWY, RULE, CLAMP, 8, true, false, false, true>(f, a.M, W, SX, SY, SZ, mx, Es, XB0, lane, wy,
                                                                           cmin, cmax, rmin, rmax, 0, Ss, nullptr, fixL,
                                                                           fixR);
    else if (fixL || fixR)
        transport_passes<K, NWY, RULE, CLAMP, 8, false, false, false, true>(f, a.M, W, SX, SY, SZ, mx, Es, XB0, lane,
                                                                            wy, cmin, cmax, rmin, rmax, 0, Ss, nullptr,
                                                                            fixL, fixR);
    else
        transport_passes<K, NWY, RULE, CLAMP, 8, false, false>(f, a.M, W, SX, SY, SZ, mx, Es, XB0, lane, wy, cmin, cmax,
                                                               rmin, rmax, 0, Ss);
    unsigned fl = 0;
    const bool tcol = c0 >= Rc && c0 < Rc + TW && c0 >= cmin && c0 <= cmax;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int r = r0 + k;
        if (r >= Rr && r < Rr + TH && r >= rmin && r <= rmax) {
            if (tcol) {
                if (CLAMP) {
                    if (mx[k] > f.U) fl |= SF_FLAG_CLAMPED;
                } else if (xmul(f.dt, mx[k]) > 1.0f) {
                    fl |= SF_FLAG_CFL;
                }
            }
            const size_t g = plane + (size_t)(gi0 + r) * f.W + (gj0 + c0);
            if (c0 >= Rc && c0 < Rc + TW && c0 >= cmin && c0 <= cmax) {
                a.foutW[g] = make_float4(W[0][k].x, W[1][k].x, W[2][k].x, W[7][k].x);
                a.foutA[g] = make_float4(W[3][k].x, W[4][k].x, W[5][k].x, W[6][k].x);
            }
            if (c0 + 1 >= Rc && c0 + 1 < Rc + TW && c0 + 1 >= cmin && c0 + 1 <= cmax) {
                a.foutW[g + 1] = make_float4(W[0][k].y, W[1][k].y, W[2][k].y, W[7][k].y);
                a.foutA[g + 1] = make_float4(W[3][k].y, W[4][k].y, W[5][k].y, W[6][k].y);
            }
        }
    }
    const unsigned any = __reduce_or_sync(FULL, fl);
    if (lane == 0 && any) atomicOr(a.flags, any);
}

// The configuration used today: RW = 64, RH = 72 (K = 6 rows x 12 warps), 384 threads, 1 CTA / SM.
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
        int R = upd ? (p.M[l] > 2 ? p.M[l] : 2) + 2 * f.S : p.M[l];
        // multiple of 4: tile origins are 16-byte aligned columns (TMA needs the innermost start
        // coordinate x 4 bytes to be a multiple of 16; the lanes own even/odd column pairs)
        p.R[l] = (R + 3) & ~3;
    }
    return p;
}

// Region shapes (both RW = 64 x RH = 72, one CTA per SM):
//   cfg 0: K = 6 rows x 12 warps (384 threads, ~168 registers)
//   cfg 1: K = 4 rows x 18 warps (576 threads, <= 112 registers)
int fused_cfg() {
    static int cfg = -1;
    if (cfg < 0) {
        const char* e = getenv("SF_FUSED_CFG");
        cfg = (e && e[0] == '1') ? 1 : 0;
    }
    return cfg;
}

template <int K, int NWY>
bool prepare_cfg() {
    using FC = Cfg<K, NWY>;
    const void* fns[] = {(const void*)k_fused<K, NWY, SF_DOM_LARGEST, true>,
                         (const void*)k_fused<K, NWY, SF_DOM_LARGEST, false>,
                         (const void*)k_fused<K, NWY, SF_DOM_PRINTED, true>,
                         (const void*)k_fused<K, NWY, SF_DOM_PRINTED, false>};
    for (const void* fn : fns)
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FC::SMEM) != cudaSuccess)
            return false;
    return true;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// Process-wide switches read once: SF_NO_TMA (cp.async staging), SF_NO_PDL (no programmatic
// dependent launch).
bool env_flag(const char* name) { return getenv(name) != nullptr; }
bool no_tma() {
    static const bool v = env_flag("SF_NO_TMA");
    return v;
}
bool no_pdl() {
    static const bool v = env_flag("SF_NO_PDL");
    return v;
}

// 3-D fp32 tensor [d2][H][W], box RW x RH x bz.  Encodings are memoised (a few host µs each;
// the per-frame inputs alternate between a handful of buffers): a small direct-mapped cache.
bool encode3d_raw(CUtensorMap* m, const float* base, int W, int H, int d2, int RW, int RH, int bz);
bool encode3d(CUtensorMap* m, const float* base, int W, int H, int d2, int RW, int RH, int bz) {
    struct Entry {
        const float* base;
        int W, H, d2, RW, RH, bz;
        bool ok;
        CUtensorMap map;
    };
    static Entry cache[16];
    static bool valid[16];
    static std::mutex mu;  // contexts may launch from several host threads
    std::lock_guard<std::mutex> lock(mu);
    const size_t h = ((reinterpret_cast<uintptr_t>(base) >> 8) ^ (size_t)(W * 31 + H * 7 + d2 * 3 + RH + bz)) & 15;
    Entry& e = cache[h];
    if (valid[h] && e.base == base && e.W == W && e.H == H && e.d2 == d2 && e.RW == RW && e.RH == RH && e.bz == bz) {
        *m = e.map;
        return e.ok;
    }
    e.ok = encode3d_raw(&e.map, base, W, H, d2, RW, RH, bz);
    e.base = base;
    e.W = W;
    e.H = H;
    e.d2 = d2;
    e.RW = RW;
    e.RH = RH;
    e.bz = bz;
    valid[h] = true;
    *m = e.map;
    return e.ok;
}

bool encode3d_raw(CUtensorMap* m, const float* base, int W, int H, int d2, int RW, int RH, int bz) {
    EncodeTiledFn fn = encode_fn();
    if (!fn || (W & 3) || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)d2};
    const cuuint64_t strides[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4};
    const cuuint32_t box[3] = {(cuuint32_t)RW, (cuuint32_t)RH, (cuuint32_t)bz};
    const cuuint32_t es[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// TMA / PDL switches shared with sf_update.cu
bool sf_tma_encode3d(CUtensorMap* m, const float* base, int W, int H, int d2, int RW, int RH, int bz) {
    return !no_tma() && encode3d(m, base, W, H, d2, RW, RH, bz);
}
bool sf_pdl_enabled() { return !no_pdl(); }

namespace {

template <int K, int NWY>
cudaError_t launch_cfg(sf_ctx* c, const float* Y, const float* D) {
    using FC = Cfg<K, NWY>;
    const FrameParams& f = c->fp;
    const Plan p = make_plan(f);
    const float4* src = c->state[c->cur];
    float4* bufs[2] = {c->pred, c->tmp};
    for (int l = 0; l < p.launches; ++l) {
        const bool upd = l == p.launches - 1;
        FusedArgs a;
        {
            static const int dbg_env = [] {
                const char* e = getenv("SF_DEBUG_SKIP");
                return e ? atoi(e) : 0;
            }();
            a.dbg_skip = dbg_env;
        }
        a.tma = !no_tma() && encode3d(&a.tmE, c->E, sf_ew(f.W), sf_eh(f.H), 6, FC::RW, FC::RH, 3) &&
                encode3d(&a.tmY, Y, f.W, f.H, f.B, FC::RW, FC::RH, 1) &&
                encode3d(&a.tmD, D, f.W, f.H, f.B, FC::RW, FC::RH, 1);
        a.y16 = ((reinterpret_cast<uintptr_t>(Y) | reinterpret_cast<uintptr_t>(D)) & 15) == 0;
        a.fin = src;
        a.sk = c->state[c->cur];
        a.fout = upd ? c->state[1 - c->cur] : bufs[l & 1];
        a.yin = c->yhat[c->cur];
        a.yout = c->yhat[1 - c->cur];
        a.Y = Y;
        a.D = D;
        a.G0 = c->G0;
        a.G1 = c->G1;
        a.G2 = c->G2;
        a.E = c->E;
        a.flags = c->flags;
        a.f = f;
        a.M = p.M[l];
        a.upd = upd ? 1 : 0;
        a.R = p.R[l];
        a.TW = FC::RW - 2 * a.R;
        a.TH = FC::RH - 2 * a.R;
        const dim3 grid((f.W + a.TW - 1) / a.TW, (f.H + a.TH - 1) / a.TH, f.B);
        void (*kern)(FusedArgs) = f.rule == SF_DOM_PRINTED
                                      ? (f.clamp ? k_fused<K, NWY, SF_DOM_PRINTED, true> : k_fused<K, NWY, SF_DOM_PRINTED, false>)
                                      : (f.clamp ? k_fused<K, NWY, SF_DOM_LARGEST, true> : k_fused<K, NWY, SF_DOM_LARGEST, false>);
        cudaLaunchConfig_t lc = {};
        lc.gridDim = grid;
        lc.blockDim = dim3(FC::NT);
        lc.dynamicSmemBytes = FC::SMEM;
        lc.stream = c->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL
        at[0].val.programmaticStreamSerializationAllowed = no_pdl() ? 0 : 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&lc, kern, a);
        if (e == cudaSuccess) e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        src = a.fout;
    }
    return cudaSuccess;
}

// Bottom-level fused prediction: ceil(N / MMAX) launches of M <= MMAX substeps; the last one
// writes (pred, Wpred), earlier ones ping-pong through (tmp, Wtmp).
constexpr int LOW_K = 5, LOW_NWY = 12;

template <int K, int NWY>
bool prepare_low() {
    using LC = LowCfg<K, NWY>;
    const void* fns[] = {(const void*)k_low<K, NWY, SF_DOM_LARGEST, true>, (const void*)k_low<K, NWY, SF_DOM_LARGEST, false>,
                         (const void*)k_low<K, NWY, SF_DOM_PRINTED, true>, (const void*)k_low<K, NWY, SF_DOM_PRINTED, false>};
    for (const void* fn : fns)
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LC::SMEM) != cudaSuccess)
            return false;
    return true;
}

template <int K, int NWY>
cudaError_t launch_low(sf_ctx* c) {
    using LC = LowCfg<K, NWY>;
    const FrameParams& f = c->fp;
    const int L = (f.N + MMAX - 1) / MMAX;
    const float4* srcA = c->state[c->cur];
    const float4* srcW = c->Wf[c->cur];
    for (int l = 0; l < L; ++l) {
        LowArgs a;
        a.M = (l < L - 1) ? MMAX : f.N - MMAX * (L - 1);
        a.R = (a.M + 3) & ~3;
        a.TW = LC::RW - 2 * a.R;
        a.TH = LC::RH - 2 * a.R;
        a.tma = !no_tma() && encode3d(&a.tmE, c->E, sf_ew(f.W), sf_eh(f.H), 6, LC::RW, LC::RH, 3);
        a.finA = srcA;
        a.finW = srcW;
        const bool last = ((L - 1 - l) & 1) == 0;
        a.foutA = last ? c->pred : c->tmp;
        a.foutW = last ? c->Wpred : c->Wtmp;
        a.G0 = c->G0;
        a.E = c->E;
        a.flags = c->flags;
        a.f = f;
        const dim3 grid((f.W + a.TW - 1) / a.TW, (f.H + a.TH - 1) / a.TH, f.B);
        void (*kern)(LowArgs) = f.rule == SF_DOM_PRINTED
                                    ? (f.clamp ? k_low<K, NWY, SF_DOM_PRINTED, true> : k_low<K, NWY, SF_DOM_PRINTED, false>)
                                    : (f.clamp ? k_low<K, NWY, SF_DOM_LARGEST, true> : k_low<K, NWY, SF_DOM_LARGEST, false>);
        cudaLaunchConfig_t lc = {};
        lc.gridDim = grid;
        lc.blockDim = dim3(LC::NT);
        lc.dynamicSmemBytes = LC::SMEM;
        lc.stream = c->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = no_pdl() ? 0 : 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&lc, kern, a);
        if (e == cudaSuccess) e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        srcA = a.foutA;
        srcW = a.foutW;
    }
    return cudaSuccess;
}

// Split step (default): ceil(N / 8) transport launches (k_trans, halo R = M) + one update launch
// (k_upd, sf_update.cu).  SF_FUSED_MODE=mono selects the single-launch k_fused (halo M + 2S).
// SF_TRANS_CFG picks the transport region shape (rows x warps) and where e1 / e2 live: 0 = 7 x 8
// with e in registers (default), 1 = 7 x 8 with e read from shared memory, 2 = 4 x 14 (shared) --
// all 64 x 56 regions.
bool fused_mono() {
    static const bool v = [] {
        const char* e = getenv("SF_FUSED_MODE");
        return e && e[0] == 'm';
    }();
    return v;
}
int trans_cfg() {
    static const int v = [] {
        const char* e = getenv("SF_TRANS_CFG");
        return e ? atoi(e) : 0;
    }();
    return v;
}

template <int K, int NWY, bool EREG>
bool prepare_trans() {
    using TC = TransCfg<K, NWY, EREG>;
    const void* fns[] = {(const void*)k_trans<K, NWY, SF_DOM_LARGEST, true, EREG>,
                         (const void*)k_trans<K, NWY, SF_DOM_LARGEST, false, EREG>,
                         (const void*)k_trans<K, NWY, SF_DOM_PRINTED, true, EREG>,
                         (const void*)k_trans<K, NWY, SF_DOM_PRINTED, false, EREG>};
    for (const void* fn : fns)
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TC::SMEM) != cudaSuccess)
            return false;
    return true;
}

// Transport launches l = 0..L-1 (M <= 8 substeps each, halo R = M rounded up to 4); the last one
// writes c->pred, earlier ones alternate through c->tmp / c->tmp2.
template <int K, int NWY, bool EREG>
cudaError_t launch_trans(sf_ctx* c, const float* Y, const float* D) {
    using TC = TransCfg<K, NWY, EREG>;
    const FrameParams& f = c->fp;
    const int L = (f.N + MMAX - 1) / MMAX;
    const float4* src = c->state[c->cur];
    for (int l = 0; l < L; ++l) {
        FusedArgs a;
        memset(&a, 0, sizeof(a));
        a.M = (l < L - 1) ? MMAX : f.N - MMAX * (L - 1);
        a.R = (a.M + 3) & ~3;
        a.TW = TC::RW - 2 * a.R;
        a.TH = TC::RH - 2 * a.R;
        a.tma = !no_tma() && encode3d(&a.tmE, c->E, sf_ew(f.W), sf_eh(f.H), 6, TC::RW, TC::RH, 3);
        a.flush = getenv("SF_NO_FLUSH") ? 0 : 1;  // (A/B switches)
        a.onebody = getenv("SF_ONEBODY") ? 1 : 0;
        a.fin = src;
        a.fout = (l == L - 1) ? c->pred : (((L - 1 - l) & 1) ? c->tmp : c->tmp2);
        const bool pf = l == 0 && Y && D && ((reinterpret_cast<uintptr_t>(Y) | reinterpret_cast<uintptr_t>(D)) & 15) == 0;
        a.Y = pf ? Y : nullptr;  // L2 prefetch of the update's inputs by the first launch
        a.D = pf ? D : nullptr;
        a.rk = l == 0 ? c->rk : nullptr;  // (state k is read by the first launch only)
        a.dslot = c->dbg_frame;
        a.G0 = c->G0;
        a.E = c->E;
        a.flags = c->flags;
        a.f = f;
        {
            static const int dbg_env = [] {
                const char* e = getenv("SF_DEBUG_SKIP");
                return e ? atoi(e) : 0;
            }();
            a.dbg_skip = dbg_env;
        }
        const dim3 grid((f.W + a.TW - 1) / a.TW, (f.H + a.TH - 1) / a.TH, f.B);
        void (*kern)(FusedArgs) =
            f.rule == SF_DOM_PRINTED
                ? (f.clamp ? k_trans<K, NWY, SF_DOM_PRINTED, true, EREG> : k_trans<K, NWY, SF_DOM_PRINTED, false, EREG>)
                : (f.clamp ? k_trans<K, NWY, SF_DOM_LARGEST, true, EREG> : k_trans<K, NWY, SF_DOM_LARGEST, false, EREG>);
        cudaLaunchConfig_t lc = {};
        lc.gridDim = grid;
        lc.blockDim = dim3(TC::NT);
        lc.dynamicSmemBytes = TC::SMEM;
        lc.stream = c->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = no_pdl() ? 0 : 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&lc, kern, a);
        if (e == cudaSuccess) e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        src = a.fout;
    }
    return cudaSuccess;
}

}  // namespace

bool sf_fused_supported(const sf_ctx* c) {
    // (sf_predict / sf_update on a fused context run k_trans / k_upd in either mode)
    if ((c->fp.N + MMAX - 1) / MMAX > 8 || !sf_update_fused_supported(c)) return false;
    bool ok;
    switch (trans_cfg()) {
        case 1: ok = prepare_trans<7, 8, false>(); break;
        case 2: ok = prepare_trans<4, 14, false>(); break;
        default: ok = prepare_trans<7, 8, true>(); break;
    }
    if (!ok || !fused_mono()) return ok;
    const Plan p = make_plan(c->fp);
    for (int l = 0; l < p.launches; ++l)
        if (64 - 2 * p.R[l] < 8 || 72 - 2 * p.R[l] < 8) return false;
    // opt in to the large dynamic shared-memory carve-out (one CTA per SM)
    return fused_cfg() == 1 ? prepare_cfg<4, 18>() : prepare_cfg<6, 12>();
}

int sf_fused_launches(const sf_ctx* c) {
    if (fused_mono()) return make_plan(c->fp).launches;
    return (c->fp.N + MMAX - 1) / MMAX + 1;
}

// The prediction alone (k_trans launches) into c->pred: sf_predict on the fused path.  Y / D
// (nullable): the next update's inputs, prefetched into L2 by the transport.
cudaError_t sf_launch_predict_fused(sf_ctx* c, const float* Y, const float* D) {
    switch (trans_cfg()) {
        case 1: return launch_trans<7, 8, false>(c, Y, D);
        case 2: return launch_trans<4, 14, false>(c, Y, D);
        default: return launch_trans<7, 8, true>(c, Y, D);
    }
}

cudaError_t sf_launch_fused_step(sf_ctx* c, const float* Y, const float* D) {
    if (fused_mono()) return fused_cfg() == 1 ? launch_cfg<4, 18>(c, Y, D) : launch_cfg<6, 12>(c, Y, D);
    cudaError_t e = sf_launch_predict_fused(c, Y, D);
    if (e != cudaSuccess) return e;
    e = sf_launch_update_fused(c, Y, D, c->pred, c->rk, 1, c->yhat[c->cur], 1, c->state[1 - c->cur],
                               c->yhat[1 - c->cur]);
    ++c->dbg_frame;
    return e;
}

bool sf_low_fused_supported(const sf_ctx* c) {
    if ((c->fp.N + MMAX - 1) / MMAX > 8) return false;
    return prepare_low<LOW_K, LOW_NWY>();
}

int sf_low_fused_launches(const sf_ctx* c) { return (c->fp.N + MMAX - 1) / MMAX; }

#ifdef SF_DEBUG_KNOBS
// Debug builds: the k_trans per-CTA timeline of trace slot `slot` (n CTAs x (entry ns, exit ns,
// by << 32 | bx << 16 | smid)).
extern "C" int sf_debug_trace_trans(int slot, unsigned long long* out, int n) {
    return cudaMemcpyFromSymbol(out, g_trace_trans, sizeof(unsigned long long) * 3 * n,
                                sizeof(unsigned long long) * 3 * 4096 * (slot & 3)) == cudaSuccess ? 0 : -1;
}
#endif

cudaError_t sf_launch_predict_low_fused(sf_ctx* c) { return launch_low<LOW_K, LOW_NWY>(c); }
