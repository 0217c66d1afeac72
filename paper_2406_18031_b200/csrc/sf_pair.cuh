// sf_pair.cuh -- device helpers of the tiled kernels (sf_fused.cu, sf_update.cu): paired float32
// ops (sm_100a f32x2: FADD2 / FMUL2 / FFMA2, each lane the IEEE float32 op), cp.async / mbarrier /
// TMA / programmatic-dependent-launch wrappers, and the cell-paired update arithmetic in the
// order of DESIGN.md section 4 (each lane of a pair computes exactly sf_internal.cuh's scalar form).
#pragma once

#include <cuda.h>
#include <stdio.h>

#include "sf_internal.cuh"

namespace sfp {

// Phase profile of one CTA (debug builds, SF_BUILD_DEBUG=1, and SF_DEBUG_SKIP with bit 8192 set in
// the launch): SF_PROF() closes a phase (a CTA barrier, then thread 0 reads clock64); SF_PROF_PRINT
// prints the phase lengths in SM cycles for CTAs (0,0) and (3,3) of batch member 0.
#ifdef SF_DEBUG_KNOBS
#define SF_PROF_DECL(on) const bool prof_on_ = (on); long long prof_t_[16]; int prof_n_ = 0
#define SF_PROF()                                                                  \
    do {                                                                           \
        if (prof_on_) {                                                            \
            __syncthreads();                                                       \
            if (threadIdx.x == 0 && prof_n_ < 16) prof_t_[prof_n_] = clock64();    \
            ++prof_n_;                                                             \
        }                                                                          \
    } while (0)
#define SF_PROF_PRINT(name)                                                                                      \
    do {                                                                                                         \
        if (prof_on_ && threadIdx.x == 0 && blockIdx.z == 0 &&                                                   \
            ((blockIdx.x == 0 && blockIdx.y == 0) || (blockIdx.x == 3 && blockIdx.y == 3))) {                    \
            long long d_[15];                                                                                    \
            for (int i_ = 0; i_ < 15; ++i_) d_[i_] = (i_ + 1 < prof_n_ && i_ + 1 < 16) ? prof_t_[i_ + 1] - prof_t_[i_] : 0; \
            printf("SFPROF %s %d,%d: %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld tot=%lld\n", name, blockIdx.x, \
                   blockIdx.y, d_[0], d_[1], d_[2], d_[3], d_[4], d_[5], d_[6], d_[7], d_[8], d_[9],                 \
                   prof_t_[min(prof_n_, 16) - 1] - prof_t_[0]);                                                   \
        }                                                                                                        \
    } while (0)
#else
#define SF_PROF_DECL(on)
#define SF_PROF() do { } while (0)
#define SF_PROF_PRINT(name) do { } while (0)
#endif

// Bounds assertions of the debug builds (SF_BUILD_DEBUG=1): a failed check traps the kernel (the
// GPU suite run on a debug build stands in for compute-sanitizer where that is unavailable).
#ifdef SF_DEBUG_KNOBS
#define SF_DASSERT(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define SF_DASSERT(cond) do { } while (0)
#endif

// Per-CTA timeline (debug builds, SF_DEBUG_SKIP bit 16384): thread 0 of every CTA records the
// globaltimer at entry and exit and its SM into slot (frame & 3) of the translation unit's trace
// array (SF_TRACE_ARRAY), read back by that unit's sf_debug_trace_* export (tools/cta_trace.py).
#ifdef SF_DEBUG_KNOBS
#define SF_TRACE_ARRAY(name) __device__ unsigned long long name[4][4096][3]
#define SF_TRACE_BEGIN(on)                                                              \
    unsigned long long trace_t0_ = 0;                                                   \
    const bool trace_on_ = (on);                                                        \
    if (trace_on_ && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(trace_t0_))
#define SF_TRACE_END(arr, slot)                                                                              \
    do {                                                                                                     \
        if (trace_on_ && threadIdx.x == 0) {                                                                 \
            unsigned long long t1_;                                                                          \
            unsigned sm_;                                                                                    \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1_));                                          \
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_));                                                 \
            const unsigned cta_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);           \
            if (cta_ < 4096) {                                                                               \
                arr[(slot) & 3][cta_][0] = trace_t0_;                                                        \
                arr[(slot) & 3][cta_][1] = t1_;                                                              \
                arr[(slot) & 3][cta_][2] = ((unsigned long long)blockIdx.y << 32) | (blockIdx.x << 16) | sm_; \
            }                                                                                                \
        }                                                                                                    \
    } while (0)
#else
#define SF_TRACE_ARRAY(name)
#define SF_TRACE_BEGIN(on)
#define SF_TRACE_END(arr, slot) do { } while (0)
#endif

// Tile of this CTA in a gridDim.x x gridDim.y tile grid, edge tiles first: CTAs are dispatched in
// linear block order as SMs free up (the first ones onto idle SMs, where they run their prologue
// while the previous kernel drains), and the edge tiles are the slow ones -- so the first 2 ny
// linear indices are the left / right tile columns, then (rows_too) the top / bottom tile rows,
// then the interior in row-major order.
#ifndef SF_EDGE_FIRST
#define SF_EDGE_FIRST 1
#endif
__device__ __forceinline__ void edge_first_tile(bool rows_too, int& tx, int& ty) {
    const int nx = gridDim.x, ny = gridDim.y;
    tx = blockIdx.x;
    ty = blockIdx.y;
    if (!SF_EDGE_FIRST || nx < 3) return;
    int I = blockIdx.x + nx * blockIdx.y;
    if (I < 2 * ny) {
        tx = (I & 1) ? nx - 1 : 0;
        ty = I >> 1;
        return;
    }
    I -= 2 * ny;
    if (rows_too && ny >= 3) {
        if (I < 2 * (nx - 2)) {
            tx = 1 + (I >> 1);
            ty = (I & 1) ? ny - 1 : 0;
            return;
        }
        I -= 2 * (nx - 2);
        tx = 1 + I % (nx - 2);
        ty = 1 + I / (nx - 2);
        return;
    }
    tx = 1 + I % (nx - 2);
    ty = I / (nx - 2);
}

// Iterate the cells of the rectangle [r0, r1] x [c0, c1] with NT threads, row-major, full lane
// utilisation and no per-iteration integer division.
#define SF_FOR_RECT(r, c, R0, R1, C0, C1, NT, tid)                                                  \
    for (int nc_ = (C1) - (C0) + 1, dr_ = (NT) / nc_, dc_ = (NT) % nc_, r = (R0) + (tid) / nc_,   \
             c = (C0) + (tid) % nc_;                                                             \
         nc_ > 0 && r <= (R1); r += dr_ + ((c + dc_ > (C1)) ? 1 : 0), c = (c + dc_ > (C1)) ? c + dc_ - nc_ : c + dc_)

constexpr unsigned FULL = 0xffffffffu;

// ---- paired float32 ops (sm_100a f32x2; each lane op is the IEEE float32 op)
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
        : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
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

__device__ __forceinline__ void cp_async4(float* sdst, const float* gsrc) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gsrc));
}
__device__ __forceinline__ void cp_async8(float* sdst, const float* gsrc) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc));
}
__device__ __forceinline__ void cp_async16(float* sdst, const float* gsrc) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---- programmatic dependent launch (griddepcontrol; no-ops without the launch attribute)
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;\n" ::); }

// ---- mbarrier + TMA (cp.async.bulk.tensor) helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::
            "r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}


// Cell-paired helpers: every float2 holds one quantity of the thread's two cells (cell 0, cell 1),
// so the per-cell arithmetic runs as f32x2 ops with no operand regrouping.
// dot2 = fma(az, z, fma(ay, y, ax x)) per cell (the order of xdot3).
__device__ __forceinline__ float2 dot2(float2 ax, float2 ay, float2 az, float2 x, float2 y, float2 z) {
    return fma2(az, z, fma2(ay, y, mul2(ax, x)));
}
// f* = fma(-dt, fma(|u_hat|, f - f_up, f q), f) per cell -- equal (up to the sign of a zero) to the
// literal fma(-dt, fma(u_hat, D, f q), f) with D the upwind difference, because
// |u_hat| (f - f_up) and u_hat D are the same exact product.
__device__ __forceinline__ float2 tr2(float2 v, float2 fu, float2 A, float2 Q, float2 T) {
    return fma2(T, fma2(A, sub2(v, fu), mul2(v, Q)), v);
}
__device__ __forceinline__ float2 sel2(bool p0, bool p1, float2 a, float2 b) {
    return make_float2(p0 ? a.x : b.x, p1 ? a.y : b.y);
}

// Cell-paired update arithmetic (the order of sf_internal.cuh's tap_g / tap_h / ls_solve3 per
// lane of the pair; reciprocals stay scalar __frcp_rn).
__device__ __forceinline__ float2 bc2(float x) { return make_float2(x, x); }
__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }
__device__ __forceinline__ float2 tap2_g(float2 x0, float2 x1, float2 x2, float2 x3, float2 x4) {
    float2 a = mul2(bc2(SF_G0), x0);
    a = fma2(bc2(SF_G1), x1, a);
    a = fma2(bc2(SF_G2), x2, a);
    a = fma2(bc2(SF_G1), x3, a);
    return fma2(bc2(SF_G0), x4, a);
}
__device__ __forceinline__ float2 tap2_h(float2 x0, float2 x1, float2 x2, float2 x3, float2 x4) {
    float2 a = mul2(bc2(SF_H0), x0);
    a = fma2(bc2(SF_H1), x1, a);
    a = fma2(bc2(0.0f), x2, a);
    a = fma2(bc2(SF_H3), x3, a);
    return fma2(bc2(SF_H4), x4, a);
}
template <bool FAST>
__device__ __forceinline__ float2 rcp2(float2 a, bool& ok) {
    return make_float2(rcp_rn<FAST>(a.x, ok), rcp_rn<FAST>(a.y, ok));
}
template <bool FAST>
__device__ __forceinline__ void ls_solve3x2_t(const float2 g[3], const float2 m[3], float2 cY, float2 cr,
                                              const float2 wp[3], float g1, float2 g2, float g3, float2 x[3], bool& ok) {
    float2 g1g[3], g2m[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        g1g[a] = mul2(bc2(g1), g[a]);
        g2m[a] = mul2(g2, m[a]);
    }
    const float2 G3 = bc2(g3);
    const float2 A00 = add2(fma2(g2m[0], m[0], mul2(g1g[0], g[0])), G3);
    const float2 A10 = fma2(g2m[1], m[0], mul2(g1g[1], g[0]));
    const float2 A11 = add2(fma2(g2m[1], m[1], mul2(g1g[1], g[1])), G3);
    const float2 A20 = fma2(g2m[2], m[0], mul2(g1g[2], g[0]));
    const float2 A21 = fma2(g2m[2], m[1], mul2(g1g[2], g[1]));
    const float2 A22 = add2(fma2(g2m[2], m[2], mul2(g1g[2], g[2])), G3);
    float2 b[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) b[a] = fma2(neg2(g2m[a]), cr, fma2(neg2(g1g[a]), cY, mul2(G3, wp[a])));
    const float2 r0 = rcp2<FAST>(A00, ok);
    const float2 l10 = mul2(A10, r0), l20 = mul2(A20, r0);
    const float2 d1 = fma2(neg2(l10), A10, A11);
    const float2 r1 = rcp2<FAST>(d1, ok);
    const float2 t = fma2(neg2(l20), A10, A21);
    const float2 l21 = mul2(t, r1);
    const float2 dd2 = fma2(neg2(l21), t, fma2(neg2(l20), A20, A22));
    const float2 r2 = rcp2<FAST>(dd2, ok);
    const float2 y1 = fma2(neg2(l10), b[0], b[1]);
    const float2 y2 = fma2(neg2(l21), y1, fma2(neg2(l20), b[0], b[2]));
    x[2] = mul2(y2, r2);
    x[1] = fma2(neg2(l21), x[2], mul2(y1, r1));
    x[0] = fma2(neg2(l20), x[2], fma2(neg2(l10), x[1], mul2(b[0], r0)));
}
// fast reciprocals; the whole solve is redone with __frcp_rn if an input left the exact range
__device__ __forceinline__ void ls_solve3x2(const float2 g[3], const float2 m[3], float2 cY, float2 cr,
                                            const float2 wp[3], float g1, float2 g2, float g3, float2 x[3]) {
    bool ok = true;
    ls_solve3x2_t<true>(g, m, cY, cr, wp, g1, g2, g3, x, ok);
    if (!ok) ls_solve3x2_t<false>(g, m, cY, cr, wp, g1, g2, g3, x, ok);
}

}  // namespace sfp

// Host: memoised 3-D fp32 TMA descriptor [d2][H][W] with box RW x RH x bz (false when TMA is off
// (SF_NO_TMA), W % 4 != 0 or the base is not 16-byte aligned); programmatic dependent launch on?
bool sf_tma_encode3d(CUtensorMap* m, const float* base, int W, int H, int d2, int RW, int RH, int bz);
bool sf_pdl_enabled();
