// sf_api.cu -- host side of the libsf C-ABI (include/sf.h): validation, device memory,
// state machine (fresh -> initialised -> prediction pending), dispatch to the kernels.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "sf_internal.cuh"

extern "C" void sf_config_default(sf_config* cfg, int32_t height, int32_t width) {
    memset(cfg, 0, sizeof(*cfg));
    cfg->abi_version = SF_ABI_VERSION;
    cfg->height = height;
    cfg->width = width;
    cfg->batch = 1;
    cfg->levels = 1;
    cfg->max_flow_px = 1.0f;
    for (int k = 0; k < 5; ++k) cfg->gamma[k] = 1.0f;
    cfg->smooth_iters = 2;
    cfg->dominant_rule = SF_DOM_LARGEST;
    cfg->source_weight = 0.5f;
    cfg->clamp_advection = 1;
    cfg->kernel = SF_KERNEL_AUTO;
}

static sf_status validate(const sf_config* c) {
    if (c->abi_version != SF_ABI_VERSION) return SF_E_CONFIG;
    if (c->height < 2 || c->width < 2 || c->batch < 1) return SF_E_CONFIG;
    if ((long long)c->height * c->width * c->batch > (1LL << 31)) return SF_E_CONFIG;
    if (!(c->max_flow_px > 0.0f) || !isfinite(c->max_flow_px) || c->max_flow_px > 4096.0f) return SF_E_CONFIG;
    for (int k = 0; k < 5; ++k)
        if (!(c->gamma[k] >= 0.0f) || !isfinite(c->gamma[k])) return SF_E_CONFIG;
    if (!(c->gamma[2] > 0.0f) || !(c->gamma[3] + c->gamma[4] > 0.0f)) return SF_E_CONFIG;
    if (c->smooth_iters < 0 || c->smooth_iters > 64) return SF_E_CONFIG;
    if (c->dominant_rule != SF_DOM_LARGEST && c->dominant_rule != SF_DOM_PRINTED) return SF_E_CONFIG;
    if (!(c->source_weight >= 0.0f) || !isfinite(c->source_weight)) return SF_E_CONFIG;
    if (c->kernel < SF_KERNEL_AUTO || c->kernel > SF_KERNEL_PASSES) return SF_E_CONFIG;
    if (c->band_own_end != 0) {  // banded mode
        const int gh = c->global_height;
        if (c->band_ext_begin < 0 || c->band_ext_begin > c->band_own_begin || c->band_own_begin >= c->band_own_end ||
            c->band_own_end > c->band_ext_begin + c->height || c->band_ext_begin + c->height > gh)
            return SF_E_CONFIG;
    } else if (c->band_ext_begin != 0 || c->band_own_begin != 0 || (c->global_height != 0 && c->global_height != c->height)) {
        return SF_E_CONFIG;
    }
    if (c->levels == 2) {
        if ((c->height & 1) || (c->width & 1) || c->height < 4 || c->width < 4) return SF_E_CONFIG;
        if (c->smooth_iters_top < 0 || c->smooth_iters_top > 64) return SF_E_CONFIG;
        if (c->band_own_end != 0) return SF_E_UNSUPPORTED;
    } else if (c->levels != 1) {
        return SF_E_UNSUPPORTED;
    }
    return SF_OK;
}

static void async_teardown(sf_ctx* c);

static void free_ctx(sf_ctx* c) {
    if (!c) return;
    void* ptrs[] = {c->G0, c->G1, c->G2, c->E, c->state[0], c->state[1], c->pred, c->tmp, c->tmp2,
                    c->yhat[0], c->yhat[1], c->HG, c->HH, c->rk, c->flags, c->hY, c->hD, c->hw, c->hr, c->eval_part,
                    c->Wf[0], c->Wf[1], c->Wpred, c->Wtmp, c->Y2, c->D2, c->mY, c->mD};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (c->top) {
        cudaStreamSynchronize(c->top->stream);
        free_ctx(c->top);
    }
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->xstream) {
        cudaStreamSynchronize(c->xstream);
        cudaStreamDestroy(c->xstream);
    }
    if (c->xev[0]) cudaEventDestroy(c->xev[0]);
    if (c->xev[1]) cudaEventDestroy(c->xev[1]);
    if (c->xhost) cudaFreeHost(c->xhost);
    if (c->async_ready) {
        cudaStreamSynchronize(c->s_in);
        cudaStreamSynchronize(c->s_out);
        async_teardown(c);
    }
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    free(c);
}

// Pyramid (levels == 2): bottom-level buffers and the top-level H = 1 context on the half grid
// (geometry level 2 follows level 1 in `geometry`).  Per-level parameters: DESIGN reading 29.
static sf_status create_top(sf_ctx* c, const sf_config* cfg, const float* geometry) {
    const FrameParams& f = c->fp;
    const int Hc = f.H / 2, Wc = f.W / 2;
    const size_t nall = (size_t)f.H * f.W * f.B, ncoarse = (size_t)Hc * Wc * f.B;
    bool ok = cudaMalloc(&c->Wf[0], nall * sizeof(float4)) == cudaSuccess &&
              cudaMalloc(&c->Wf[1], nall * sizeof(float4)) == cudaSuccess &&
              cudaMalloc(&c->Wpred, nall * sizeof(float4)) == cudaSuccess &&
              cudaMalloc(&c->Wtmp, nall * sizeof(float4)) == cudaSuccess &&
              cudaMalloc(&c->Y2, ncoarse * sizeof(float)) == cudaSuccess &&
              cudaMalloc(&c->D2, ncoarse * sizeof(float)) == cudaSuccess &&
              cudaMemsetAsync(c->Wf[0], 0, nall * sizeof(float4), c->stream) == cudaSuccess;
    if (!ok) return SF_E_CUDA;
    const float* g2 = geometry + (size_t)f.H * f.W * 10;
    float ds1 = 0.0f, ds2 = 0.0f;  // centre pixel separations (host or device geometry)
    if (cudaMemcpy(&ds1, geometry + ((size_t)(f.H / 2) * f.W + f.W / 2) * 10 + 9, sizeof(float), cudaMemcpyDefault) !=
            cudaSuccess ||
        cudaMemcpy(&ds2, g2 + ((size_t)(Hc / 2) * Wc + Wc / 2) * 10 + 9, sizeof(float), cudaMemcpyDefault) != cudaSuccess)
        return SF_E_CUDA;
    if (!(ds1 > 0.0f) || !(ds2 > 0.0f)) return SF_E_DATA;
    sf_config t = *cfg;
    t.levels = 1;
    t.height = Hc;
    t.width = Wc;
    t.max_flow_px = cfg->max_flow_px * 0.5f;
    t.smooth_iters = cfg->smooth_iters_top > 0 ? cfg->smooth_iters_top : 4;
    t.smooth_iters_top = 0;
    const double r = (double)ds1 / (double)ds2, r2 = r * r;
    t.gamma[0] = (float)((double)cfg->gamma[0] * r2);
    t.gamma[1] = (float)((double)cfg->gamma[1] * r2);
    t.stream = nullptr;  // own stream: the top level overlaps the bottom-level prediction
    if (cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess)
        return SF_E_CUDA;
    return sf_create(&t, g2, &c->top);
}

extern "C" sf_status sf_create(const sf_config* cfg, const float* geometry, sf_ctx** out) {
    SF_NVTX("sf_create");
    if (!cfg || !out) return SF_E_DATA;
    *out = nullptr;
    sf_status st = validate(cfg);
    if (st != SF_OK) return st;
    if (!geometry) return SF_E_DATA;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || cfg->device < 0 || cfg->device >= ndev) return SF_E_CUDA;
    SfDeviceGuard guard(cfg->device);  // the caller's current device is restored on return
    sf_ctx* c = (sf_ctx*)calloc(1, sizeof(sf_ctx));
    if (!c) return SF_E_CUDA;
    c->cfg = *cfg;
    c->device = cfg->device;
    FrameParams& f = c->fp;
    f.H = cfg->height;
    f.W = cfg->width;
    f.B = cfg->batch;
    f.N = (int)ceilf(cfg->max_flow_px);
    if (f.N < 1) f.N = 1;
    f.S = cfg->smooth_iters;
    f.rule = cfg->dominant_rule;
    f.clamp = cfg->clamp_advection ? 1 : 0;
    f.is_inv = cfg->input_is_inverse_depth ? 1 : 0;
    f.U = cfg->max_flow_px;
    f.dt = 1.0f / (float)f.N;
    f.sigma = cfg->source_weight;
    f.g1 = cfg->gamma[0];
    f.g2 = cfg->gamma[1];
    f.g3 = cfg->gamma[2];
    {
        volatile float g45 = cfg->gamma[3] + cfg->gamma[4];  // float32 sum, then IEEE division
        f.kappa = cfg->gamma[3] / g45;
    }
    if (cfg->band_own_end != 0) {
        c->ext_begin = cfg->band_ext_begin;
        c->own_begin = cfg->band_own_begin;
        c->own_end = cfg->band_own_end;
        c->global_h = cfg->global_height;
    } else {
        c->ext_begin = 0;
        c->own_begin = 0;
        c->own_end = f.H;
        c->global_h = f.H;
    }
    f.fr0 = c->own_begin - c->ext_begin;
    f.fr1 = c->own_end - c->ext_begin;
    if (cfg->stream) {
        c->stream = (cudaStream_t)cfg->stream;
    } else {
        if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
            free_ctx(c);
            return SF_E_CUDA;
        }
        c->own_stream = true;
    }
    const size_t npix = (size_t)f.H * f.W, nall = npix * f.B;
    bool ok = cudaMalloc(&c->G0, npix * sizeof(float4)) == cudaSuccess &&
              cudaMalloc(&c->G1, npix * sizeof(float4)) == cudaSuccess &&
              cudaMalloc(&c->G2, npix * sizeof(float4)) == cudaSuccess &&
              cudaMalloc(&c->E, 6 * (size_t)sf_ew(f.W) * sf_eh(f.H) * sizeof(float)) == cudaSuccess &&
              cudaMalloc(&c->state[0], nall * sizeof(float4)) == cudaSuccess &&
              cudaMalloc(&c->state[1], nall * sizeof(float4)) == cudaSuccess &&
              cudaMalloc(&c->pred, nall * sizeof(float4)) == cudaSuccess &&
              cudaMalloc(&c->tmp, nall * sizeof(float4)) == cudaSuccess &&
              cudaMalloc(&c->tmp2, nall * sizeof(float4)) == cudaSuccess &&
              cudaMalloc(&c->yhat[0], nall * sizeof(float)) == cudaSuccess &&
              cudaMalloc(&c->yhat[1], nall * sizeof(float)) == cudaSuccess &&
              cudaMalloc(&c->HG, nall * sizeof(float)) == cudaSuccess &&
              cudaMalloc(&c->HH, nall * sizeof(float)) == cudaSuccess &&
              cudaMalloc(&c->rk, nall * sizeof(float)) == cudaSuccess &&
              cudaMalloc(&c->flags, sizeof(unsigned)) == cudaSuccess;
    if (!ok) {
        free_ctx(c);
        return SF_E_CUDA;
    }
    // geometry: host or device pointer
    cudaPointerAttributes attr;
    const float* gsrc = geometry;
    float* gtmp = nullptr;
    if (cudaPointerGetAttributes(&attr, geometry) != cudaSuccess || attr.type != cudaMemoryTypeDevice) {
        cudaGetLastError();
        if (cudaMalloc(&gtmp, npix * 10 * sizeof(float)) != cudaSuccess ||
            cudaMemcpy(gtmp, geometry, npix * 10 * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess) {
            if (gtmp) cudaFree(gtmp);
            free_ctx(c);
            return SF_E_CUDA;
        }
        gsrc = gtmp;
    }
    ok = cudaMemsetAsync(c->flags, 0, sizeof(unsigned), c->stream) == cudaSuccess &&
         cudaMemsetAsync(c->state[0], 0, nall * sizeof(float4), c->stream) == cudaSuccess &&
         cudaMemsetAsync(c->yhat[0], 0, nall * sizeof(float), c->stream) == cudaSuccess &&
         sf_launch_geometry(c, gsrc) == cudaSuccess && cudaStreamSynchronize(c->stream) == cudaSuccess;
    if (gtmp) cudaFree(gtmp);
    if (!ok) {
        free_ctx(c);
        return SF_E_CUDA;
    }
    c->levels = cfg->levels;
    if (c->levels == 2) {
        st = create_top(c, cfg, geometry);
        if (st != SF_OK) {
            free_ctx(c);
            return st;
        }
        // bottom level: fused prediction unless the pass kernels are requested; update on passes
        c->low_fused = cfg->kernel != SF_KERNEL_PASSES && sf_low_fused_supported(c);
        // the bottom-level update [dU] by the tiled k_upd (default), launched after the top level has
        // joined (with the reconstruction in its store stage), or by the per-pass kernels
        // (SF_UPD_LOW_PASSES=1): 51.6 vs 52.2 us/frame at 512^2, 8 px
        c->upd_fused = cfg->kernel != SF_KERNEL_PASSES && !getenv("SF_UPD_LOW_PASSES") && sf_update_fused_supported(c);
        c->kernel = c->low_fused ? SF_KERNEL_FUSED : SF_KERNEL_PASSES;
        *out = c;
        return SF_OK;
    }
    c->kernel = (cfg->kernel != SF_KERNEL_PASSES && sf_fused_supported(c)) ? SF_KERNEL_FUSED : SF_KERNEL_PASSES;
    if (cfg->kernel == SF_KERNEL_FUSED && c->kernel != SF_KERNEL_FUSED) {
        free_ctx(c);
        return SF_E_UNSUPPORTED;
    }
    *out = c;
    return SF_OK;
}

extern "C" void sf_destroy(sf_ctx* c) {
    SF_NVTX("sf_destroy");
    if (!c) return;
    SF_DEVICE_GUARD(c);
    cudaStreamSynchronize(c->stream);
    free_ctx(c);
}

extern "C" sf_status sf_predict(sf_ctx* c) {
    SF_NVTX("sf_predict");
    if (!c) return SF_E_DATA;
    SF_DEVICE_GUARD(c);
    if (c->levels == 2) return SF_E_UNSUPPORTED;
    if (!c->initialized || c->pending) return SF_E_STATE;
    SF_TRY(c->kernel == SF_KERNEL_FUSED ? sf_launch_predict_fused(c) : sf_launch_predict_passes(c));
    c->pending = true;
    return SF_OK;
}

extern "C" sf_status sf_update(sf_ctx* c, const float* Y, const float* D) {
    SF_NVTX("sf_update");
    if (!c || !Y || !D) return SF_E_DATA;
    SF_DEVICE_GUARD(c);
    if (c->levels == 2) return SF_E_UNSUPPORTED;
    if (!c->initialized) {
        SF_TRY(sf_launch_update_passes(c, Y, D, true));
        c->initialized = true;
        return SF_OK;
    }
    if (!c->pending) return SF_E_STATE;
    if (c->kernel == SF_KERNEL_FUSED)
        SF_TRY(sf_launch_update_fused(c, Y, D, c->pred, c->rk, 1, c->yhat[c->cur], 1, c->state[1 - c->cur],
                                      c->yhat[1 - c->cur]));  // (rho^k: written by sf_predict's k_trans)
    else
        SF_TRY(sf_launch_update_passes(c, Y, D, false));
    c->cur = 1 - c->cur;
    c->pending = false;
    return SF_OK;
}

// One frame of the two-level filter (Fig. 3): top level on the down-sampled inputs, bottom
// level predict [P_[]] + update [dU], reconstruction [R] with the new top flow.
// The top level (down-sampling + H = 1 step) runs on its own stream, forked from and joined
// back into the context stream (capturable into CUDA graphs): it only meets the bottom level at
// the reconstruction, so it overlaps the bottom-level prediction and update.
static sf_status pyr_step(sf_ctx* c, const float* Y, const float* D) {
    cudaStream_t ts = c->top->stream;
    SF_TRY(cudaEventRecord(c->ev_fork, c->stream));
    SF_TRY(cudaStreamWaitEvent(ts, c->ev_fork, 0));
    {
        cudaStream_t keep = c->stream;  // k_down2 on the top stream
        c->stream = ts;
        const cudaError_t e = sf_launch_down2(c, Y, D);
        c->stream = keep;
        SF_TRY(e);
    }
    sf_status st = sf_step(c->top, c->Y2, c->D2);
    if (st != SF_OK) return st;
    SF_TRY(cudaEventRecord(c->ev_join, ts));
    const bool init = !c->initialized;
    // the reconstruction rides on the bottom update's last box pass where there is one (one kernel
    // and one hand-off less on the bottom chain, the frame's critical path); else k_up2_add
    static const bool separate = getenv("SF_PYR_UP2_SEPARATE") != nullptr;  // (A/B switch)
    const bool fuse = !init && sf_update_low_defers(c) && !separate;
    if (init) {
        SF_TRY(sf_launch_update_low(c, Y, D, true));
    } else {
        SF_TRY(c->low_fused ? sf_launch_predict_low_fused(c) : sf_launch_predict_low(c));
        SF_TRY(sf_launch_update_low(c, Y, D, false, fuse));
    }
    SF_TRY(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    const float4* w2 = c->top->state[c->top->cur];
    const int nxt = init ? c->cur : 1 - c->cur;
    if (fuse)
        SF_TRY(sf_launch_update_low_last(c, Y, D, w2, c->Wf[nxt]));
    else
        SF_TRY(sf_launch_up2_add(c, w2, c->state[nxt], c->yhat[0], c->Wf[nxt]));
    c->cur = nxt;
    c->initialized = true;
    return SF_OK;
}

extern "C" sf_status sf_step(sf_ctx* c, const float* Y, const float* D) {
    SF_NVTX("sf_step");
    if (!c || !Y || !D) return SF_E_DATA;
    SF_DEVICE_GUARD(c);
    if (c->levels == 2) return pyr_step(c, Y, D);
    if (!c->initialized) return sf_update(c, Y, D);
    if (c->pending) return SF_E_STATE;
    if (c->kernel == SF_KERNEL_FUSED) {
        SF_TRY(sf_launch_fused_step(c, Y, D));
        c->cur = 1 - c->cur;
        return SF_OK;
    }
    sf_status st = sf_predict(c);
    if (st != SF_OK) return st;
    return sf_update(c, Y, D);
}

extern "C" sf_status sf_step_timed(sf_ctx* c, const float* Y, const float* D, float* ms_predict, float* ms_update) {
    SF_NVTX("sf_step_timed");
    if (!c || !Y || !D || !ms_predict || !ms_update) return SF_E_DATA;
    SF_DEVICE_GUARD(c);
    if (c->levels == 2 || c->kernel != SF_KERNEL_FUSED) return SF_E_UNSUPPORTED;
    if (!c->initialized || c->pending) return SF_E_STATE;
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
    sf_status st = SF_OK;
    for (int i = 0; i < 3 && st == SF_OK; ++i)
        if (cudaEventCreate(&ev[i]) != cudaSuccess) st = SF_E_CUDA;
    // (a 100 us device spin first: the launches below are queued before the GPU reaches them, so the
    // events time the kernels and not the host's launch latency)
    if (st == SF_OK &&
        (sf_launch_spin(c, 100000) != cudaSuccess || cudaEventRecord(ev[0], c->stream) != cudaSuccess ||
         sf_launch_predict_fused(c, Y, D) != cudaSuccess ||
         cudaEventRecord(ev[1], c->stream) != cudaSuccess ||
         sf_launch_update_fused(c, Y, D, c->pred, c->rk, 1, c->yhat[c->cur], 1, c->state[1 - c->cur],
                                c->yhat[1 - c->cur]) != cudaSuccess ||
         cudaEventRecord(ev[2], c->stream) != cudaSuccess || cudaEventSynchronize(ev[2]) != cudaSuccess ||
         cudaEventElapsedTime(ms_predict, ev[0], ev[1]) != cudaSuccess ||
         cudaEventElapsedTime(ms_update, ev[1], ev[2]) != cudaSuccess))
        st = SF_E_CUDA;
    if (st == SF_OK) c->cur = 1 - c->cur;
    for (int i = 0; i < 3; ++i)
        if (ev[i]) cudaEventDestroy(ev[i]);
    return st;
}

extern "C" sf_status sf_kernel_times(sf_ctx* c, const float* Y, const float* D, int32_t reps, float* ms_predict,
                                     float* ms_update) {
    SF_NVTX("sf_kernel_times");
    if (!c || !Y || !D || !ms_predict || !ms_update || reps < 1 || reps > 1000) return SF_E_DATA;
    SF_DEVICE_GUARD(c);
    if (c->levels == 2 || c->kernel != SF_KERNEL_FUSED) return SF_E_UNSUPPORTED;
    if (!c->initialized || c->pending) return SF_E_STATE;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    sf_status st = SF_OK;
    for (int i = 0; i < 4 && st == SF_OK; ++i)
        if (cudaEventCreate(&ev[i]) != cudaSuccess) st = SF_E_CUDA;
    bool ok = st == SF_OK && sf_launch_spin(c, 100000) == cudaSuccess && cudaEventRecord(ev[0], c->stream) == cudaSuccess;
    for (int r = 0; ok && r < reps; ++r) ok = sf_launch_predict_fused(c, Y, D) == cudaSuccess;
    ok = ok && cudaEventRecord(ev[1], c->stream) == cudaSuccess && cudaEventRecord(ev[2], c->stream) == cudaSuccess;
    for (int r = 0; ok && r < reps; ++r)
        ok = sf_launch_update_fused(c, Y, D, c->pred, c->rk, 1, c->yhat[c->cur], 1, c->state[1 - c->cur],
                                    c->yhat[1 - c->cur]) == cudaSuccess;
    ok = ok && cudaEventRecord(ev[3], c->stream) == cudaSuccess && cudaEventSynchronize(ev[3]) == cudaSuccess &&
         cudaEventElapsedTime(ms_predict, ev[0], ev[1]) == cudaSuccess &&
         cudaEventElapsedTime(ms_update, ev[2], ev[3]) == cudaSuccess;
    if (st == SF_OK && !ok) st = SF_E_CUDA;
    if (st == SF_OK) {
        *ms_predict /= (float)reps;
        *ms_update /= (float)reps;
        c->cur = 1 - c->cur;
    }
    for (int i = 0; i < 4; ++i)
        if (ev[i]) cudaEventDestroy(ev[i]);
    return st;
}

extern "C" sf_status sf_step_host(sf_ctx* c, const float* Yh, const float* Dh, float* wh, float* rh) {
    SF_NVTX("sf_step_host");
    if (!c || !Yh || !Dh) return SF_E_DATA;
    SF_DEVICE_GUARD(c);
    const size_t n = (size_t)c->fp.B * c->fp.H * c->fp.W;
    if (!c->hY) {  // staging buffers, committed only when all four allocations succeed
        float* b[4] = {nullptr, nullptr, nullptr, nullptr};
        const size_t sz[4] = {n, n, 3 * n, n};
        for (int i = 0; i < 4; ++i)
            if (cudaMalloc(&b[i], sz[i] * sizeof(float)) != cudaSuccess) {
                for (int j = 0; j < 4; ++j)
                    if (b[j]) cudaFree(b[j]);
                return SF_E_CUDA;
            }
        c->hY = b[0];
        c->hD = b[1];
        c->hw = b[2];
        c->hr = b[3];
    }
    SF_TRY(cudaMemcpyAsync(c->hY, Yh, n * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    SF_TRY(cudaMemcpyAsync(c->hD, Dh, n * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    sf_status st = sf_step(c, c->hY, c->hD);
    if (st != SF_OK) return st;
    if (wh || rh) {
        if (c->levels == 2)
            SF_TRY(sf_launch_unpack_pyr(c, wh ? c->hw : nullptr, rh ? c->hr : nullptr, nullptr));
        else
            SF_TRY(sf_launch_unpack(c, c->state[c->cur], wh ? c->hw : nullptr, rh ? c->hr : nullptr));
        if (wh) SF_TRY(cudaMemcpyAsync(wh, c->hw, 3 * n * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
        if (rh) SF_TRY(cudaMemcpyAsync(rh, c->hr, n * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    }
    SF_TRY(cudaStreamSynchronize(c->stream));
    return SF_OK;
}

// Pipelined host-buffer frames: frame k's input copies (stream s_in), step + unpack (the
// context stream) and output copies (stream s_out) overlap frame k-1's output copies and
// frame k+1's input copies; slot k % 2 holds the device staging of frame k.
static void async_teardown(sf_ctx* c) {
    for (int i = 0; i < 2; ++i) {
        if (c->aY[i]) cudaFree(c->aY[i]);
        if (c->aD[i]) cudaFree(c->aD[i]);
        if (c->aw[i]) cudaFree(c->aw[i]);
        if (c->ar[i]) cudaFree(c->ar[i]);
        if (c->ev_in[i]) cudaEventDestroy(c->ev_in[i]);
        if (c->ev_done[i]) cudaEventDestroy(c->ev_done[i]);
        if (c->ev_out[i]) cudaEventDestroy(c->ev_out[i]);
        c->aY[i] = c->aD[i] = c->aw[i] = c->ar[i] = nullptr;
        c->ev_in[i] = c->ev_done[i] = c->ev_out[i] = nullptr;
    }
    if (c->s_in) cudaStreamDestroy(c->s_in);
    if (c->s_out) cudaStreamDestroy(c->s_out);
    c->s_in = c->s_out = nullptr;
}

static sf_status async_setup(sf_ctx* c) {
    const size_t n = (size_t)c->fp.B * c->fp.H * c->fp.W;
    bool ok = true;
    for (int i = 0; i < 2 && ok; ++i) {
        ok = cudaMalloc(&c->aY[i], n * sizeof(float)) == cudaSuccess && cudaMalloc(&c->aD[i], n * sizeof(float)) == cudaSuccess &&
             cudaMalloc(&c->aw[i], 3 * n * sizeof(float)) == cudaSuccess &&
             cudaMalloc(&c->ar[i], n * sizeof(float)) == cudaSuccess &&
             cudaEventCreateWithFlags(&c->ev_in[i], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&c->ev_done[i], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&c->ev_out[i], cudaEventDisableTiming) == cudaSuccess &&
             // "previous use finished" is true initially
             cudaEventRecord(c->ev_done[i], c->stream) == cudaSuccess && cudaEventRecord(c->ev_out[i], c->stream) == cudaSuccess;
    }
    ok = ok && cudaStreamCreateWithFlags(&c->s_in, cudaStreamNonBlocking) == cudaSuccess &&
         cudaStreamCreateWithFlags(&c->s_out, cudaStreamNonBlocking) == cudaSuccess;
    if (!ok) {  // nothing half-made survives: the next call retries from scratch
        cudaStreamSynchronize(c->stream);
        async_teardown(c);
        return SF_E_CUDA;
    }
    c->async_ready = true;
    c->slot = 0;
    return SF_OK;
}

extern "C" sf_status sf_step_host_async(sf_ctx* c, const float* Yh, const float* Dh, float* wh, float* rh) {
    SF_NVTX("sf_step_host_async");
    if (!c || !Yh || !Dh) return SF_E_DATA;
    SF_DEVICE_GUARD(c);
    if (!c->async_ready) {
        sf_status st = async_setup(c);
        if (st != SF_OK) return st;
    }
    const size_t n = (size_t)c->fp.B * c->fp.H * c->fp.W;
    const int i = c->slot;
    c->slot ^= 1;
    // inputs: wait until the step that last read slot i is done, then copy in
    SF_TRY(cudaStreamWaitEvent(c->s_in, c->ev_done[i], 0));
    SF_TRY(cudaMemcpyAsync(c->aY[i], Yh, n * sizeof(float), cudaMemcpyHostToDevice, c->s_in));
    SF_TRY(cudaMemcpyAsync(c->aD[i], Dh, n * sizeof(float), cudaMemcpyHostToDevice, c->s_in));
    SF_TRY(cudaEventRecord(c->ev_in[i], c->s_in));
    // step on the context stream
    SF_TRY(cudaStreamWaitEvent(c->stream, c->ev_in[i], 0));
    sf_status st = sf_step(c, c->aY[i], c->aD[i]);
    if (st != SF_OK) return st;
    if (wh || rh) {
        SF_TRY(cudaStreamWaitEvent(c->stream, c->ev_out[i], 0));  // slot i's outputs drained
        if (c->levels == 2) {
            SF_TRY(sf_launch_unpack_pyr(c, wh ? c->aw[i] : nullptr, rh ? c->ar[i] : nullptr, nullptr));
        } else {
            SF_TRY(sf_launch_unpack(c, c->state[c->cur], wh ? c->aw[i] : nullptr, rh ? c->ar[i] : nullptr));
        }
    }
    SF_TRY(cudaEventRecord(c->ev_done[i], c->stream));
    if (wh || rh) {
        SF_TRY(cudaStreamWaitEvent(c->s_out, c->ev_done[i], 0));
        if (wh) SF_TRY(cudaMemcpyAsync(wh, c->aw[i], 3 * n * sizeof(float), cudaMemcpyDeviceToHost, c->s_out));
        if (rh) SF_TRY(cudaMemcpyAsync(rh, c->ar[i], n * sizeof(float), cudaMemcpyDeviceToHost, c->s_out));
        SF_TRY(cudaEventRecord(c->ev_out[i], c->s_out));
    }
    return SF_OK;
}

extern "C" sf_status sf_wait(sf_ctx* c) {
    SF_NVTX("sf_wait");
    if (!c) return SF_E_DATA;
    SF_DEVICE_GUARD(c);
    if (c->async_ready) {
        SF_TRY(cudaStreamSynchronize(c->s_in));
        SF_TRY(cudaStreamSynchronize(c->s_out));
    }
    SF_TRY(cudaStreamSynchronize(c->stream));
    return SF_OK;
}

extern "C" sf_status sf_get_fields(sf_ctx* c, int32_t which, float* w, float* rho, float* yhat) {
    SF_NVTX("sf_get_fields");
    if (!c) return SF_E_DATA;
    SF_DEVICE_GUARD(c);
    if (!c->initialized) return SF_E_STATE;
    const size_t n = (size_t)c->fp.B * c->fp.H * c->fp.W;
    if (c->levels == 2) {
        if (which != SF_FIELDS_STATE) return which == SF_FIELDS_PREDICTED ? SF_E_UNSUPPORTED : SF_E_CONFIG;
        SF_TRY(sf_launch_unpack_pyr(c, w, rho, yhat));
        return SF_OK;
    }
    const float4* src;
    if (which == SF_FIELDS_STATE) {
        src = c->state[c->cur];
    } else if (which == SF_FIELDS_PREDICTED) {
        if (!c->pending) return SF_E_STATE;
        src = c->pred;
    } else {
        return SF_E_CONFIG;
    }
    if (w || rho) SF_TRY(sf_launch_unpack(c, src, w, rho));
    if (yhat) SF_TRY(cudaMemcpyAsync(yhat, c->yhat[c->cur], n * sizeof(float), cudaMemcpyDeviceToDevice, c->stream));
    return SF_OK;
}

extern "C" sf_status sf_set_fields(sf_ctx* c, const float* w, const float* rho, const float* yhat) {
    SF_NVTX("sf_set_fields");
    if (!c || !w || !rho) return SF_E_DATA;
    SF_DEVICE_GUARD(c);
    if (c->levels == 2) return SF_E_UNSUPPORTED;
    const size_t n = (size_t)c->fp.B * c->fp.H * c->fp.W;
    SF_TRY(sf_launch_pack(c, w, rho, c->state[c->cur]));
    if (yhat)
        SF_TRY(cudaMemcpyAsync(c->yhat[c->cur], yhat, n * sizeof(float), cudaMemcpyDeviceToDevice, c->stream));
    else
        SF_TRY(cudaMemsetAsync(c->yhat[c->cur], 0, n * sizeof(float), c->stream));
    c->initialized = true;
    c->pending = false;
    return SF_OK;
}

extern "C" sf_status sf_status_flags(sf_ctx* c, uint32_t* flags, int32_t clear) {
    SF_NVTX("sf_status_flags");
    if (!c || !flags) return SF_E_DATA;
    SF_DEVICE_GUARD(c);
    unsigned h = 0, ht = 0;
    SF_TRY(cudaMemcpyAsync(&h, c->flags, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
    if (c->top) SF_TRY(cudaMemcpyAsync(&ht, c->top->flags, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
    SF_TRY(cudaStreamSynchronize(c->stream));
    h |= ht;
    if (clear) {
        SF_TRY(cudaMemsetAsync(c->flags, 0, sizeof(unsigned), c->stream));
        if (c->top) SF_TRY(cudaMemsetAsync(c->top->flags, 0, sizeof(unsigned), c->stream));
    }
    *flags = h;
    return (h & SF_FLAG_CFL) ? SF_E_STABILITY : SF_OK;
}

extern "C" sf_status sf_set_motion(sf_ctx* c, const float* omega, const float* accel) {
    if (!c) return SF_E_DATA;
    if (c->levels == 2) return SF_E_UNSUPPORTED;
    FrameParams& f = c->fp;
    if (!omega && !accel) {
        f.imu = 0;
        return SF_OK;
    }
    float om[3], ac[3];  // validated before anything is committed (a failure leaves the context unchanged)
    for (int k = 0; k < 3; ++k) {
        om[k] = omega ? omega[k] : 0.0f;
        ac[k] = accel ? accel[k] : 0.0f;
        if (!isfinite(om[k]) || !isfinite(ac[k])) return SF_E_CONFIG;
    }
    for (int k = 0; k < 3; ++k) {
        f.om[k] = om[k];
        f.ac[k] = ac[k];
    }
    f.imu = 1;
    return SF_OK;
}

extern "C" int32_t sf_kernel_in_use(const sf_ctx* c) { return c ? c->kernel : 0; }

extern "C" int32_t sf_launches_per_step(const sf_ctx* c) {
    if (!c) return 0;
    if (c->levels == 2)  // down2 + top + bottom prediction + update + S box + up2
        return 1 + sf_launches_per_step(c->top) + (c->low_fused ? sf_low_fused_launches(c) : 2 * c->fp.N) +
               (c->upd_fused ? 1 : 1 + c->fp.S) + 1;
    if (c->kernel == SF_KERNEL_FUSED) return sf_fused_launches(c);
    return 2 * c->fp.N + 1 + c->fp.S;
}

extern "C" const char* sf_error_string(sf_status s) {
    switch (s) {
        case SF_OK: return "ok";
        case SF_E_DATA: return "invalid pointer argument";
        case SF_E_STABILITY: return "CFL stability condition violated (clamp_advection = 0)";
        case SF_E_CONFIG: return "invalid configuration";
        case SF_E_STATE: return "call not valid in the current context state";
        case SF_E_CUDA: return "CUDA runtime error";
        case SF_E_NCCL: return "halo exchange error";
        case SF_E_UNSUPPORTED: return "unsupported configuration";
    }
    return "unknown status";
}
