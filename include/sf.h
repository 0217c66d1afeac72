/*
 * sf.h -- C-ABI of libsf, the B200 (sm_100a) structure-flow predictor-update loop.
 *
 * Method: Adarve & Mahony, "Real-time Structure Flow", arXiv 2406.18031.  Line numbers
 * below cite /root/reference/PAPER.md ("P:L"); readings of ambiguous passages are the
 * numbered rows of DESIGN.md section 3.
 *
 * The filter estimates, per Spherepix pixel, the structure flow w (3-vector, rad/frame;
 * eq:homogeneous_flow P:L194-198) and the inverse depth rho (eq:inv_depth P:L167-173)
 * recursively from brightness Y and depth lambda frames (problem statement P:L360,
 * Fig. 3a).  One context holds B independent sequences on one grid.
 *
 * Conventions (all calls):
 *  - Every call returns sf_status; SF_OK = 0.  Validation failures return synchronously
 *    and leave the context unchanged.
 *  - Field pointers are DEVICE pointers unless the name ends in _host.  Layout is C
 *    row-major float32: scalar planes [B][H][W], 3-vectors [B][H][W][3].  The caller owns
 *    every buffer it passes; libsf reads/writes them asynchronously on the context stream
 *    and the caller keeps them alive until that stream has passed the call.
 *  - Device anomalies never fail a call: they set sticky flags (SF_FLAG_*) read by
 *    sf_status_flags, the only call that synchronises the stream.
 *  - One context is single-writer; distinct contexts are independent.
 *  - Arithmetic is IEEE float32 in the fixed order of DESIGN.md section 4 (no FTZ, no
 *    implicit contraction), so results are bitwise reproducible and equal to the CPU
 *    oracle's float32 build.
 */
#ifndef SF_H
#define SF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SF_ABI_VERSION 1

typedef enum {
    SF_OK = 0,
    SF_E_DATA = 2,        /* NULL or misaligned pointer argument                        */
    SF_E_STABILITY = 3,   /* sf_status_flags: CFL violated with clamp_advection = 0     */
    SF_E_CONFIG = 4,      /* invalid sf_config field                                    */
    SF_E_STATE = 5,       /* call not valid in the context's current state              */
    SF_E_CUDA = 6,        /* a CUDA runtime call failed                                 */
    SF_E_NCCL = 7,        /* halo exchange failed (banded mode)                         */
    SF_E_UNSUPPORTED = 8  /* valid request this build does not implement (levels > 2 ...) */
} sf_status;

/* Dominant-flow rule (DESIGN reading 1). */
enum { SF_DOM_LARGEST = 0, SF_DOM_PRINTED = 1 };
/* Which fields sf_get_fields returns. */
enum { SF_FIELDS_STATE = 0, SF_FIELDS_PREDICTED = 1 };
/* Sticky device flags. */
enum {
    SF_FLAG_CLAMPED = 1u,   /* |u_hat| or |v_hat| exceeded max_flow and was clamped (reading 12) */
    SF_FLAG_NONFINITE = 2u, /* non-finite brightness input, or a non-finite solved field       */
    SF_FLAG_CFL = 4u        /* clamp_advection = 0 and dt*|u_hat| > 1 (eq:numerical_stability)  */
};
/* Kernel strategy. */
enum {
    SF_KERNEL_AUTO = 0,   /* fused when available for the configuration, else passes     */
    SF_KERNEL_FUSED = 1,  /* one on-chip kernel per frame (predict + update)             */
    SF_KERNEL_PASSES = 2  /* one kernel per pass / stage (2N + 1 + S launches per frame)  */
};

typedef struct sf_ctx sf_ctx; /* opaque; owns all device state */

typedef struct {
    int32_t abi_version;            /* == SF_ABI_VERSION                                              */
    int32_t height, width;          /* grid H x W, each >= 2                                          */
    int32_t batch;                  /* B >= 1 independent sequences sharing the grid                  */
    int32_t levels;                 /* pyramid levels H: 1, or 2 (see "Pyramid" below)   */
    float max_flow_px;              /* > 0. N = ceil(max_flow_px) substeps, dt = 1/N;
                                       also the clamp bound on u_hat, v_hat (reading 12)              */
    float gamma[5];                 /* gamma1..gamma5 exactly as in eq:cost_top and
                                       eq:cost_invdepth; all >= 0, gamma3 > 0, g4+g5 > 0    */
    int32_t smooth_iters;           /* S >= 0 box passes after the solve (paper H=1: 2)       */
    int32_t dominant_rule;          /* SF_DOM_LARGEST (default) or SF_DOM_PRINTED                     */
    float source_weight;            /* sigma, weight of -f<s,w> per pass (reading 2): 0.5 default     */
    int32_t clamp_advection;        /* 1 (default): clamp u_hat to +-max_flow; 0: literal + CFL flag  */
    int32_t input_is_inverse_depth; /* 0: depth lambda in metres; 1: rho given directly      */
    int32_t device;                 /* CUDA device ordinal                                            */
    void* stream;                   /* cudaStream_t for all work (cudaStreamLegacy allowed); NULL: the
                                       context creates its own non-blocking stream                     */
    int32_t kernel;                 /* SF_KERNEL_*                                                    */
    /* Banded mode (row-band decomposition of a tall grid over several contexts / GPUs,
     * DESIGN.md section 10).  All zero: the context is the whole grid.  Otherwise the context
     * holds rows [band_ext_begin, band_ext_begin + height) of a global grid of global_height
     * rows and OWNS rows [band_own_begin, band_own_end): the others are halo rows refreshed by
     * sf_halo_exchange_* before each sf_step (see sf_band_partition). */
    int32_t band_ext_begin;
    int32_t band_own_begin;
    int32_t band_own_end;
    int32_t global_height;
    int32_t smooth_iters_top;       /* levels = 2: box passes S_2 of the top level; 0 = 4 (Table 3)   */
    int32_t reserved[2];            /* zero                                                           */
} sf_config;

/* Pyramid (levels = 2; DESIGN readings 24-30).  height and
 * width even.  The geometry passed to sf_create holds level 1 ([H][W][10]) followed by level 2
 * ([H/2][W/2][10], the Spherepix grid of the same patch at half resolution).  The context runs
 * the top level as an H = 1 filter on the half grid with 2x2-mean inputs, max flow
 * max_flow_px / 2, S_2 = smooth_iters_top box passes and gains gamma1,2 scaled by
 * (ds1 / ds2)^2 (centre pixel separations; gamma3..5 unchanged), and the bottom level as the
 * increment filter (8-field transport by the reconstructed flow, increment LS with
 * smooth_iters passes, reconstruction w = up(w^2) + dw).  The state seen through the API is the
 * bottom level: w = reconstructed flow, rho = bottom-level inverse depth, Yhat = its brightness
 * model.  Only sf_step / sf_step_host advance a pyramid context (sf_predict, sf_update,
 * sf_set_fields, SF_FIELDS_PREDICTED and banded mode return SF_E_UNSUPPORTED). */

/* Fill *cfg with defaults for an H x W grid (batch 1, max flow 1 px, S = 2, sigma = 0.5,
 * LARGEST, clamp on, gamma = {1,1,1,1,1}, device 0, own stream, AUTO kernel). */
void sf_config_default(sf_config* cfg, int32_t height, int32_t width);

/* Create a context.  geometry: the Spherepix grid as [H][W][10] float32 =
 * (s.xyz, b1.xyz, b2.xyz, ds): unit direction s, basis columns b1 (towards (i,j+1)) and
 * b2 (towards (i+1,j)), pixel separation ds = ||P(s_ij) s_{i,j+1}||.  Host or
 * device pointer (detected); copied, so the caller may free it after the call returns.
 * The state is "fresh": the first sf_update / sf_step initialises it.
 * Errors: SF_E_CONFIG (bad field), SF_E_DATA (NULL), SF_E_CUDA (allocation). */
sf_status sf_create(const sf_config* cfg, const float* geometry, sf_ctx** out);

/* Release all device memory (synchronises the context stream).  NULL is a no-op. */
void sf_destroy(sf_ctx* ctx);

/* Prediction k -> k+ (section "State prediction" P:L501-523, numerical scheme
 * P:L623-690): N substeps of a column pass then a row pass of the upwind transport of
 * (w, rho) with source -f<s,w>.  Keeps the state (w^k, rho^k) and stores the prediction.
 * Errors: SF_E_STATE on a fresh context or when a prediction is already pending. */
sf_status sf_predict(sf_ctx* ctx);

/* Update k+ -> k+1 (section "State update" P:L546-621) from brightness Y and depth
 * (device [B][H][W]): brightness model, inverse-depth model,
 * per-pixel 3x3 LS (eq:LS_update P:L583-588), S box smoothings, rho fusion
 * (P:L617-621).  On a fresh context it initialises the state instead: w = 0, rho = 1/lambda
 * (0 where invalid), Yhat = brightness model of Y.
 * Errors: SF_E_DATA (NULL), SF_E_STATE (initialised context without a pending prediction). */
sf_status sf_update(sf_ctx* ctx, const float* Y, const float* depth);

/* One frame: sf_predict then sf_update (bitwise identical results), using the fused
 * kernel when selected.  On a fresh context: initialisation only.  Errors: as above. */
sf_status sf_step(sf_ctx* ctx, const float* Y, const float* depth);

/* End-to-end variant with HOST buffers: copies Y_host, depth_host ([B][H][W]) to the
 * device, runs sf_step, copies the new state to w_host ([B][H][W][3]) and rho_host
 * ([B][H][W]) (either may be NULL), and synchronises the stream before returning. */
sf_status sf_step_host(sf_ctx* ctx, const float* Y_host, const float* depth_host, float* w_host, float* rho_host);

/* Pipelined variant of sf_step_host for a stream of frames: enqueues the input copies (own
 * copy-in stream), the step and the output copies (own copy-out stream) and returns without
 * synchronising, so frame k's copies overlap frame k-1's output copies and frame k+1's input
 * copies (two device staging slots, ordered by events).  Host buffers must be pinned
 * (cudaHostAlloc / torch pin_memory) and stay untouched until sf_wait; w_host / rho_host
 * receive frame k's new state.  Errors: as sf_step. */
sf_status sf_step_host_async(sf_ctx* ctx, const float* Y_host, const float* depth_host, float* w_host,
                             float* rho_host);

/* Wait for every frame enqueued by sf_step_host_async (and all context work). */
sf_status sf_wait(sf_ctx* ctx);

/* Copy fields out (asynchronously, canonical layout): which = SF_FIELDS_STATE (w^k, rho^k,
 * Yhat^k) or SF_FIELDS_PREDICTED (w^{k+}, rho^{k+}; needs a pending prediction).  Any
 * output pointer may be NULL.  Errors: SF_E_STATE (fresh, or no prediction). */
sf_status sf_get_fields(sf_ctx* ctx, int32_t which, float* w, float* rho, float* yhat);

/* Overwrite the state (checkpoint / test hook); marks the context initialised and drops a
 * pending prediction.  yhat may be NULL (zeros).  Errors: SF_E_DATA. */
sf_status sf_set_fields(sf_ctx* ctx, const float* w, const float* rho, const float* yhat);

/* Read (and optionally clear) the sticky device flags; synchronises the stream.  Returns
 * SF_E_STABILITY if SF_FLAG_CFL is set, else SF_OK. */
sf_status sf_status_flags(sf_ctx* ctx, uint32_t* flags, int32_t clear);

/* ---- inertial source terms -------------------------------------------
 * Camera motion for the following frames (until changed): omega = camera angular velocity
 * Omega (rad per frame), accel = camera linear acceleration a_c (per frame^2, the units of
 * rho a_c being those of w per frame), both host float[3] in the camera frame; NULL = zero.
 * With either given, every prediction substep ends with the explicit stage
 * w += dt (rho a_c - 2 Omega x w - Omega x (Omega x s)) of the terms eq:assumption drops
 * (-Omega x w + a_w, eq:hflow_conservation, eq:totaldev_hflow P:L258-280, P:L341-345;
 * DESIGN reading 32); both NULL switches them off (the paper's predictor).  One motion for
 * all batch members.  Errors: SF_E_DATA, SF_E_CONFIG (non-finite), SF_E_UNSUPPORTED (levels 2). */
sf_status sf_set_motion(sf_ctx* ctx, const float* omega, const float* accel);

/* ---- evaluation outputs ----------------------------------------------
 * Tangent and normal flow of the current state w^k in pixels per frame: tangent [B][H][W][2] =
 * B^T P(s) w / ds (eq:tangent_flow), evaluated as (e1 . t, e2 . t) with
 * t = w - s <s,w> and the filter's e_k = b_k / ds (DESIGN reading 23); normal [B][H][W] =
 * <s,w> / ds (eq:normal_flow).  Device pointers, either may be NULL; asynchronous
 * on the context stream.  Errors: SF_E_DATA (ctx NULL), SF_E_STATE (fresh context). */
sf_status sf_flow_px(sf_ctx* ctx, float* tangent, float* normal);

/* Accuracy of the current state against a ground truth w_gt ([B][H][W][3] float32, device):
 * per-pixel RMSE = || (w_gt - w) / ds || in px/frame (eq:RMSE_vel; float32
 * [B][H][W]) and AAE in degrees (P:L731-734 with DESIGN reading 22: Barron's homogeneous form
 * with squared norms on w/ds; computed in double, [B][H][W]); either raster may be NULL.
 * mean_rmse / mean_aae: HOST double [B] (may be NULL) receive each batch member's mean over
 * its owned rows (all rows unless banded); when either is given the call synchronises the
 * stream.  Errors: SF_E_DATA (ctx or w_gt NULL), SF_E_STATE (fresh context), SF_E_CUDA. */
sf_status sf_eval(sf_ctx* ctx, const float* w_gt, float* rmse, double* aae_deg, double* mean_rmse, double* mean_aae);

/* ---- Spherepix input mapping -----------------------------------------
 * Resample a pinhole camera's measurements onto the context's grid (inside the paper's
 * timed region; operator: DESIGN reading 31).  Ycam, Zcam: device [B][cam_height][cam_width]
 * float32 brightness and z-DEPTH (distance along the optical axis; <= 0 or non-finite = no
 * measurement).  K = {fx, fy, cx, cy} (host, pixel centres at integer coordinates); Rcg: host
 * row-major 3x3 rotation grid -> camera frame, or NULL for the identity.  Per grid pixel s:
 * t = Rcg s, (u, v) = (fx t.x/t.z + cx, fy t.y/t.z + cy); Y = bilinear brightness at (u, v)
 * clamped to the image; lambda = bilinear z-depth / t.z (range along s), NaN (invalid) when
 * t.z <= 0, (u, v) is outside the pixel footprint or a sample is invalid.  Outputs Y, D: device
 * [B][H][W] (the inputs of sf_step).  Asynchronous on the context stream.
 * Errors: SF_E_DATA (NULL pointer), SF_E_CONFIG (bad camera size or intrinsics). */
sf_status sf_map_inputs(sf_ctx* ctx, const float* Ycam, const float* Zcam, int32_t cam_height, int32_t cam_width,
                        const float* K, const float* Rcg, float* Y, float* D);

/* One frame straight from camera images (arguments as sf_map_inputs): sf_map_inputs into the
 * context's own grid buffers, then sf_step.  Errors: as sf_map_inputs and sf_step. */
sf_status sf_step_camera(sf_ctx* ctx, const float* Ycam, const float* Zcam, int32_t cam_height, int32_t cam_width,
                         const float* K, const float* Rcg);

/* ---- banded mode -------------------------------------------------------------------------
 * Halo rows a band needs so that its owned rows are exact after one sf_step: the transport
 * moves information N rows per frame (eq:numerical_stability), the update reads +-2 rows of
 * brightness and +-1 of depth and S box passes reach +-2S: halo = max(N, 2) + 2S. */
int32_t sf_band_halo(const sf_config* cfg);

/* Even split of global_height rows into nbands bands; band b owns [*own_begin, *own_end) and
 * its context holds [*ext_begin, *ext_end) (owned rows + `halo` rows each side, clipped to the
 * grid).  Errors: SF_E_CONFIG (a band thinner than the halo, bad indices). */
sf_status sf_band_partition(int32_t global_height, int32_t nbands, int32_t band, int32_t halo, int32_t* ext_begin,
                            int32_t* own_begin, int32_t* own_end, int32_t* ext_end);

/* Refresh this band's halo rows of the state (w, rho, Yhat^k) from the neighbouring bands'
 * contexts in this process (device-to-device copies on ctx's stream; up / down NULL at the grid
 * edges).  All bands must share a stream or be ordered by the caller. */
sf_status sf_halo_exchange_peer(sf_ctx* ctx, const sf_ctx* up, const sf_ctx* down);

/* The same exchange across processes: ncclSend / ncclRecv of the boundary rows with ranks
 * rank - 1 and rank + 1 (band index == rank) on ctx's stream.  nccl_comm: an ncclComm_t from
 * sf_nccl_comm_init (or any communicator of the same NCCL library).  Errors: SF_E_NCCL. */
sf_status sf_halo_exchange_nccl(sf_ctx* ctx, void* nccl_comm, int32_t rank, int32_t nranks);

/* ---- per-substep banded exchange (the north star's banded split) --------
 * A band context created with band_own_begin / band_own_end and 2 halo rows on every cut side
 * (sf_band_partition(..., sf_band_halo_substep(cfg), ...)) runs a frame with the halo rows
 * refreshed at each point that reads across a row boundary: after every column pass (1 row of
 * (w*, rho*), before the row pass) and before every box pass (2 rows of w) --
 * N + S exchanges per frame instead of sf_halo_exchange_*'s one deep exchange.  Transport and box
 * run on the per-pass kernels; Y / depth cover the band's rows (halo included).  The owned rows
 * equal a whole-grid context's bit for bit.
 * The transport is the caller's: xfer(user, send_up, recv_up, send_down, recv_down, n_up, n_down)
 * is called once per batch member at every exchange point; send_* point at the rows to send to the
 * neighbour above / below, recv_* at the rows to fill from it (n_* floats each; NULL / 0 where
 * the band has no neighbour on that side).  host_staged = 1: the pointers are pinned host memory
 * (libsf copies the rows out before and in after the call, synchronously); 0: device pointers
 * into the context's buffers, the callee enqueues the transfer in the context stream's order.
 * xfer returns 0 on success.  Errors: SF_E_DATA, SF_E_STATE, SF_E_CONFIG (halo rows missing or a
 * band thinner than 4 rows), SF_E_UNSUPPORTED (pyramid), SF_E_NCCL (xfer failed), SF_E_CUDA. */
typedef int32_t (*sf_halo_xfer_fn)(void* user, const float* send_up, float* recv_up, const float* send_down,
                                   float* recv_down, size_t n_up, size_t n_down);
int32_t sf_band_halo_substep(const sf_config* cfg);
sf_status sf_step_banded(sf_ctx* ctx, const float* Y_dev, const float* depth_dev, sf_halo_xfer_fn xfer, void* user,
                         int32_t host_staged);
/* The same over NCCL (band index == rank): every exchange is an ncclGroup of ncclSend / ncclRecv
 * with ranks rank - 1 and rank + 1; the row pass's inner rows run while the transport exchange is
 * in flight on a side stream (interior first), the rows next to the cut edges after it. */
sf_status sf_step_banded_nccl(sf_ctx* ctx, const float* Y_dev, const float* depth_dev, void* nccl_comm, int32_t rank,
                              int32_t nranks);

/* NCCL plumbing (libnccl.so.2 is loaded at first use): rank 0 makes a 128-byte unique id, the
 * caller broadcasts it (e.g. torch.distributed), every rank creates its communicator. */
sf_status sf_nccl_unique_id(char id[128]);
sf_status sf_nccl_comm_init(int32_t nranks, const char id[128], int32_t rank, void** comm);
void sf_nccl_comm_destroy(void* comm);

/* Kernel strategy actually used by sf_step (SF_KERNEL_FUSED or SF_KERNEL_PASSES). */
int32_t sf_kernel_in_use(const sf_ctx* ctx);

/* Number of kernel launches one sf_step issues (for the bench's gpu_launches count). */
int32_t sf_launches_per_step(const sf_ctx* ctx);

/* Per-kernel timing of one frame (measurement hook): sf_step's kernels on
 * the context stream with CUDA events between the prediction (the k_trans launches) and the
 * update (k_upd): *ms_predict / *ms_update receive the two durations in milliseconds (the event
 * between them also removes the programmatic-launch overlap of the two kernels; a short device
 * spin queued first keeps host launch latency out of the timings).  Y / depth as in
 * sf_step.  Synchronises the stream.  Fused H = 1 contexts with a pending-free, initialised state
 * only; errors: SF_E_DATA (null pointer), SF_E_STATE, SF_E_UNSUPPORTED (passes kernels, pyramid),
 * SF_E_CUDA. */
sf_status sf_step_timed(sf_ctx* ctx, const float* Y_dev, const float* depth_dev, float* ms_predict, float* ms_update);

/* Average launch durations of the split step's two kernels (measurement hook, DESIGN.md section
 * 9): after a short device spin, `reps` back-to-back launches of the prediction (k_trans; each
 * one recomputes the same w^{k+}, rho^{k+} from state k) between two CUDA events, then `reps`
 * back-to-back launches of the update (k_upd; each one recomputes the same state k+1) between
 * two more; consecutive launches of a kernel overlap through programmatic dependent launch as
 * in sf_step.  *ms_predict / *ms_update receive elapsed / reps in milliseconds.  The context then
 * holds state k+1 exactly as after one sf_step (the repeated launches are idempotent).  Y / depth
 * as in sf_step; reps in [1, 1000].  Synchronises the stream.  Fused H = 1 contexts, initialised,
 * no pending prediction; errors: SF_E_DATA (null pointer, reps out of range), SF_E_STATE,
 * SF_E_UNSUPPORTED (passes kernels, pyramid), SF_E_CUDA. */
sf_status sf_kernel_times(sf_ctx* ctx, const float* Y_dev, const float* depth_dev, int32_t reps, float* ms_predict,
                          float* ms_update);

/* Static description of a status code. */
const char* sf_error_string(sf_status s);

#ifdef __cplusplus
}
#endif
#endif /* SF_H */
