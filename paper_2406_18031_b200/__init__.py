"""paper_2406_18031_b200 -- B200-native structure-flow predictor-update loop.

Thin ctypes binding over libsf.so (include/sf.h): the same entry points, argument
marshalling only.  Every step of the filter runs in the CUDA kernels of libsf; there
is no CPU or PyTorch fallback -- importing this package without a built libsf.so raises.
PyTorch is used only for device memory, streams and process groups.

Method: Adarve & Mahony, "Real-time Structure Flow", arXiv 2406.18031.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SF_LIB: an alternative build of the same library (A/B measurements of two builds in one run)
LIB_PATH = os.environ.get("SF_LIB") or os.path.join(HERE, "libsf.so")

SF_OK, SF_E_DATA, SF_E_STABILITY, SF_E_CONFIG, SF_E_STATE, SF_E_CUDA, SF_E_NCCL, SF_E_UNSUPPORTED = 0, 2, 3, 4, 5, 6, 7, 8
SF_DOM_LARGEST, SF_DOM_PRINTED = 0, 1
SF_FIELDS_STATE, SF_FIELDS_PREDICTED = 0, 1
SF_FLAG_CLAMPED, SF_FLAG_NONFINITE, SF_FLAG_CFL = 1, 2, 4
SF_KERNEL_AUTO, SF_KERNEL_FUSED, SF_KERNEL_PASSES = 0, 1, 2
SF_ABI_VERSION = 1

EXPORTS = ("sf_config_default", "sf_create", "sf_destroy", "sf_predict", "sf_update", "sf_step", "sf_step_host",
           "sf_get_fields", "sf_set_fields", "sf_status_flags", "sf_kernel_in_use", "sf_launches_per_step",
           "sf_error_string", "sf_band_halo", "sf_band_partition", "sf_halo_exchange_peer", "sf_halo_exchange_nccl",
           "sf_nccl_unique_id", "sf_nccl_comm_init", "sf_nccl_comm_destroy", "sf_flow_px", "sf_eval", "sf_map_inputs", "sf_set_motion", "sf_step_host_async", "sf_wait",
           "sf_step_camera", "sf_step_timed", "sf_kernel_times", "sf_band_halo_substep", "sf_step_banded",
           "sf_step_banded_nccl")


class sf_config(C.Structure):
    _fields_ = [("abi_version", C.c_int32), ("height", C.c_int32), ("width", C.c_int32), ("batch", C.c_int32),
                ("levels", C.c_int32), ("max_flow_px", C.c_float), ("gamma", C.c_float * 5),
                ("smooth_iters", C.c_int32), ("dominant_rule", C.c_int32), ("source_weight", C.c_float),
                ("clamp_advection", C.c_int32), ("input_is_inverse_depth", C.c_int32), ("device", C.c_int32),
                ("stream", C.c_void_p), ("kernel", C.c_int32), ("band_ext_begin", C.c_int32),
                ("band_own_begin", C.c_int32), ("band_own_end", C.c_int32), ("global_height", C.c_int32),
                ("smooth_iters_top", C.c_int32), ("reserved", C.c_int32 * 2)]


class SFError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"{where}: {sf_error_string(status)} (status {status})")
        self.status = status


# sf_halo_xfer_fn (include/sf.h): (user, send_up, recv_up, send_down, recv_down, n_up, n_down) -> 0
HALO_XFER_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                           C.c_size_t)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libsf.so not built at {LIB_PATH}: run `python paper_2406_18031_b200/build.py` "
                          "(there is no fallback path)")
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    lib.sf_config_default.argtypes = [C.POINTER(sf_config), C.c_int32, C.c_int32]
    lib.sf_config_default.restype = None
    lib.sf_create.argtypes = [C.POINTER(sf_config), P, C.POINTER(P)]
    lib.sf_destroy.argtypes = [P]
    lib.sf_destroy.restype = None
    lib.sf_predict.argtypes = [P]
    lib.sf_update.argtypes = [P, P, P]
    lib.sf_step.argtypes = [P, P, P]
    lib.sf_step_host.argtypes = [P, P, P, P, P]
    lib.sf_get_fields.argtypes = [P, C.c_int32, P, P, P]
    lib.sf_set_fields.argtypes = [P, P, P, P]
    lib.sf_status_flags.argtypes = [P, C.POINTER(C.c_uint32), C.c_int32]
    lib.sf_kernel_in_use.argtypes = [P]
    lib.sf_launches_per_step.argtypes = [P]
    lib.sf_error_string.argtypes = [C.c_int]
    lib.sf_error_string.restype = C.c_char_p
    lib.sf_band_halo.argtypes = [C.POINTER(sf_config)]
    I = C.POINTER(C.c_int32)
    lib.sf_band_partition.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, I, I, I, I]
    lib.sf_halo_exchange_peer.argtypes = [P, P, P]
    lib.sf_halo_exchange_nccl.argtypes = [P, P, C.c_int32, C.c_int32]
    lib.sf_nccl_unique_id.argtypes = [C.c_char_p]
    lib.sf_nccl_comm_init.argtypes = [C.c_int32, C.c_char_p, C.c_int32, C.POINTER(P)]
    lib.sf_nccl_comm_destroy.argtypes = [P]
    lib.sf_nccl_comm_destroy.restype = None
    lib.sf_flow_px.argtypes = [P, P, P]
    lib.sf_eval.argtypes = [P, P, P, P, P, P]
    lib.sf_map_inputs.argtypes = [P, P, P, C.c_int32, C.c_int32, P, P, P, P]
    lib.sf_set_motion.argtypes = [P, P, P]
    lib.sf_step_host_async.argtypes = [P, P, P, P, P]
    lib.sf_wait.argtypes = [P]
    lib.sf_step_camera.argtypes = [P, P, P, C.c_int32, C.c_int32, P, P]
    lib.sf_step_timed.argtypes = [P, P, P, C.POINTER(C.c_float), C.POINTER(C.c_float)]
    lib.sf_kernel_times.argtypes = [P, P, P, C.c_int32, C.POINTER(C.c_float), C.POINTER(C.c_float)]
    lib.sf_band_halo_substep.argtypes = [C.POINTER(sf_config)]
    lib.sf_step_banded.argtypes = [P, P, P, HALO_XFER_FN, P, C.c_int32]
    lib.sf_step_banded_nccl.argtypes = [P, P, P, P, C.c_int32, C.c_int32]
    for name in ("sf_create", "sf_predict", "sf_update", "sf_step", "sf_step_host", "sf_get_fields",
                 "sf_set_fields", "sf_status_flags", "sf_kernel_in_use", "sf_launches_per_step", "sf_band_halo",
                 "sf_band_partition", "sf_halo_exchange_peer", "sf_halo_exchange_nccl", "sf_nccl_unique_id",
                 "sf_nccl_comm_init", "sf_flow_px", "sf_eval", "sf_map_inputs", "sf_set_motion", "sf_step_host_async", "sf_wait",
                 "sf_step_camera", "sf_step_timed", "sf_kernel_times", "sf_band_halo_substep", "sf_step_banded",
                 "sf_step_banded_nccl"):
        getattr(lib, name).restype = C.c_int
    return lib


_lib = _load()


# ----------------------------------------------------------------------------- C-ABI names
def sf_error_string(status: int) -> str:
    return _lib.sf_error_string(int(status)).decode()


def _check(st: int, where: str) -> None:
    if st != SF_OK:
        raise SFError(st, where)


def sf_config_default(height: int, width: int) -> sf_config:
    cfg = sf_config()
    _lib.sf_config_default(C.byref(cfg), height, width)
    return cfg


def sf_create(cfg: sf_config, geometry_ptr: int) -> int:
    h = C.c_void_p()
    _check(_lib.sf_create(C.byref(cfg), C.c_void_p(geometry_ptr), C.byref(h)), "sf_create")
    return h.value


def sf_destroy(ctx: int) -> None:
    _lib.sf_destroy(C.c_void_p(ctx))


def sf_predict(ctx: int) -> None:
    _check(_lib.sf_predict(C.c_void_p(ctx)), "sf_predict")


def sf_update(ctx: int, Y_ptr: int, depth_ptr: int) -> None:
    _check(_lib.sf_update(C.c_void_p(ctx), C.c_void_p(Y_ptr), C.c_void_p(depth_ptr)), "sf_update")


def sf_step(ctx: int, Y_ptr: int, depth_ptr: int) -> None:
    _check(_lib.sf_step(C.c_void_p(ctx), C.c_void_p(Y_ptr), C.c_void_p(depth_ptr)), "sf_step")


def sf_step_host(ctx: int, Y_ptr: int, depth_ptr: int, w_ptr: int | None, rho_ptr: int | None) -> None:
    _check(_lib.sf_step_host(C.c_void_p(ctx), C.c_void_p(Y_ptr), C.c_void_p(depth_ptr), C.c_void_p(w_ptr),
                             C.c_void_p(rho_ptr)), "sf_step_host")


def sf_step_host_async(ctx: int, Y_ptr: int, depth_ptr: int, w_ptr: int | None, rho_ptr: int | None) -> None:
    _check(_lib.sf_step_host_async(C.c_void_p(ctx), C.c_void_p(Y_ptr), C.c_void_p(depth_ptr), C.c_void_p(w_ptr),
                                   C.c_void_p(rho_ptr)), "sf_step_host_async")


def sf_wait(ctx: int) -> None:
    _check(_lib.sf_wait(C.c_void_p(ctx)), "sf_wait")


def sf_get_fields(ctx: int, which: int, w_ptr: int | None, rho_ptr: int | None, yhat_ptr: int | None) -> None:
    _check(_lib.sf_get_fields(C.c_void_p(ctx), which, C.c_void_p(w_ptr), C.c_void_p(rho_ptr), C.c_void_p(yhat_ptr)),
           "sf_get_fields")


def sf_flow_px(ctx: int, tangent_ptr: int | None, normal_ptr: int | None) -> None:
    _check(_lib.sf_flow_px(C.c_void_p(ctx), C.c_void_p(tangent_ptr), C.c_void_p(normal_ptr)), "sf_flow_px")


def sf_eval(ctx: int, wgt_ptr: int, rmse_ptr: int | None, aae_ptr: int | None, mean_rmse_ptr: int | None,
            mean_aae_ptr: int | None) -> None:
    _check(_lib.sf_eval(C.c_void_p(ctx), C.c_void_p(wgt_ptr), C.c_void_p(rmse_ptr), C.c_void_p(aae_ptr),
                        C.c_void_p(mean_rmse_ptr), C.c_void_p(mean_aae_ptr)), "sf_eval")


def sf_map_inputs(ctx: int, ycam_ptr: int, zcam_ptr: int, cam_height: int, cam_width: int, K, Rcg,
                  y_ptr: int, d_ptr: int) -> None:
    """K: 4 floats (fx, fy, cx, cy); Rcg: 9 floats (row-major grid -> camera) or None."""
    Kc = (C.c_float * 4)(*[float(x) for x in K])
    Rc = (C.c_float * 9)(*[float(x) for x in list(Rcg)]) if Rcg is not None else None
    _check(_lib.sf_map_inputs(C.c_void_p(ctx), C.c_void_p(ycam_ptr), C.c_void_p(zcam_ptr), cam_height, cam_width,
                              C.cast(Kc, C.c_void_p), C.cast(Rc, C.c_void_p) if Rc is not None else None,
                              C.c_void_p(y_ptr), C.c_void_p(d_ptr)), "sf_map_inputs")


def sf_set_motion(ctx: int, omega=None, accel=None) -> None:
    """omega, accel: 3 floats each (camera frame) or None."""
    om = (C.c_float * 3)(*[float(x) for x in omega]) if omega is not None else None
    ac = (C.c_float * 3)(*[float(x) for x in accel]) if accel is not None else None
    _check(_lib.sf_set_motion(C.c_void_p(ctx), C.cast(om, C.c_void_p) if om is not None else None,
                              C.cast(ac, C.c_void_p) if ac is not None else None), "sf_set_motion")


def sf_step_camera(ctx: int, ycam_ptr: int, zcam_ptr: int, cam_height: int, cam_width: int, K, Rcg=None) -> None:
    Kc = (C.c_float * 4)(*[float(x) for x in K])
    Rc = (C.c_float * 9)(*[float(x) for x in list(Rcg)]) if Rcg is not None else None
    _check(_lib.sf_step_camera(C.c_void_p(ctx), C.c_void_p(ycam_ptr), C.c_void_p(zcam_ptr), cam_height, cam_width,
                               C.cast(Kc, C.c_void_p), C.cast(Rc, C.c_void_p) if Rc is not None else None),
           "sf_step_camera")


def sf_set_fields(ctx: int, w_ptr: int, rho_ptr: int, yhat_ptr: int | None) -> None:
    _check(_lib.sf_set_fields(C.c_void_p(ctx), C.c_void_p(w_ptr), C.c_void_p(rho_ptr), C.c_void_p(yhat_ptr)),
           "sf_set_fields")


def sf_status_flags(ctx: int, clear: bool = False) -> tuple[int, int]:
    """Returns (status, flags); status is SF_E_STABILITY when SF_FLAG_CFL is set."""
    f = C.c_uint32()
    st = _lib.sf_status_flags(C.c_void_p(ctx), C.byref(f), int(clear))
    if st not in (SF_OK, SF_E_STABILITY):
        raise SFError(st, "sf_status_flags")
    return st, f.value


def sf_kernel_in_use(ctx: int) -> int:
    return _lib.sf_kernel_in_use(C.c_void_p(ctx))


def sf_launches_per_step(ctx: int) -> int:
    return _lib.sf_launches_per_step(C.c_void_p(ctx))


def sf_band_halo_substep(cfg) -> int:
    return _lib.sf_band_halo_substep(C.byref(cfg))


def sf_step_banded(ctx: int, Y_ptr: int, D_ptr: int, xfer, host_staged: int = 1) -> None:
    """One frame of a band context with the per-substep halo exchange through the caller's
    transport `xfer(send_up, recv_up, send_down, recv_down, n_up, n_down)` (addresses as ints,
    None where there is no neighbour; host pointers when host_staged)."""
    def _cb(user, su, ru, sd, rd, nu, nd):
        try:
            xfer(su, ru, sd, rd, nu, nd)
            return 0
        except Exception:  # reported as SF_E_NCCL by the library
            import traceback
            traceback.print_exc()
            return 1
    fn = HALO_XFER_FN(_cb)
    _check(_lib.sf_step_banded(C.c_void_p(ctx), C.c_void_p(Y_ptr), C.c_void_p(D_ptr), fn, None, int(host_staged)),
           "sf_step_banded")


def sf_step_banded_nccl(ctx: int, Y_ptr: int, D_ptr: int, comm: int, rank: int, nranks: int) -> None:
    _check(_lib.sf_step_banded_nccl(C.c_void_p(ctx), C.c_void_p(Y_ptr), C.c_void_p(D_ptr), C.c_void_p(comm),
                                    int(rank), int(nranks)), "sf_step_banded_nccl")


def sf_step_timed(ctx: int, Y_ptr: int, D_ptr: int):
    """One fused frame with CUDA events between its prediction and update kernels (sf.h):
    returns (ms_predict, ms_update)."""
    a, b = C.c_float(), C.c_float()
    _check(_lib.sf_step_timed(C.c_void_p(ctx), C.c_void_p(Y_ptr), C.c_void_p(D_ptr), C.byref(a), C.byref(b)),
           "sf_step_timed")
    return a.value, b.value


def sf_kernel_times(ctx: int, Y_ptr: int, D_ptr: int, reps: int):
    """Average launch durations of the split step's kernels, `reps` back-to-back launches of each
    (sf.h): returns (ms_predict, ms_update); the context advances by one frame."""
    a, b = C.c_float(), C.c_float()
    _check(_lib.sf_kernel_times(C.c_void_p(ctx), C.c_void_p(Y_ptr), C.c_void_p(D_ptr), int(reps), C.byref(a),
                                C.byref(b)), "sf_kernel_times")
    return a.value, b.value


def sf_band_halo(cfg: sf_config) -> int:
    return _lib.sf_band_halo(C.byref(cfg))


def sf_band_partition(global_height: int, nbands: int, band: int, halo: int) -> tuple[int, int, int, int]:
    """(ext_begin, own_begin, own_end, ext_end) of band `band`."""
    v = [C.c_int32() for _ in range(4)]
    _check(_lib.sf_band_partition(global_height, nbands, band, halo, *[C.byref(x) for x in v]), "sf_band_partition")
    return tuple(x.value for x in v)


def sf_halo_exchange_peer(ctx: int, up: int | None, down: int | None) -> None:
    _check(_lib.sf_halo_exchange_peer(C.c_void_p(ctx), C.c_void_p(up), C.c_void_p(down)), "sf_halo_exchange_peer")


def sf_halo_exchange_nccl(ctx: int, comm: int, rank: int, nranks: int) -> None:
    _check(_lib.sf_halo_exchange_nccl(C.c_void_p(ctx), C.c_void_p(comm), rank, nranks), "sf_halo_exchange_nccl")


def sf_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib.sf_nccl_unique_id(buf), "sf_nccl_unique_id")
    return buf.raw


def sf_nccl_comm_init(nranks: int, uid: bytes, rank: int) -> int:
    h = C.c_void_p()
    _check(_lib.sf_nccl_comm_init(nranks, C.create_string_buffer(uid, 128), rank, C.byref(h)), "sf_nccl_comm_init")
    return h.value


def sf_nccl_comm_destroy(comm: int) -> None:
    _lib.sf_nccl_comm_destroy(C.c_void_p(comm))


# ----------------------------------------------------------------------------- torch convenience
class StructureFlow:
    """One libsf context over torch CUDA tensors (marshalling only).

    geometry: [H][W][10] float32 (s, b1, b2, ds), host numpy or torch tensor; or a list
    [level 1, level 2] of them for the H = 2 pyramid (level 2 = the half-resolution grid).
    params: any object with max_flow, gamma, smooth_iters, sigma, dominant_rule,
    clamp_advection, input_is_inverse_depth (e.g. sfgen.Params).
    """

    def __init__(self, geometry, params, batch: int = 1, device: int = 0, stream=None, kernel: int = SF_KERNEL_AUTO,
                 band: tuple | None = None, smooth_iters_top: int = 0):
        """band: None, or (ext_begin, own_begin, own_end, global_height) for a row-band context
        whose geometry holds the global rows [ext_begin, ext_begin + H)."""
        import numpy as np
        import torch

        self.torch = torch

        def dev(x):
            t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
            return t.to(dtype=torch.float32, device=f"cuda:{device}").contiguous()

        levels = len(geometry) if isinstance(geometry, (list, tuple)) else 1
        if levels == 1:
            g = dev(geometry)
            H, W, ch = g.shape
        else:
            parts = [dev(x) for x in geometry]
            H, W, ch = parts[0].shape
            assert all(p.shape == (H >> h, W >> h, 10) for h, p in enumerate(parts))
            g = torch.cat([p.reshape(-1) for p in parts])
        assert ch == 10
        self.H, self.W, self.B, self.device = H, W, batch, torch.device(f"cuda:{device}")
        cfg = sf_config_default(H, W)
        cfg.batch = batch
        cfg.max_flow_px = float(params.max_flow)
        for k in range(5):
            cfg.gamma[k] = float(params.gamma[k])
        cfg.smooth_iters = int(params.smooth_iters)
        cfg.dominant_rule = int(params.dominant_rule)
        cfg.source_weight = float(params.sigma)
        cfg.clamp_advection = int(params.clamp_advection)
        cfg.input_is_inverse_depth = int(params.input_is_inverse_depth)
        cfg.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        # torch's default stream has handle 0, which sf_create reads as "make your own";
        # pass cudaStreamLegacy (0x1) so libsf orders with torch's work on that stream.
        cfg.stream = self.stream.cuda_stream or 1
        cfg.kernel = kernel
        cfg.levels = levels
        cfg.smooth_iters_top = smooth_iters_top
        self.levels = levels
        self._geometry = g  # keep the device copy alive until sf_create has read it
        if band is not None:
            cfg.band_ext_begin, cfg.band_own_begin, cfg.band_own_end, cfg.global_height = (int(x) for x in band)
        self.cfg = cfg
        torch.cuda.synchronize(self.device)
        self.ctx = sf_create(cfg, g.data_ptr())
        if getattr(params, "omega", None) is not None or getattr(params, "accel", None) is not None:
            sf_set_motion(self.ctx, params.omega or (0.0, 0.0, 0.0), params.accel or (0.0, 0.0, 0.0))

    def __del__(self):
        ctx = getattr(self, "ctx", None)
        if ctx and callable(globals().get("sf_destroy")):  # (module globals are gone at interpreter exit)
            sf_destroy(ctx)
            self.ctx = None

    def _in(self, x):
        t = self.torch
        assert isinstance(x, t.Tensor) and x.is_cuda and x.dtype == t.float32 and x.is_contiguous()
        assert x.numel() == self.B * self.H * self.W
        return x.data_ptr()

    def step(self, Y, depth):
        sf_step(self.ctx, self._in(Y), self._in(depth))

    def predict(self):
        sf_predict(self.ctx)

    def update(self, Y, depth):
        sf_update(self.ctx, self._in(Y), self._in(depth))

    def get_fields(self, which: int = SF_FIELDS_STATE):
        t = self.torch
        w = t.empty((self.B, self.H, self.W, 3), dtype=t.float32, device=self.device)
        rho = t.empty((self.B, self.H, self.W), dtype=t.float32, device=self.device)
        yhat = t.empty((self.B, self.H, self.W), dtype=t.float32, device=self.device) if which == SF_FIELDS_STATE else None
        sf_get_fields(self.ctx, which, w.data_ptr(), rho.data_ptr(), yhat.data_ptr() if yhat is not None else None)
        return w, rho, yhat

    def flow_px(self):
        """(tangent [B][H][W][2], normal [B][H][W]) of the current state in pixels (sf_flow_px)."""
        t = self.torch
        tg = t.empty((self.B, self.H, self.W, 2), dtype=t.float32, device=self.device)
        nm = t.empty((self.B, self.H, self.W), dtype=t.float32, device=self.device)
        sf_flow_px(self.ctx, tg.data_ptr(), nm.data_ptr())
        return tg, nm

    def evaluate(self, w_gt, rasters: bool = True):
        """RMSE (px/frame) and AAE (degrees) against w_gt (device [B][H][W][3]) -> dict with the
        per-pixel rasters (if asked) and the per-batch-member means (sf_eval)."""
        t = self.torch
        rm = t.empty((self.B, self.H, self.W), dtype=t.float32, device=self.device) if rasters else None
        aa = t.empty((self.B, self.H, self.W), dtype=t.float64, device=self.device) if rasters else None
        mr = (C.c_double * self.B)()
        ma = (C.c_double * self.B)()
        sf_eval(self.ctx, self._in3(w_gt), rm.data_ptr() if rasters else None, aa.data_ptr() if rasters else None,
                C.addressof(mr), C.addressof(ma))
        return {"rmse": rm, "aae_deg": aa, "mean_rmse": list(mr), "mean_aae_deg": list(ma)}

    def map_inputs(self, Ycam, Zcam, K, Rcg=None):
        """Camera brightness / z-depth (device [B][Hc][Wc]) -> grid (Y, depth) device tensors."""
        t = self.torch
        assert Ycam.is_cuda and Ycam.dtype == t.float32 and Ycam.is_contiguous() and Zcam.shape == Ycam.shape
        Hc, Wc = Ycam.shape[-2:]
        Y = t.empty((self.B, self.H, self.W), dtype=t.float32, device=self.device)
        D = t.empty_like(Y)
        Rf = None if Rcg is None else [float(x) for x in (Rcg.flatten() if hasattr(Rcg, "flatten") else Rcg)]
        sf_map_inputs(self.ctx, Ycam.data_ptr(), Zcam.contiguous().data_ptr(), Hc, Wc, K, Rf, Y.data_ptr(),
                      D.data_ptr())
        return Y, D

    def set_fields(self, w, rho, yhat=None):
        sf_set_fields(self.ctx, self._in3(w), self._in(rho), self._in(yhat) if yhat is not None else None)

    def _in3(self, x):
        t = self.torch
        assert isinstance(x, t.Tensor) and x.is_cuda and x.dtype == t.float32 and x.is_contiguous()
        assert x.numel() == 3 * self.B * self.H * self.W
        return x.data_ptr()

    def flags(self, clear: bool = False) -> int:
        return sf_status_flags(self.ctx, clear)[1]

    @property
    def kernel(self) -> int:
        return sf_kernel_in_use(self.ctx)

    @property
    def launches_per_step(self) -> int:
        return sf_launches_per_step(self.ctx)
