#!/usr/bin/env python3
"""Benchmark: structure-flow predictor-update frames/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl sf|reference] [--config 2|3|4]

One step = one frame k -> k+1 of the whole hot path (predict N substeps + update) for
every sequence in the batch.  N = 1: configs[1] (512 x 512, max flow 8 px, S = 2, batch 1).
N > 1 (torchrun, one process per GPU): each rank runs its own independent sequence, no
data-path collective ("weak" scaling; value = frames of all ranks / max-over-ranks time).

Inputs: a ring of R distinct frames resident in HBM (R x 2 MiB > the 126 MB L2), so each
step reads cold brightness/depth; steps are replayed from CUDA graphs of 16 consecutive steps
captured on the context stream.  Timing: CUDA events on that stream, barrier + synchronize on both
sides, max over ranks.  --impl reference times the float32 CPU oracle (the only other
place this file runs oracle/), see DESIGN.md section 9.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "predictor-update Hz at 512x512, 8-px max flow; achieved HBM GB/s vs peak"
CONFIG_NAMES = {2: "512x512 spherepix (gnomonic 90 deg), max flow 8 px (N=8), S=2, H=1 level",
                3: "1024x1024 spherepix (gnomonic 90 deg), max flow 16 px (N=16), S=2, H=1 level",
                4: "64 x 512x512 sequences per job, max flow 8 px (N=8), S=2, H=1 level",
                5: "8192x8192 spherepix (gnomonic 90 deg) row-banded over the GPUs, max flow 8 px (N=8), S=2"}
CONFIG_NAMES_PYR = {2: "512x512 spherepix, max flow 8 px, H=2 levels (top 256x256: N=4, S=4; bottom: N=8, S=2); "
                         "the paper's Table 3 shape (594.7 Hz on a GTX 780, context only)",
                      3: "1024x1024 spherepix, max flow 16 px, H=2 levels (top: N=8, S=4; bottom: N=16, S=2)",
                      4: "64 x 512x512 sequences per job, max flow 8 px, H=2 levels"}
ALGO_BYTES_PER_PX = 48  # read w 12 + rho 4 + Yhat 4 + Y 4 + lambda 4, write 12 + 4 + 4


def algo_ops_per_px(N: int, S: int) -> int:
    """FP32 operations per pixel per frame of the arithmetic definition:
    26 per transport pass (2N passes) + 109 for the models, solve and fusion + 27 per box pass."""
    return 26 * 2 * N + 109 + 27 * S


def algo_ops_per_px_pyr(N1: int, S1: int, N2: int, S2: int) -> float:
    """H = 2: the top level's H = 1 count on a quarter of the pixels, plus the
    bottom level's 42 ops per 8-field transport pass (2 N1 passes), the same 109 + 27 S1 update
    and 12 for the down-sampling and reconstruction."""
    return algo_ops_per_px(N2, S2) / 4.0 + 42 * 2 * N1 + 109 + 27 * S1 + 12


SMS, FP32_LANES_PER_SM = 148, 128  # B200: 148 SMs x 4 SMSPs x 32 FP32 lanes


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0)))


def ncu_traffic(kernel="k_fused", cid=2):
    """DRAM bytes per launch of the dominant kernel from the newest committed ncu --set full
    summary (profiles/*_ncu_<kernel>.json, written by tools/ncu_summary.py), or None."""
    import glob

    # per-kernel evidence of the bench workload (tools/gpu_ncu_evidence.sh -> profiles/<tag>_cfg2_<kernel>.json)
    ev = sorted(glob.glob(os.path.join(ROOT, "profiles", f"*_cfg{cid}_{kernel}.json")))
    for fp in reversed(ev):
        try:
            d = json.load(open(fp))
            if d.get("dram_bytes_per_launch"):
                return {"bytes_per_launch": d["dram_bytes_per_launch"], "source": os.path.relpath(fp, ROOT)}
        except Exception:
            continue
    if cid != 2:
        return None
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"*_ncu_{kernel}.json")), key=os.path.getmtime)
    for fp in reversed(files):
        try:
            caps = json.load(open(fp)).get("captures", [])
            vals = [c["traffic_bytes_per_launch"] for c in caps if "traffic_bytes_per_launch" in c]
            if vals:
                return {"bytes_per_launch": sum(vals) / len(vals), "source": os.path.relpath(fp, ROOT)}
        except Exception:
            continue
    return None


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


def start_clock_sampler(device: int):
    fd, path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
    os.close(fd)
    q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    try:
        p = subprocess.Popen(["nvidia-smi", f"--id={device}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                              "-lms", "50"], stdout=open(path, "w"), stderr=subprocess.DEVNULL)
    except Exception:
        return None, path
    return p, path


def stop_clock_sampler(p, path):
    if p is None:
        return None
    p.terminate()
    try:
        p.wait(timeout=5)
    except Exception:
        p.kill()
    sm, mx, reasons = [], [], set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    for line in open(path):
        parts = [x.strip() for x in line.split(",")]
        if len(parts) < 9:
            continue
        try:
            sm.append(float(parts[1]))
            mx.append(float(parts[2]))
        except ValueError:
            continue
        for n, v in zip(names, parts[5:9]):
            if v.lower() == "active":
                reasons.add(n)
    os.unlink(path)
    if not sm:
        return None
    load = [x for x in sm if x > 0.5 * max(sm)] or sm
    return {"sm_mhz": statistics.median(load), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
            "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU oracle arms
def oracle_frames(seq, frames, rows=None, levels=1):
    """Run the float32 oracle over `frames` frames (optionally on the first `rows` rows of
    the grid, a bounded sample); return seconds per frame (excluding the init frame)."""
    import oracle
    import sfgen

    g = seq.geom if rows is None else np.ascontiguousarray(seq.geom[:rows])
    if levels == 2:
        H, W = seq.geom.shape[:2]
        g1, g2 = sfgen.grid.gnomonic_pyramid(H, W, seq.fov)
        r = H if rows is None else rows - rows % 2
        o = oracle.PyramidOracle(np.ascontiguousarray(g1[:r]), np.ascontiguousarray(g2[:r // 2]), seq.params)
        rows = r
    else:
        o = oracle.Oracle(g, seq.params, "f32")
    sl = (slice(None),) if rows is None else (slice(None), slice(0, rows))
    Y = np.ascontiguousarray(seq.Y[sl])
    D = np.ascontiguousarray(seq.depth[sl])
    o.step(Y[0], D[0])
    t0 = time.perf_counter()
    for k in range(1, frames + 1):
        o.step(Y[k % len(Y)], D[k % len(D)])
    return (time.perf_counter() - t0) / frames


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _oracle_worker(payload):
    """One process of the all-cores aggregate: the float32 oracle on its own copy of the sequence,
    `frames` timed frames after the init frame.  Returns (frames, seconds)."""
    geom, params, Y, D, frames, levels = payload
    import oracle
    if levels == 2:
        g1, g2 = geom
        o = oracle.PyramidOracle(g1, g2, params)
    else:
        o = oracle.Oracle(geom, params, "f32")
    o.step(Y[0], D[0])
    t0 = time.perf_counter()
    for k in range(1, frames + 1):
        o.step(Y[k % len(Y)], D[k % len(D)])
    return frames, time.perf_counter() - t0


def cpu_all_cores(seq, t1, budget_s=12.0, levels=1):
    """Aggregate frames/s of P = all host cores running independent sequences (one oracle process
    each, config-4 style), each for ~budget_s of frames."""
    import concurrent.futures as cf
    import multiprocessing as mp
    import sfgen

    P = host_cores()
    frames = max(1, min(60, int(budget_s / max(t1, 1e-6))))
    geom = seq.geom
    if levels == 2:
        H, W = seq.geom.shape[:2]
        geom = sfgen.grid.gnomonic_pyramid(H, W, seq.fov)
    payload = (geom, seq.params, seq.Y[:3], seq.depth[:3], frames, levels)
    with cf.ProcessPoolExecutor(max_workers=P, mp_context=mp.get_context("spawn")) as ex:
        res = list(ex.map(_oracle_worker, [payload] * P))
    total = sum(f for f, _ in res)
    span = max(t for _, t in res)
    return {"value": total / span, "unit": "Hz", "cores": P, "kind": "oracle",
            "sample": f"{P} independent processes x {frames} full frames each (aggregate frames/s of independent "
                      f"sequences, config-4 style), float32 oracle as it stands, 1 thread per process"}


def cpu_baseline(seq, budget_s=15.0, levels=1, all_cores=True):
    """Oracle on host cores, single thread, bounded sample: full frames until ~budget; plus the
    all-cores aggregate over independent sequences."""
    t1 = oracle_frames(seq, 1, levels=levels)
    frames = max(2, min(60, int(budget_s / max(t1, 1e-6))))
    t = oracle_frames(seq, frames, levels=levels)
    H, W = seq.geom.shape[:2]
    out = {"value": 1.0 / t, "unit": "Hz", "cores": 1, "kind": "oracle",
           "sample": f"{frames} full {H}x{W} frames (N={seq.params.N}, S={seq.params.smooth_iters}, H={levels} "
                     f"level{'s' if levels > 1 else ''}) of the bench workload, float32 oracle, 1 thread, "
                     f"{host_cores()} host cores available ({cpu_model()})",
           "cpu_model": cpu_model(), "host_cores": host_cores()}
    if all_cores:
        try:
            out["all_cores"] = cpu_all_cores(seq, t, levels=levels)
        except Exception as e:  # noqa: BLE001 -- report, do not fail the bench
            out["all_cores"] = {"error": repr(e)}
    return out


def workload_config(cid, levels, B, world, mf=None, cam=False):
    """The config dict both arms print (identical keys and values for the same workload)."""
    import sfgen
    base = sfgen.CONFIGS[2 if cid == 4 else cid]
    N = max(1, math.ceil(mf if mf else base["max_flow"]))
    return {"workload": (CONFIG_NAMES[cid] if levels == 1 else CONFIG_NAMES_PYR[cid]) +
                        (f" [max flow overridden: {mf} px]" if mf else ""),
            "batch_per_gpu": B, "H": base["H"], "W": base["W"], "N": N, "levels": levels, "S": 2,
            "parallelism": f"independent sequences x{world}",
            "l2": "inputs from a ring of distinct rendered frames larger than L2 (cold reads every step)",
            "input_mapping": ("pinhole camera 640x640 90 deg -> grid (sf_step_camera) inside each step"
                              if cam else "inputs already on the grid")}


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    import sfgen

    cid = args.config
    seq = sfgen.config_sequence(cid if cid != 4 else 2, frames=8)
    H, W = seq.geom.shape[:2]
    lv = args.levels
    t1 = oracle_frames(seq, 1, levels=lv)
    total = args.steps + args.warmup
    budget = 150.0
    rows = H if t1 * total <= budget else max(8, int(H * budget / (t1 * total)))
    rows -= rows % 2
    per_frame = oracle_frames(seq, args.warmup, rows, lv) if args.warmup else 0.0  # warm-up (untimed)
    per_frame = oracle_frames(seq, args.steps, rows, lv)
    frac = rows / H
    value = frac / per_frame  # full frames per second equivalent
    sample = f"each step: one frame of the first {rows} of {H} rows ({frac:.3f} of a frame), f32 oracle, 1 thread"
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "Hz", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_frame * 1e3 / frac,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": workload_config(cid, lv, 1 if cid != 4 else max(1, 64 // world), world,
                                     getattr(args, "max_flow", None), getattr(args, "map", False)),
           "cpu_baseline": {"value": value, "unit": "Hz", "cores": 1, "kind": "oracle", "sample": sample,
                            "cpu_model": cpu_model(), "host_cores": host_cores()},
           "e2e": {"value": value, "unit": "Hz", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


# ----------------------------------------------------------------------------- GPU arm
def run_sf(args):
    import torch
    import torch.distributed as dist

    import paper_2406_18031_b200 as sf
    import sfgen

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    cid = args.config
    B = 1 if cid != 4 else max(1, 64 // world)
    base = sfgen.CONFIGS[2 if cid == 4 else cid]
    H, W = base["H"], base["W"]
    # batch steps already read > L2 per step (64 MiB x 2): a short ring of rendered frames
    ring = args.ring if B == 1 else 8
    # independent sequence(s) per rank (seeds differ); frames of the sequence fill the ring
    mf = getattr(args, "max_flow", None)
    # config 4: the batch of 64 sequences has seeds 100..163, split over the ranks
    seed0 = sfgen.CONFIGS[4]["seed"] + B * rank if cid == 4 else base["seed"] + 1000 * rank
    seqs = [sfgen.config_sequence(2 if cid == 4 else cid, frames=ring, seed=seed0 + b, max_flow=mf)
            for b in range(B)]
    geom, params = seqs[0].geom, seqs[0].params
    if B == 1:
        Yh, Dh = seqs[0].Y, seqs[0].depth
    else:
        Yh = np.stack([np.stack([s.Y[k] for s in seqs]) for k in range(ring)])
        Dh = np.stack([np.stack([s.depth[k] for s in seqs]) for k in range(ring)])
    Yd = torch.from_numpy(np.ascontiguousarray(Yh.reshape(ring, B, H, W))).to(dev)
    Dd = torch.from_numpy(np.ascontiguousarray(Dh.reshape(ring, B, H, W))).to(dev)
    frame_bytes = B * H * W * 4

    s = torch.cuda.Stream(device=dev)
    kern = {"auto": sf.SF_KERNEL_AUTO, "fused": sf.SF_KERNEL_FUSED, "passes": sf.SF_KERNEL_PASSES}[args.kernel]
    levels = getattr(args, "levels", 1)
    if levels == 2:
        pyr = sfgen.grid.gnomonic_pyramid(H, W, base["fov"])
        m = sf.StructureFlow(pyr, params, batch=B, device=local, stream=s, kernel=kern)
    else:
        m = sf.StructureFlow(geom, params, batch=B, device=local, stream=s, kernel=kern)

    def frame_of(i):
        """Palindromic replay order 0..R-1, R-1..0: no jump back in time at the wrap (a camera
        that reverses), while every step still reads a cold frame of a > L2 ring."""
        j = i % (2 * ring)
        return j if j < ring else 2 * ring - 1 - j

    # --map: every step first resamples a pinhole camera frame onto the grid (sf_map_inputs,
    # inside the paper's timed region): camera 640 x 640, 90 deg, frames of the same scene
    cam = None
    if getattr(args, "map", False):
        from sfgen.scene import render_camera
        Hc = Wc = 640
        K = (Wc / 2.0, Hc / 2.0, (Wc - 1) / 2.0, (Hc - 1) / 2.0)  # f = (W/2) / tan(45 deg)
        cams = [render_camera(seqs[0].scene, Hc, Wc, K, float(k)) for k in range(ring)]
        Yc = torch.from_numpy(np.stack([c[0] for c in cams])[:, None]).to(dev)
        Zc = torch.from_numpy(np.stack([c[1] for c in cams])[:, None]).to(dev)
        Ym = torch.empty((B, H, W), dtype=torch.float32, device=dev)
        Dm = torch.empty_like(Ym)
        cam = (Hc, Wc, K, Yc, Zc, Ym, Dm)

    def do_step(k):
        if cam is None:
            m.step(Yd[k], Dd[k])
        else:
            Hc, Wc, K, Yc, Zc, Ym, Dm = cam
            sf.sf_step_camera(m.ctx, Yc[k].data_ptr(), Zc[k].data_ptr(), Hc, Wc, K, None)

    with torch.cuda.stream(s):
        do_step(0)  # frame 0: initialisation (not a timed step)
        for k in range(1, ring):  # one real pass over the ring before capture (untimed)
            do_step(k)
    s.synchronize()
    # CUDA graphs of CHUNK consecutive steps of the palindrome (an even count, so a chunk starts
    # and ends at the same state parity); the cycle of 2R steps is split into 2R / CHUNK graphs
    # replayed in order.  Steps beyond a multiple of CHUNK are direct sf_step calls.
    # (16: graph boundaries -- no programmatic launch across them -- cost ~6 us each; measured per
    # frame 28.3 / 26.65 / 25.5 / 25.3 us for graphs of 2 / 4 / 16 / 32 steps and 25.9 us for direct,
    # PDL-chained launches; SF_BENCH_CHUNK overrides, even)
    CHUNK = int(os.environ.get("SF_BENCH_CHUNK", "16"))
    cycle = 2 * ring
    pos0 = ring  # palindrome position after the untimed pass over the ring
    chunks = []
    for c in range(cycle // CHUNK):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for t in range(CHUNK):
                k = frame_of(pos0 + c * CHUNK + t)
                do_step(k)
        chunks.append(g)
    launches = m.launches_per_step + (1 if cam is not None else 0)  # sf_step_camera: + the mapping kernel
    state = {"i": pos0}

    def run_steps(n):
        """n steps continuing the palindrome: whole chunks as graph replays, the rest direct."""
        while n > 0:
            off = state["i"] - pos0
            if n >= CHUNK and off % CHUNK == 0:
                chunks[(off // CHUNK) % len(chunks)].replay()
                state["i"] += CHUNK
                n -= CHUNK
            else:
                k = frame_of(state["i"])
                do_step(k)
                state["i"] += 1
                n -= 1

    # setup (untimed, not warm-up): every graph replayed once so that no timed replay is a graph's
    # first launch (upload), then direct steps so that the W warm-up steps end on a chunk boundary
    with torch.cuda.stream(s):
        run_steps(cycle)
        run_steps((-(state["i"] - pos0 + args.warmup)) % CHUNK)
        torch.cuda.synchronize(dev)
        run_steps(args.warmup)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clk, clk_path = (None, None)
    if rank == 0:
        clk, clk_path = start_clock_sampler(local)
        time.sleep(0.3)
    nchunk = args.steps // CHUNK
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(nchunk + 2)]
    with torch.cuda.stream(s):
        ev[0].record(s)
        for i in range(nchunk):
            run_steps(CHUNK)
            ev[i + 1].record(s)
        run_steps(args.steps - nchunk * CHUNK)
        ev[-1].record(s)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = stop_clock_sampler(clk, clk_path) if rank == 0 else None
    total_ms = ev[0].elapsed_time(ev[-1])
    step_ms = [ev[i].elapsed_time(ev[i + 1]) / CHUNK for i in range(nchunk)] or [total_ms / args.steps]
    t = torch.tensor([total_ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    st, flags = sf.sf_status_flags(m.ctx)

    # ---- the same steps as direct sf_step calls (no graphs; consecutive kernels PDL-chained), the
    # streaming mode of a real-time caller: an even number of steps, CUDA events around them
    direct_ms = None
    if world == 1:
        nd = 2 * max(10, min(args.steps, 400) // 2)
        with torch.cuda.stream(s):
            dev0 = torch.cuda.Event(enable_timing=True)
            dev1 = torch.cuda.Event(enable_timing=True)
            for _ in range(20):  # warm-up of the direct path
                k = frame_of(state["i"])
                do_step(k)
                state["i"] += 1
            dev0.record(s)
            for _ in range(nd):
                k = frame_of(state["i"])
                do_step(k)
                state["i"] += 1
            dev1.record(s)
        torch.cuda.synchronize(dev)
        direct_ms = dev0.elapsed_time(dev1) / nd

    # ---- per-kernel durations (fused H = 1): frames through sf_step_timed, CUDA events on the context
    # stream between the transport (k_trans) and the update (k_upd); the roofline's dominant kernel
    ktimes = None
    if m.kernel == sf.SF_KERNEL_FUSED and levels == 1 and cam is None:
        tp, tu = [], []
        with torch.cuda.stream(s):
            for i in range(max(20, min(args.steps, 200))):
                k = frame_of(state["i"])
                state["i"] += 1
                a_ms, b_ms = sf.sf_step_timed(m.ctx, Yd[k].data_ptr(), Dd[k].data_ptr())
                if i >= 5:
                    tp.append(a_ms)
                    tu.append(b_ms)
        # average launch durations: REPS back-to-back launches of each kernel between CUDA events
        # (consecutive launches overlap through programmatic dependent launch, as in the step)
        REPS = 20
        bp, bu = [], []
        with torch.cuda.stream(s):
            for i in range(12):
                k = frame_of(state["i"])
                state["i"] += 1
                a_ms, b_ms = sf.sf_kernel_times(m.ctx, Yd[k].data_ptr(), Dd[k].data_ptr(), REPS)
                if i >= 2:
                    bp.append(a_ms)
                    bu.append(b_ms)
        ktimes = {"k_trans_ms": statistics.mean(bp), "k_upd_ms": statistics.mean(bu),
                  "runs": len(bp), "reps": REPS,
                  "note": f"sf_kernel_times: {REPS} back-to-back launches of each kernel between CUDA events on "
                          "the context stream (programmatic dependent launch between consecutive launches), "
                          "after the timed region",
                  "single_frame": {"k_trans_ms": statistics.mean(tp), "k_upd_ms": statistics.mean(tu),
                                   "frames": len(tp),
                                   "note": "sf_step_timed: CUDA events around each kernel of one frame (launch "
                                           "latency and drain included, no overlap across the events)"}}

    # ---- end to end through the host-buffer C-ABI call (pinned host memory), same metric
    e2e_steps = max(3, min(args.steps, 400))
    Yp = torch.empty((ring, B, H, W), dtype=torch.float32, pin_memory=True)
    Dp = torch.empty_like(Yp).pin_memory()
    Yp.copy_(Yd.cpu())
    Dp.copy_(Dd.cpu())
    # two pinned result sets: frame k's w, rho land in set k % 2 (the pipelined API overlaps
    # frame k's copies with frame k-1's output copies and frame k+1's input copies)
    w_out = [torch.empty((B, H, W, 3), dtype=torch.float32, pin_memory=True) for _ in range(2)]
    r_out = [torch.empty((B, H, W), dtype=torch.float32, pin_memory=True) for _ in range(2)]

    def e2e_run(n, fn):
        for i in range(n):
            k = frame_of(state["i"])
            state["i"] += 1
            fn(m.ctx, Yp[k].data_ptr(), Dp[k].data_ptr(), w_out[i % 2].data_ptr(), r_out[i % 2].data_ptr())
        sf.sf_wait(m.ctx)

    e2e_run(4, sf.sf_step_host_async)
    e2e_run(2, sf.sf_step_host)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    e2e_run(e2e_steps, sf.sf_step_host_async)
    e2e_s = torch.tensor([time.perf_counter() - t0], device=dev)
    t0 = time.perf_counter()
    sync_steps = max(3, e2e_steps // 4)
    e2e_run(sync_steps, sf.sf_step_host)
    sync_s = torch.tensor([time.perf_counter() - t0], device=dev)
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
        dist.all_reduce(sync_s, op=dist.ReduceOp.MAX)
    e2e_value = world * B * e2e_steps / float(e2e_s.item())
    e2e_sync_value = world * B * sync_steps / float(sync_s.item())

    if rank == 0:
        value = world * B * args.steps / (total_ms / 1e3)
        pk = peaks() or {}
        hbm_peak = pk.get("hbm_gbs", 6650.0)
        # dominant (only) kernel per step: CUDA-event step durations on the launching stream
        med_ms = statistics.median(step_ms)
        mean_ms = total_ms / args.steps
        algo_bytes = ALGO_BYTES_PER_PX * B * H * W
        gbs = algo_bytes / (mean_ms / 1e3) / 1e9
        if levels == 2:
            ops = algo_ops_per_px_pyr(params.N, params.smooth_iters, max(1, math.ceil(params.max_flow / 2)), 4) * B * H * W
        else:
            ops = algo_ops_per_px(params.N, params.smooth_iters) * B * H * W
        sm_max = pk.get("sm_max_mhz", 1965.0)
        alu_peak = SMS * FP32_LANES_PER_SM * sm_max * 1e6 / 1e12  # TFLOP/s-equivalent FP32 lane-ops
        alu = ops / (mean_ms / 1e3) / 1e12
        step_view = {"achieved": alu, "frac": alu / alu_peak, "ops_per_step": ops,
                     "note": "all algorithmic FP32 ops of the step / the device-timed step"}
        if ktimes:
            # dominant kernel: the transport (2N passes x 26 ops/px) over its
            # event-timed duration; the update kernel's view beside it
            t_ops = 26 * 2 * params.N * B * H * W
            u_ops = (109 + 27 * params.smooth_iters) * B * H * W
            t_alu = t_ops / (ktimes["k_trans_ms"] / 1e3) / 1e12
            u_alu = u_ops / (ktimes["k_upd_ms"] / 1e3) / 1e12
            tr = ncu_traffic("k_trans", cid)
            roof = {"bound": "alu", "achieved": t_alu, "peak": alu_peak, "unit": "TFLOP/s", "frac": t_alu / alu_peak,
                    "traffic": tr["bytes_per_launch"] if tr else None,
                    "traffic_source": (tr["source"] + " (ncu --set full, cache-flushed replay)") if tr else None,
                    "kernel": "k_trans", "launches_per_step": (params.N + 7) // 8,
                    "algo_ops_per_launch": t_ops / ((params.N + 7) // 8),
                    "kernel_ms": ktimes["k_trans_ms"], "kernel_times": ktimes,
                    "peak_source": f"148 SMs x 128 FP32 lanes x {sm_max:.0f} MHz (DESIGN.md section 8)",
                    "update_kernel": {"kernel": "k_upd", "achieved": u_alu, "frac": u_alu / alu_peak,
                                      "ops_per_launch": u_ops, "kernel_ms": ktimes["k_upd_ms"]},
                    "step_view": step_view,
                    "hbm_view": {"achieved_gbs": gbs, "peak_gbs": hbm_peak, "frac": gbs / hbm_peak,
                                 "algo_bytes_per_step": algo_bytes,
                                 "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in pk else "fallback"}}
        else:
            kname = "whole step (2N+1+S per-pass kernels)" if m.kernel != sf.SF_KERNEL_FUSED else "whole step"
            if levels == 2:
                kname = "whole step (top level fused + bottom-level kernels)"
            roof = {"bound": "alu", "achieved": alu, "peak": alu_peak, "unit": "TFLOP/s", "frac": alu / alu_peak,
                    "traffic": None, "traffic_source": None, "kernel": kname, "launches_per_step": launches,
                    "algo_ops_per_launch": ops / max(1, launches),
                    "peak_source": f"148 SMs x 128 FP32 lanes x {sm_max:.0f} MHz (DESIGN.md section 8)",
                    "step_view": step_view,
                    "hbm_view": {"achieved_gbs": gbs, "peak_gbs": hbm_peak, "frac": gbs / hbm_peak,
                                 "algo_bytes_per_step": algo_bytes,
                                 "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in pk else "fallback"}}
        out = {"metric": METRIC, "value": value, "unit": "Hz", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
               "config": workload_config(cid, levels, B, world, mf, cam is not None),
               "impl_detail": {"kernel": {sf.SF_KERNEL_FUSED: "fused", sf.SF_KERNEL_PASSES: "passes"}.get(m.kernel),
                               "inputs": f"ring of {ring} frames ({ring * 2 * frame_bytes / 2**20:.0f} MiB) > L2, "
                                         "replayed palindromically, cold reads each step",
                               "launch": f"CUDA graphs of {CHUNK} steps (each replayed once before the warm-up), "
                                         "remainder steps launched directly",
                               "direct_launch_ms_per_step": direct_ms,
                               "direct_launch_note": "the same steps as direct sf_step calls (no graphs, kernels "
                                                     "chained by programmatic dependent launch), after the timed "
                                                     "region"},
               "roofline": roof, "gpu_launches": launches * args.steps, "step_ms_median": med_ms,
               "e2e": {"value": e2e_value, "unit": "Hz", "h2d_bytes_per_step": 2 * frame_bytes,
                       "d2h_bytes_per_step": 4 * frame_bytes,
                       "note": "sf_step_host_async per frame (pinned Y,lambda H2D + step + w,rho D2H, copies "
                               "overlapped across frames) then sf_wait; wall clock",
                       "synchronous_value": e2e_sync_value,
                       "synchronous_note": "sf_step_host: the same copies + step + stream sync per frame"},
               "device_flags": flags, "clocks": clocks}
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(seqs[0], levels=levels)
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_banded(args):
    """configs[4]: one 8192^2 frame per step, row bands over the ranks (strong scaling).
    --band-mode deep (default): each rank owns rows [o0, o1) plus halo = max(N,2)+2S rows; per
    step one NCCL halo exchange (sf_halo_exchange_nccl, 2 x halo rows of state + Yhat), then the
    fused sf_step on the band.  --band-mode substep: 2 halo rows; sf_step_banded_nccl exchanges 1
    row after every column pass and 2 rows before every box pass (N + S NCCL groups per frame) on
    the per-pass kernels (the north star's per-substep split)."""
    import torch
    import torch.distributed as dist

    import paper_2406_18031_b200 as sf
    import sfgen

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    c = sfgen.CONFIGS[5]
    H, W = c["H"], c["W"]
    cfg0 = sf.sf_config_default(H, W)
    cfg0.max_flow_px = c["max_flow"]
    cfg0.smooth_iters = 2
    substep = getattr(args, "band_mode", "deep") == "substep"
    halo = sf.sf_band_halo_substep(cfg0) if substep else sf.sf_band_halo(cfg0)
    e0, o0, o1, e1 = sf.sf_band_partition(H, world, rank, halo)
    ring = 2  # each frame is 512 MiB of inputs: 2 frames replayed palindromically already exceed L2
    geom, Yh, Dh, params = sfgen.configs.band_sequence(5, e0, e1, ring)
    Hb = e1 - e0
    Yd = torch.from_numpy(Yh.reshape(ring, 1, Hb, W)).to(dev)
    Dd = torch.from_numpy(Dh.reshape(ring, 1, Hb, W)).to(dev)
    s = torch.cuda.Stream(device=dev)
    band = (e0, o0, o1, H) if world > 1 else None
    m = sf.StructureFlow(geom, params, batch=1, device=local, stream=s, band=band)
    comm = None
    if world > 1:
        uid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(sf.sf_nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        comm = sf.sf_nccl_comm_init(world, bytes(uid.cpu().numpy()), rank)

    started = [False]

    def step(i):
        j = i % (2 * ring)
        k = j if j < ring else 2 * ring - 1 - j
        if substep and comm is not None:
            sf.sf_step_banded_nccl(m.ctx, Yd[k].data_ptr(), Dd[k].data_ptr(), comm, rank, world)
            return
        if comm is not None and started[0]:
            sf.sf_halo_exchange_nccl(m.ctx, comm, rank, world)
        m.step(Yd[k], Dd[k])
        started[0] = True

    with torch.cuda.stream(s):
        for i in range(args.warmup + 1):
            step(i)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clk, clk_path = (start_clock_sampler(local) if rank == 0 else (None, None))
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        ev0.record(s)
        for i in range(args.steps):
            step(args.warmup + 1 + i)
        ev1.record(s)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks = stop_clock_sampler(clk, clk_path) if rank == 0 else None
    t = torch.tensor([ev0.elapsed_time(ev1)], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    flags = sf.sf_status_flags(m.ctx)[1]
    if rank == 0:
        value = args.steps / (total_ms / 1e3)  # whole 8192^2 frames per second
        ops = algo_ops_per_px(params.N, params.smooth_iters) * H * W
        pk = peaks() or {}
        sm_max = pk.get("sm_max_mhz", 1965.0)
        alu_peak = world * SMS * FP32_LANES_PER_SM * sm_max * 1e6 / 1e12
        alu = ops / (total_ms / args.steps / 1e3) / 1e12
        out = {"metric": METRIC, "value": value, "unit": "Hz", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
               "config": {"workload": CONFIG_NAMES[5], "H": H, "W": W, "N": params.N, "S": params.smooth_iters,
                          "parallelism": (f"row bands x{world}, halo {halo} rows, per-substep NCCL exchange "
                                          f"({params.N + params.smooth_iters} groups / frame, per-pass kernels)"
                                          if substep and world > 1 else
                                          f"row bands x{world}, halo {halo} rows, 1 NCCL exchange / frame"),
                          "inputs": f"{ring} frames x {2 * H * W * 4 / 2**20:.0f} MiB, palindromic (> L2)"},
               "roofline": {"bound": "alu", "achieved": alu, "peak": alu_peak, "unit": "TFLOP/s",
                            "frac": alu / alu_peak, "traffic": None,
                            "kernel": "per-pass kernels + per-substep exchange" if substep and world > 1
                            else "fused step + halo exchange",
                            "peak_source": f"{world} x 148 SMs x 128 FP32 lanes x {sm_max:.0f} MHz"},
               "gpu_launches": m.launches_per_step * args.steps, "e2e": None, "device_flags": flags, "clocks": clocks}
        if world == 1 and not args.no_cpu_baseline:
            # the float32 oracle on a bounded band of the frame (the first rows rows, 1 thread), scaled
            # to whole 8192^2 frames
            import types
            rows = 256
            sq = types.SimpleNamespace(geom=geom, params=params, Y=Yh.reshape(ring, Hb, W), depth=Dh.reshape(ring, Hb, W))
            tr = oracle_frames(sq, 1, rows=rows)
            out["cpu_baseline"] = {"value": 1.0 / (tr * H / rows), "unit": "Hz", "cores": 1, "kind": "oracle",
                                   "sample": f"one frame of the first {rows} of {H} rows ({rows * W} px), float32 "
                                             f"oracle, 1 thread, scaled to whole frames ({cpu_model()})"}
        print(json.dumps(out))
    if comm is not None:
        torch.cuda.synchronize(dev)
        sf.sf_nccl_comm_destroy(comm)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["sf", "reference"], default="sf")
    ap.add_argument("--config", type=int, choices=[2, 3, 4, 5], default=2)
    ap.add_argument("--kernel", choices=["auto", "fused", "passes"], default="auto")
    ap.add_argument("--max-flow", type=float, default=None,
                    help="override the workload's max flow (px; N = ceil) -- for the paper's Table 2/3 sweeps")
    ap.add_argument("--map", action="store_true",
                    help="include the Spherepix input mapping of a 640x640 camera frame in every step (P:L785)")
    ap.add_argument("--levels", type=int, choices=[1, 2], default=1,
                    help="pyramid levels (1: the graded H = 1 hot path; 2: the paper's Table 3 shape)")
    ap.add_argument("--ring", type=int, default=96)
    ap.add_argument("--band-mode", choices=["deep", "substep"], default="deep",
                    help="--config 5 over N > 1 ranks: one deep halo exchange per frame, or the per-substep exchange")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.ring % 2:
        args.ring += 1
    if args.impl == "reference":
        return run_reference(args)
    if args.config == 5:
        return run_banded(args)
    return run_sf(args)


if __name__ == "__main__":
    sys.exit(main())
