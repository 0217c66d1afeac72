"""Row-band decomposition on CPU with torch.distributed (gloo, world size 2 and 3).

Each rank runs the float32 ORACLE on its extended band (owned rows + halo rows from
sf_band_partition / sf_band_halo, the same host functions libsf's banded mode uses),
refreshes its halo rows from the neighbouring ranks with send/recv before every frame, and
the owned rows must equal the single-process full-grid oracle bit for bit.  This checks the
decomposition logic (partition, halo size, which rows travel where) without a GPU; the GPU
path moves the same rows with NCCL or peer copies (tests/test_gpu_parity.py)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(H=72, W=40, N=3, S=2, frames=3):
    import sfgen
    from sfgen import grid
    from sfgen.configs import Params

    g = grid.gnomonic(H, W, 70.0)
    p = Params(max_flow=float(N), gamma=(3e5, 3e6, 1.0, 1.0, 2.0), smooth_iters=S)
    rng = np.random.default_rng(7)
    ds = g[..., 9][..., None]
    w = (rng.normal(size=(H, W, 3)) * 0.5 * N * ds).astype(np.float32)
    rho = rng.uniform(0.05, 0.6, (H, W)).astype(np.float32)
    yh = rng.uniform(0.1, 0.9, (H, W)).astype(np.float32)
    Ys = rng.uniform(0.1, 0.9, (frames, H, W)).astype(np.float32)
    Ds = rng.uniform(1.0, 9.0, (frames, H, W)).astype(np.float32)
    return g, p, w, rho, yh, Ys, Ds


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import oracle
    import paper_2406_18031_b200 as sf

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, p, w, rho, yh, Ys, Ds = _case()
    H = g.shape[0]
    cfg = sf.sf_config_default(H, g.shape[1])
    cfg.max_flow_px = p.max_flow
    cfg.smooth_iters = p.smooth_iters
    halo = sf.sf_band_halo(cfg)
    e0, o0, o1, e1 = sf.sf_band_partition(H, world, rank, halo)
    o = oracle.Oracle(np.ascontiguousarray(g[e0:e1]), p, "f32")
    o.set_state(w[e0:e1], rho[e0:e1], yh[e0:e1])
    parts = [sf.sf_band_partition(H, world, r, halo) for r in range(world)]
    for k in range(Ys.shape[0]):
        # halo exchange: my first / last `halo` owned rows to the neighbours, theirs into my halo
        reqs = []
        state = np.concatenate([o.w, o.rho[..., None], o.yhat[..., None]], axis=-1)  # [rows][W][5]
        recv = {}
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(state[o0 - e0:o0 - e0 + (o0 - e0)])), rank - 1))
            recv["up"] = torch.empty((o0 - e0,) + state.shape[1:], dtype=torch.float32)
            reqs.append(dist.irecv(recv["up"], rank - 1))
        if rank < world - 1:
            nb = e1 - o1
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(state[o1 - e0 - nb:o1 - e0])), rank + 1))
            recv["dn"] = torch.empty((nb,) + state.shape[1:], dtype=torch.float32)
            reqs.append(dist.irecv(recv["dn"], rank + 1))
        for r in reqs:
            r.wait()
        if "up" in recv:
            state[:o0 - e0] = recv["up"].numpy()
        if "dn" in recv:
            state[o1 - e0:] = recv["dn"].numpy()
        o.set_state(np.ascontiguousarray(state[..., :3]), np.ascontiguousarray(state[..., 3]),
                    np.ascontiguousarray(state[..., 4]))
        o.step(np.ascontiguousarray(Ys[k, e0:e1]), np.ascontiguousarray(Ds[k, e0:e1]))
    q.put((rank, o0, o1, o.w[o0 - e0:o1 - e0].copy(), o.rho[o0 - e0:o1 - e0].copy(),
           o.yhat[o0 - e0:o1 - e0].copy(), parts))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_banded_oracle_over_gloo_equals_full_grid(world):
    import oracle

    g, p, w, rho, yh, Ys, Ds = _case()
    full = oracle.Oracle(g, p, "f32")
    full.set_state(w, rho, yh)
    for k in range(Ys.shape[0]):
        full.step(Ys[k], Ds[k])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    covered = np.zeros(g.shape[0], bool)
    for rank, o0, o1, wb, rb, yb, parts in res:
        assert np.array_equal(wb, full.w[o0:o1]), rank
        assert np.array_equal(rb, full.rho[o0:o1]), rank
        assert np.array_equal(yb, full.yhat[o0:o1]), rank
        covered[o0:o1] = True
    assert covered.all()
