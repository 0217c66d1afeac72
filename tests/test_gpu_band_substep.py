"""Banded split with the per-substep halo exchange (north star: "row bands with a per-substep halo
exchange") driven through libsf's sf_step_banded on one GPU:

* band contexts in threads of one process, the transport a host-staged queue exchange;
* two PROCESSES on the same GPU with a gloo host-staged transport (NCCL refuses two ranks on
  one device; the rows exchanged are selected by the same library code as the NCCL transport).

Owned rows must equal a whole-grid context bit for bit, flags included; the whole-grid context
itself is checked against the float32 oracle on the small grid.
"""
import ctypes as C
import os
import queue
import socket
import threading

import numpy as np
import pytest

import oracle
from sfgen import grid
from sfgen.configs import Params

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")]


def _sf():
    import paper_2406_18031_b200 as sf
    return sf


def _problem(H, W, N, S, frames, seed):
    g = grid.gnomonic(H, W, 80.0)
    p = Params(max_flow=float(N) - 0.25, gamma=(3e5, 3e6, 1.0, 1.0, 2.0), smooth_iters=S)
    rng = np.random.default_rng(seed)
    ds = g[..., 9][None, ..., None]
    w = (rng.normal(size=(1, H, W, 3)) * 0.5 * N * ds).astype(np.float32)
    rho = rng.uniform(0.05, 0.6, (1, H, W)).astype(np.float32)
    yh = rng.uniform(0.1, 0.9, (1, H, W)).astype(np.float32)
    Ys = rng.uniform(0.1, 0.9, (frames, 1, H, W)).astype(np.float32)
    Ds = rng.uniform(1.0, 9.0, (frames, 1, H, W)).astype(np.float32)
    Ds[:, :, ::11, ::7] = np.nan
    return g, p, w, rho, yh, Ys, Ds


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _fields(m):
    w, rho, yh = m.get_fields()
    torch.cuda.synchronize()
    return w.cpu().numpy(), rho.cpu().numpy(), yh.cpu().numpy()


def _full_run(g, p, w, rho, yh, Ys, Ds, check_oracle=False):
    sf = _sf()
    full = sf.StructureFlow(g, p)
    full.set_fields(_dev(w), _dev(rho), _dev(yh))
    o = None
    if check_oracle:
        o = oracle.Oracle(g, p, "f32")
        o.set_state(w[0], rho[0], yh[0])
    for k in range(len(Ys)):
        full.step(_dev(Ys[k]), _dev(Ds[k]))
        if o is not None:
            o.step(Ys[k][0], Ds[k][0])
    ref = _fields(full)
    if o is not None:
        for x, y in zip(ref, (o.w, o.rho, o.yhat)):
            assert np.array_equal(x[0], y)
    return ref, sf.sf_status_flags(full.ctx)[1]


def _host(addr, n):
    return np.ctypeslib.as_array((C.c_float * n).from_address(addr))


@pytest.mark.parametrize("H,W,nb,N,S", [(150, 61, 3, 8, 2), (97, 130, 2, 5, 1), (64, 48, 4, 2, 3)])
def test_banded_substep_threads_equal_single_context(H, W, nb, N, S):
    """nb band contexts, one thread each, per-substep exchange through queues (host-staged):
    owned rows bitwise the whole-grid context (itself bitwise the oracle), flags equal."""
    sf = _sf()
    frames = 3
    g, p, w, rho, yh, Ys, Ds = _problem(H, W, N, S, frames, H + W + nb)
    ref, ref_flags = _full_run(g, p, w, rho, yh, Ys, Ds, check_oracle=True)
    halo = 2
    parts = [sf.sf_band_partition(H, nb, b, halo) for b in range(nb)]
    # channel[(src, dst)]: rows band src sends to band dst
    chan = {(a, b): queue.Queue() for a in range(nb) for b in range(nb) if abs(a - b) == 1}
    results, errors = [None] * nb, []

    def run(b):
        try:
            e0, o0, o1, e1 = parts[b]
            torch.cuda.set_device(0)
            stream = torch.cuda.Stream()
            m = sf.StructureFlow(g[e0:e1], p, stream=stream, band=(e0, o0, o1, H))
            with torch.cuda.stream(stream):
                m.set_fields(_dev(w[:, e0:e1]), _dev(rho[:, e0:e1]), _dev(yh[:, e0:e1]))

            def xfer(su, ru, sd, rd, nu, nd):
                if su:
                    chan[(b, b - 1)].put(_host(su, nu).copy())
                if sd:
                    chan[(b, b + 1)].put(_host(sd, nd).copy())
                if ru:
                    _host(ru, nu)[:] = chan[(b - 1, b)].get(timeout=60)
                if rd:
                    _host(rd, nd)[:] = chan[(b + 1, b)].get(timeout=60)

            for k in range(frames):
                with torch.cuda.stream(stream):
                    Yb, Db = _dev(Ys[k][:, e0:e1]), _dev(Ds[k][:, e0:e1])
                    stream.synchronize()
                    sf.sf_step_banded(m.ctx, Yb.data_ptr(), Db.data_ptr(), xfer, host_staged=1)
            stream.synchronize()
            results[b] = (_fields(m), sf.sf_status_flags(m.ctx)[1])
        except Exception as ex:  # surfaced in the main thread
            errors.append(repr(ex))

    th = [threading.Thread(target=run, args=(b,)) for b in range(nb)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errors, errors
    fl = 0
    for b, (e0, o0, o1, e1) in enumerate(parts):
        got, flags = results[b]
        fl |= flags
        for name, x, y in zip(("w", "rho", "yhat"), ref, got):
            assert np.array_equal(y[:, o0 - e0:o1 - e0], x[:, o0:o1]), (name, b)
    assert fl == ref_flags


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, H, W, N, S, frames, out_dir):
    import torch.distributed as dist

    import paper_2406_18031_b200 as sf

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    g, p, w, rho, yh, Ys, Ds = _problem(H, W, N, S, frames, 7)
    e0, o0, o1, e1 = sf.sf_band_partition(H, world, rank, 2)
    m = sf.StructureFlow(g[e0:e1], p, band=(e0, o0, o1, H))
    m.set_fields(_dev(w[:, e0:e1]), _dev(rho[:, e0:e1]), _dev(yh[:, e0:e1]))

    def xfer(su, ru, sd, rd, nu, nd):
        ops = []
        if su:
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(_host(su, nu).copy()), rank - 1))
        if sd:
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(_host(sd, nd).copy()), rank + 1))
        bu = torch.empty(nu) if ru else None
        bd = torch.empty(nd) if rd else None
        if ru:
            ops.append(dist.P2POp(dist.irecv, bu, rank - 1))
        if rd:
            ops.append(dist.P2POp(dist.irecv, bd, rank + 1))
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        if ru:
            _host(ru, nu)[:] = bu.numpy()
        if rd:
            _host(rd, nd)[:] = bd.numpy()

    for k in range(frames):
        Yb, Db = _dev(Ys[k][:, e0:e1]), _dev(Ds[k][:, e0:e1])
        torch.cuda.synchronize()
        sf.sf_step_banded(m.ctx, Yb.data_ptr(), Db.data_ptr(), xfer, host_staged=1)
    got = _fields(m)
    np.savez(os.path.join(out_dir, f"band{rank}.npz"), w=got[0], rho=got[1], yh=got[2],
             flags=np.array([sf.sf_status_flags(m.ctx)[1]]), rows=np.array([e0, o0, o1, e1]))
    dist.barrier()
    dist.destroy_process_group()


def test_banded_substep_two_processes_gloo(tmp_path):
    """Two processes on one GPU (ranks = bands), gloo host-staged transport: each process's owned
    rows equal the whole-grid context bit for bit after 3 frames (N = 8, S = 2), flags equal."""
    import torch.multiprocessing as mp

    H, W, N, S, frames = 120, 72, 8, 2, 3
    g, p, w, rho, yh, Ys, Ds = _problem(H, W, N, S, frames, 7)
    ref, ref_flags = _full_run(g, p, w, rho, yh, Ys, Ds)
    mp.start_processes(_gloo_worker, args=(2, _free_port(), H, W, N, S, frames, str(tmp_path)), nprocs=2,
                       join=True, start_method="spawn")
    fl = 0
    for rank in range(2):
        d = np.load(tmp_path / f"band{rank}.npz")
        e0, o0, o1, e1 = d["rows"]
        fl |= int(d["flags"][0])
        for x, y in zip(ref, (d["w"], d["rho"], d["yh"])):
            assert np.array_equal(y[:, o0 - e0:o1 - e0], x[:, o0:o1]), rank
    assert fl == ref_flags
