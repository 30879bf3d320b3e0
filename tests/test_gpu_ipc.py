"""The cross-PROCESS combine on one GPU: R processes, each
its own CUDA context on cuda:0, exchange their mailbox handles through a gloo
process group (Comm.from_process_group: jf_comm_create / export / connect with
real cudaIpcOpenMemHandle) and run a sharded pass and a sharded fit of one
image.  Every rank must return the identical result, equal to the oracle
(pass: 1e-10 normalised) and to the single-process fit (counts, x to 1e-6)."""
import os
import socket

import numpy as np
import pytest

import datagen as dg

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


W, H, SEED = 384, 385, 15


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    import paper_2208_12187_b200 as jf
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    pr = dg.make_gauss2d(W, H=H, seed=SEED)
    r0, r1 = dg.shard_rows(H, world, rank)
    z = torch.as_tensor(pr.z[r0 * W:r1 * W]).cuda()
    comm = jf.Comm.from_process_group(rank, world, 0, dist)
    comm.set_timeout(30000)
    torch.cuda.synchronize()
    dist.barrier()
    p = jf.jpass(pr.model, z, pr.p0, grid=(W, r1 - r0, r0), comm=comm, m_global=pr.m)
    f = jf.curve_fit(pr.model, z, p0=pr.p0, grid=(W, r1 - r0, r0), comm=comm, m_global=0)
    sm, us = comm.bench(float(rank + 1), reps=200)
    dist.barrier()
    comm.destroy()
    out[rank] = (p[0], p[1], p[2], p[3], f.status, f.nfev, f.njev, f.nit, f.x, f.cost, sm, us)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_cross_process_ipc_combine(world):
    import torch.multiprocessing as mp
    from oracle import passes as orp
    import paper_2208_12187_b200 as jf
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    pr = dg.make_gauss2d(W, H=H, seed=SEED)
    cr, gr, Gr, _ = orp.jpass(pr.model, pr.coords(), pr.z, pr.p0)
    d = np.sqrt(np.diag(Gr))
    ref = jf.curve_fit(pr.model, pr.z, p0=pr.p0, grid=pr.grid)
    for r in range(world):
        c, g, G, bad, st, nfev, njev, nit, x, cost, sm, us = out[r]
        assert bad == 0 and abs(c - cr) <= 1e-10 * cr
        assert np.all(np.abs(g - gr) <= 1e-10 * d * np.sqrt(2 * cr))
        assert np.all(np.abs(G - Gr) <= 1e-10 * np.outer(d, d))
        assert (st, nfev, njev, nit) == (ref.status, ref.nfev, ref.njev, ref.nit)
        assert np.allclose(x, ref.x, rtol=1e-6)
        assert sm == world * (world + 1) / 2
        assert np.array_equal(x, out[0][8]) and cost == out[0][9]
        print(f"rank {r}: combine {us:.2f} us over {world} processes")
