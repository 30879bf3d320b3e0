"""Multi-rank host logic on CPU (gloo, world_size 2): the row-band partition
used by bench.py and the sharded fit, the handle exchange used by
Comm.from_process_group, and the identity the in-kernel cross-rank combine
relies on — the K-vector of the whole image is the rank-order sum of the
shards' K-vectors (checked with the oracle's passes)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import datagen as dg


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    from oracle import passes as orp
    from paper_2208_12187_b200.api import exchange_handles
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    W, H = 64, 45
    pr = dg.make_gauss2d(W, H=H, seed=9)
    r0, r1 = dg.shard_rows(H, world, rank)
    X, Y = dg.grid_coords(W, r1 - r0, r0)
    c, g, G, bad = orp.jpass(pr.model, (X, Y), pr.z[r0 * W:r1 * W], pr.p0)
    vec = torch.tensor(np.concatenate([[c], g, G.ravel(), [bad]]), dtype=torch.float64)
    parts = [torch.zeros_like(vec) for _ in range(world)]
    dist.all_gather(parts, vec)
    blob = bytes([rank]) * 256
    allb = exchange_handles(blob, dist)
    out[rank] = (r0, r1, [p.numpy() for p in parts], allb)
    dist.destroy_process_group()


def test_two_rank_partition_and_exchange():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    bands = sorted((out[r][0], out[r][1]) for r in range(world))
    assert bands[0][0] == 0 and bands[-1][1] == 45 and bands[0][1] == bands[1][0]
    for r in range(world):
        assert out[r][3] == bytes([0]) * 256 + bytes([1]) * 256
    from oracle import passes as orp
    pr = dg.make_gauss2d(64, H=45, seed=9)
    c, g, G, bad = orp.jpass(pr.model, pr.coords(), pr.z, pr.p0)
    full = np.concatenate([[c], g, G.ravel(), [bad]])
    summed = out[0][2][0] + out[0][2][1]
    assert np.allclose(summed, full, rtol=1e-13, atol=0)
    assert np.array_equal(out[0][2][0], out[1][2][0])


def test_shard_helpers_cover_exactly():
    for H in (1, 7, 4096, 8191):
        for R in (1, 2, 3, 8):
            bands = [dg.shard_rows(H, R, k) for k in range(R)]
            assert bands[0][0] == 0 and bands[-1][1] == H
            assert all(bands[k][1] == bands[k + 1][0] for k in range(R - 1))


def _run_ref(env_extra):
    import subprocess
    import sys
    import json
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, env=env, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    return [json.loads(ln) for ln in lines]


def test_reference_arm_rank_nonzero_is_silent():
    """bench.py --impl reference under torchrun: ranks other than 0 exit 0 without work or output."""
    assert _run_ref({"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"}) == []


def test_reference_arm_line_at_n2_carries_the_c5_metric():
    """At N > 1 the reference arm reports our arm's metric (C5 row bands, n = 13) with the contract keys."""
    (d,) = _run_ref({"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert "n=13, C5 row bands" in d["metric"] and d["unit"] == "points/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
