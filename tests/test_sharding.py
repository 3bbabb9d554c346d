"""Multi-rank time sharding (gloo, world size 2 and 3, CPU): the host logic
of paper_2108_07126_b200.sharding — partition, halo rows, global validation,
all-gather and ordered product — reproduces the unsharded oracle.  The
per-rank block compute is injected (the oracle) because this tier has no GPU;
the GPU block path is covered by tests/test_sharding_gpu.py."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from cases import qubit_inputs, random_inputs

from paper_2108_07126_b200.sharding import ordered_product, partition, shard_rows


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_partition_and_rows():
    assert partition(10, 3) == [(0, 3), (3, 6), (6, 10)]
    assert partition(2, 4) == [(0, 0), (0, 1), (1, 1), (1, 2)]
    assert shard_rows("midpoint", 3, 6) == (3, 6)
    # slice j reads rows 2j..2j+2: slices [3, 6) read rows 6..12 inclusive
    assert shard_rows("simpson", 3, 6) == (6, 13)
    assert shard_rows("magnus", 2, 2) == (0, 0)


def test_ordered_product_orders():
    rng = np.random.default_rng(3)
    mats = [rng.standard_normal((3, 3)) + 1j * rng.standard_normal((3, 3)) for _ in range(5)]
    seq = mats[4] @ mats[3] @ mats[2] @ mats[1] @ mats[0]
    assert np.allclose(ordered_product(mats, "sequential"), seq)
    assert np.allclose(ordered_product(mats, "pairwise"), seq)


def _worker(rank, world, port, mode, case, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import paper_2108_07126_b200 as sp
    from paper_2108_07126_b200.sharding import equiprop_sharded
    dist.init_process_group("gloo", rank=rank, world_size=world)
    h0, hs, values, dt = case
    ctx = sp.create()
    ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=mode == "magnus",
                        quadrature=None if mode == "magnus" else mode)
    amps = sp.ControlAmplitudes(values, dt)

    def block(sub):
        u, _, _ = oracle.equiprop(h0, hs, sub.values, dt, mode=mode)
        return u

    res = equiprop_sharded(ctx, amps, block_fn=block)
    np.save(f"{result_path}.{rank}.npy", res.u)
    # a bad sample on any rank raises on every rank (no collective deadlock)
    bad = values.copy()
    bad[-1, 0] = 2.0
    try:
        equiprop_sharded(ctx, sp.ControlAmplitudes(bad, dt), block_fn=block)
        raise SystemExit(3)
    except sp.AmplitudeBoundError:
        pass
    dist.destroy_process_group()


@pytest.mark.parametrize("world,mode,kind", [(2, "midpoint", "qubit"), (2, "magnus", "qubit"),
                                             (3, "simpson", "random"), (2, "midpoint", "random")])
def test_sharded_matches_unsharded(tmp_path, world, mode, kind):
    if kind == "qubit":
        case = qubit_inputs(201 if mode != "midpoint" else 200, mode)
    else:
        case = random_inputs(6, 2, 41, 5)
    path = str(tmp_path / "u")
    mp.spawn(_worker, args=(world, _free_port(), mode, case, path), nprocs=world, join=True)
    h0, hs, values, dt = case
    ref, _, _ = oracle.equiprop(h0, hs, values, dt, mode=mode)
    for r in range(world):
        u = np.load(f"{path}.{r}.npy")
        assert np.linalg.norm(u - ref) / np.linalg.norm(ref) <= 1e-12
