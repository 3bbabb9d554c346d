"""Device path of the time sharding on one B200: NCCL process group of size
1, sp_product_device ordered products, and the halo-sliced per-rank blocks
recombined on the device reproduce the unsharded propagation."""

import os
import socket

import numpy as np
import pytest

import paper_2108_07126_b200 as sp
from cases import qubit_inputs, random_inputs
from helpers import haar_unitary

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("reduction", ["pairwise", "sequential"])
@pytest.mark.parametrize("d,count", [(2, 1), (2, 9), (5, 7), (32, 8), (128, 3)])
def test_product_device(rng, d, count, reduction):
    import torch
    mats = np.stack([haar_unitary(rng, d) for _ in range(count)])
    ctx = sp.create()
    ctx.set_hamiltonian(sp.ControlSystem(np.zeros((d, d))))
    dm = torch.from_numpy(mats).cuda()
    out = torch.empty((d, d), dtype=torch.complex128, device="cuda")
    ctx.product_device_ptr(count, dm.data_ptr(), out.data_ptr(), reduction=reduction)
    torch.cuda.synchronize()
    ref = np.eye(d, dtype=complex)
    for m in mats:
        ref = m @ ref
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-13


@pytest.mark.parametrize("mode,case", [("midpoint", random_inputs(128, 4, 64, 9)),
                                       ("magnus", qubit_inputs(2001, "magnus")),
                                       ("simpson", random_inputs(32, 2, 257, 10))])
def test_blocks_recombine_on_device(mode, case):
    """Emulate P = 4 ranks on one GPU: per-rank halo-sliced blocks, ordered
    product on the device, equal to the unsharded result."""
    import torch
    from paper_2108_07126_b200.sharding import partition, shard_rows
    h0, hs, values, dt = case
    ctx = sp.create()
    ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=mode == "magnus",
                        quadrature=None if mode == "magnus" else mode)
    full = ctx.equiprop(sp.ControlAmplitudes(values, dt)).u
    n = ctx.slice_count(values.shape[0])
    d = h0.shape[0]
    plan = ctx.plan_for(dt)
    blocks = torch.empty((4, d, d), dtype=torch.complex128, device="cuda")
    for r, (a, b) in enumerate(partition(n, 4)):
        lo, hi = shard_rows(ctx.mode, a, b)
        loc = torch.from_numpy(np.ascontiguousarray(values[lo:hi])).cuda()
        ctx.equiprop_device_ptr(loc.data_ptr(), hi - lo, len(hs), dt, blocks[r].data_ptr(),
                                plan=plan)
    out = torch.empty((d, d), dtype=torch.complex128, device="cuda")
    ctx.product_device_ptr(4, blocks.data_ptr(), out.data_ptr())
    torch.cuda.synchronize()
    assert np.linalg.norm(out.cpu().numpy() - full) / np.linalg.norm(full) <= 1e-12


def test_nccl_world_of_one():
    import torch
    import torch.distributed as dist
    from paper_2108_07126_b200.sharding import equiprop_sharded_device
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        h0, hs, values, dt = random_inputs(64, 2, 100, 11)
        ctx = sp.create()
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
        ref = ctx.equiprop(sp.ControlAmplitudes(values, dt)).u
        out, plan, n = equiprop_sharded_device(ctx, torch.from_numpy(values).cuda(), dt, 100)
        torch.cuda.synchronize()
        assert np.linalg.norm(out.cpu().numpy() - ref) / np.linalg.norm(ref) <= 1e-13
    finally:
        dist.destroy_process_group()


def _world_of_one():
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    return dist


def test_sharded_device_fp32_and_side_stream():
    """complex64 contexts through the device sharded path (block in the
    working dtype, gathered as complex128, result complex64) on a
    non-current stream (stream ordering of the collective)."""
    import torch
    from paper_2108_07126_b200.sharding import equiprop_sharded_device
    dist = _world_of_one()
    try:
        h0, hs, values, dt = random_inputs(4, 2, 300, 21)
        ctx = sp.create(precision="fp32")
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
        ref = ctx.equiprop(sp.ControlAmplitudes(values, dt)).u
        side = torch.cuda.Stream()
        out, _, _ = equiprop_sharded_device(ctx, torch.from_numpy(values).cuda(), dt, 300,
                                            stream=side)
        side.synchronize()
        got = out.cpu().numpy()
        assert got.dtype == np.complex64
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-6
    finally:
        dist.destroy_process_group()


def test_sharded_device_validates_before_the_gather():
    import torch
    from paper_2108_07126_b200.sharding import equiprop_sharded_device
    dist = _world_of_one()
    try:
        h0, hs, values, dt = random_inputs(8, 2, 100, 22)
        values = values.copy()
        values[37, 1] = 3.0
        ctx = sp.create()
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
        with pytest.raises(sp.AmplitudeBoundError) as exc:
            equiprop_sharded_device(ctx, torch.from_numpy(values).cuda(), dt, 100)
        assert "sample 37, control 1" in str(exc.value)
    finally:
        dist.destroy_process_group()


def test_two_ranks_raise_the_same_violation():
    """gloo world of 2 folded onto one GPU (torchrun): the bad sample sits in
    rank 1's shard, and BOTH ranks raise the same AmplitudeBoundError instead
    of rank 0 blocking in the gather."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", str(_free_port()),
                        os.path.join(root, "tests", "_sharded_worker.py")],
                       cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    import re
    found = dict(re.findall(r"RANK(\d):(control amplitude .*?lies outside \[-1, 1\]|no error)",
                            r.stdout))
    assert set(found) == {"0", "1"}, r.stdout
    assert found["0"] == found["1"] and "sample 70, control 0" in found["0"]
