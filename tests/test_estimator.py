"""Estimator and the multi-rank reduction (gloo, world 2)."""

import math
import os

import numpy as np
import pytest

import paper_2604_13144_b200 as tb
from paper_2604_13144_b200.estimator import FIX, SampleRecord, aggregate, aggregate_fixed, quantize


def test_spec_examples():
    r = aggregate([SampleRecord(0, 1, 2.0, 1.0), SampleRecord(1, -1, 2.0, 1.0)])
    assert r.mean == 0.0
    assert r.var_o == pytest.approx(4 * r.var_v) and r.var_v == pytest.approx(2.0)
    same = aggregate([SampleRecord(i, 1, 1.0, 0.3) for i in range(5)])
    assert same.var_o == 0.0 and same.mean == pytest.approx(0.3)
    with pytest.raises(ValueError):
        aggregate([])
    with pytest.raises(ValueError):
        aggregate([SampleRecord(0, 1, 1.0, 0.1), SampleRecord(1, 1, 1.5, 0.1)])


def test_fixed_point_matches_float_statistics():
    rng = np.random.default_rng(0)
    vals = rng.uniform(-1, 1, size=(500, 3, 4))
    signs = rng.choice([-1, 1], size=(500, 3, 1))
    g = np.array([1.1, 1.3, 1.7])
    sv = quantize(signs * vals).sum(axis=0)
    sv2 = quantize(vals**2).sum(axis=0)
    st = aggregate_fixed(sv, sv2, 500, g)
    v = signs * vals
    np.testing.assert_allclose(st["estimate"], g[:, None] * v.mean(axis=0), atol=1e-12)
    np.testing.assert_allclose(st["var_v"], v.var(axis=0, ddof=1), atol=1e-10)
    np.testing.assert_allclose(st["var_o"], g[:, None] ** 2 * st["var_v"], rtol=1e-15)
    rec = aggregate([SampleRecord(i, int(signs[i, 0, 0]), g[0], vals[i, 0, 0]) for i in range(500)])
    assert rec.mean == pytest.approx(st["estimate"][0, 0], abs=1e-12)
    assert rec.var_o == pytest.approx(st["var_o"][0, 0], rel=1e-9)


def test_partial_sums_are_order_and_shard_independent():
    rng = np.random.default_rng(1)
    v = rng.uniform(-1, 1, size=(1000, 2))
    q = quantize(v)
    full = q.sum(axis=0)
    for world in (1, 2, 4, 8):
        parts = [q[tb.shard_range(1000, r, world).start: tb.shard_range(1000, r, world).stop].sum(axis=0)
                 for r in range(world)]
        assert np.array_equal(np.sum(parts[::-1], axis=0), full)
    assert abs(full[0] / FIX - v[:, 0].sum()) < 1000 * 2.0**-41


def test_shard_range_covers_everything():
    for n in (0, 1, 7, 100001):
        for w in (1, 2, 3, 8):
            ids = [i for r in range(w) for i in tb.shard_range(n, r, w)]
            assert ids == list(range(n))


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(7)
    v = rng.uniform(-1, 1, size=(101, 2, 3))
    ids = tb.shard_range(101, rank, world)
    local = v[ids.start: ids.stop]
    run = tb.EnsembleRun(len(ids), None, None, None, quantize(local).sum(axis=0), quantize(local**2).sum(axis=0),
                         np.ones(2), 0.0, 0.0, 0.0)
    red = tb.allreduce_sums(run)
    if rank == 0:
        out.put((red.n_samples, red.sum_v.tolist(), quantize(v).sum(axis=0).tolist()))
    dist.destroy_process_group()


def test_gloo_world2_allreduce_is_exact():
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 2000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ns, got, want = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert ns == 101 and got == want


def _bcast_worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    st = None
    if rank == 0:
        st = tb.MPSState(3)
        st.ensure_capacity(2)
        st.dims = np.array([1, 2, 2, 1])
        st.buf[:] = np.arange(st.buf.size).reshape(st.buf.shape) * (1 + 0.5j)
        st.center = 1
        st.discarded_weight = 1e-9
    got = tb.broadcast_state(st, 0)
    if rank == 1:
        out.put((got.bond_dims, got.center, got.discarded_weight, [t.tolist() for t in got.tensors]))
    else:
        out.put(("src", st.bond_dims, [t.tolist() for t in st.tensors]))
    dist.destroy_process_group()


def test_gloo_world2_snapshot_broadcast():
    """Config-5 fan-out: the t0 MPS reaches every rank intact (snapshot format)."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31500 + (os.getpid() % 2000)
    procs = [ctx.Process(target=_bcast_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120), q.get(timeout=120)]
    for p in procs:
        p.join(timeout=60)
    src = [r for r in res if r[0] == "src"][0]
    dst = [r for r in res if r[0] != "src"][0]
    assert dst[0] == src[1] and dst[1] == 1 and dst[2] == 1e-9 and dst[3] == src[2]
