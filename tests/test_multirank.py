"""Multi-rank determinism of the sharded slot pipeline (
SURVEY.md §8(e)): world 2 over gloo gives BIT-IDENTICAL fixed-point sums to
world 1 on the same total id set.  The CPU test injects the oracle for the
device call; the GPU test runs the real engine (both ranks on cuda:0)."""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "_multirank_worker.py")


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _launch(world, engine, slots, out, timeout):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", WORKER, "--engine", engine, "--slots", str(slots),
           "--out", out]
    env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1")
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    return np.load(out)


def _check(tmp_path, engine, slots, timeout):
    one = _launch(1, engine, slots, str(tmp_path / "w1.npz"), timeout)
    two = _launch(2, engine, slots, str(tmp_path / "w2.npz"), timeout)
    assert int(one["n"]) == int(two["n"]) == 2 * slots
    np.testing.assert_array_equal(one["counts"], np.full(10, 2 * slots))
    np.testing.assert_array_equal(two["counts"], one["counts"])
    np.testing.assert_array_equal(two["sum_v"], one["sum_v"])
    np.testing.assert_array_equal(two["sum_v2"], one["sum_v2"])
    assert np.any(one["sum_v"] != 0)


def test_world2_gloo_bit_identical_to_world1_oracle_engine(tmp_path):
    _check(tmp_path, "oracle", 4, 600)


@pytest.mark.gpu
def test_world2_gloo_bit_identical_to_world1_gpu_engine(tmp_path):
    _check(tmp_path, "gpu", 16, 900)
