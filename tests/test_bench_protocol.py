"""bench.py's measurement protocol on the CPU: the capacity search (the
reference's capacity rule, inc/simulator.hpp:804-820: largest offered rate
with on-time >= 0.90), the timed-region step-down, and the N > 1 metric
reductions over gloo at world size 2 (the same code path NCCL takes on the
GPU box, with CPU tensors)."""
import os
import socket
import sys
from pathlib import Path

import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def knee(cap):
    """A served-on-time curve with its 0.90 crossing at `cap`."""
    return lambda rate, i: 1.0 if rate <= cap else max(0.0, 0.9 - (rate - cap) / cap)


@pytest.mark.parametrize("cap,est", [(45000.0, 50000.0), (45000.0, 200000.0), (45000.0, 9000.0), (107000.0, 122000.0)])
def test_capacity_search_brackets_the_knee(cap, est):
    rate, runs = bench.capacity_search(knee(cap), est, min_runs=4)
    assert rate <= cap  # never reports a rate that missed the bar
    assert rate >= 0.94 * cap  # bisection to within 6%
    assert len(runs) >= 4 and len(runs) <= 14
    assert all((r <= cap) == (x >= 0.90) for r, x in runs)


def test_capacity_search_never_passing_returns_lowest_probe():
    rate, runs = bench.capacity_search(lambda r, i: 0.0, 1000.0, min_runs=3)
    assert len(runs) == 14 and rate == runs[-1][0] * 0.6


def test_step_down_is_proportional_to_the_miss():
    assert bench.step_down(1000.0, 0.85) == pytest.approx(960.0)
    assert bench.step_down(1000.0, 0.6) == pytest.approx(850.0)
    assert bench.step_down(1000.0, 0.1) == pytest.approx(700.0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _reduce_worker(rank, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE="2",
                      BENCH_DIST_BACKEND="gloo")
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method="env://")
    # per-rank values as in run_ours: served counts summed, device time maxed
    s = bench.allreduce_sum(100.0 + rank, 2)
    m = bench.allreduce_max(7.0 * (rank + 1), 2)
    bench.barrier(2)
    out[rank] = (s, m)
    dist.destroy_process_group()


def test_metric_reductions_world2_gloo():
    port = _free_port()
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        ps = [ctx.Process(target=_reduce_worker, args=(r, port, out)) for r in range(2)]
        for p in ps:
            p.start()
        for p in ps:
            p.join(120)
            assert p.exitcode == 0
        assert out[0] == out[1] == (201.0, 14.0)
