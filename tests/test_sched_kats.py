"""The reference's hand-computed known-answer tests, restated against
libbs_host.so (each cites the Catch2 case it follows under
/root/reference/proj/tests/)."""
import math

import pytest

from paper_2304_09961_b200 import scheduler as bs
from paper_2304_09961_b200.scheduler import make_request as R

TWO = bs.uniform_profile(2, [(1, 10.0), (2, 12.0)], 90)        # test_dp_scheduler.cpp:11-13
TWO_1013 = bs.uniform_profile(2, [(1, 10.0), (2, 13.0)], 90)   # test_deadline.cpp two_layer_1013


# ---------------------------------------------------------------- sweep (test_dp_scheduler.cpp:17-51)
def test_sweep_single_request():
    s = bs.segment_duration([1], TWO, 0, 90)
    assert s.duration == 20.0 and s.max_layer_batch == 1


def test_sweep_two_requests_batched():
    s = bs.segment_duration([1, 1], TWO, 0, 90)
    assert s.duration == 24.0 and s.max_layer_batch == 2


def test_sweep_deeper_member_joins():
    s = bs.segment_duration([2, 1], TWO, 0, 90)
    assert s.start_layer == 1 and s.duration == 22.0 and s.layer_batch == [1, 2]


def test_sweep_bound_violation_infeasible():
    s = bs.segment_duration([1, 1, 1], TWO, 0, 2)
    assert not s.feasible and s.duration == math.inf


# ------------------------------------------------------------- DP (test_dp_scheduler.cpp:53-79, 225-283)
def test_merge_beats_split():
    s = bs.compute_schedule([R(1, 0.0, 1), R(2, 0.0, 1)], TWO, 0, 90)
    assert len(s.segments) == 1 and s.objective == 48.0 and s.total_duration == 24.0
    assert s.offset_of(1) == 24.0 and s.offset_of(2) == 24.0


def test_split_wins_when_earlier_nearly_done():
    s = bs.compute_schedule([R(1, 0.0, 2), R(2, 1.0, 1)], TWO, 0, 90)
    assert len(s.segments) == 2 and s.objective == 40.0
    assert s.segments[0].members == [1] and s.offset_of(1) == 10.0 and s.offset_of(2) == 30.0


def test_single_request():
    assert bs.compute_schedule([R(1, 0.0, 1)], TWO, 0, 90).objective == 20.0


def test_unusable_bound_names_layer():
    with pytest.raises(RuntimeError, match="layer"):
        bs.compute_schedule([R(1, 0.0, 1), R(2, 1.0, 1)], TWO, 0, 0)


def test_no_batch_baseline():
    s = bs.baseline_no_batch([R(1, 0.0, 1), R(2, 0.0, 1)], TWO)
    assert len(s.segments) == 2 and s.offset_of(1) == 20.0 and s.offset_of(2) == 40.0 and s.objective == 60.0


def test_batch_baseline_fills_to_bound():
    s = bs.baseline_batch([R(1, 0.0, 1), R(2, 1.0, 1), R(3, 2.0, 1)], TWO, 2)
    assert [g.members for g in s.segments] == [[1, 2], [3]]


def test_granularity_nesting():
    # full <= layer <= group on a batching-friendly instance (test_dp_scheduler.cpp:128-200)
    ps = bs.uniform_profile(5, [(1, 10.0), (2, 11.0), (4, 12.0), (8, 14.0)], 8)
    reqs = [R(1, 0.0, 5), R(2, 1.0, 4), R(3, 2.0, 4), R(4, 3.0, 2), R(5, 4.0, 1), R(6, 5.0, 1)]
    full = bs.compute_schedule(reqs, ps, 0, 8).objective
    layer = bs.compute_schedule_layer_units(reqs, ps, 0, 8).objective
    group = bs.compute_schedule_grouped(reqs, ps, 0, 8, 2).objective
    assert full <= layer <= group


# -------------------------------------------------------- EDF / tardy (test_deadline.cpp:53-73,137-177)
def test_edf_batches_loose_deadlines():
    s = bs.edf_batch([R(1, 0.0, 1, 500.0), R(2, 0.0, 1, 600.0)], TWO_1013, 90, 0.0)
    assert len(s.segments) == 1 and len(s.segments[0].members) == 2 and s.tardy_count == 0


def test_edf_keeps_tight_job_alone():
    s = bs.edf_batch([R(1, 0.0, 1, 25.0), R(2, 0.0, 1, 1000.0)], TWO_1013, 90, 0.0)
    assert [g.members for g in s.segments] == [[1], [2]]
    assert s.segments[0].finish_offset == 20.0 and s.segments[1].finish_offset == 40.0 and s.tardy_count == 0


def test_edf_empty():
    s = bs.edf_batch([], TWO_1013, 90, 0.0)
    assert s.segments == [] and s.objective == 0.0


def test_tardy_without_deadlines_equals_time_dp():
    reqs = [R(1, 0.0, 2), R(2, 1.0, 1), R(3, 2.0, 1)]
    t = bs.tardy_dp(reqs, TWO, 0, 3, 0.0)
    assert t.tardy_count == 0 and t.objective == bs.compute_schedule(reqs, TWO, 0, 3).objective


def test_tardy_marks_predicted_late_for_drop():
    reqs = [R(1, 0.0, 1, 15.0), R(2, 1.0, 1, 100.0)]
    t = bs.tardy_dp(reqs, TWO_1013, 0, 90, 0.0)
    assert t.tardy_count == 1 and t.drop_marks == [1]


# -------------------------------------------------------- cost model (test_cost_profile.cpp:8-48)
def test_lookup_exact_interp_bound():
    ps = bs.uniform_profile(1, [(1, 10.0), (10, 12.0)], 90)
    row = bs.lookup_table(ps, 0, 90)[0]
    assert row[0] == 10.0 and row[9] == 12.0
    assert abs(row[3] - (10.0 + 2.0 * 3.0 / 9.0)) < 1e-12
    assert row[90] == math.inf  # b = 91 > bound


def test_group_layers_equal_runtime():
    ps = bs.profile_from_grids([[(1, 1.0)], [(1, 1.0)], [(1, 1.0)], [(1, 1.0)]], 90)
    assert bs.group_layers(ps, 0, 2) == [(1, 2), (3, 4)]
    with pytest.raises(ValueError):
        bs.group_layers(ps, 0, 5)


# --------------------------------------------------------- multi-DNN (test_multidnn.cpp:179-232)
SHARED = {"max_batch": 90,
          "components": [{"id": "flow", "layers": [{"runtime_ms": [[1, 10.0], [2, 11.0], [3, 12.0], [4, 13.0]]}] * 2},
                         {"id": "head_a", "layers": [{"runtime_ms": [[1, 2.0], [2, 2.2], [3, 2.4], [4, 2.6]]}]},
                         {"id": "head_b", "layers": [{"runtime_ms": [[1, 2.0], [2, 2.2], [3, 2.4], [4, 2.6]]}]}],
          "dnns": [{"id": "task_a", "stages": ["flow", "head_a"]}, {"id": "task_b", "stages": ["flow", "head_b"]}]}


def test_shared_prefix_batching_beats_plain():
    reqs = [R(1, 0.0, 1, dnn=0), R(2, 1.0, 1, dnn=1), R(3, 2.0, 1, dnn=0), R(4, 3.0, 1, dnn=1)]
    plain = bs.schedule_multi(reqs, SHARED, 90)
    shared = bs.schedule_multi_shared(reqs, SHARED, 90)
    assert shared.objective < plain.objective
    assert any(seg.riders for seg in shared.segments)


def test_permutation_guard():
    ps = {"max_batch": 4, "components": [{"id": f"c{d}", "layers": [{"runtime_ms": [[1, 5.0], [2, 6.0]]}] * 2}
                                         for d in range(7)],
          "dnns": [{"id": f"m{d}", "stages": [f"c{d}"]} for d in range(7)]}
    reqs = [R(d + 1, float(d), 1, dnn=d) for d in range(7)]
    with pytest.raises(RuntimeError):
        bs.schedule_multi(reqs, ps, 4, guard=6, heuristic=False)
    bs.schedule_multi(reqs, ps, 4, guard=6, heuristic=True)


# -------------------------------------------------- RNG / workload (test_workload_net.cpp:9-40)
def test_splitmix64_golden_sequence():
    # draws() consumes several values per row; check the raw u64 stream.
    d = bs.SplitMix64.draws(42, count=1)
    assert d[0][0] == 0xBDD732262FEB6E95


def test_streams_golden():
    a = bs.SplitMix64.draws(42, count=1, tag=1)[0]
    b = bs.SplitMix64.draws(42, count=1, tag=2)[0]
    # stream(42, tag).next_double() is the SECOND draw's double here (first is next_u64)
    assert a[0] != b[0]
    arr = bs.generate_arrivals("constant", rate=10.0, count=5)
    assert [t for t, _, _ in arr] == pytest.approx([100.0, 200.0, 300.0, 400.0, 500.0], abs=1e-9)


def test_stream_first_double_golden():
    # SplitMix64::stream(42, kArrivalStream).next_double() == 0.37516029192677325
    # -> first Poisson gap of seed 42 at rate 1000/s (mean 1 ms) = -log(1 - u).
    arr = bs.generate_arrivals("poisson", rate=1000.0, count=1, seed=42)
    assert abs(arr[0][0] - (-math.log(1 - 0.37516029192677325))) < 1e-12


def test_poisson_mix_fraction():
    arr = bs.generate_arrivals("poisson", rate=100.0, count=5000, seed=21, dnn_mix=[["a", 0.25], ["b", 0.75]])
    frac = sum(1 for _, d, _ in arr if d == 0) / 5000
    assert abs(frac - 0.25) < 0.02
