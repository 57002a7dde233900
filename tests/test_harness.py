"""The reference's overhead / scaling harness restated for the GPU path
(reference proj/core/src/harness.cpp:15-20, 125-167, 188-201): the tests
mirror proj/tests/unit/test_harness.cpp:110-132 and the exactness check of
the acceptance gate (proj/tests/acceptance/acceptance_main.cpp:742-749)."""
import io

import pytest

from paper_2210_06437_b200 import hydro as H


def test_sweep_validates_counts():
    for bad in ([], [0], [2, 1], [1, 1]):
        with pytest.raises(ValueError):
            H.sweep_rows_from_times(512, 3, bad, [1.0] * len(bad), [1.0] * len(bad))
    with pytest.raises(ValueError, match="one time per arm"):
        H.sweep_rows_from_times(512, 3, [1, 2], [1.0], [1.0, 2.0])
    with pytest.raises(ValueError, match="positive"):
        H.sweep_rows_from_times(512, 3, [1], [0.0], [1.0])
    with pytest.raises(ValueError, match="baseline must be positive"):
        H.compute_overhead(1, 1.0, 0.0)


def test_single_count_rows_are_exactly_recomputable():
    rows = H.sweep_rows_from_times(512, 7, [1], [0.25], [0.2])
    assert len(rows) == 1
    r = rows[0]
    assert r.n == 1 and r.speedup_with == 1.0 and r.speedup_without == 1.0
    assert r.o_percent == H.compute_overhead(1, r.time_with_s, r.time_without_s)
    cells = 512.0 * 7
    assert r.cells_per_second_with == cells / r.time_with_s
    assert r.cells_per_second_without == cells / r.time_without_s


def test_speedups_are_relative_to_the_smallest_count():
    rows = H.sweep_rows_from_times(4096 * 512, 10, [1, 2, 4], [4.0, 2.1, 1.1], [3.9, 2.0, 1.0])
    assert [r.speedup_with for r in rows] == [1.0, 4.0 / 2.1, 4.0 / 1.1]
    assert [r.speedup_without for r in rows] == [1.0, 3.9 / 2.0, 3.9 / 1.0]
    assert rows[1].o_percent == (2.1 / 2.0) * 100.0 - 100.0


def test_sweep_csv_round_trips_exactly():
    """acceptance_main.cpp:742-749: every derived column recomputes exactly
    from the written text (%.17g)."""
    rows = H.sweep_rows_from_times(2097152, 20, [1, 2, 4], [0.0111, 0.00589, 0.00306],
                                   [0.0110, 0.00583, 0.00302])
    buf = io.StringIO()
    H.write_sweep_csv(buf, rows)
    lines = buf.getvalue().splitlines()
    assert lines[0] == ("n,time_with,time_without,cells_per_second_with,cells_per_second_without,"
                        "o_percent,speedup_with,speedup_without")
    back = [[float(v) for v in ln.split(",")] for ln in lines[1:]]
    cells = 2097152.0 * 20
    for r, b in zip(rows, back):
        assert int(b[0]) == r.n
        assert b[3] == cells / b[1] and b[4] == cells / b[2]
        assert b[5] == H.compute_overhead(r.n, b[1], b[2])
        assert b[6] == back[0][1] / b[1] and b[7] == back[0][2] / b[2]


@pytest.mark.gpu
def test_timing_hook_overhead_on_the_gpu():
    """measure_arm on the B200: the 'full' arm stamps one record per launch,
    the 'disabled' arm none; the sweep row of the two times is well formed."""
    mesh = H.uniform_mesh(8, 8, 8)
    dev = H.CudaDevice(H.HydroConfig(dx=1.0 / 64))
    session = H.WorkloadSession(mesh, dev, H.StepConfig(num_steps=5))
    session.load_problem("sedov")
    dev.step(2)
    dev.synchronize()
    dev.flush_activity()
    dev.set_profiling(False)
    dev.step(2)
    dev.synchronize()
    assert dev.flush_activity() == []
    dev.set_profiling(True)
    dev.step(1)
    dev.synchronize()
    assert len([r for r in dev.flush_activity() if r.kind == "kernel"]) >= 3
    t_with = H.measure_arm(session, True, repetitions=3)
    t_without = H.measure_arm(session, False, repetitions=3)
    rows = H.sweep_rows_from_times(mesh.total_cells(), 5, [1], [t_with], [t_without])
    assert rows[0].cells_per_second_with > 1e8
    assert abs(rows[0].o_percent) < 50.0
    dev.close()
