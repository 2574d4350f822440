"""§8(f) on the GPU: the CUDA-event layer profiler feeds the bit-exact
scheduler through the profile v1 file, and the bandwidth-throttled sync mode
reproduces the simulator's exposed-sync prediction."""
import os

import numpy as np
import pytest

from oracle import pyoracle as O

pytestmark = pytest.mark.gpu


def test_profiler_writes_a_schedulable_profile(tmp_path):
    from paper_2502_11058_b200.lab import (Lab, LabDesc, schedule_from_profile, sync_mask,
                                           write_profile)
    L, dim, K = 12, 600000, 4
    curv, sizes = O.make_quadratic(dim, L)
    lab = Lab(LabDesc(dim=dim, block_sizes=list(sizes), workers_total=K, sigma=1.0))
    lab.seed(3)
    lab.fill(0.5)
    w_before = lab.get_params()
    rng_before = [lab.rng_text(k) for k in range(K)]
    t_bp, t_comm = lab.profile(reps=3)
    assert np.all(t_bp > 0) and np.all(t_comm < 0)          # single rank, no link: not measured
    assert np.array_equal(lab.get_params(), w_before)        # profiling leaves the state alone
    assert [lab.rng_text(k) for k in range(K)] == rng_before
    # measured times are proportional to layer size (HBM-bound local step)
    big = t_bp[np.argmax(sizes)]
    assert big >= 0.5 * t_bp.max()
    path = str(tmp_path / "measured.profile")
    write_profile(path, [int(s) * 8 for s in sizes], np.zeros(L), t_bp, None,
                  bandwidth=1e9, latency=2e-6)
    sets, fills, obj, text = schedule_from_profile(path, 4)
    assert text.startswith("dreamsched-schedule v1") and len(sets) == 4
    assert sorted(l for s in sets for l in s) == list(range(1, L + 1))
    # the measured schedule drives the step
    for r in range(4):
        lab.step(O.learning_rate(r, 1.0, 2.0, 4), sync_mask("partial", 4, r, L, sets, fills))
    lab.sync()
    lab.close()


def test_throttled_link_exposes_the_modelled_comm():
    """On a 1 GB/s emulated link the synced layers' transfers occupy the FIFO
    sync stream after their local step; the measured exposed time matches the
    closed form max(bp_total, comm finish) - bp_total within scheduling noise."""
    from paper_2502_11058_b200.lab import Lab, LabDesc, sync_mask
    L, dim, K, H = 8, 400000, 4, 2
    curv, sizes = O.make_quadratic(dim, L)
    lab = Lab(LabDesc(dim=dim, block_sizes=list(sizes), workers_total=K, sigma=0.0))
    lab.seed(1)
    lab.fill(0.0)
    bw, lat = 1e9, 50e-6
    lab.set_link(bw, lat)
    lab.set_instrument(True)
    sets = O.enp(L, H)
    times = []
    for r in range(2 * H):
        lab.step(O.learning_rate(r, 1.0, 2.0, H), sync_mask("partial", H, r, L, sets))
        times.append(lab.last_step_times())
    lab.set_link(0.0, 0.0)
    # phase 1 syncs layers 8..5 (ENP): modelled comm = 4 * (lat + 50000*8/bw)
    comm = sum(lat + sizes[l - 1] * 8 / bw for l in sets[0])
    step_ms, sync_ms, exposed_ms = times[2][0], times[2][1], times[2][2]
    assert sync_ms * 1e-3 == pytest.approx(comm, rel=0.15, abs=50e-6)
    assert exposed_ms > 0.0
    # without the link the same step is much shorter
    lab.set_instrument(True)
    lab.step(O.learning_rate(9, 1.0, 2.0, H), sync_mask("partial", H, 9, L, sets))
    assert lab.last_step_times()[0] < step_ms
    lab.close()
