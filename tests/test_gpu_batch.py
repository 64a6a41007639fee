"""BASELINE C5 shape: a batch of independent Air3D tubes sharing grid and
dynamics runs in lockstep as one stacked state; every member must equal its
own single-problem solve bit for bit."""
import numpy as np
import pytest

import paper_2411_03501_b200 as hj

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("stage_kernel")]


@pytest.mark.parametrize("scheme", ["weno5", "eno2"])
def test_batch_members_equal_single_solves(scheme):
    g = hj.air3d_grid((33, 31, 24))
    cfg = hj.air3d_term_config(scheme=scheme)
    rng = np.random.default_rng(0)
    targets = []
    for _ in range(4):
        cx, cy = rng.uniform(-2.0, 2.0, 2)
        targets.append(hj.cylinder(g, 2, (cx, cy, 0.0), rng.uniform(3.0, 6.0)))
    snaps, times = hj.solve_tube_batch(g, targets, cfg, 0.2, 2, order=3)
    assert snaps.shape == (3, 4) + g.counts
    for b, tgt in enumerate(targets):
        res = hj.solve_tube(g, tgt, cfg, 0.2, 2, order=3)
        assert tuple(res.times) == times
        for k, s in enumerate(res.snapshots):
            assert np.array_equal(s.values, snaps[k, b]), (b, k)


@pytest.mark.parametrize("scheme", ["weno5", "eno2"])
def test_batch_final_states_streamed(scheme):
    """keep_snapshots=False over one interval runs one stream per problem
    (copies of one problem overlapping the stages of the others): the final
    states equal the lockstep batch's bit for bit, and a non-finite target
    raises the reference's ValueError."""
    g = hj.air3d_grid((33, 31, 24))
    cfg = hj.air3d_term_config(scheme=scheme)
    rng = np.random.default_rng(1)
    targets = []
    for _ in range(3):
        cx, cy = rng.uniform(-2.0, 2.0, 2)
        targets.append(hj.cylinder(g, 2, (cx, cy, 0.0), rng.uniform(3.0, 6.0)).values)
    final, times = hj.solve_tube_batch(g, targets, cfg, 0.05, 1, order=3, keep_snapshots=False)
    snaps, times2 = hj.solve_tube_batch(g, targets, cfg, 0.05, 1, order=3)
    assert tuple(times) == tuple(times2)
    assert final.shape == (3,) + g.counts
    assert np.array_equal(final, snaps[-1])
    bad = [t.copy() for t in targets]
    bad[1][3, 4, 5] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        hj.solve_tube_batch(g, bad, cfg, 0.05, 1, order=3, keep_snapshots=False)
