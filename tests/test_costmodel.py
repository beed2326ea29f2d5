"""NEXT-1 / NEXT-3 model-based planner (paper_2304_11745_b200/costmodel.py)
on hand-built lookup tables: the deployment model of Eq. 1, the residue of
Eq. 2/3 with the pointer penalty of Eq. 8, the largest-residue spatial
heuristic of §4.2 (l.688-695) and Algorithm 1's search vs brute force."""
import itertools

import pytest

from paper_2304_11745_b200 import costmodel as CM
from paper_2304_11745_b200.planner import all_pointer_matrices


def tenant(ops, batch=2, n_orig=None):
    """ops: list of {b: (W, T[, Wb])} per fused op; fused op f = original op f."""
    n = len(ops)
    tm = CM.TenantModel(batch=batch, n_orig=n_orig or n, last_member=list(range(n)),
                        first_member=list(range(n)), decomposable=[True] * n)
    for f, tab in enumerate(ops):
        for b, v in tab.items():
            tm.cost[(f, b)] = CM.OpCost(*v)
    return tm


def test_two_ops_that_do_not_fit_run_back_to_back():
    """W 0.6 + 0.6 > S_GPU: the second is moved to the next cycle
    (l.438-444); R = residue 0.4 over 10 us twice (Eq. 3)."""
    A = tenant([{2: (0.6, 10.0)}])
    B = tenant([{2: (0.6, 10.0)}])
    sim = CM.simulate([A, B], ((), ()), {}, t_sw=1.0)
    assert sim.makespan == pytest.approx(20.0)
    assert sim.R == pytest.approx(0.4 * 10 + 0.4 * 10)


def test_ops_that_fit_share_the_cycle_and_pointer_penalty():
    A = tenant([{2: (0.5, 10.0)}, {2: (0.5, 10.0)}])
    B = tenant([{2: (0.5, 20.0)}])
    sim = CM.simulate([A, B], ((), ()), {}, t_sw=1.5)
    assert sim.makespan == pytest.approx(20.0) and sim.R == pytest.approx(0.0)
    # a pointer after A's first op and none in B (cut 0 = B in cluster 1):
    # cluster 0 = {A1}, cluster 1 = {A2, B}; Eq. 8 adds |P| * S_GPU * T_SW
    sim = CM.simulate([A, B], ((1,), (0,)), {}, t_sw=1.5)
    assert sim.makespan == pytest.approx(30.0)
    assert sim.R == pytest.approx(0.5 * 10 + 0.5 * 10 + 1 * 1.5)


def test_largest_residue_split_fits_the_residue():
    """§4.2: the biggest residue (0.4 while A runs) is filled by a chunk of
    the waiting operator whose W fits it (b = 1, W = 0.3); the split lowers R
    (hand-computed: 0.1*6 + 0.1*4 + 0.7*2 = 2.4 vs 8)."""
    A = tenant([{2: (0.6, 10.0)}])
    B = tenant([{2: (0.6, 10.0), 1: (0.3, 6.0)}])
    sim = CM.simulate([A, B], ((), ()), {}, t_sw=0.0)
    d2 = CM.largest_residue_split([A, B], sim, {})
    assert d2 == {(1, 0): (1, 1)}
    sim2 = CM.simulate([A, B], ((), ()), d2, t_sw=0.0)
    assert sim2.makespan == pytest.approx(12.0)
    assert sim2.R == pytest.approx(2.4)
    res = CM.model_based_search([A, B], t_sw=0.0, max_pointers=1)
    assert res.decomposition == {(1, 0): (1, 1)} and res.R == pytest.approx(2.4)


def test_bandwidth_as_second_resource():
    """NEXT-3: two HBM-bound ops with small SM shares fit by SM (0.2 + 0.2)
    but not by bandwidth (0.7 + 0.7 > 1): bandwidth-aware, they serialise."""
    A = tenant([{2: (0.2, 10.0, 0.7)}])
    B = tenant([{2: (0.2, 10.0, 0.7)}])
    assert CM.simulate([A, B], ((), ()), {}, 0.0).makespan == pytest.approx(10.0)
    sim = CM.simulate([A, B], ((), ()), {}, 0.0, bandwidth=True)
    assert sim.makespan == pytest.approx(20.0)


def test_search_matches_brute_force_over_matrix_p():
    """Algorithm 1's coordinate descent + pointer escalation finds the
    brute-force optimum of Eq. 8 over every Matrix_P with <= 2 pointers on a
    small instance (no decomposition)."""
    A = tenant([{2: (0.7, 10.0)}, {2: (0.3, 5.0)}, {2: (0.8, 8.0)}, {2: (0.2, 4.0)}])
    B = tenant([{2: (0.3, 12.0)}, {2: (0.6, 6.0)}, {2: (0.4, 9.0)}])
    ts = [A, B]
    best = min(CM.simulate(ts, p, {}, 0.5).R
               for k in range(3) for p in all_pointer_matrices([4, 3], k))
    res = CM.model_based_search(ts, t_sw=0.5, max_pointers=2, rounds=2, spatial_steps=0)
    assert res.R == pytest.approx(best)
    assert res.R <= CM.simulate(ts, ((), ()), {}, 0.5).R


def test_interpolated_costs_between_profiled_batches():
    A = tenant([{2: (0.4, 10.0), 8: (1.0, 22.0)}], batch=8)
    c = A.op_cost(0, 4)
    assert c.T == pytest.approx(10.0 + (2 / 6) * 12.0) and 0.4 < c.W < 1.0
