"""Algorithm 1 (§4.4, l.832-855) search logic, host-only: the
coordinate-descent / stop-rule search against a brute-force oracle on tiny
instances (SPEC.md search module), plus the Matrix_P move
primitives.  The objective here is synthetic; on the GPU it is the measured
executor makespan (tests/test_gpu_planner.py)."""
import itertools

import numpy as np
import pytest

from paper_2304_11745_b200 import planner as P


def test_add_pointer_midpoint_rule():
    # SPEC S:277 examples (midpoint of the largest segment, equal counts)
    assert P.add_pointer(((),), [5]) == ((3,),)
    assert P.add_pointer(((2, 8),), [12]) == ((2, 5, 8),)
    assert P.add_pointer(((),), [1]) == ((1,),)
    assert P.add_pointer(((), ()), [4, 10]) == ((2,), (5,))


def test_coordinate_moves_legal_and_incumbent():
    moves = P.coordinate_moves(((2,),), 0, 0, 5)
    assert [m[0][0] for m in moves] == [0, 1, 2, 3, 4, 5]
    # squeezed between neighbours 3 and 5 (non-decreasing cuts, reading Q7)
    moves = P.coordinate_moves(((3, 4, 5),), 0, 1, 9)
    assert [m[0][1] for m in moves] == [3, 4, 5]
    # other models untouched, every candidate a valid matrix
    for m in P.coordinate_moves(((1, 2), (0, 3)), 1, 0, 6):
        assert m[0] == (1, 2) and list(m[1]) == sorted(m[1]) and 0 <= m[1][0] <= 3


def _separable(targets, penalty):
    def ev(ptrs, dec):
        r = penalty * sum(len(p) for p in ptrs)
        for cuts, tg in zip(ptrs, targets):
            k = min(len(cuts), len(tg))
            r += sum(abs(a - b) for a, b in zip(cuts[:k], tg[:k])) + 3.0 * abs(len(cuts) - len(tg))
        for t, ch in dec:
            r += 0.0 if ch == 1 else 0.5
        return r
    return ev


@pytest.mark.parametrize("seed", range(6))
def test_search_matches_brute_force(seed):
    rng = np.random.default_rng(seed)
    n_ops = [int(rng.integers(3, 7)), int(rng.integers(3, 7))]
    k = int(rng.integers(0, 3))
    targets = [tuple(sorted(int(v) for v in rng.integers(0, n + 1, size=k))) for n in n_ops]
    ev = _separable(targets, penalty=0.05)
    res = P.granularity_aware_search(ev, n_ops, P.SearchConfig(max_pointers=3, rounds=2))
    r_opt, p_opt, _ = P.brute_force_oracle(ev, n_ops, 3)
    assert res.R == pytest.approx(r_opt)
    assert ev(res.pointers, res.decomposition) == pytest.approx(res.R)


def test_stop_rule_returns_zero_pointers_when_they_only_cost():
    n_ops = [4, 5]
    ev = _separable([(), ()], penalty=100.0)
    res = P.granularity_aware_search(ev, n_ops, P.SearchConfig(max_pointers=3))
    assert res.pointers == ((), ())
    assert set(res.records) == {0, 1}          # one escalation attempt, then the stop rule


def test_spatial_moves_only_when_strictly_better():
    n_ops = [3, 3]

    def ev(ptrs, dec):
        d = dict(dec)
        return 10.0 - (1.0 if d[1] == 2 else 0.0) + 5.0 * sum(len(p) for p in ptrs)
    res = P.granularity_aware_search(ev, n_ops, P.SearchConfig(max_pointers=1))
    assert dict(res.decomposition) == {0: 1, 1: 2}
    assert res.R == 9.0


def test_memoised_each_plan_evaluated_once():
    calls = {}

    def ev(ptrs, dec):
        k = (ptrs, dec)
        calls[k] = calls.get(k, 0) + 1
        return float(sum(sum(p) for p in ptrs)) + 1.0
    P.granularity_aware_search(ev, [4, 4], P.SearchConfig(max_pointers=2, rounds=3))
    assert max(calls.values()) == 1


def test_brute_force_guard():
    with pytest.raises(ValueError):
        P.brute_force_oracle(lambda p, d: 0.0, [60, 60, 60], 3)


def test_all_pointer_matrices_count():
    # non-decreasing k-subsets with repetition of {0..n}: C(n+k, k) per model
    from math import comb
    mats = P.all_pointer_matrices([4, 2], 2)
    assert len(mats) == comb(6, 2) * comb(4, 2)
    assert all(list(r) == sorted(r) for m in mats for r in m)
    assert len(set(mats)) == len(mats)
    assert ((0, 0), (2, 2)) in mats and ((4, 4), (0, 2)) in mats
    assert itertools  # (module used by the planner's enumeration)
