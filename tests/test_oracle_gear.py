"""Pins for oracle G1: the online local search of the clock gears
on the simulator of reading R7.

Pinned to the simulator's closed forms (default gears give objective 1; a memory-bound
workload's time does not depend on the SM clock; the cap penalty), to brute force (the
exhaustive argmin over every gear pair of noiseless convex landscapes: the search ends within
2 SM gears of the argmin at its memory gear, memory gear exact, at most 12 probes per domain),
and to the bracket rules (a prediction at the optimum is kept; a monotone landscape ends at the
domain boundary).
"""
import numpy as np
import pytest

import oracle as O

SM = np.arange(510, 1966, 15, dtype=np.float64)  # 98 gears
MEM = np.array([405.0, 810.0, 1600.0, 2619.0, 3996.0])
# bracket: doubling strides on both sides (<= 2 (ceil(log2 n) + 1)), golden section (<= 2 per
# iteration, 12 iterations), the <= 3 gears left
MAXP = 2 * (int(np.ceil(np.log2(len(SM)))) + 1) + 2 * 12 + 3


def _w(rng, noise=0.0):
    return O.gear_workload(compute_work=rng.uniform(0.5e9, 3e9), memory_work=rng.uniform(0.5e9, 3e9),
                           overhead=rng.uniform(0.01, 0.1), p_static=rng.uniform(80, 150), c_sm=rng.uniform(0.01, 0.05),
                           c_mem=rng.uniform(0.005, 0.03), u_c=rng.uniform(0.2, 1.0), u_m=rng.uniform(0.2, 1.0),
                           noise=noise, seed=int(rng.integers(1 << 62)))


def test_default_gears_objective_is_one():
    w = _w(np.random.default_rng(0))
    assert O.gear_objective(w, SM, MEM, 0.05, len(SM) - 1, len(MEM) - 1) == pytest.approx(1.0, abs=1e-15)


def test_memory_bound_time_ignores_sm_clock_and_penalty():
    # memory-bound: Wm/fm dominates at every SM gear, so time_rel = 1 and the objective is the
    # energy ratio, which falls with the SM clock (power ~ fs^1.8): the lowest SM gear wins
    w = O.gear_workload(compute_work=1e7, memory_work=4e9, overhead=0.0, p_static=100.0, c_sm=0.01, c_mem=0.0,
                        u_c=1.0, u_m=0.0, noise=0.0, seed=1)
    o = [O.gear_objective(w, SM, MEM, 0.05, g, len(MEM) - 1) for g in range(len(SM))]
    assert np.all(np.diff(o) > 0)
    p_lo = 100.0 + 0.01 * SM[0] ** 1.8
    p_hi = 100.0 + 0.01 * SM[-1] ** 1.8
    assert o[0] == pytest.approx(p_lo / p_hi, rel=1e-12)
    r = O.gear_search(w, SM, MEM, 0.05, 50, len(MEM) - 1)
    assert r["sm_gear"] == 0  # monotone landscape: the bracket runs to the boundary


def _smooth(rng):
    # compute-bound (Wm/fm << Wc/fs at every gear pair) and a cap that never binds: the SM
    # objective (Ps + c fs^1.8)(Wc/fs + t0) is smooth and strictly convex; memory only adds
    # power (monotone: gear 0)
    return O.gear_workload(compute_work=rng.uniform(1e9, 3e9), memory_work=1e6, overhead=rng.uniform(0.01, 0.1),
                           p_static=rng.uniform(60, 150), c_sm=rng.uniform(2e-4, 1e-3), c_mem=rng.uniform(0.005, 0.03),
                           u_c=rng.uniform(0.5, 1.0), u_m=rng.uniform(0.2, 1.0), noise=0.0,
                           seed=int(rng.integers(1 << 62)))


@pytest.mark.parametrize("seed", range(50))
def test_search_against_brute_force_on_convex_landscapes(seed):
    rng = np.random.default_rng(100 + seed)
    w = _smooth(rng)
    cap = 10.0
    ps, pm = int(rng.integers(0, len(SM))), int(rng.integers(0, len(MEM)))
    r = O.gear_search(w, SM, MEM, cap, ps, pm)
    assert r["probes_sm"] <= MAXP and r["probes_mem"] <= len(MEM)
    obj = np.array([[O.gear_objective(w, SM, MEM, cap, a, b) for b in range(len(MEM))] for a in range(len(SM))])
    gs, gm = np.unravel_index(obj.argmin(), obj.shape)
    assert r["mem_gear"] == gm
    assert abs(r["sm_gear"] - gs) <= 2, (r, gs)


@pytest.mark.parametrize("seed", range(20))
def test_search_invariants_on_kinked_landscapes(seed):
    # the general simulator (max() of compute and memory time, the cap penalty) has kinks where
    # a quadratic fit can miss the argmin: check only the procedure's invariants
    rng = np.random.default_rng(500 + seed)
    w = _w(rng)
    ps, pm = int(rng.integers(0, len(SM))), int(rng.integers(0, len(MEM)))
    r = O.gear_search(w, SM, MEM, 0.05, ps, pm)
    assert 0 <= r["sm_gear"] < len(SM) and 0 <= r["mem_gear"] < len(MEM)
    assert r["probes_sm"] <= MAXP and r["probes_mem"] <= len(MEM)
    assert r["objective"] == O.gear_objective(w, SM, MEM, 0.05, r["sm_gear"], r["mem_gear"])


def test_prediction_at_optimum_is_kept():
    rng = np.random.default_rng(7)
    for _ in range(10):
        w = _w(rng)
        om = [O.gear_objective(w, SM, MEM, 0.05, len(SM) - 1, g) for g in range(len(MEM))]
        gm = int(np.argmin(om))
        os_ = [O.gear_objective(w, SM, MEM, 0.05, g, gm) for g in range(len(SM))]
        gs = int(np.argmin(os_))
        if gs in (0, len(SM) - 1):
            continue
        r = O.gear_search(w, SM, MEM, 0.05, gs, gm)
        assert r["mem_gear"] == gm and abs(r["sm_gear"] - gs) <= 1
