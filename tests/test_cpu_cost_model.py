"""CPU checks of the sampled reference-cost model behind bench.py's
cpu_baseline and --impl reference (oracle/cost_model.py): exact work counts,
the step functions equal the oracle's loops, and a small end-to-end estimate
lands near a complete run of the oracle (the full-size validation is
tools/validate_cost_model.py on the GPU box's host)."""
import time

import numpy as np

from oracle import bse_oracle as orc
from oracle import cost_model as cm
from paper_1501_03830_b200 import configs


def test_work_count_closed_forms():
    for m in (5, 64, 257):
        assert cm.sum_prod(m) == sum((m - j) * (j + 1) for j in range(m))
        L = m - 2
        assert cm._sum_sq(m - L, m - 1) == sum((m - j - 1) ** 2 for j in range(L))


def test_loop_estimate_is_exact_for_proportional_cost():
    calls = []
    loop = cm.Loop("synthetic", 100, lambda j: calls.append(j), lambda j: j + 1,
                   sum(j + 1 for j in range(100)))
    loop.t_sum, loop.w_sum = 2.0, 4.0  # 0.5 s per unit of work
    assert loop.estimate() == 0.5 * 5050
    loop2 = cm.Loop("synthetic", 100, lambda j: None, lambda j: 1, 100)
    loop2.sample(4, 0.5)
    assert loop2.samples == 4 and loop2.w_sum == 4


def test_step_functions_reproduce_the_oracle():
    rng = np.random.default_rng(0)
    g = rng.standard_normal((12, 12))
    w = g - g.T
    d, sub, store, taus = orc.tridiagonalize(w, skew=True)
    a = w.copy()
    st2, t2, s2 = np.zeros_like(store), np.zeros_like(taus), np.zeros_like(sub)
    for k in range(10):
        orc.tridiagonalize_step(a, st2, t2, s2, k, True)
    assert np.array_equal(st2, store) and np.array_equal(t2, taus)
    spd = g @ g.T + 12 * np.eye(12)
    f = spd.copy()
    for j in range(12):
        orc.cholesky_column(f, j)
    assert np.array_equal(np.tril(f), orc.cholesky(spd))


def test_small_estimate_near_full_run():
    n = 96
    a, b, _ = configs.config_operator(2, n=n, seed=2)
    t0 = time.perf_counter()
    orc.solve_complex(a, b)
    full = time.perf_counter() - t0
    smp = cm.SolveComplexCost(a, b, (0.1, 100.0))
    for u in cm.offsets(3):
        smp.round(points=2, u=u)
    est = smp.estimate()
    assert set(smp.phases()) == {"build_m", "cholesky", "congruence", "tridiagonalize",
                                 "tridiag_eig", "back_transform"}
    # tiny sizes are dominated by interpreter overhead the model neglects
    assert 0.2 * full <= est <= 5.0 * full, (est, full)
