"""Sampled full-size cost of the reference's ``solve_complex`` on host cores.
MEASUREMENT INFRASTRUCTURE ONLY: imported by bench.py's ``cpu_baseline`` leg
and ``--impl reference`` arm (and by the tools/tests that validate it); never
by the product package.

Why sampled.  The reference (bse-solver 0.1.0, pure Python + numpy) needs
~10^4-10^5 s at BASELINE cfg2 (n = 16384; its solve_complex works on the
2n = 32768 embedding, solvers.py:29-77), while a bench run must end in
minutes.  Every stage of that solve is either a BLAS-3 product, an
elementwise pass, or a Python loop whose step ``j`` does value-independent
work on full-size arrays.  So instead of extrapolating from small n, this
module runs the reference's OWN step bodies -- the oracle's restatements
``bse_oracle.cholesky_column`` (kernels.py:56-64), ``tridiagonalize_step``
(kernels.py:102-117), ``reflect_rows`` (kernels.py:131-136), ``sturm_counts``
(kernels.py:262-272), ``lu_shifted`` / ``lu_solve`` (kernels.py:302-356),
``start_vectors`` (kernels.py:362-369), ``reorthogonalize_column``
(kernels.py:421-443) -- on arrays of the FULL workload size, for a
stratified sample of step indices, and prices each loop as

    time(loop) = (sum of measured step times) / (sum of their work units)
                 x (exact work units of the whole loop),

with the work unit of step j the number of array elements it streams
(Cholesky: (m - j) j, tridiagonal reduction: (m - k - 1)^2, reorthogonalisation:
m j, reflector application: (m - k - 1) n).  BLAS-3 products are timed on a
column block and scaled by the column count, elementwise stages on a row
block.  Successive rounds (bench steps) use new stratum offsets and pool
their samples.

Model assumptions (stated in ``notes()``):
  * one irreducible tridiagonal block (no splits; true for the seeded dense
    BASELINE inputs), no inverse-iteration retries, per-step interpreter
    overhead neglected (< 1e-3 of a step at m = 32768);
  * bisection iteration count = min(160, ceil(log2(W0 / (4 eps lam_min))) + 1)
    with W0 = 4 lam_max, from the caller's eigenvalue bounds (an upper bound:
    the loop in kernels.py:284-298 stops once every bracket is 2 eps relative).
Validated against complete oracle runs where they finish
(tools/validate_cost_model.py -> profiles/r02/cost_model_validation*.json).
"""
from __future__ import annotations

import math
import time

import numpy as np

from . import bse_oracle as orc


def _t(fn, *args, **kw):
    t0 = time.perf_counter()
    fn(*args, **kw)
    return time.perf_counter() - t0


def offsets(count: int):
    """Low-discrepancy stratum offsets for successive rounds (golden ratio)."""
    g = (math.sqrt(5.0) - 1.0) / 2.0
    return [((0.5 + i * g) % 1.0) for i in range(count)]


class Loop:
    """A Python loop of the reference, priced by sampled steps."""

    def __init__(self, name, length, step, work, total_work, warm_bytes_limit=256 << 20):
        self.name = name
        self.length = length
        self.step = step              # step(j): runs the reference's step body j
        self.work = work              # work(j): array elements streamed by step j
        self.total_work = float(total_work)
        self.warm_limit = warm_bytes_limit
        self.t_sum = 0.0
        self.w_sum = 0.0
        self.samples = 0

    def sample(self, points, u):
        for i in range(max(1, min(points, self.length))):
            j = min(self.length - 1, int((i + u) * self.length / max(1, points)))
            if j > 0 and 8 * self.work(j) < self.warm_limit:
                self.step(j - 1)  # the cache state of the loop (small working sets only)
            self.t_sum += _t(self.step, j)
            self.w_sum += self.work(j)
            self.samples += 1

    def estimate(self):
        return self.t_sum / self.w_sum * self.total_work if self.w_sum > 0.0 else 0.0


def _sum_sq(lo, hi):
    """sum_{x=lo}^{hi} x^2 (0 if hi < lo)."""
    if hi < lo:
        return 0.0
    f = lambda x: x * (x + 1) * (2 * x + 1) / 6.0  # noqa: E731
    return f(hi) - f(lo - 1)


class SolveComplexCost:
    """Full-size sampler for the reference solve_complex at block size n
    (working dimension m = 2n).  ``a``, ``b``: the complex128 n x n operator
    blocks (BseOperator stores both kinds as complex128, core.py:45-75).
    ``lam_bounds``: (lam_min, lam_max) bounds of the positive spectrum (for the
    bisection iteration count)."""

    def __init__(self, a, b, lam_bounds, seed: int = 0):
        self.a = np.ascontiguousarray(a, dtype=np.complex128)
        self.b = np.ascontiguousarray(b, dtype=np.complex128)
        self.n = n = self.a.shape[0]
        self.m = m = 2 * n
        self.k = k = n  # kept (positive) eigenpairs
        self.lam_min, self.lam_max = (float(x) for x in lam_bounds)
        self.rng = np.random.default_rng(seed)
        # One full-size m x m buffer serves as the Cholesky factor, the matrix
        # being tridiagonalized and the reflector store, and one m x k buffer
        # as the inverse-iteration vectors / back-transform operand: a loop
        # step only needs arrays of the right shapes (its cost does not depend
        # on the values), so they are refilled from small random tiles before
        # each phase (keeps the values finite and normal across rounds).
        self.F = np.empty((m, m))
        self.V = np.empty((m, k))
        self.taus = self.rng.uniform(0.5, 1.5, m)
        # tau_k = 2 / |v_k|^2 for tile-filled store columns (|v_k|^2 ~ (m-k-1)/3),
        # so the sampled reflections stay (nearly) orthogonal
        self.taus_q = 6.0 / np.maximum(1.0, m - 1.0 - np.arange(m))
        self.sub = np.zeros(m)
        self.d = np.zeros(m)
        self.e = self.rng.uniform(0.5, 1.5, m - 1) * self.lam_max / 2
        self.pivmin = orc.pivmin_of(self.e)
        self.lams = np.sort(self.rng.uniform(self.lam_min, self.lam_max, k))
        idx = np.arange(k)
        F, V, d, e, lams = self.F, self.V, self.d, self.e, self.lams
        L = max(m - 2, 0)
        self.loops = {
            # column j: GEMV over (m - j) x j, then (m - j) scaling
            "cholesky": Loop("cholesky", m, lambda j: orc.cholesky_column(F, j, "M", False),
                             lambda j: (m - j) * (j + 1),
                             sum_prod(m)),
            # reflector k: GEMV + two outer-product updates of the (m-k-1)^2 trail
            "tridiagonalize": Loop("tridiagonalize", L,
                                   lambda j: orc.tridiagonalize_step(F, F, self.taus, self.sub, j,
                                                                     True),
                                   lambda j: (m - j - 1) ** 2, _sum_sq(m - L, m - 1)),
            # vector j: two CGS passes against j previous vectors of length m
            "reorthogonalize": Loop("reorthogonalize", k,
                                    lambda j: orc.reorthogonalize_column(V, j, d, e, lams, idx, 0,
                                                                         self.pivmin, False),
                                    lambda j: m * (j + 1), m * k * (k + 1) / 2.0),
            # apply_q walks the reflectors backwards (kernels.py:130): step j is
            # reflector m - 3 - j, a rank-1 update of (j + 2) x k rows
            "apply_q": Loop("apply_q", L,
                            lambda j: orc.reflect_rows(V, F, self.taus_q, m - 3 - j),
                            lambda j: (j + 2) * k, k * (L * (L + 1) / 2.0 + L)),
        }
        self.fixed = None  # single-shot phases, measured in the first round
        self.rounds = 0

    def _fill_f(self):
        m = self.m
        tile = self.rng.uniform(-1.0, 1.0, (m, 64))
        if m % 64 == 0:
            self.F.reshape(m, -1, 64)[:] = tile[:, None, :]
        else:
            self.F[:] = self.rng.uniform(-1.0, 1.0, (m, m))

    def _fill_v(self):
        m, k = self.m, self.k
        tile = self.rng.standard_normal((m, 64))
        tile /= np.linalg.norm(tile, axis=0)
        if k % 64 == 0:
            self.V.reshape(m, -1, 64)[:] = tile[:, None, :]
        else:
            self.V[:] = self.rng.standard_normal((m, k)) / math.sqrt(m)

    # -- phases without a per-step loop (BLAS-3 / elementwise / vectorised) --
    def _fixed_phases(self):
        n, m, k = self.n, self.m, self.k
        F, V, d, e = self.F, self.V, self.d, self.e
        ph = {}
        q = max(1, n // 4)  # build_m: elementwise, a q x q corner scaled by area
        ph["build_m"] = _t(orc.build_m, self.a[:q, :q], self.b[:q, :q]) * (n / q) ** 2
        r = max(1, m // 16)
        ph["cholesky_tril"] = _t(np.tril, F[:r]) * m / r
        r = max(1, n // 8)
        ph["congruence_stack"] = _t(lambda: np.vstack([F[n:n + r], -F[:r]])) * n / r
        c = max(1, m // 64)
        g = np.ascontiguousarray(F[:, :c])
        ph["congruence_gemm"] = _t(lambda: F.T @ g) * m / c
        qq = max(1, m // 4)
        blk = F[:qq, :qq]
        ph["congruence_skew"] = _t(lambda: 0.5 * (blk - blk.T)) * (m / qq) ** 2
        r = max(1, m // 16)
        ph["tridiag_copy"] = _t(np.array, F[:r]) * m / r
        # tridiag_eig: split scan, bisection sweeps, tagging/sorting
        rr = max(2, min(m, 256))
        ph["split_points"] = _t(orc.split_points, d[:rr], e[:rr - 1]) * m / rr
        lo = np.full(m, -self.lam_max)
        hi = np.full(m, self.lam_max)
        mid = 0.5 * (lo + hi)
        rows = max(2, min(m, 64))
        sweep = _t(orc.sturm_counts, d[:rows], e[:rows - 1], mid, self.pivmin) * m / rows
        idx_all = np.arange(m)

        def vec_ops():
            np.any(hi - lo > 2.0 * orc.EPS * (np.abs(lo) + np.abs(hi)) + 2.0 * orc.TINY)
            left = (idx_all + 1) > idx_all
            np.where(left, mid, hi)
            np.where(left, lo, mid)
        ph["bisection"] = self.bisection_iterations() * (sweep + _t(vec_ops))
        vals = np.sort(np.concatenate([-self.lams, self.lams]))

        def tag_sort():
            tagged = [(v, 0, li) for li, v in enumerate(vals)]
            tagged.sort(key=lambda t: (t[0], t[1], t[2]))
            return tagged[m // 2:][::-1]
        ph["tag_sort"] = _t(tag_sort)
        # inverse iteration: start vectors, batched LU + 3 solves, normalisations
        ks = max(1, min(k, 128))
        ph["start_vectors"] = _t(orc.start_vectors, m, 0, np.arange(ks)) * k / ks
        rows = max(3, min(m, 64))
        ph["lu_shifted"] = _t(orc.lu_shifted, d[:rows], e[:rows - 1], self.lams,
                              self.pivmin) * m / rows
        fact = orc.lu_shifted(d[:rows], e[:rows - 1], self.lams, self.pivmin)
        ph["lu_solve"] = 3 * _t(orc.lu_solve, fact, V[:rows]) * m / rows
        cs = max(1, k // 16)
        blk = np.ascontiguousarray(V[:, :cs])

        def norms():
            v = blk / np.linalg.norm(blk, axis=0)
            for _ in range(3):
                amax = np.max(np.abs(v), axis=0)
                amax = np.where(amax == 0.0, orc.TINY, amax)
                v = v / amax
                nrm = np.linalg.norm(v, axis=0)
                nrm = np.where(nrm == 0.0, 1.0, nrm)
                np.minimum(amax, 1e300) * nrm
                v = v / nrm
        ph["iterate_norms"] = _t(norms) * k / cs
        kc = min(k, 256)
        out = np.zeros((m, kc))

        def scatter():  # out[:, c] = cols[bi][li] (kernels.py:528-533)
            cols = {li: V[:, li] for li in range(kc)}
            for c2 in range(kc):
                out[:, c2] = cols[c2]
        ph["vector_scatter"] = _t(scatter) * k / kc

        def phase_split():  # zr / zi from D V+ (solvers.py:56-62)
            zr = np.zeros_like(blk)
            zi = np.zeros_like(blk)
            zr[0::4], zr[2::4] = blk[0::4], -blk[2::4]
            zi[1::4], zi[3::4] = blk[1::4], -blk[3::4]
        ph["phase_split"] = _t(phase_split) * k / cs
        r = max(1, m // 16)
        ph["apply_q_copy"] = 2 * _t(np.array, V[:r]) * m / r
        c = max(1, k // 32)
        blk2 = np.ascontiguousarray(V[:, :c])
        ph["recover_gemm"] = 2 * _t(lambda: F @ blk2) * k / c  # gr = L zr, gi = L zi
        rr = max(1, n // 16)
        lam = self.lams[::-1]

        def combine():  # Q action and Lambda^-1/2 scaling (solvers.py:67-72)
            top = ((V[:rr] + V[n:n + rr]) + 1j * (V[:rr] - V[n:n + rr])) / math.sqrt(2.0)
            bot = ((V[:rr] - V[n:n + rr]) + 1j * (V[:rr] + V[n:n + rr])) / math.sqrt(2.0)
            scale = 1.0 / np.sqrt(lam)
            top * scale
            -bot * scale
        ph["combine"] = _t(combine) * n / rr
        return ph

    def bisection_iterations(self):
        w0 = 4.0 * self.lam_max
        need = math.log2(w0 / (4.0 * orc.EPS * self.lam_min)) if self.lam_min > 0 else 160
        return int(min(160, math.ceil(need) + 1))

    # -- rounds ---------------------------------------------------------------
    def round(self, points: int = 1, u: float = 0.5):
        """One sampling round (one bench step): every loop sampled at
        ``points`` stratified step indices with offset ``u``; the single-shot
        phases are measured in the first round.  Returns the seconds spent
        running reference code (buffer refills excluded)."""
        spent = 0.0
        self._fill_f()
        self._fill_v()
        t0 = time.perf_counter()
        if self.fixed is None:
            self.fixed = self._fixed_phases()
        self.loops["cholesky"].sample(points, u)
        self.loops["tridiagonalize"].sample(points, u)
        spent += time.perf_counter() - t0
        self._fill_f()  # fresh values for the next phases
        self._fill_v()
        t0 = time.perf_counter()
        self.loops["reorthogonalize"].sample(points, u)
        spent += time.perf_counter() - t0
        self._fill_v()
        t0 = time.perf_counter()
        self.loops["apply_q"].sample(points, u)
        spent += time.perf_counter() - t0
        self.rounds += 1
        return spent

    def phases(self):
        """Estimated seconds per reference stage (solvers.py:46-72 order)."""
        f = self.fixed or {}
        L = self.loops

        def s(*keys):
            return sum(f.get(x, 0.0) for x in keys)
        return {
            "build_m": s("build_m"),
            "cholesky": L["cholesky"].estimate() + s("cholesky_tril"),
            "congruence": s("congruence_stack", "congruence_gemm", "congruence_skew"),
            "tridiagonalize": s("tridiag_copy") + L["tridiagonalize"].estimate(),
            "tridiag_eig": s("split_points", "bisection", "tag_sort", "start_vectors",
                             "lu_shifted", "lu_solve", "iterate_norms", "vector_scatter")
                           + L["reorthogonalize"].estimate(),
            "back_transform": s("phase_split", "apply_q_copy", "recover_gemm", "combine")
                              + 2 * L["apply_q"].estimate(),
        }

    def estimate(self):
        return float(sum(self.phases().values()))

    def notes(self) -> str:
        return (f"reference solve_complex (solvers.py:29-77) at m = {self.m}: the oracle's "
                f"restated step bodies timed at full size on stratified step indices "
                f"({sum(lp.samples for lp in self.loops.values())} loop steps over {self.rounds} "
                f"rounds) and priced by exact per-loop work counts; BLAS-3 products on column "
                f"blocks; {self.bisection_iterations()} bisection iterations (bound from lam in "
                f"[{self.lam_min:.3g}, {self.lam_max:.3g}]); one tridiagonal block, no "
                f"inverse-iteration retries")


def sum_prod(m):
    """sum_{j=0}^{m-1} (m - j) (j + 1) = m (m + 1) (m + 2) / 6."""
    return m * (m + 1) * (m + 2) / 6.0
