"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU).

Each test names the oracle part it pins (P1..P12) and the
passage it follows.  None of these re-types the oracle's formula: they use exact
rational derivations, closed forms, library routines (numpy/scipy) on special
cases, brute force on tiny inputs, invariants, and the paper's printed numbers.
"""
from __future__ import annotations

import math
import os
from fractions import Fraction

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as fh:
        for line in fh:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


# --------------------------------------------------------------------------- P1
def _not_a_knot_cardinal_integrals(K, a, b):
    """Exact integrals over [a,b] of the cardinal functions of the not-a-knot cubic
    spline through t = 0..K (unit spacing), in rational arithmetic (Eq. 15 conditions).
    K <= 2: the not-a-knot spline degenerates to the interpolating polynomial."""
    out = []
    for j in range(K + 1):
        data = [Fraction(int(i == j)) for i in range(K + 1)]
        if K <= 2:
            # interpolating polynomial: integrate Lagrange basis exactly via monomial moments
            # build coefficients of the Lagrange basis polynomial l_j
            coeffs = [Fraction(1)]
            denom = Fraction(1)
            for m in range(K + 1):
                if m == j:
                    continue
                coeffs = [(coeffs[k - 1] if k >= 1 else 0) - m * (coeffs[k] if k < len(coeffs) else 0)
                          for k in range(len(coeffs) + 1)]
                denom *= (j - m)
            integ = sum(c * (Fraction(b) ** (k + 1) - Fraction(a) ** (k + 1)) / (k + 1)
                        for k, c in enumerate(coeffs)) / denom
            out.append(integ)
            continue
        # moments: M_{i-1} + 4 M_i + M_{i+1} = 6 (F_{i-1} - 2 F_i + F_{i+1}), i = 1..K-1,
        # not-a-knot: M_0 - 2 M_1 + M_2 = 0, M_{K-2} - 2 M_{K-1} + M_K = 0 (s''' continuous)
        n = K + 1
        A = [[Fraction(0)] * n for _ in range(n)]
        r = [Fraction(0)] * n
        A[0][0], A[0][1], A[0][2] = Fraction(1), Fraction(-2), Fraction(1)
        A[K][K - 2], A[K][K - 1], A[K][K] = Fraction(1), Fraction(-2), Fraction(1)
        for i in range(1, K):
            A[i][i - 1], A[i][i], A[i][i + 1] = Fraction(1), Fraction(4), Fraction(1)
            r[i] = 6 * (data[i - 1] - 2 * data[i] + data[i + 1])
        # Gaussian elimination, exact
        for c in range(n):
            p = next(k for k in range(c, n) if A[k][c] != 0)
            A[c], A[p] = A[p], A[c]
            r[c], r[p] = r[p], r[c]
            for k in range(n):
                if k != c and A[k][c] != 0:
                    f = A[k][c] / A[c][c]
                    A[k] = [x - f * y for x, y in zip(A[k], A[c])]
                    r[k] -= f * r[c]
        M = [r[i] / A[i][i] for i in range(n)]
        # integral of the cubic spline over cell [i, i+1]: (F_i + F_{i+1})/2 - (M_i + M_{i+1})/24
        tot = Fraction(0)
        for i in range(a, b):
            tot += (data[i] + data[i + 1]) / 2 - (M[i] + M[i + 1]) / 24
        out.append(tot)
    return out


def test_P1_gamma_tables_printed_equal_not_a_knot_derivation():
    """Tables 1-2 are (1/K) int_0^K and int_0^1 of the temporal
    not-a-knot spline's cardinal functions (Eq. 8-15)."""
    for row in _golden("gamma_tables.txt"):
        table, K = int(row[0]), int(row[1])
        printed = [Fraction(v) for v in row[2:]]
        assert len(printed) == K + 1
        if table == 1:
            derived = [v / K for v in _not_a_knot_cardinal_integrals(K, 0, K)]
        else:
            derived = _not_a_knot_cardinal_integrals(K, 0, 1)
        assert derived == printed, (table, K, derived, printed)
        assert sum(printed) == 1


def test_P1_oracle_gamma_equals_printed(oracle_mod):
    for row in _golden("gamma_tables.txt"):
        table, K = int(row[0]), int(row[1])
        printed = np.array([float(Fraction(v)) for v in row[2:]])
        got = oracle_mod.gamma_row(K, "y" if table == 1 else "z")
        assert np.array_equal(got, printed)


def test_P1_worked_example_Ky3():
    """K_y = 3 worked example PAPER.md:222-228: 3/8, 9/8, 9/8, 3/8 == Ky * gamma."""
    g = _not_a_knot_cardinal_integrals(3, 0, 3)
    assert g == [Fraction(3, 8), Fraction(9, 8), Fraction(9, 8), Fraction(3, 8)]


# --------------------------------------------------------------------------- P2
@pytest.mark.parametrize("L", [1, 2, 3, 5, 8, 16, 32, 64])
def test_P2_gauss_hermite_exactness(oracle_mod, L):
    """Eq. 21 rule: exact for monomials of degree <= 2L-1 against e^{-a^2}."""
    a, w = oracle_mod.gauss_hermite(L)
    assert np.all(w > 0) and np.all(np.diff(a) > 0)
    assert abs(w.sum() - math.sqrt(math.pi)) < 1e-14
    for k in range(0, min(2 * L, 40)):
        exact = 0.0 if k % 2 else math.gamma((k + 1) / 2)
        terms = w * a.astype(np.longdouble) ** k
        got = float(np.sum(terms))
        scale = float(np.sum(np.abs(terms)))
        assert abs(got - exact) <= 1e-13 * max(1.0, scale), (L, k, got, exact)


def test_P2_gauss_hermite_textbook_values(oracle_mod):
    a, w = oracle_mod.gauss_hermite(2)
    assert np.allclose(a, [-1 / math.sqrt(2), 1 / math.sqrt(2)], rtol=0, atol=1e-15)
    assert np.allclose(w, [math.sqrt(math.pi) / 2] * 2, rtol=1e-15)
    a, w = oracle_mod.gauss_hermite(3)
    assert np.allclose(a, [-math.sqrt(1.5), 0.0, math.sqrt(1.5)], atol=1e-15)
    assert np.allclose(w, [math.sqrt(math.pi) / 6, 2 * math.sqrt(math.pi) / 3, math.sqrt(math.pi) / 6], rtol=1e-14)
    for L, amax in [(8, 2.930637420257244), (16, 4.688738939305818), (32, 7.125813909830728)]:
        a, _ = oracle_mod.gauss_hermite(L)
        assert abs(a[-1] - amax) < 1e-13


@pytest.mark.parametrize("L", [4, 8, 16, 32, 64])
def test_P2_gauss_hermite_vs_numpy(oracle_mod, L):
    a, w = oracle_mod.gauss_hermite(L)
    ra, rw = np.polynomial.hermite.hermgauss(L)
    assert np.allclose(a, ra, rtol=0, atol=1e-13)
    assert np.allclose(w, rw, rtol=1e-10, atol=1e-300)


# --------------------------------------------------------------------------- P3/P4
def test_P4_thomas_dense(oracle_mod):
    rng = np.random.Generator(np.random.PCG64(1909135600))
    n = 64
    a = rng.uniform(-1, 1, n)
    c = rng.uniform(-1, 1, n)
    b = 3.0 + rng.uniform(0, 1, n)
    r = rng.uniform(-1, 1, n)
    x = oracle_mod.thomas(a, b, c, r)
    A = np.diag(b) + np.diag(a[1:], -1) + np.diag(c[:-1], 1)
    assert np.max(np.abs(A @ x - r)) <= 1e-12 * (1 + np.max(np.abs(r)))
    assert np.allclose(x, np.linalg.solve(A, r), rtol=1e-13, atol=1e-14)


def test_P3_spline_reproduces_cubics(oracle_mod):
    rng = np.random.Generator(np.random.PCG64(1909135601))
    for P in [4, 5, 7, 33, 200]:
        x = np.linspace(-3.0, 5.0, P)
        c = rng.uniform(-1, 1, 4)
        f = lambda t: c[0] + c[1] * t + c[2] * t ** 2 + c[3] * t ** 3  # noqa: E731
        F = f(x)
        M = oracle_mod.spline_moments(F, x[1] - x[0])
        assert np.allclose(M, 2 * c[2] + 6 * c[3] * x, rtol=1e-9, atol=1e-9)
        X = rng.uniform(-3.0, 5.0, 100)
        got = oracle_mod.spline_eval(F, M, -3.0, x[1] - x[0], X)
        assert np.max(np.abs(got - f(X))) <= 1e-12 * np.max(np.abs(F)) * 10


def test_P3_spline_equals_scipy_not_a_knot(oracle_mod):
    from scipy.interpolate import CubicSpline
    rng = np.random.Generator(np.random.PCG64(1909135602))
    for P in [4, 6, 50, 1000]:
        dx = 0.125                      # exactly representable grid, so both sides see the same knots
        x = -16.0 + dx * np.arange(P)
        F = np.sin(x) + rng.normal(size=P) * 0.1
        M = oracle_mod.spline_moments(F, dx)
        cs = CubicSpline(x, F, bc_type="not-a-knot")
        assert np.allclose(M, cs(x, 2), rtol=0, atol=1e-12 * np.max(np.abs(M)))
        X = rng.uniform(x[0], x[-1], 300)
        assert np.allclose(oracle_mod.spline_eval(F, M, -16, dx, X), cs(X), rtol=0, atol=1e-13)
        # clamping: outside the box the boundary value
        assert oracle_mod.spline_eval(F, M, -16, dx, [-40.0])[0] == F[0]
        assert abs(oracle_mod.spline_eval(F, M, -16, dx, [x[-1] + 40.0])[0] - F[-1]) <= 1e-14 * max(1, abs(F[-1]))


def test_P3_spline_linear_constant(oracle_mod):
    x = np.linspace(0, 1, 9)
    M = oracle_mod.spline_moments(2 * x + 1, x[1] - x[0])
    assert np.max(np.abs(M)) < 1e-10
    M = oracle_mod.spline_moments(np.full(9, 3.5), x[1] - x[0])
    assert np.max(np.abs(M)) == 0.0


# --------------------------------------------------------------------------- balance rule
def test_balance_rule_reproduces_printed_M(oracle_mod):
    """Reading R3: M = 2 ceil(X/dx), dx = dt^{(q+1)/4}, q = min{Ky+1, Kz, 3}; all printed M."""
    for row in _golden("balance_M.txt"):
        _, half, T, K, N, M = row
        P = oracle_mod.balance_npts(2 * float(half), float(T) / int(N), int(K), int(K), 4)
        assert P == int(M) + 1, row


# --------------------------------------------------------------------------- closed forms (P11)
def test_P11_closed_forms_match_printed(oracle_mod):
    from paper_1909_13560_b200 import workloads as W
    from scipy.stats import norm
    # Ex. 1 (Eq. 23) and Ex. 2 (Eq. 25)
    y, z = oracle_mod.exact(W.ex1(3, 8), 0.0, [0.0])
    assert y == 0.5 and z[0] == 0.25
    y, z = oracle_mod.exact(W.ex2(3, 8), 0.0, [0.0])
    assert abs(y - math.log(3)) < 1e-15 and abs(z[0] - 1 / 3) < 1e-15
    # Black-Scholes (Eq. 31, delta in d1: reading R13) vs the printed 4.3671 / 10.0950
    bs = W.black_scholes(3, 32)
    y, z = oracle_mod.exact(bs, 0.0, [0.0])
    assert round(y, 4) == 4.3671 and round(z[0], 4) == 10.0950
    S, K, r, q, s, T = 100.0, 100.0, 0.03, 0.04, 0.2, 0.33
    d1 = (math.log(S / K) + (r - q + s * s / 2) * T) / (s * math.sqrt(T))
    ref = S * math.exp(-q * T) * norm.cdf(d1) - K * math.exp(-r * T) * norm.cdf(d1 - s * math.sqrt(T))
    assert abs(y - ref) < 1e-12
    # Ex. 4 (Eq. 35)
    y, z = oracle_mod.exact(W.ex4_2d(3, 8), 0.0, [0.0, 0.0])
    assert abs(y) < 1e-15 and np.allclose(z, [1, 1])
    # Ex. 5 Margrabe (Eq. 37) at T=1 (reading R12) vs printed 15.48076, -12.6779
    y, z = oracle_mod.exact(W.exchange_2d(3, 8), 0.0, [0.0, 0.0])
    assert round(y, 5) == 15.48076 and round(z[1], 4) == -12.6779 and round(z[0], 4) == 14.4351


def test_closed_forms_are_exact_at_terminal_and_solve_pde(oracle_mod):
    """u(T, w) = g(w), and u_t + 1/2 Laplace u + f(t, u, grad u) = 0 (Eq. 5) by finite differences."""
    from paper_1909_13560_b200 import workloads as W
    specs = [W.ex1(3, 8), W.ex2(3, 8), W.black_scholes(3, 8), W.diff_rates(3, 8, P=64),
             W.ex4_2d(3, 8), W.exchange_2d(3, 8), W.basket_3d(P=8), W.ex1_3d(P=8)]
    for spec in specs:
        d = spec["d"]
        w = np.array([0.13, -0.21, 0.07][:d])
        t = 0.4 * spec["T"]
        h = 1e-3
        y, z = oracle_mod.exact(spec, t, w)
        yt = (oracle_mod.exact(spec, t + h, w)[0] - oracle_mod.exact(spec, t - h, w)[0]) / (2 * h)
        lap = 0.0
        for a in range(d):
            e = np.zeros(d)
            e[a] = h
            yp, zp = oracle_mod.exact(spec, t, w + e)
            ym, zm = oracle_mod.exact(spec, t, w - e)
            lap += (yp - 2 * y + ym) / h ** 2
            assert abs((yp - ym) / (2 * h) - z[a]) < 1e-5 * max(1, abs(z[a])), spec["name"]
        f = oracle_mod.driver(spec, t, y, z)
        res = yt + 0.5 * lap + f
        assert abs(res) < 2e-4 * max(1.0, abs(y)), (spec["name"], res)


# --------------------------------------------------------------------------- P6/P7/P8
@pytest.mark.parametrize("K", [1, 2, 3, 4, 5, 6])
def test_P6_heat_polynomial_exact_1d(oracle_mod, K):
    """f = 0, g = x^3: y = x^3 + 3x(T-t), z = 3x^2 + 3(T-t) for every K, away from the box edge."""
    from paper_1909_13560_b200 import workloads as W
    spec = W.heat_poly(1, K, N=8, P=513, T=0.25, box=16.0, L=16)
    o = oracle_mod.Oracle(spec, nthreads=4)
    o.solve()
    x = np.linspace(-16, 16, 513)
    m = np.abs(x) <= 6
    y, z = o.layer(0), o.layer(1)
    assert np.max(np.abs(y[m] - (x[m] ** 3 + 3 * x[m] * 0.25))) <= 3e-13 * 216
    assert np.max(np.abs(z[m] - (3 * x[m] ** 2 + 0.75))) <= 3e-13 * 108


def test_P6_heat_polynomial_exact_2d(oracle_mod):
    from paper_1909_13560_b200 import workloads as W
    spec = W.heat_poly(2, 3, N=5, P=65, T=0.25, box=16.0, L=8)
    o = oracle_mod.Oracle(spec, nthreads=4)
    o.solve()
    x = np.linspace(-16, 16, 65)
    X1, X2 = np.meshgrid(x, x, indexing="ij")
    m = (np.abs(X1) <= 5) & (np.abs(X2) <= 5)
    tau = 0.25
    y = o.layer(0)
    yex = X1 ** 3 * X2 + 3 * X1 * X2 * tau
    z1ex = 3 * X1 ** 2 * X2 + 3 * X2 * tau
    z2ex = X1 ** 3 + 3 * X1 * tau
    assert np.max(np.abs(y[m] - yex[m])) <= 1e-12 * 625
    assert np.max(np.abs(o.layer(1)[m] - z1ex[m])) <= 1e-12 * 375
    assert np.max(np.abs(o.layer(2)[m] - z2ex[m])) <= 1e-12 * 125


@pytest.mark.parametrize("Ky,Kz", [(Ky, Kz) for Ky in range(1, 7) for Kz in range(1, 7)])
def test_P8_constant_solution_invariant(oracle_mod, Ky, Kz):
    """f = 0, g = c  =>  y = c, z = 0 everywhere, including the boundary (all 36 pairs)."""
    from paper_1909_13560_b200 import workloads as W
    spec = W.constant(1, Ky, Kz, N=10, P=40, c=2.5, L=8)
    o = oracle_mod.Oracle(spec, nthreads=2)
    o.solve()
    assert np.max(np.abs(o.layer(0) - 2.5)) <= 1e-14
    assert np.max(np.abs(o.layer(1))) <= 1e-14


@pytest.mark.parametrize("K", [1, 2, 3, 4, 6])
def test_P7_scalar_recurrence(oracle_mod, K):
    """f = -r y, constant data: y^n (1 + K dt gamma_0 r) = y^{n+K} - r K dt sum_j gamma_j y^{n+j}
    in exact rational arithmetic (Eq. 20 with E[c] = c); initial layers exact c e^{-r(T-t)}."""
    from paper_1909_13560_b200 import workloads as W
    rate, N, c = 0.7, 12, 2.5
    spec = W.constant(1, K, K, N=N, P=16, c=c, L=4, rate=rate)
    o = oracle_mod.Oracle(spec, nthreads=1)
    y0, _ = o.solve()
    gam = [Fraction(v) for v in _golden("gamma_tables.txt")[K - 1][2:]]
    dt = Fraction(1, N)
    r = Fraction(rate)
    ys = {}
    for m in range(N, N - K, -1):
        ys[m] = c * math.exp(-rate * float((N - m) * dt))
    ys = {m: Fraction(v) for m, v in ys.items()}
    for n in range(N - K, -1, -1):
        rhs = ys[n + K] - r * K * dt * sum(gam[j] * ys[n + j] for j in range(1, K + 1))
        ys[n] = rhs / (1 + K * dt * gam[0] * r)
    assert abs(y0 - float(ys[0])) <= 2e-15 * abs(float(ys[0]))


def test_P7_picard_closed_form(oracle_mod):
    """f = -y, K_y = 1, one step from g = c: the fixed point of the Picard map of Eq. 20,
    y = c + dt (-c/2 - y/2), i.e. y = c (1 - dt/2) / (1 + dt/2)."""
    from paper_1909_13560_b200 import workloads as W
    spec = dict(W.constant(1, 1, 1, N=1, P=8, c=3.0, L=2, rate=1.0), T=0.02)
    o = oracle_mod.Oracle(spec, nthreads=1)
    y0, _ = o.solve()
    assert abs(y0 - 3.0 * 0.99 / 1.01) <= 2e-15
    assert np.all(o.picard_counts() == 30)


# --------------------------------------------------------------------------- P9/P10 printed rows
def _rows(example, maxN):
    return [r for r in _golden("printed_errors.txt") if r[0] == example and int(r[2]) <= maxN]


@pytest.mark.parametrize("row", _rows("ex1", 256) + _rows("ex2", 256), ids=lambda r: f"{r[0]}_K{r[1]}_N{r[2]}")
def test_P9_printed_rows_1d(oracle_mod, row):
    from paper_1909_13560_b200 import workloads as W
    ex, K, N, M, ye, ze, _ = row
    K, N = int(K), int(N)
    if N > 512 and K > 1:
        pytest.skip("too slow for the CPU suite")
    spec = (W.ex1 if ex == "ex1" else W.ex2)(K, N)
    o = oracle_mod.Oracle(spec, nthreads=os.cpu_count())
    assert o.shape == (int(M) + 1,)
    y0, z0 = o.solve()
    ref = W.reference_solution(spec)
    ey, ez = abs(y0 - ref[0]), abs(z0[0] - ref[1][0])
    assert abs(ey / float(ye) - 1) <= 0.03, (ey, ye)
    assert abs(ez / float(ze) - 1) <= 0.03, (ez, ze)


@pytest.mark.parametrize("row", _rows("ex4", 16), ids=lambda r: f"{r[0]}_K{r[1]}_N{r[2]}")
def test_P10_printed_rows_2d(oracle_mod, row):
    from paper_1909_13560_b200 import workloads as W
    _, K, N, M, ye, ze, _ = row
    K, N = int(K), int(N)
    spec = W.ex4_2d(K, N)
    o = oracle_mod.Oracle(spec, nthreads=os.cpu_count())
    assert o.shape == (int(M) + 1,) * 2
    y0, z0 = o.solve()
    ey = abs(y0 - 0.0)
    ez = float(np.linalg.norm(np.asarray(z0) - 1.0))   # Euclidean norm (reading R15)
    tol_z = 0.05 if K == 1 else 0.03
    assert abs(ey / float(ye) - 1) <= 0.03, (ey, ye)
    assert abs(ez / float(ze) - 1) <= tol_z, (ez, ze)


# --------------------------------------------------------------------------- P12 orders
def _order(errs, Ns):
    return -np.polyfit(np.log(Ns), np.log(errs), 1)[0]


def test_P12_convergence_orders(oracle_mod):
    """Theorems 1-2 on the balanced grid: K=1 -> order ~1, K=3 -> ~3 (Ex. 2)."""
    from paper_1909_13560_b200 import workloads as W
    for K, Ns, lo in [(1, [64, 128, 256], 0.65), (3, [32, 64, 128], 2.65)]:
        ey, ez = [], []
        for N in Ns:
            o = oracle_mod.Oracle(W.ex2(K, N), nthreads=os.cpu_count())
            y0, z0 = o.solve()
            ey.append(abs(y0 - math.log(3)))
            ez.append(abs(z0[0] - 1 / 3))
        assert _order(ey, Ns) >= lo and _order(ez, Ns) >= lo, (K, ey, ez)


# --------------------------------------------------------------------------- determinism, bootstrap, smoothing
def test_determinism_thread_count(oracle_mod):
    from paper_1909_13560_b200 import workloads as W
    spec = W.diff_rates(4, N=12, P=301)
    a = oracle_mod.Oracle(spec, nthreads=1)
    a.solve()
    b = oracle_mod.Oracle(spec, nthreads=os.cpu_count())
    b.solve()
    assert np.array_equal(a.layers(), b.layers())


def test_bootstrap_converges_to_exact_start(oracle_mod):
    """Reading R9: the one-step start with S_b sub-steps approaches the exact-start result."""
    from paper_1909_13560_b200 import workloads as W
    spec = W.ex1(3, 32)
    exact0, _ = oracle_mod.Oracle(spec, nthreads=os.cpu_count()).solve()
    errs = []
    for sb in [1, 4, 16]:
        s = dict(spec, bootstrap=1, bootstrap_substeps=sb)
        y, _ = oracle_mod.Oracle(s, nthreads=os.cpu_count()).solve()
        errs.append(abs(y - exact0))
    assert errs[0] > errs[1] > errs[2]
    assert errs[2] < 0.2 * errs[0]


def test_smoothing_is_the_cell_average(oracle_mod):
    """Reading R11: smoothed y^N at kink cells equals the cell average of g (scipy quad)."""
    from scipy.integrate import quad, dblquad
    from paper_1909_13560_b200 import workloads as W
    spec = dict(W.black_scholes(1, 4, L=4, npts=101), N=1, Ky=1, Kz=1)
    o = oracle_mod.Oracle(spec, nthreads=1)
    x = np.linspace(-16, 16, 101)
    h = x[1] - x[0]
    y = o.layer(0)
    smoothed = 0
    for i, xi in enumerate(x):
        g = lambda w: oracle_mod.terminal(spec, [w])[0]  # noqa: E731
        if (g(xi - h / 2) == 0) != (g(xi + h / 2) == 0):
            S0, K, mu, sg = spec["terminal_params"][:4]
            wk = (math.log(K / S0) - (mu - sg * sg / 2) * spec["T"]) / sg    # kink of (S_T(w) - K)^+
            avg = quad(g, xi - h / 2, xi + h / 2, points=[wk], limit=200, epsabs=1e-14, epsrel=1e-14)[0] / h
            assert abs(y[i] - avg) < 1e-10 * max(1, abs(avg))
            smoothed += 1
        else:
            assert y[i] == g(xi)
    assert smoothed == 1
    spec2 = dict(W.exchange_2d(1, 4, npts=33), N=1)
    o2 = oracle_mod.Oracle(spec2, nthreads=4)
    x = np.linspace(-8, 8, 33)
    h = x[1] - x[0]
    y2 = o2.layer(0)
    i, j = 16, 16   # x = (0, 0): S1 = S2 at the origin -> kink through the cell
    g2 = lambda b, a: oracle_mod.terminal(spec2, [a, b])[0]  # noqa: E731
    avg = dblquad(g2, x[i] - h / 2, x[i] + h / 2, x[j] - h / 2, x[j] + h / 2, epsabs=1e-12)[0] / h ** 2
    assert abs(y2[i, j] - avg) < 2e-4 * abs(avg)
