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
def _rows(example, maxN, minN=0):
    """Gated rows of tests/golden/printed_tables.txt (every printed row of Tables 4, 5, 9 with the
    reason of each exclusion: R10 for K = 2, the rounding floor for y < 1e-12, Table 9 K=1 N=8 z)."""
    return [r for r in _golden("printed_tables.txt")
            if r[0] == example and minN <= int(r[2]) <= maxN and r[7] != "-"]


def _check_row(row, ey, ez):
    _, K, N, M, ye, ze, line, gate, _ = row
    if "y" in gate:
        assert abs(ey / float(ye) - 1) <= 0.03, (ey, ye, line)
    if "z" in gate:
        assert abs(ez / float(ze) - 1) <= 0.03, (ez, ze, line)


@pytest.mark.parametrize("row", _rows("ex1", 128) + _rows("ex2", 128) +
                         [r for r in _rows("ex1", 256, 256) + _rows("ex2", 256, 256) if r[1] == "1"],
                         ids=lambda r: f"{r[0]}_K{r[1]}_N{r[2]}")
def test_P9_printed_rows_1d(oracle_mod, row):
    """Printed rows of Tables 4 and 5 (Ex. 1, Ex. 2) reproduced to 3 % by the oracle (the CPU suite
    runs N <= 128 and the K = 1, N = 256 rows; the GPU suite runs every gated row)."""
    from paper_1909_13560_b200 import workloads as W
    ex, K, N, M = row[0], int(row[1]), int(row[2]), int(row[3])
    spec = (W.ex1 if ex == "ex1" else W.ex2)(K, N)
    o = oracle_mod.Oracle(spec, nthreads=os.cpu_count())
    assert o.shape == (M + 1,)
    y0, z0 = o.solve()
    ref = W.reference_solution(spec)
    _check_row(row, abs(y0 - ref[0]), abs(z0[0] - ref[1][0]))


@pytest.mark.parametrize("row", _rows("ex4", 16), ids=lambda r: f"{r[0]}_K{r[1]}_N{r[2]}")
def test_P10_printed_rows_2d(oracle_mod, row):
    """Table 9 (Ex. 4) with the tensor spline (north_star, reading R14)."""
    from paper_1909_13560_b200 import workloads as W
    K, N, M = int(row[1]), int(row[2]), int(row[3])
    spec = W.ex4_2d(K, N)
    o = oracle_mod.Oracle(spec, nthreads=os.cpu_count())
    assert o.shape == (M + 1,) * 2
    y0, z0 = o.solve()
    _check_row(row, abs(y0 - 0.0), float(np.linalg.norm(np.asarray(z0) - 1.0)))   # Euclidean z (R15)


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


# --------------------------------------------------------------------------- d = 3 pins
# The 3-D oracle path (tensor spline by successive Thomas passes in build_spline /
# eval_spline, the L^3 tensor tap loop of point_step, the GL16^3 smoothing box_avg) is
# pinned against: exact polynomial solutions (P6), the constant invariant (P8), the 1-D
# oracle on data that vary along one axis only (the tensor spline of such data is the 1-D
# spline, the tensor GH rule of such a function is the 1-D rule), scipy's tensor-product
# not-a-knot B-spline interpolant (library), and nested scipy quad of the payoff (smoothing).

def _poly3_spec(K, factors, N=4, P=17, T=0.25, box=4.0, L=4):
    """f = 0, g = prod_a p_a(x_a) with cubic factors p_a (coefficients c0..c3 per axis)."""
    from paper_1909_13560_b200 import workloads as W
    s = W.heat_poly(3, K, N=N, P=P, T=T, box=box, L=L)
    s["terminal_params"] = [float(c) for f in factors for c in f]
    return s


def _heat_cubic(c, x, tau):
    """E[p(x + W_tau)] and its x-derivative for a cubic p (W_tau ~ N(0, tau)):
    E[(x+W)^2] = x^2 + tau, E[(x+W)^3] = x^3 + 3 x tau."""
    v = c[0] + c[1] * x + c[2] * (x * x + tau) + c[3] * (x ** 3 + 3 * x * tau)
    dv = c[1] + 2 * c[2] * x + 3 * c[3] * (x * x + tau)
    return v, dv


@pytest.mark.parametrize("K", [1, 2, 3])
def test_P6_heat_polynomial_exact_3d(oracle_mod, K):
    """P6, d = 3: f = 0, g = p1(x1) p2(x2) p3(x3) with factors of degree 3, 2, 3 (distinct per
    axis, so a swapped axis, stride or corner weight breaks exactness).  The tensor not-a-knot
    spline reproduces g, the L = 4 tensor Gauss-Hermite rule integrates degree <= 7 per axis
    exactly, so y = prod_a E[p_a(x_a + W)] and z_a = dE[p_a]/dx_a prod_{b != a} E[p_b] hold to
    rounding at every point whose taps stay inside the box (Eq. 20-21).
    N = K: one sweep step from K exact levels (closed-form initial layers, reading R9), so the
    clamped boundary taps of earlier steps cannot leak inward through the spline's global
    coupling (0.268^k per cell); multi-step propagation in 3-D is pinned by the 1-D embedding
    test below."""
    factors = [[0.0, 0.0, 0.0, 1.0], [0.5, 1.0, 1.0, 0.0], [0.0, -2.0, 0.0, 1.0]]
    spec = _poly3_spec(K, factors, N=K)
    o = oracle_mod.Oracle(spec, nthreads=os.cpu_count())
    o.solve()
    x = np.linspace(-4.0, 4.0, 17)
    tau = spec["T"]
    vals = [_heat_cubic(f, x, tau) for f in factors]
    m = np.abs(x) <= 2.5                                   # taps reach sqrt(2 T) a_max = 1.17 < 4 - 2.5
    X = np.ix_(m, m, m)
    v = [vals[a][0][m] for a in range(3)]
    dv = [vals[a][1][m] for a in range(3)]
    y_ex = np.einsum("i,j,k->ijk", v[0], v[1], v[2])
    z_ex = [np.einsum("i,j,k->ijk", dv[0], v[1], v[2]), np.einsum("i,j,k->ijk", v[0], dv[1], v[2]),
            np.einsum("i,j,k->ijk", v[0], v[1], dv[2])]
    L = o.layers()
    assert np.max(np.abs(L[0][X] - y_ex)) <= 1e-12 * np.max(np.abs(y_ex))
    for a in range(3):
        assert np.max(np.abs(L[1 + a][X] - z_ex[a])) <= 1e-12 * np.max(np.abs(z_ex[a])), a


@pytest.mark.parametrize("Ky,Kz", [(1, 1), (1, 3), (3, 1), (2, 2), (3, 3), (2, 4)])
def test_P8_constant_solution_invariant_3d(oracle_mod, Ky, Kz):
    """P8, d = 3: f = 0, g = c gives y = c, z = 0 at every point, boundary included."""
    from paper_1909_13560_b200 import workloads as W
    spec = dict(W.constant(3, Ky, Kz, N=6, P=6, c=2.5, L=3), npts=[5, 6, 7])
    o = oracle_mod.Oracle(spec, nthreads=2)
    o.solve()
    L = o.layers()
    assert np.max(np.abs(L[0] - 2.5)) <= 1e-14
    assert np.max(np.abs(L[1:])) <= 1e-14


def _embedded_pair(K, Ky, Kz, axis, driver):
    """A 1-D problem and the same problem embedded in 3-D along `axis` (data constant along
    the other two axes, transverse sizes 5 and 6)."""
    from paper_1909_13560_b200 import workloads as W
    if driver == "diff_rates":                     # z-dependent nonlinear driver, call payoff (x_0 only)
        s1 = W.diff_rates(K, N=6, P=41, L=6, smoothing=0)
    else:                                          # Ex. 1 driver, bounded cubic terminal
        s1 = dict(W.ex1(K, 6, L=6, npts=41), terminal="poly", terminal_params=[0.5, 0.08, 0.004, -0.0015])
    s1 = dict(s1, Ky=Ky, Kz=Kz, T=0.5, xlo=[-6.0], xhi=[6.0], bootstrap=1, bootstrap_substeps=2)
    shape = [5, 6, 6]
    shape[axis] = 41
    s3 = dict(s1, d=3, npts=shape, xlo=[-3.0, -2.0, -4.0], xhi=[3.0, 2.5, 4.0])
    s3["xlo"][axis], s3["xhi"][axis] = -6.0, 6.0
    if driver == "diff_rates":
        dp = list(s1["driver_params"])
        s3["driver_params"] = [dp[0], dp[1], dp[2], 0.0, 0.0, dp[5], 0.0, 0.0]
    else:
        tp = [1.0, 0.0, 0.0, 0.0] * 3
        tp[4 * axis:4 * axis + 4] = s1["terminal_params"][:4]
        s3["terminal_params"] = tp
    return s1, s3


@pytest.mark.parametrize("driver,axis,K,Ky,Kz", [("diff_rates", 0, 3, 3, 3), ("ex1", 0, 2, 2, 1),
                                                  ("ex1", 1, 3, 2, 3), ("ex1", 2, 3, 3, 3),
                                                  ("ex1", 2, 1, 1, 1)])
def test_3d_oracle_equals_1d_oracle_on_axis_data(oracle_mod, driver, axis, K, Ky, Kz):
    """Data varying along one axis only: the tensor spline (moments of constant lines are 0)
    is the 1-D spline of that axis, and the L^3 tensor Gauss-Hermite rule of a function of
    x_axis is the 1-D rule times sum_b w_b sum_c w_c / pi = 1.  So every layer of the 3-D
    oracle restricted to one transverse line equals the 1-D oracle's layer (to rounding), z of
    the other two axes vanishes, and this holds for a nonlinear, z-dependent driver (Eq. 20
    with Eq. 21), the bootstrap and Ky != Kz.  A mask -> axis, stride, corner
    weight or dW-axis mistake in the 3-D path shows up as an O(1) difference."""
    s1, s3 = _embedded_pair(K, Ky, Kz, axis, driver)
    o1 = oracle_mod.Oracle(s1, nthreads=os.cpu_count())
    o1.solve()
    o3 = oracle_mod.Oracle(s3, nthreads=os.cpu_count())
    o3.solve()
    L1, L3 = o1.layers(), o3.layers()
    y3 = np.moveaxis(L3[0], axis, -1).reshape(-1, 41)
    z3 = np.moveaxis(L3[1 + axis], axis, -1).reshape(-1, 41)
    for row in range(y3.shape[0]):
        assert np.max(np.abs(y3[row] - L1[0])) <= 1e-13 * np.max(np.abs(L1[0])), row
        assert np.max(np.abs(z3[row] - L1[1])) <= 1e-13 * np.max(np.abs(L1[1])), row
    for b in range(3):
        if b != axis:
            assert np.max(np.abs(L3[1 + b])) <= 1e-13 * np.max(np.abs(L1[1]))


def test_P3_spline_3d_equals_scipy_tensor_not_a_knot(oracle_mod):
    """The oracle's 3-D tensor spline (values + moments, successive Thomas passes) equals
    scipy's tensor-product not-a-knot cubic B-spline interpolant (make_interp_spline along each
    axis, NdBSpline), on a non-cubic grid with distinct sizes and boxes per axis, at random
    points inside and outside the box (clamped per coordinate)."""
    from scipy.interpolate import make_interp_spline, NdBSpline
    from paper_1909_13560_b200 import workloads as W
    spec = dict(W.ex1_3d(K=1, N=4, L=2, P=9), npts=[9, 11, 13], xlo=[-4.0, -3.0, -5.0], xhi=[4.0, 2.0, 3.0])
    o = oracle_mod.Oracle(spec, nthreads=2)
    V = o.layers()
    axes = [np.linspace(lo, hi, n) for lo, hi, n in zip(spec["xlo"], spec["xhi"], spec["npts"])]
    rng = np.random.Generator(np.random.PCG64(1909135600))
    pts = [[rng.uniform(lo - 1, hi + 1) for lo, hi in zip(spec["xlo"], spec["xhi"])] for _ in range(100)]
    got = np.array([o.eval_newest(x) for x in pts])
    for f in range(4):
        c, ts = V[f], []
        for a in range(3):
            sp = make_interp_spline(axes[a], c, k=3, axis=a)      # not-a-knot for k = 3
            c = np.moveaxis(sp.c, 0, a)
            ts.append(sp.t)
        nd = NdBSpline(tuple(ts), c, 3)
        ref = nd(np.clip(pts, spec["xlo"], spec["xhi"]))
        assert np.max(np.abs(got[:, f] - ref)) <= 1e-13 * np.max(np.abs(V[f])), f


def test_smoothing_3d_is_the_cell_average(oracle_mod):
    """Reading R11 in 3-D: at a grid point whose cell meets the payoff kink, y^N is the cell
    average of g (geometric-basket call).  Reference: nested scipy quad with the
    kink plane (log G is affine in w) passed as a break point.  The oracle's GL16^3 rule of a
    kinked integrand is accurate to ~1e-4 of the payoff scale; a wrong operator (point value,
    shifted cell) is off by O(1) of it."""
    import math
    from scipy.integrate import quad
    from paper_1909_13560_b200 import workloads as W
    spec = dict(W.basket_3d(K=1, N=2, L=2, P=9), npts=[9, 9, 9])
    o = oracle_mod.Oracle(spec, nthreads=2)
    V = o.layers()
    p = spec["terminal_params"]
    S0, K, mu, sg, T = p[:3], p[3], p[4], p[5:8], spec["T"]
    alpha = sum(math.log(S0[k]) + (mu - 0.5 * sg[k] ** 2) * T for k in range(3)) / 3
    beta = [s / 3 for s in sg]

    def g(a, b, c):
        return max(math.exp(alpha + beta[0] * a + beta[1] * b + beta[2] * c) - K, 0.0)

    def kink(b, c):
        return (math.log(K) - alpha - beta[1] * b - beta[2] * c) / beta[0]

    x = np.linspace(-8, 8, 9)
    h = x[1] - x[0]
    i, j, k = 0, 3, 7                                     # the kink plane crosses this cell
    lo = [x[i] - h / 2, x[j] - h / 2, x[k] - h / 2]
    hi = [x[i] + h / 2, x[j] + h / 2, x[k] + h / 2]
    corners = [g(a, b, c) for a in (lo[0], hi[0]) for b in (lo[1], hi[1]) for c in (lo[2], hi[2])]
    assert min(corners) == 0.0 < max(corners)

    def inner(b, c):
        kp = min(max(kink(b, c), lo[0]), hi[0])
        return quad(lambda a: g(a, b, c), lo[0], hi[0], points=[kp], epsabs=1e-12, epsrel=1e-12)[0]

    mid = lambda c: quad(lambda b: inner(b, c), lo[1], hi[1], epsabs=1e-10, epsrel=1e-10)[0]  # noqa: E731
    avg = quad(mid, lo[2], hi[2], epsabs=1e-10, epsrel=1e-10)[0] / h ** 3
    assert abs(V[0][i, j, k] - avg) <= 1e-3 * max(corners), (V[0][i, j, k], avg)
    # away from the kink the terminal layer is g itself
    assert abs(V[0][8, 8, 8] - g(x[8], x[8], x[8])) <= 1e-14 * V[0][8, 8, 8] and V[0][0, 0, 0] == 0.0


# --------------------------------------------------------------------------- forward SDE (Eq. 1)
# The FBSDE of Eq. 1 with the forward process approximated "by using the
# Euler-Scheme": the level-j sample from x_i is x_i + a(x_i) j dt + b(x_i) dW_j.

def _fsde_spec(sde, sp, terminal, tp, driver="zero", dp=(), K=1, N=2, P=257, box=(-8.0, 8.0), T=0.1, L=8):
    return dict(d=1, t0=0.0, T=T, N=N, Ky=K, Kz=K, L=L, npts=[P], xlo=[box[0]], xhi=[box[1]], r=4,
                driver=driver, driver_params=list(dp), terminal=terminal, terminal_params=list(tp),
                sde=sde, sde_params=list(sp), bootstrap=1, bootstrap_substeps=2, picard_max=30, name=f"fsde_{sde}")


def test_fsde_brownian_special_case_is_the_bsde_path(oracle_mod):
    """OU with kappa = 0, sigma = 1 is X = W: the Euler sample x + 0 * j dt + 1 * dW is bitwise
    x + dW, so every layer equals the X = W solve of Eq. 2 (Ex. 2 driver, K = 3, bootstrap)."""
    from paper_1909_13560_b200 import workloads as W
    s = dict(W.ex2(3, 16, npts=801), bootstrap=1, bootstrap_substeps=2)
    a = oracle_mod.Oracle(s, nthreads=os.cpu_count())
    a.solve()
    b = oracle_mod.Oracle(dict(s, sde="ou", sde_params=[0.0] * 6 + [1.0] * 3), nthreads=os.cpu_count())
    b.solve()
    assert np.array_equal(a.layers(), b.layers())


def test_fsde_gbm_linear_payoff_exact(oracle_mod):
    """GBM dX = mu X dt + sigma X dW, f = 0, g = x, K = 1: E[X_{n+1} | x] = x (1 + mu dt) for one
    Euler step, the spline reproduces linear data and the Gauss-Hermite rule integrates linear
    functions exactly, so y^n = x (1 + mu dt)^(N-n) and z^n = sigma x (1 + mu dt)^(N-n)
    (z = b grad u, Eq. 1; z^N = sigma x) at every point whose samples stay inside the box."""
    mu, sig, N = 0.35, 0.4, 4
    spec = _fsde_spec("gbm", [mu, 0, 0, sig, 0, 0, 0, 0, 0, 1.0], "poly", [0.0, 1.0, 0.0, 0.0], N=N, P=321,
                      box=(0.0, 16.0), T=0.2)
    o = oracle_mod.Oracle(spec, nthreads=2)
    o.solve()
    x = np.linspace(0.0, 16.0, 321)
    m = x <= 3.0                      # the clamped samples near x = 16 leak through the spline to ~x = 8
    fac = (1.0 + mu * spec["T"] / N) ** N
    assert np.max(np.abs(o.layer(0)[m] - x[m] * fac)) <= 1e-13 * 8
    assert np.max(np.abs(o.layer(1)[m] - sig * x[m] * fac)) <= 1e-13 * 8


def _gauss_compose(coef, alpha, beta, s):
    """Coefficients (ascending) of x -> E[p(alpha x + beta + s Z)], Z ~ N(0, 1), for the polynomial
    p with ascending coefficients coef; E[Z^m] = (m-1)!! for even m, 0 for odd m."""
    from numpy.polynomial import polynomial as Pn
    out = np.zeros(1)
    lin = np.array([beta, alpha])
    for k, ck in enumerate(coef):
        acc = np.zeros(1)
        for m in range(0, k + 1, 2):
            ez = float(np.prod(np.arange(m - 1, 0, -2))) if m else 1.0
            acc = Pn.polyadd(acc, math.comb(k, m) * s ** m * ez * Pn.polypow(lin, k - m))
        out = Pn.polyadd(out, ck * acc)
    return out


def test_fsde_ou_cubic_exact_discrete_solution(oracle_mod):
    """OU dX = kappa (theta - X) dt + sigma dW, f = 0, g = x^3 - x, K = 1: one Euler step maps
    x to alpha x + beta + sigma sqrt(dt) Z with alpha = 1 - kappa dt, beta = kappa theta dt, so the
    discrete solution stays a cubic, y^n(x) = E[y^{n+1}(alpha x + beta + sigma sqrt(dt) Z)] and
    z^n = E[z^{n+1}(...)] from z^N = sigma g'(x) (Eq. 20 with K = 1, f = 0) -- computed here by
    polynomial algebra.  The spline reproduces cubics, L = 4 Gauss-Hermite is exact to degree 7."""
    from numpy.polynomial import polynomial as Pn
    kap, th, sig, N, T = 0.7, 0.3, 0.5, 3, 0.15
    spec = _fsde_spec("ou", [kap, 0, 0, th, 0, 0, sig, 0, 0, 0.0], "poly", [0.0, -1.0, 0.0, 1.0], N=N, P=257, T=T, L=4)
    o = oracle_mod.Oracle(spec, nthreads=2)
    o.solve()
    dt = T / N
    y = np.array([0.0, -1.0, 0.0, 1.0])
    z = sig * Pn.polyder(y)
    for _ in range(N):
        y = _gauss_compose(y, 1 - kap * dt, kap * th * dt, sig * math.sqrt(dt))
        z = _gauss_compose(z, 1 - kap * dt, kap * th * dt, sig * math.sqrt(dt))
    x = np.linspace(-8.0, 8.0, 257)
    m = np.abs(x) <= 3.0
    assert np.max(np.abs(o.layer(0)[m] - Pn.polyval(x[m], y))) <= 1e-12 * 27
    assert np.max(np.abs(o.layer(1)[m] - Pn.polyval(x[m], z))) <= 1e-12 * 27


def test_fsde_gbm_black_scholes_in_price_space(oracle_mod):
    """Black-Scholes call (Ex. 3 parameters without dividend) solved in price space:
    X = S is a GBM with drift mu, f = -(r y + theta z), theta = (mu - r)/sigma (Eq. 29-30).
    Accuracy, not parity: y0 at S0 = K = 100 within 0.5 % of the closed form and z0 within 2 %
    (the Euler forward step is weak order 1; a wrong drift would be off by ~|mu - r| T S0 ~ 0.7)."""
    from scipy.stats import norm
    S0, Kst, r, mu, sig, T = 100.0, 100.0, 0.03, 0.05, 0.2, 0.33
    d1 = (math.log(S0 / Kst) + (r + 0.5 * sig ** 2) * T) / (sig * math.sqrt(T))
    ey = S0 * norm.cdf(d1) - Kst * math.exp(-r * T) * norm.cdf(d1 - sig * math.sqrt(T))
    ez = sig * S0 * norm.cdf(d1)
    spec = _fsde_spec("gbm", [mu, 0, 0, sig, 0, 0, 0, 0, 0, S0], "call_x", [0.0, Kst], driver="affine",
                      dp=[-r, -(mu - r) / sig, 0, 0, 0], K=3, N=32, P=1601, box=(0.0, 400.0), T=T, L=16)
    o = oracle_mod.Oracle(spec, nthreads=os.cpu_count())
    y0, z0 = o.solve()
    assert abs(y0 - ey) <= 5e-3 * ey and abs(z0[0] - ez) <= 2e-2 * ez, (y0, ey, z0, ez)


# --------------------------------------------------------------------------- FD-bicubic 2-D interpolation
# "bicubic interpolation for 2-dimensional cases ... first and mixed derivatives
# ... approximated using finite difference schemes of the fourth order of accuracy (central,
# forward and backward) ... a matrix vector multiplication ... for each point".

def test_fd_weights_are_the_fourth_order_stencils(oracle_mod):
    """The 5-point derivative weights (Fornberg's tables): central (1, -8, 0, 8, -1)/12, one-sided
    (-25, 48, -36, 16, -3)/12 and (-3, -10, 18, -6, 1)/12; derivatives exact on quartics (also at
    the ends) and 4th order on a quintic (error ratio ~16 per halving of h)."""
    assert np.allclose(oracle_mod.fd_weights([-2, -1, 0, 1, 2]) * 12, [1, -8, 0, 8, -1], atol=1e-13)
    assert np.allclose(oracle_mod.fd_weights([0, 1, 2, 3, 4]) * 12, [-25, 48, -36, 16, -3], atol=1e-12)
    assert np.allclose(oracle_mod.fd_weights([-1, 0, 1, 2, 3]) * 12, [-3, -10, 18, -6, 1], atol=1e-12)
    x = np.linspace(-1.0, 2.0, 13)
    assert np.max(np.abs(oracle_mod.fd_deriv(x ** 4 - 2 * x ** 3 + x, x[1] - x[0]) - (4 * x ** 3 - 6 * x ** 2 + 1))) <= 1e-12
    errs = []
    for n in (17, 33):
        x = np.linspace(0.0, 1.0, n)
        errs.append(np.max(np.abs(oracle_mod.fd_deriv(x ** 5, x[1] - x[0]) - 5 * x ** 4)))
    assert 12 < errs[0] / errs[1] < 40


def test_bicubic_reproduces_bicubic_polynomials(oracle_mod):
    """With f = x1^3 x2^2 + x1 x2 the 4th-order differences are exact (degree <= 4 per axis), so
    the 16-coefficient cells reproduce f at random points (SPEC examples: xy reproduced, corner
    value = sample), inside and outside the box (clamped)."""
    from paper_1909_13560_b200 import workloads as W
    spec = dict(W.heat_poly(2, 1, N=2, P=9, T=0.25, box=2.0, L=2), npts=[9, 13], xlo=[-2.0, -1.0],
                xhi=[2.0, 3.0], interp="fd_bicubic")
    spec["terminal_params"] = [0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 1.0, 0.0]       # x1^3 * x2^2
    o = oracle_mod.Oracle(spec, nthreads=1)
    rng = np.random.Generator(np.random.PCG64(1909135600))
    for _ in range(100):
        x = [rng.uniform(-2.5, 2.5), rng.uniform(-1.5, 3.5)]
        xc = np.clip(x, [-2.0, -1.0], [2.0, 3.0])
        v = o.eval_newest(x)
        assert abs(v[0] - xc[0] ** 3 * xc[1] ** 2) <= 1e-12 * 72
        assert abs(v[1] - 3 * xc[0] ** 2 * xc[1] ** 2) <= 1e-11 * 108      # z_1 = d/dx1 of g
        assert abs(v[2] - 2 * xc[0] ** 3 * xc[1]) <= 1e-11 * 48


def test_P6_heat_polynomial_exact_2d_bicubic(oracle_mod):
    """P6 with the FD-bicubic interpolation: g = x1^3 x2 is in the bicubic space and its FD
    derivatives are exact, so every K reproduces y = x1^3 x2 + 3 x1 x2 (T-t) away from the edge."""
    from paper_1909_13560_b200 import workloads as W
    spec = dict(W.heat_poly(2, 3, N=5, P=65, T=0.25, box=16.0, L=8), interp="fd_bicubic")
    o = oracle_mod.Oracle(spec, nthreads=os.cpu_count())
    o.solve()
    x = np.linspace(-16, 16, 65)
    X1, X2 = np.meshgrid(x, x, indexing="ij")
    m = (np.abs(X1) <= 5) & (np.abs(X2) <= 5)
    assert np.max(np.abs(o.layer(0)[m] - (X1 ** 3 * X2 + 0.75 * X1 * X2)[m])) <= 1e-12 * 625
    assert np.max(np.abs(o.layer(1)[m] - (3 * X1 ** 2 * X2 + 0.75 * X2)[m])) <= 1e-12 * 375


@pytest.mark.parametrize("row", [r for r in _rows("ex4", 16)], ids=lambda r: f"ex4_K{r[1]}_N{r[2]}")
def test_P10_printed_rows_2d_bicubic(oracle_mod, row):
    """Table 9 was computed with the FD-bicubic interpolation: the oracle's
    bicubic path reproduces the gated printed rows within 3 % (y and Euclidean z, reading R15)."""
    from paper_1909_13560_b200 import workloads as W
    spec = dict(W.ex4_2d(int(row[1]), int(row[2])), interp="fd_bicubic")
    o = oracle_mod.Oracle(spec, nthreads=os.cpu_count())
    y0, z0 = o.solve()
    _check_row(row, abs(y0), float(np.linalg.norm(np.asarray(z0) - 1.0)))
