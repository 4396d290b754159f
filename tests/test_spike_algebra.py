"""The algebra of the SPIKE slab spline (R29, host.cu spike_setup / kernels.cu
spike_correct), checked in numpy against a dense solve of the global not-a-knot moment system:
local solves with zero coupling at the slab interfaces, the 2(R-1) interface system built from the
closed-form spike vectors S^L_k = (rho^{k+1} - rho^{2n+1-k}) / (1 - rho^{2n+2}), and the
correction m = m_loc + m(r0 - 1) S^L + m(r1) S^R reproduce the global moments exactly."""
import numpy as np
import pytest

RHO = np.sqrt(3.0) - 2.0


def _solve(r, fa, fb, ma, mb):
    n = fb - fa - 1
    A = np.diag(4.0 * np.ones(n)) + np.diag(np.ones(n - 1), 1) + np.diag(np.ones(n - 1), -1)
    rr = r[fa:fb - 1].copy()            # rows fa+1 .. fb-1 (r[i] is the row i+1 right-hand side)
    rr[0] -= ma
    rr[-1] -= mb
    return np.linalg.solve(A, rr)


def _sl(n, k):
    return (RHO ** (k + 1) - RHO ** (2 * n + 1 - k)) / (1.0 - RHO ** (2 * n + 2))


@pytest.mark.parametrize("P,R", [(200, 2), (200, 4), (257, 5), (64, 3)])
def test_spike_reproduces_global_moments(P, R):
    rng = np.random.default_rng(1909135600)
    F = rng.standard_normal(P)
    m1 = F[0] - 2 * F[1] + F[2]
    mP2 = F[P - 3] - 2 * F[P - 2] + F[P - 1]
    r = 6.0 * (F[:-2] - 2 * F[1:-1] + F[2:])
    mg = _solve(r, 1, P - 2, m1, mP2)                        # rows 2 .. P-3
    bounds = [p * P // R for p in range(R + 1)]              # host.cu rank_rows
    fa = [1 if p == 0 else bounds[p] - 1 for p in range(R)]
    fb = [P - 2 if p == R - 1 else bounds[p + 1] for p in range(R)]
    loc = [_solve(r, fa[p], fb[p], m1 if p == 0 else 0.0, mP2 if p == R - 1 else 0.0) for p in range(R)]
    n = [fb[p] - fa[p] - 1 for p in range(R)]
    sA = [_sl(n[p], 0) for p in range(R)]
    sB = [_sl(n[p], n[p] - 1) for p in range(R)]
    M = 2 * (R - 1)
    A = np.zeros((M, M))
    rhs = np.zeros(M)
    for i in range(R - 1):                                   # host.cu spike_setup
        A[2 * i, 2 * i] = 1.0
        A[2 * i, 2 * i + 1] = -sA[i]
        if i > 0:
            A[2 * i, 2 * (i - 1)] = -sB[i]
        rhs[2 * i] = loc[i][-1]
        A[2 * i + 1, 2 * i + 1] = 1.0
        A[2 * i + 1, 2 * i] = -sA[i + 1]
        if i + 1 < R - 1:
            A[2 * i + 1, 2 * (i + 1) + 1] = -sB[i + 1]
        rhs[2 * i + 1] = loc[i + 1][0]
    X = np.linalg.solve(A, rhs)
    for p in range(R):
        xl = X[2 * (p - 1)] if p > 0 else 0.0
        xr = X[2 * p + 1] if p < R - 1 else 0.0
        k = np.arange(n[p])
        m = loc[p] + xl * _sl(n[p], k) + xr * _sl(n[p], n[p] - 1 - k)
        rows = np.arange(fa[p] + 1, fb[p])
        assert np.max(np.abs(m - mg[rows - 2])) <= 1e-13 * max(1.0, np.max(np.abs(mg)))


def test_recursive_filter_is_the_toeplitz_inverse():
    """R30: -rho (1 - rho z)^-1 (1 - rho z^-1)^-1 inverts (1, 4, 1) (impulse response
    -rho^{|d|+1} / (1 - rho^2)); truncating both filters 32 rows out changes the result by < 1e-18."""
    rng = np.random.default_rng(7)
    n = 400
    r = rng.standard_normal(n)
    A = np.diag(4.0 * np.ones(n)) + np.diag(np.ones(n - 1), 1) + np.diag(np.ones(n - 1), -1)
    u = np.zeros(n)
    acc = 0.0
    for k in range(n):
        acc = r[k] + RHO * acc
        u[k] = acc
    v = np.zeros(n)
    acc = 0.0
    for k in range(n - 1, -1, -1):
        acc = u[k] + RHO * acc
        v[k] = acc
    m = -RHO * v
    # interior rows agree with the infinite-line (here: zero-extended) inverse
    exact = np.linalg.solve(A, r)
    assert np.max(np.abs(m[40:-40] - exact[40:-40])) <= 1e-14 * np.max(np.abs(exact))
    assert abs(RHO) ** 32 < 5.1e-19
