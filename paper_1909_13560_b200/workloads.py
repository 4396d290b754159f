"""Workload specifications: the paper's examples and BASELINE.json's five configs.

This module holds problem *parameters* only -- no arithmetic of the method.  A
spec is a plain dict understood by both the CUDA library binding
(``paper_1909_13560_b200.bsde``) and the CPU oracle binding (``oracle``); each
side translates it into its own config struct.  Grid sizes are left at 0 where
the paper's balance rule applies so that each side computes them itself.

Closed-form reference solutions at (t0, x=0) are given for accuracy reporting
(Eq. 23, 25, 31, 35, 37; R21) -- they are the exact solutions of the
continuous problem, not outputs of the scheme.
"""
from __future__ import annotations

import math

# --- Black-Scholes parameters of Ex. 3 ---------------------------
BS = dict(S0=100.0, K=100.0, r=0.03, mu=0.05, delta=0.04, sigma=0.2, T=0.33)


def _base(d, T, N, K, L, box, **kw):
    spec = dict(d=d, t0=0.0, T=float(T), N=int(N), Ky=int(K), Kz=int(K), L=int(L),
                npts=[0] * d, xlo=[-box] * d, xhi=[box] * d, r=4,
                picard_max=30, picard_tol=0.0, bootstrap=0, bootstrap_substeps=1, smoothing=0)
    spec.update(kw)
    return spec


def ex1(K, N, L=32, npts=None):
    """Example 1 (Eq. 22), T=1, [-16,16], L=32, p=30."""
    s = _base(1, 1.0, N, K, L, 16.0, driver="ex1", terminal="logistic", name=f"ex1_K{K}_N{N}")
    if npts:
        s["npts"] = [int(npts)]
    return s


def ex2(K, N, L=32, npts=None):
    """Example 2 (Eq. 24), T=1, [-16,16], L=32."""
    s = _base(1, 1.0, N, K, L, 16.0, driver="ex2", terminal="ex2", name=f"ex2_K{K}_N{N}")
    if npts:
        s["npts"] = [int(npts)]
    return s


def _bs_driver(p):
    theta = (p["mu"] - p["r"] + p["delta"]) / p["sigma"]
    return [-p["r"], -theta, 0.0, 0.0, 0.0]


def black_scholes(K, N, L=32, npts=None, smoothing=1, T=None):
    """Example 3 (Eq. 30) in W-space (reading R20): f = -(r y + theta z)."""
    p = dict(BS)
    if T is not None:
        p["T"] = T
    s = _base(1, p["T"], N, K, L, 16.0, driver="affine", driver_params=_bs_driver(p),
              terminal="call_w", terminal_params=[p["S0"], p["K"], p["mu"], p["sigma"]],
              smoothing=smoothing, name=f"bs_K{K}_N{N}")
    if npts:
        s["npts"] = [int(npts)]
    return s


def diff_rates(K, N=256, P=65536, L=16, R=0.06, smoothing=1):
    """BASELINE cfg 2: call under different borrowing/lending rates (reading R21).
    f = -(r y + theta z) + (R - r) max(z/sigma - y, 0), theta = (mu - r + delta)/sigma."""
    p = dict(BS)
    theta = (p["mu"] - p["r"] + p["delta"]) / p["sigma"]
    dp = [p["r"], R, theta, 0.0, 0.0, 1.0 / p["sigma"], 0.0, 0.0]
    return _base(1, p["T"], N, K, L, 16.0, npts=[int(P)], driver="diff_rates", driver_params=dp,
                 terminal="call_w", terminal_params=[p["S0"], p["K"], p["mu"], p["sigma"]],
                 smoothing=smoothing, name=f"diffrates_K{K}_N{N}_P{P}")


def cfg1():
    """BASELINE cfg 1: 1-D Black-Scholes, K=2, N=32, P=256, L=8."""
    s = black_scholes(2, 32, L=8, npts=256)
    s["name"] = "cfg1_bs_K2_N32_P256_L8"
    return s


def cfg2(K=6):
    s = diff_rates(K)
    s["name"] = f"cfg2_diffrates_K{K}_N256_P65536_L16"
    return s


def ex4_2d(K, N, L=8, npts=None):
    """Example 4 (Eq. 34): f = y - (z1 + z2)/2, g = sin(w1 + w2 + T), [-8,8]^2, L=8."""
    s = _base(2, 1.0, N, K, L, 8.0, driver="affine", driver_params=[1.0, -0.5, -0.5, 0.0, 0.0],
              terminal="sin_sum", name=f"ex4_K{K}_N{N}")
    if npts:
        s["npts"] = [int(npts)] * 2
    return s


EXCHANGE = dict(S0=(100.0, 100.0), sigma=(0.25, 0.3), rho=0.0, r=0.05, mu=(0.1, 0.1), T=1.0)


def exchange_2d(K, N, L=8, npts=None, smoothing=1, T=None):
    """Example 5 (Eq. 36) in W-space, T=1 (reading R12): f = -(r y + z A^{-1} (mu - r)^T)."""
    p = dict(EXCHANGE)
    if T is not None:
        p["T"] = T
    s1, s2 = p["sigma"]
    rho = p["rho"]
    a11, a21, a22 = s1, rho * s2, s2 * math.sqrt(1.0 - rho * rho)
    m1, m2 = p["mu"][0] - p["r"], p["mu"][1] - p["r"]
    # A^{-1} M^T for lower-triangular A
    v1 = m1 / a11
    v2 = (m2 - a21 * v1) / a22
    spec = _base(2, p["T"], N, K, L, 8.0, driver="affine", driver_params=[-p["r"], -v1, -v2, 0.0, 0.0],
                 terminal="exchange_w",
                 terminal_params=[p["S0"][0], p["S0"][1], p["mu"][0], p["mu"][1], s1, s2, rho],
                 smoothing=smoothing, name=f"exchange_K{K}_N{N}")
    if npts:
        spec["npts"] = [int(npts)] * 2
    return spec


def cfg4(P=4096):
    s = exchange_2d(4, 128, L=8, npts=P)
    s["name"] = f"cfg4_exchange_K4_N128_P{P}^2_L8"
    return s


BASKET = dict(S0=(100.0, 100.0, 100.0), sigma=(0.2, 0.25, 0.3), mu=0.05, r=0.01, R=0.06, K=100.0, T=0.5)


def basket_3d(K=3, N=64, L=8, P=512, smoothing=1):
    """BASELINE cfg 5: 3-D geometric basket call, differential rates (reading R21)."""
    p = dict(BASKET)
    th = [(p["mu"] - p["r"]) / sg for sg in p["sigma"]]
    pi = [1.0 / sg for sg in p["sigma"]]
    spec = _base(3, p["T"], N, K, L, 8.0, npts=[int(P)] * 3, driver="diff_rates",
                 driver_params=[p["r"], p["R"]] + th + pi,
                 terminal="geo_basket_w",
                 terminal_params=list(p["S0"]) + [p["K"], p["mu"]] + list(p["sigma"]),
                 smoothing=smoothing, name=f"basket3d_K{K}_N{N}_P{P}^3")
    return spec


def ex1_3d(K=3, N=64, L=8, P=512):
    """3-D smooth control for cfg 5: u = logistic((w1+w2+w3)/sqrt(3) + t), Ex. 1 driver."""
    return _base(3, 1.0, N, K, L, 8.0, npts=[int(P)] * 3, driver="ex1", terminal="logistic",
                 name=f"ex1_3d_K{K}_N{N}_P{P}^3")


def heat_poly(d, K, N, P, T=0.25, box=16.0, L=16):
    """Exactness pin P6: f = 0, g = x^3 (d=1) or x1^3 x2 (d=2)."""
    tp = [0.0, 0.0, 0.0, 1.0] + ([0.0, 1.0, 0.0, 0.0] if d >= 2 else []) + ([1.0, 0, 0, 0] if d >= 3 else [])
    return _base(d, T, N, K, L, box, npts=[int(P)] * d, driver="zero", terminal="poly", terminal_params=tp,
                 name=f"heatpoly{d}d_K{K}")


def constant(d, Ky, Kz, N, P, c=2.5, L=8, box=8.0, rate=None):
    """Invariant P8 (f = 0, g = c) or P7 (f = -r y, g = c)."""
    s = _base(d, 1.0, N, max(Ky, Kz), L, box, npts=[int(P)] * d, terminal="const", terminal_params=[c],
              driver="zero" if rate is None else "affine",
              driver_params=[] if rate is None else [-rate, 0.0, 0.0, 0.0, 0.0], name="const")
    s["Ky"], s["Kz"] = int(Ky), int(Kz)
    return s


# ------------------------------------------------------------------ closed forms
def _ncdf(x):
    return 0.5 * math.erfc(-x / math.sqrt(2.0))


def bs_price(S, K, r, q, sig, tau):
    st = sig * math.sqrt(tau)
    d1 = (math.log(S / K) + (r - q + 0.5 * sig * sig) * tau) / st
    d2 = d1 - st
    return S * math.exp(-q * tau) * _ncdf(d1) - K * math.exp(-r * tau) * _ncdf(d2), S * math.exp(-q * tau) * _ncdf(d1)


def reference_solution(spec):
    """(y0, z0) of the continuous problem at t0 = 0, W = 0, or None."""
    d = spec["d"]
    if spec["terminal"] == "logistic" and spec["driver"] == "ex1":
        return 0.5, [0.25 / math.sqrt(d)] * d
    if spec["terminal"] == "ex2":
        return math.log(3.0), [1.0 / 3.0]
    if spec["terminal"] == "call_w":
        S0, K, mu, sig = spec["terminal_params"][:4]
        T = spec["T"]
        if spec["driver"] == "affine":
            r, th = -spec["driver_params"][0], -spec["driver_params"][1]
            rate = r
        else:
            r, rate, th = spec["driver_params"][0], spec["driver_params"][1], spec["driver_params"][2]
        q = th * sig - mu + r
        V, SdV = bs_price(S0, K, rate, q, sig, T)
        return V, [sig * SdV]
    if spec["terminal"] == "sin_sum":
        return 0.0, [1.0] * d  # sin(0), cos(0): Eq. 35 at t=0, W=0
    if spec["terminal"] == "exchange_w":
        S1, S2, _, _, s1, s2, rho = spec["terminal_params"][:7]
        T = spec["T"]
        st = math.sqrt(s1 * s1 + s2 * s2 - 2 * rho * s1 * s2)
        d1 = (math.log(S1 / S2) + 0.5 * st * st * T) / (st * math.sqrt(T))
        d2 = d1 - st * math.sqrt(T)
        n1, n2 = _ncdf(d1), _ncdf(d2)
        a21, a22 = rho * s2, s2 * math.sqrt(1 - rho * rho)
        return S1 * n1 - S2 * n2, [s1 * S1 * n1 - a21 * S2 * n2, -a22 * S2 * n2]
    if spec["terminal"] == "geo_basket_w":
        p = spec["terminal_params"]
        S0, K, sig = p[:d], p[3], p[5:5 + d]
        R = spec["driver_params"][1]
        T = spec["T"]
        G = math.exp(sum(math.log(s) for s in S0) / d)
        ss = sum(s * s for s in sig)
        sg = math.sqrt(ss) / d
        qg = ss / (2 * d) - 0.5 * sg * sg
        V, GdV = bs_price(G, K, R, qg, sg, T)
        return V, [GdV * s / d for s in sig]
    return None
