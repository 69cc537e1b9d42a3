"""Pins for the weight function S(r) (Fig. 4c/d; reading G1).

* the constants rho = 2^(-1/d) against high-precision evaluation;
* the zero-moment condition  int S(r) r^(d-1) dr = 0 by quadrature;
* plateau values -1 / +1 / 0 and the inner ramp width dr = dR/cbrt(2);
* S_r, S_R against central finite differences of S.
"""
from decimal import Decimal, getcontext

import numpy as np
import pytest
from scipy import integrate


def _nearest_double(d: Decimal) -> float:
    f = float(d)
    cands = [np.nextafter(f, -np.inf), f, np.nextafter(f, np.inf)]
    return float(min(cands, key=lambda x: abs(Decimal(float(x)) - d)))


def test_rho_constants_are_correctly_rounded(ora):
    getcontext().prec = 60
    k = ora.constants()
    assert k["rho3"] == _nearest_double(Decimal(2) ** (Decimal(-1) / Decimal(3)))
    assert k["rho2"] == _nearest_double(Decimal(2) ** (Decimal(-1) / Decimal(2)))
    assert k["rho2_3d"] == _nearest_double(Decimal(2) ** (Decimal(-2) / Decimal(3)))
    assert k["rho2_2d"] == 0.5


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("R,dR", [(1.2, 2.0), (3.0, 1.0), (8.8, 2.0), (12.6, 2.0), (15.0, 2.52),
                                  (20.0, 1.0)])
def test_zero_moment(ora, dim, R, dR):
    """int_0^inf S(r) r^(d-1) dr = 0 (relative to the positive lobe)."""
    rho = 2 ** (-1 / dim)
    brk = sorted({max(0.0, x) for x in [rho * (R - dR / 2), rho * (R + dR / 2), R - dR / 2,
                                        R + dR / 2]})
    top = R + dR / 2
    f = lambda r: ora.weight(r, R, dR, dim)[0] * r ** (dim - 1)
    mom, _ = integrate.quad(f, 0.0, top, points=brk, limit=400, epsabs=1e-14, epsrel=1e-13)
    pos, _ = integrate.quad(lambda r: max(f(r), 0.0), 0.0, top, points=brk, limit=400,
                            epsabs=1e-14, epsrel=1e-13)
    assert abs(mom) / pos < 1e-10


@pytest.mark.parametrize("dim", [2, 3])
def test_plateaus_and_ramp_widths(ora, dim):
    R, dR = 12.0, 2.0
    rho = 2 ** (-1 / dim)
    w = lambda r: ora.weight(r, R, dR, dim)
    assert w(0.0)[0] == -1.0 and w(0.0)[1] == 0.0 and w(0.0)[2] == 0.0
    # inner ramp spans [rho (R - dR/2), rho (R + dR/2)] — width rho dR = dR / 2^(1/d)
    assert w(rho * (R - dR / 2) - 1e-9)[0] == -1.0
    assert w(rho * (R + dR / 2) + 1e-9)[0] == pytest.approx(1.0, abs=1e-12)
    assert -1.0 < w(rho * R)[0] < 1.0
    assert w(rho * R)[0] == pytest.approx(0.0, abs=1e-12)   # ramp midpoint
    # annulus plateau +1 (gain exactly 1, G1), outer ramp to 0 across [R - dR/2, R + dR/2]
    mid = 0.5 * (rho * (R + dR / 2) + (R - dR / 2))
    assert w(mid)[0] == 1.0 and w(mid)[1] == 0.0
    assert w(R)[0] == pytest.approx(0.5, abs=1e-12)
    assert w(R + dR / 2)[0] == 0.0 and w(R + dR / 2 + 3.0)[0] == 0.0


@pytest.mark.parametrize("dim", [2, 3])
def test_partials_match_finite_differences(ora, dim):
    rng = np.random.default_rng(1)
    h = 1e-6
    for _ in range(200):
        R = rng.uniform(3, 20)
        dR = rng.uniform(0.5, 3)
        r = rng.uniform(0, R + dR)
        S, S_r, S_R = ora.weight(r, R, dR, dim)
        fd_r = (ora.weight(r + h, R, dR, dim)[0] - ora.weight(r - h, R, dR, dim)[0]) / (2 * h)
        fd_R = (ora.weight(r, R + h, dR, dim)[0] - ora.weight(r, R - h, dR, dim)[0]) / (2 * h)
        assert abs(S_r - fd_r) < 1e-5 * (1 + abs(S_r))
        assert abs(S_R - fd_R) < 1e-5 * (1 + abs(S_R))
