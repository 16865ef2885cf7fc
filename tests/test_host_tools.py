"""Host-side checks of the product path's generated code (no GPU): the digamma / lnGamma remainder
polynomials of the Dirichlet kernel (scripts/gen_digamma_u_poly.py -> csrc/digamma_u_poly.cuh) are in
sync with their generator, and their float32 evaluation meets the accuracy DESIGN R14 states.  The
reference values come from scipy, not from oracle/ (the product path and the oracle share nothing)."""
import os
import subprocess
import sys

import numpy as np
import pytest
from scipy.special import digamma, gammaln

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GEN = os.path.join(ROOT, "scripts", "gen_digamma_u_poly.py")
HDR = os.path.join(ROOT, "paper_1206_6468_b200", "csrc", "digamma_u_poly.cuh")


def _coeffs(name, text):
    """Monomial coefficients (t^0 first) of the scalar Horner function `name` in the header text."""
    import re
    line = next(l for l in text.splitlines() if f"float {name}(float t)" in l)
    vals = [float(v.rstrip("f")) for v in re.findall(r"[-+]?\d\.\d+e[-+]\d+f", line)]
    return np.array(vals[::-1], dtype=np.float32)   # innermost (highest degree) appears first


def _horner32(c, t):
    r = np.float32(c[-1]) * np.ones_like(t)
    for v in c[-2::-1]:
        r = (r * t + np.float32(v)).astype(np.float32)
    return r


def test_header_in_sync_with_generator():
    out = subprocess.run([sys.executable, GEN], capture_output=True, text=True, check=True).stdout
    assert out == open(HDR).read()


@pytest.mark.parametrize("lo,hi,tol", [(1, 6, 2.0e-7), (6, 1e3, 6e-7), (1e3, 1e6, 1.1e-6)])
def test_psi_float32_accuracy(lo, hi, tol):
    """psi(x) = ln x - u/2 - u^2 G(2u-1), u = 1/x, evaluated in float32 (the kernel's arithmetic)."""
    G = _coeffs("dig_G", open(HDR).read())
    x = np.geomspace(lo, hi, 200001).astype(np.float32)
    u = (np.float32(1) / x).astype(np.float32)
    t = (np.float32(2) * u - np.float32(1)).astype(np.float32)
    psi = (np.log(x).astype(np.float32) - (np.float32(0.5) * u + u * u * _horner32(G, t))).astype(np.float32)
    assert np.max(np.abs(psi.astype(np.float64) - digamma(x.astype(np.float64)))) <= tol


def test_lngamma_remainder_and_gtilde():
    """lnGamma(x) = (x - 1/2) ln x - x + ln(2 pi)/2 + u H(2u-1) (degree-3 H: ~3e-7, enough for the bound
    term, whose tolerance is ~1e-3 per element); g~(x) = lnG(x) - (x-1) psi(x) + x is then
    ln(x)/2 + ln(2 pi)/2 + 1/2 + u (H - 1/2) + (u - u^2) G (the identity the Dirichlet kernel uses)."""
    txt = open(HDR).read()
    G, H = _coeffs("dig_G", txt).astype(np.float64), _coeffs("lng_H", txt).astype(np.float64)
    x = np.geomspace(1, 1e6, 100001)
    u = 1 / x
    t = 2 * u - 1
    Gv = np.polynomial.polynomial.polyval(t, G)
    Hv = np.polynomial.polynomial.polyval(t, H)
    lng = (x - 0.5) * np.log(x) - x + 0.5 * np.log(2 * np.pi) + u * Hv
    assert np.max(np.abs(lng - gammaln(x)) / np.maximum(1, np.abs(gammaln(x)))) < 5e-7
    gt = 0.5 * np.log(x) + 0.5 * np.log(2 * np.pi) + 0.5 + u * (Hv - 0.5) + (u - u * u) * Gv
    ref = gammaln(x) - (x - 1) * digamma(x) + x
    assert np.max(np.abs(gt - ref)) < 1e-6


def _table(name, text):
    import re
    line = next(l for l in text.splitlines() if l.startswith(f"#define {name} "))
    return np.array([float(v.rstrip("f")) for v in re.findall(r"[-+]?\d\.\d+e[-+]\d+f", line)], dtype=np.float32)


def test_psi_u_form_float32_accuracy():
    """The round-2 Dirichlet kernel's form: psi(x) = E ln 2 + ln m - r, r = u/2 + u^2 G(u) with G as a
    polynomial in u (DIG_GNU_COEF = -G, highest degree first), evaluated in float32."""
    txt = open(HDR).read()
    Gn = _table("DIG_GNU_COEF", txt)
    x = np.concatenate([np.linspace(1, 20, 100001), np.geomspace(20, 1e6, 100001)]).astype(np.float32)
    u = (np.float32(1) / x).astype(np.float32)
    r = np.float32(Gn[0]) * np.ones_like(u)
    for c in Gn[1:]:
        r = (r * u + np.float32(c)).astype(np.float32)
    w = (u * r + np.float32(-0.5)).astype(np.float32)          # w' = u (-G) - 1/2
    rn = (u * w).astype(np.float32)                             # -r
    m, e = np.frexp(x.astype(np.float64))                       # x = m 2^e, m in [0.5, 1)
    lnm = np.log((2 * m).astype(np.float32)).astype(np.float32)
    psi = (e - 1) * np.log(2.0) + lnm.astype(np.float64) + rn.astype(np.float64)
    assert np.max(np.abs(psi - digamma(x.astype(np.float64)))) <= 4e-7
