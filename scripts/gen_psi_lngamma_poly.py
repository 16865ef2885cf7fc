"""Generate the per-unit-interval polynomial tables of psi(x) and lnGamma(x), x in [1, 6), used by the
Dirichlet kernel (paper_1206_6468_b200/csrc/dirichlet.cu).  Chebyshev least-squares fits in the variable
v = 2 (x - n - 1/2) in [-1, 1] on [n, n+1), n = 1..5, converted to monomials; the float32 Horner error is
printed (product-path code generation; scipy is only the reference for the fit)."""
import numpy as np
import numpy.polynomial.chebyshev as C
from scipy.special import digamma, gammaln

DEG = 10


def fit(fn):
    rows = []
    for n in range(1, 6):
        x = np.linspace(n, n + 1, 8001)
        v = 2 * (x - (n + 0.5))
        rows.append(C.cheb2poly(C.chebfit(v, fn(x), DEG)))
    return np.array(rows)


def horner32(coef, v):
    r = np.float32(coef[-1])
    for c in coef[-2::-1]:
        r = np.float32(r * v + np.float32(c))
    return r


if __name__ == "__main__":
    out = []
    for name, fn in (("kPsiPoly", digamma), ("kLgPoly", gammaln)):
        P = fit(fn)
        err = 0.0
        for n in range(1, 6):
            x = np.linspace(n, n + 1, 20001, endpoint=False)
            v = (2 * (x - (n + 0.5))).astype(np.float32)
            err = max(err, np.max(np.abs(horner32(P[n - 1], v).astype(np.float64) - fn(x))))
        out.append(f"// {name}: max |float32 Horner - exact| on [1,6) = {err:.2e}")
        out.append(f"__device__ __constant__ float {name}[5][{DEG + 1}] = {{")
        for row in P:
            out.append("    {" + ", ".join(f"{c:.9e}f" for c in row) + "},")
        out.append("};")
    print("\n".join(out))
