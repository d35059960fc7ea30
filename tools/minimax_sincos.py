"""Coefficients of the sin(x)/x and cos(x) polynomials in z = x^2 used by
common.cuh (sinc_cos_series): near-minimax Chebyshev fits (mpmath chebyfit,
50 digits) on [0, (pi/4)^2] (narrow: degrees 6 / 7) and [0, (pi/2)^2] (wide:
8 / 8), rounded to double.  Prints the fit error and the float64 Horner error
on a grid, then the coefficients (highest degree first).

    python tools/minimax_sincos.py
"""
import mpmath as mp
import numpy as np

mp.mp.dps = 50
ZN, ZW = (mp.pi / 4) ** 2, (mp.pi / 2) ** 2


def sinc(z):
    return mp.sin(mp.sqrt(z)) / mp.sqrt(z) if z != 0 else mp.mpf(1)


def cosf(z):
    return mp.cos(mp.sqrt(z))


for name, f, Z, d in (("sinc narrow", sinc, ZN, 6), ("cos narrow", cosf, ZN, 7),
                      ("sinc wide", sinc, ZW, 8), ("cos wide", cosf, ZW, 8)):
    poly, err = mp.chebyfit(f, [0, Z], d + 1, error=True)
    c = [float(x) for x in poly]
    worst = 0.0
    for z in np.linspace(0, float(Z), 3001):
        v = c[0]
        for ck in c[1:]:
            v = v * z + ck
        worst = max(worst, abs(float(v - f(mp.mpf(z)))))
    print(f"{name}: degree {d}, fit error {mp.nstr(err, 2)}, float64 Horner error {worst:.2e}")
    print("   ", ", ".join(repr(x) for x in c))
