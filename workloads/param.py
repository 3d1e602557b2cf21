"""Second-stage coefficient-parameter homotopy.

Stage 1 (the polyhedral homotopy) solves a start system G with the supports of the target F
and generic coefficients c_G (generic coefficients reach the mixed volume).  Stage 2
deforms G into F:

    H(x, t) = (1 - t) G(x) + t F(x) = sum_a [ c_G x^a t^0 + (c_F - c_G) x^a t^1 ],

which is again a lifted system in the parameter t = e^tau (two terms per monomial, liftings 0
and 1), so the same evaluator, solver and tracker run it unchanged.  With complex generic c_G
the paths t in [0, 1) stay regular with probability one; paths whose endpoints leave (C*)^n or
go to infinity (the target's solution count is below the mixed volume) do not converge.

Workload preparation only (no arithmetic of the method): builds the term table.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from .systems import System

# stage-2 start parameter: t0 = e^-37 ~ 8.5e-17, so the stage-1 endpoints (G(x) = 0) are on the
# stage-2 paths to within ~1e-16 relative (the same margin as the polyhedral tau0, reading R22)
TAU0 = -37.0


def parameter_homotopy(start: System, target_coeffs) -> System:
    """H(x, t) = (1 - t) G + t F for G = `start` (its coefficients) and F = the same supports with
    `target_coeffs` (same term order as `start`).  Terms with c_F = c_G keep only the t^0 term."""
    cF = np.asarray(target_coeffs, np.complex128)
    if cF.shape != start.coeffs.shape:
        raise ValueError("target coefficients must follow the start system's term order")
    offs, exps, coeffs, lift = [0], [], [], []
    for k in range(start.n):
        for i in start.terms_of(k):
            exps.append(start.exps[i])
            coeffs.append(start.coeffs[i])
            lift.append(0.0)
            d = cF[i] - start.coeffs[i]
            if d != 0:
                exps.append(start.exps[i])
                coeffs.append(d)
                lift.append(1.0)
        offs.append(len(exps))
    return dataclasses.replace(start, name=start.name + "-param", offsets=np.asarray(offs, np.int64),
                               exps=np.asarray(exps, np.int32).reshape(len(exps), start.n),
                               coeffs=np.asarray(coeffs, np.complex128), lifting=np.asarray(lift, np.float64))
