"""Benchmark systems shaped like the paper's workloads.

A system is the data of the polyhedral homotopy, Eq. (1):
    h_k(x,t) = sum_{a in S_k} c_{k,a} x^a t^{omega_k(a)},   k = 1..n
stored as per-equation term segments (a mixed system, ledger A5/A6):
    offsets[k] .. offsets[k+1]   terms of equation k
    exps[i]     integer exponent vector a (Laurent, may be negative)
    coeffs[i]   complex coefficient c_{k,a}
    lifting[i]  omega_k(a) >= 0 (integer-valued, ledger A4)

Coefficients are random points of the unit circle (generic coefficients,
ledger A29) unless ``coeffs="native"`` asks for the target system's own
coefficients (used to pin H(x,1) = F(x)).

Supports:
  * cyclic-n   (paper's cyclic-14 has 184 monomials)
  * chandra-n  (paper's chandra-24 has 324 distinct monomials)
  * katsura-n, noon-n, random dense Laurent: [ext] definitions, SURVEY §8(d).

RNG: numpy PCG64, master seed 211114317. Draw order: coefficients
(equation-major, term order), then liftings.
"""
from __future__ import annotations

import dataclasses
from typing import List, Sequence, Tuple

import numpy as np

MASTER_SEED = 211114317

Term = tuple  # (exponents, native coefficient[, lifting])


@dataclasses.dataclass
class System:
    name: str
    n: int                    # equations == variables (square system)
    offsets: np.ndarray       # int64 [n+1]
    exps: np.ndarray          # int32 [M, n]
    coeffs: np.ndarray        # complex128 [M]
    lifting: np.ndarray       # float64 [M]

    @property
    def M(self) -> int:
        return int(self.offsets[-1])

    def terms_of(self, k: int) -> range:
        return range(int(self.offsets[k]), int(self.offsets[k + 1]))

    def nnz(self) -> int:
        return int(np.count_nonzero(self.exps))

    def union_support_size(self) -> int:
        return len({tuple(int(v) for v in row) for row in self.exps})

    def with_coeffs(self, coeffs: np.ndarray) -> "System":
        return dataclasses.replace(self, coeffs=np.asarray(coeffs, np.complex128).copy())

    def with_lifting(self, lifting: np.ndarray) -> "System":
        return dataclasses.replace(self, lifting=np.asarray(lifting, np.float64).copy())


def _graded_lex_key(a: Sequence[int]):
    # graded lexicographic order: higher total degree first, then lex.
    return (-sum(a), tuple(-v for v in a))


def from_terms(name: str, n: int, equations: List[List[Term]], *, coeffs: str = "random",
               lift_max: int = 10, seed: int = MASTER_SEED) -> System:
    """Pack per-equation term lists into a System.

    equations[k] = [(exponent tuple, native coefficient[, lifting]), ...]; duplicate
    exponents in one equation are merged (their native coefficients added), mirroring
    SPEC S:52's "no duplicate monomial" rule.  If every term carries its own lifting
    value it is used, otherwise liftings are drawn ~ U{0..lift_max}.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    offs = [0]
    exps: List[Tuple[int, ...]] = []
    native: List[complex] = []
    given_lift: List[float] = []
    all_lifted = True
    for eq in equations:
        merged: dict = {}
        lifted: dict = {}
        for term in eq:
            a, c = term[0], term[1]
            a = tuple(int(v) for v in a)
            if len(a) != n:
                raise ValueError("exponent length mismatch")
            merged[a] = merged.get(a, 0) + c
            if len(term) > 2:
                lifted[a] = float(term[2])
            else:
                all_lifted = False
        keys = sorted(merged, key=_graded_lex_key)
        if not keys:
            raise ValueError("empty equation")
        exps.extend(keys)
        native.extend(merged[a] for a in keys)
        given_lift.extend(lifted.get(a, 0.0) for a in keys)
        offs.append(len(exps))
    M = len(exps)
    lifting = given_lift if all_lifted else None
    if coeffs == "native":
        c = np.asarray(native, np.complex128)
    elif coeffs == "random":
        c = np.exp(2j * np.pi * rng.random(M))
    else:
        raise ValueError(coeffs)
    if lifting is not None:
        lift = np.asarray(lifting, np.float64)
    else:
        lift = rng.integers(0, lift_max + 1, size=M).astype(np.float64)
    return System(name=name, n=n, offsets=np.asarray(offs, np.int64),
                  exps=np.asarray(exps, np.int32).reshape(M, n), coeffs=c, lifting=lift)


def cyclic_terms(n: int) -> List[List[Term]]:
    """cyclic-n: f_k = sum_i prod_{j<k} x_{(i+j) mod n}, k=1..n-1; f_n = x_1...x_n - 1."""
    eqs = []
    for k in range(1, n):
        eq = []
        for i in range(n):
            a = [0] * n
            for j in range(k):
                a[(i + j) % n] += 1
            eq.append((tuple(a), 1.0))
        eqs.append(eq)
    eqs.append([(tuple([1] * n), 1.0), (tuple([0] * n), -1.0)])
    return eqs


def katsura_terms(n: int) -> List[List[Term]]:
    """katsura-n [ext]: variables x_0..x_n (n+1 of them).

    x_0 + 2 sum_{i=1}^n x_i - 1 = 0, and for m = 0..n-1:
    sum_{l=-n}^{n} x_{|l|} x_{|m-l|} - x_m = 0   (indices > n dropped).
    """
    N = n + 1
    eqs = []
    lin = []
    for i in range(N):
        a = [0] * N
        a[i] = 1
        lin.append((tuple(a), 1.0 if i == 0 else 2.0))
    lin.append((tuple([0] * N), -1.0))
    eqs.append(lin)
    for m in range(n):
        eq = []
        for l in range(-n, n + 1):
            i, j = abs(l), abs(m - l)
            if i > n or j > n:
                continue
            a = [0] * N
            a[i] += 1
            a[j] += 1
            eq.append((tuple(a), 1.0))
        a = [0] * N
        a[m] = 1
        eq.append((tuple(a), -1.0))
        eqs.append(eq)
    return eqs


def noon_terms(n: int) -> List[List[Term]]:
    """noon-n [ext]: x_i * sum_{j != i} x_j^2 - 1.1 x_i + 1 = 0."""
    eqs = []
    for i in range(n):
        eq = []
        for j in range(n):
            if j == i:
                continue
            a = [0] * n
            a[i] += 1
            a[j] += 2
            eq.append((tuple(a), 1.0))
        a = [0] * n
        a[i] = 1
        eq.append((tuple(a), -1.1))
        eq.append((tuple([0] * n), 1.0))
        eqs.append(eq)
    return eqs


def chandra_terms(n: int, c: float = 0.51) -> List[List[Term]]:
    """chandra-n: 2n x_k - c x_k sum_{j=1}^{n-1} (k/(k+j)) x_j - 2n = 0."""
    eqs = []
    for k in range(1, n + 1):
        eq = []
        a = [0] * n
        a[k - 1] = 1
        eq.append((tuple(a), 2.0 * n))
        for j in range(1, n):
            a = [0] * n
            a[k - 1] += 1
            a[j - 1] += 1
            eq.append((tuple(a), -c * k / (k + j)))
        eq.append((tuple([0] * n), -2.0 * n))
        eqs.append(eq)
    return eqs


def cyclic(n: int, **kw) -> System:
    return from_terms(f"cyclic-{n}", n, cyclic_terms(n), **kw)


def katsura(n: int, **kw) -> System:
    return from_terms(f"katsura-{n}", n + 1, katsura_terms(n), **kw)


def noon(n: int, **kw) -> System:
    return from_terms(f"noon-{n}", n, noon_terms(n), **kw)


def chandra(n: int, c: float = 0.51, **kw) -> System:
    return from_terms(f"chandra-{n}", n, chandra_terms(n, c), **kw)


def random_dense(n: int = 20, terms_per_eq: int = 50, emax: int = 2, *, seed: int = MASTER_SEED,
                 lift_max: int = 10) -> System:
    """Random generic dense Laurent system (BJ.configs[4]): per equation `terms_per_eq`
    distinct exponent vectors with entries ~ U{-emax..emax}."""
    rng = np.random.Generator(np.random.PCG64(seed + 1_000_003))
    eqs = []
    for _ in range(n):
        seen = set()
        while len(seen) < terms_per_eq:
            seen.add(tuple(int(v) for v in rng.integers(-emax, emax + 1, size=n)))
        eqs.append([(a, 1.0) for a in sorted(seen)])
    return from_terms(f"random-dense-{n}x{terms_per_eq}", n, eqs, seed=seed, lift_max=lift_max)


def diagonal(d: Sequence[int], b: Sequence[complex], omega: Sequence[int]) -> System:
    """Diagonal system h_k = x_k^{d_k} - b_k t^{omega_k} with closed-form paths
    x_k(t) = (b_k t^{omega_k})^{1/d_k} (SURVEY §8(c) O3/O4 pins)."""
    n = len(d)
    eqs = []
    for k in range(n):
        a = [0] * n
        a[k] = int(d[k])
        eqs.append([(tuple(a), 1.0, 0.0), (tuple([0] * n), -complex(b[k]), float(omega[k]))])
    return from_terms("diagonal", n, eqs, coeffs="native")
