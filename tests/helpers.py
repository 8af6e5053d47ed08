"""Test helpers: golden-fixture loading and exact-arithmetic brute force.

Nothing here is imported by the product path or by oracle/. The brute force is
an independent formulation (dense, exact rational fma) used to pin the oracle.
"""
from __future__ import annotations

import json
import os
from fractions import Fraction

import numpy as np

from synth import Ell

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name: str) -> list[dict]:
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)["cases"]


def ell_from_entries(spec: dict, w: int | None = None) -> Ell:
    n = spec["n"]
    rows: list[list[tuple[int, float]]] = [[] for _ in range(n)]
    for i, j, v in spec["entries"]:
        rows[i].append((j, float(v)))
    mx = max([len(r) for r in rows] + [1])
    if w is None:
        w = mx + (mx & 1)
    e = Ell.empty(n, w)
    for i, r in enumerate(rows):
        r.sort()
        for q, (j, v) in enumerate(r):
            e.col[i, q] = j
            e.val[i, q] = v
        e.nnz[i] = len(r)
    return e


def entries_of(e: Ell) -> list[tuple[int, int, float]]:
    out = []
    for i in range(e.n):
        for q in range(int(e.nnz[i])):
            out.append((i, int(e.col[i, q]), float(e.val[i, q])))
    return out


def same_bits(a: Ell, b: Ell) -> bool:
    """Pattern and values identical bit for bit (padding ignored)."""
    if a.n != b.n or not np.array_equal(a.nnz, b.nnz):
        return False
    for i in range(a.n):
        k = int(a.nnz[i])
        if not np.array_equal(a.col[i, :k], b.col[i, :k]):
            return False
        if not np.array_equal(a.val[i, :k].view(np.uint64), b.val[i, :k].view(np.uint64)):
            return False
    return True


def fma_exact(a: float, b: float, c: float) -> float:
    """Correctly rounded fma via exact rationals (int/int true division is correctly rounded)."""
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def brute_multiply(A: np.ndarray, B: np.ndarray, Cold: np.ndarray, alpha: float, beta: float,
                   tau: float) -> np.ndarray:
    """Dense brute force of C <- drop(alpha*A*B + beta*C_old) with the same ascending-k fma
    chain as the definition (zero terms add exactly nothing), exact-rational fma. Returns the
    dense kept result (dropped entries are 0)."""
    n = A.shape[0]
    out = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            s = 0.0
            if alpha != 0.0:
                for k in range(n):
                    if A[i, k] != 0.0 and B[k, j] != 0.0:
                        s = fma_exact(A[i, k], B[k, j], s)
            t = float(Fraction(beta) * Fraction(Cold[i, j])) if (beta != 0.0 and Cold[i, j] != 0.0) else 0.0
            c = fma_exact(alpha, s, t)
            if abs(c) > tau:
                out[i, j] = c
    return out


def random_dense_sparse(rng: np.random.Generator, n: int, density: float, sym: bool = False,
                        dyadic: bool = False) -> np.ndarray:
    m = (rng.random((n, n)) < density)
    v = rng.standard_normal((n, n))
    if dyadic:
        v = np.round(v * 8) / 8
    d = np.where(m, v, 0.0)
    if sym:
        d = np.triu(d) + np.triu(d, 1).T
    return d
