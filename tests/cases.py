"""Seeded random case generators shared by the parity tests.

They draw the same kinds of cases as the reference's property tests
(tests/oracle.hpp:109-173 in /root/reference/proj: uniform T_w mantissas,
random exponents, random sparse CSR rows, gammas with a chosen binade) with
Python's own PRNG (the reference's std::uniform_int_distribution stream is
libstdc++-specific and not needed: parity is GPU vs oracle on the SAME inputs).
"""
import random
from fractions import Fraction

from oracle import pyref as P


class Rng:
    def __init__(self, seed: int):
        self.r = random.Random(seed)

    def uniform(self, lo: int, hi: int) -> int:
        return self.r.randint(lo, hi)

    def in_width(self, w: int) -> int:
        return self.r.randrange(-(1 << (w - 1)), 1 << (w - 1))

    def random_vec(self, n, q, e_lo=-8, e_hi=8, normalized=True) -> P.Block:
        b = P.Block([self.in_width(q) for _ in range(n)], q, self.uniform(e_lo, e_hi))
        return P.normalize(b) if normalized else b

    def random_csr(self, rows, cols, max_nnz, q, e_lo=-8, e_hi=8) -> P.Csr:
        rowptr, col, m = [0], [], []
        for _ in range(rows):
            nnz = self.uniform(0, min(max_nnz, cols))
            picks = sorted(self.r.sample(range(cols), nnz))
            for c in picks:
                col.append(c)
                m.append(self.in_width(q))
            rowptr.append(len(col))
        return P.Csr(rows, cols, rowptr, col, m, q, self.uniform(e_lo, e_hi))

    def gamma_with_binade(self, window: int, q: int = 16) -> P.Block:
        lo = 1 << (q - 2)
        return P.Block.scalar(lo + self.r.randrange(lo), q, window - q)

    def scalar(self, w: int, q: int, e_lo=-4, e_hi=4) -> P.Block:
        return P.Block.scalar(self.in_width(w), q, self.uniform(e_lo, e_hi))


def values(b: P.Block):
    return b.values()


def rational_axpby(a: P.Block, x, b: P.Block, y):
    av, bv = a.values()[0], b.values()[0]
    return [av * xi + bv * yi for xi, yi in zip(x, y)]


def rational_spmv(A: P.Csr, x):
    ea = Fraction(2) ** A.e
    out = []
    for i in range(A.rows):
        s = Fraction(0)
        for k in range(A.rowptr[i], A.rowptr[i + 1]):
            s += Fraction(A.m[k]) * ea * x[A.col[k]]
        out.append(s)
    return out
