"""Brute-force checks of §3.3's results (oracle; test infrastructure only).

A reduce tree for one block (proof of Theorem 1): N initial copies are combined
by operations O_0..O_{h-1}, O_i of fan-in f_i >= 2, into one.  These are exactly the
multifurcating rooted trees with N labelled leaves (every internal node >= 2 children);
there are 1, 4, 26, 236, 2752 of them for N = 2..6 (OEIS A000311, Schröder's 4th problem).

For each tree we check, exactly:
  Eq. 12  N − 1 = Σ (f_i − 1)
  Eq. 13/14  memory = Σ (f_i + 1)·S/N = (N − 1 + 2h)·S/N
  Theorem 1  the minimum over trees is (N + 1)·S/N, attained iff h = 1
  Theorem 2  for every w_t < N: no tree is both δ-optimal (h = 1) and ε-optimal
             (max f_i <= w_t); for w_t >= N the one-step tree (CPS) is both.
"""
from __future__ import annotations

from fractions import Fraction


def set_partitions(items):
    """All partitions of a list into non-empty blocks."""
    if not items:
        yield []
        return
    first, rest = items[0], items[1:]
    for part in set_partitions(rest):
        for i in range(len(part)):
            yield part[:i] + [[first] + part[i]] + part[i + 1:]
        yield [[first]] + part


def reduce_trees(leaves):
    """All multifurcating trees over `leaves`; each tree = list of fan-ins of its
    internal nodes (the operations O_i)."""
    if len(leaves) == 1:
        yield []
        return
    for part in set_partitions(list(leaves)):
        if len(part) < 2:
            continue
        # product over blocks of their subtrees
        def rec(i):
            if i == len(part):
                yield []
                return
            for sub in reduce_trees(part[i]):
                for tail in rec(i + 1):
                    yield sub + tail
        for inner in rec(0):
            yield [len(part)] + inner


def check_theorems(N: int, S=Fraction(1)):
    """Run every check on all reduce trees over N leaves; returns a summary dict."""
    trees = list(reduce_trees(list(range(N))))
    best = None
    for f in trees:
        h = len(f)
        assert N - 1 == sum(x - 1 for x in f), "Eq. 12"
        mem = sum((x + 1) * Fraction(S) / N for x in f)
        assert mem == (N - 1 + 2 * h) * Fraction(S) / N, "Eq. 14"
        best = mem if best is None else min(best, mem)
    lower = Fraction(N + 1, N) * S
    assert best == lower, "Theorem 1 bound"
    for f in trees:
        mem = sum((x + 1) * Fraction(S) / N for x in f)
        assert (mem == lower) == (len(f) == 1), "Theorem 1 iff h = 1"
    for w_t in range(1, N + 3):
        both = [f for f in trees if len(f) == 1 and max(f) <= w_t]
        if w_t < N:
            assert not both, "Theorem 2"
        else:
            assert both == [[N]], "CPS is both when N <= w_t"
    return {"N": N, "trees": len(trees), "min_memory": best}
