"""Hopscotch series (Def. 1) by plain enumeration — test oracle only.

H(a, b): all strictly increasing integer sequences from a to b, one per subset
of the interior integers (Def. 1 read as "all subsets of the interior",
DESIGN.md C17).  |H(a, b)| = 2^(b-a-1) (Prop. 1).
"""
from itertools import combinations


def hopscotch_series(a, b):
    """List of tuples, longest first then lexicographic, as in Ex. 1's listing."""
    if a >= b:
        return []  # H(a0, a0) is empty
    interior = list(range(a + 1, b))
    out = []
    for k in range(len(interior), -1, -1):
        for sub in combinations(interior, k):
            out.append((a,) + sub + (b,))
    return out


def hopscotch_count(a, b):
    return len(hopscotch_series(a, b))
