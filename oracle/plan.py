"""The paper's temporal-regulation semantics -- TEST INFRASTRUCTURE ONLY.

Eq. 7 (§4.3 l.742-753): M_1 = [O_{1,1..12}] + P_1:(2,8) = Seg(M_1);
"each number in P represents the position at which the pointer is inserted"
and "each P has the same number of pointers".  Eq. 6 (l.723-739): "the same
index segments from different models are divided into the same cluster which
can be deployed simultaneously".  Reading SURVEY §8(c) Q7: cuts are
non-decreasing with 0 <= p <= n_ops; cut p is the boundary after operator p;
0 / repeated cuts give empty segments (Eq. 6 shows M_2's first segment as
[None], i.e. P_2 = (0, 4)).
"""
from __future__ import annotations

from typing import List, Sequence


def segments(n_ops: int, cuts: Sequence[int]) -> List[List[int]]:
    """Eq. 7: the 1-based operator indices of each segment, in order."""
    bounds = [0] + list(cuts) + [n_ops]
    for a, b in zip(bounds, bounds[1:]):
        if not (0 <= a <= b <= n_ops):
            raise ValueError("cuts must be non-decreasing within [0, n_ops]")
    return [list(range(a + 1, b + 1)) for a, b in zip(bounds, bounds[1:])]


def clusters(n_ops: Sequence[int], matrix_p: Sequence[Sequence[int]]):
    """Eq. 6: cluster k = [segment k of model 1, ..., segment k of model n].
    Returns a list over clusters of lists over models of 1-based op indices."""
    if len({len(p) for p in matrix_p}) > 1:
        raise ValueError("each P has the same number of pointers (l.753)")
    segs = [segments(n, p) for n, p in zip(n_ops, matrix_p)]
    n_clusters = len(matrix_p[0]) + 1 if matrix_p else 1
    return [[s[k] for s in segs] for k in range(n_clusters)]


def op_cluster(n_ops: int, cuts: Sequence[int]) -> List[int]:
    """Cluster index of every operator (1-based op i -> out[i-1])."""
    out = []
    for k, seg in enumerate(segments(n_ops, cuts)):
        out.extend([k] * len(seg))
    return out


def format_clusters(n_ops, matrix_p) -> str:
    """Render Eq. 6's listing, e.g. "[O_{1,1},O_{1,2}], [None]"."""
    lines = []
    for cl in clusters(n_ops, matrix_p):
        parts = []
        for m, seg in enumerate(cl, start=1):
            parts.append("[None]" if not seg else
                         "[" + ",".join(f"O_{{{m},{i}}}" for i in seg) + "]")
        lines.append(", ".join(parts))
    return "\n".join(lines)
