"""Granularity-aware regulation search (§4.4, Algorithm 1, l.832-855).

The paper searches Matrix_P (temporal regulation: equal-count pointer lists,
Eq. 6/7) and the decomposition mask / list_B (spatial regulation, Eq. 5) by
greedy alternation, minimising the residue R of Eq. 8 computed from a
profiled lookup table.  On B200 the objective is MEASURED instead: R is the
median makespan of executor rounds under the candidate plan, which already
contains the real residue and the device pointer cost T_SW (Eq. 8's penalty
term is physically present rather than modelled).

Host-side planning only: every candidate plan is installed through the C ABI
(`gacer_set_regulation`) and timed on the executor; the hot path itself is
unchanged.  The search logic is pure Python over an `evaluate` callable so
that it is testable on the CPU against a brute-force oracle (SPEC.md
search module).

Readings: pointers are non-decreasing in [0, n_ops] (Q7);
spatial moves are binary batch splits of every decomposable op of one tenant
(SPEC's binary-chunk decision) accepted only if R strictly drops; a new
pointer starts at the midpoint of the model's largest segment.
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple

Pointers = Tuple[Tuple[int, ...], ...]          # per tenant: non-decreasing cuts
Decomp = Tuple[Tuple[int, int], ...]            # per tenant: (tenant, n_chunks), n_chunks 1 = none


def _key(ptrs: Pointers, dec: Decomp) -> Tuple:
    return (tuple(tuple(p) for p in ptrs), tuple(dec))


def coordinate_moves(ptrs: Pointers, n: int, j: int, n_ops: int, stride: int = 1) -> List[Pointers]:
    """All legal positions of pointer slot j of model n with every other entry
    fixed (§4.4 "coordinate descent ... takes the pointer number in Matrix_P
    as different coordinates"): positions in [previous cut, next cut]
    (non-decreasing, Q7), subsampled every `stride` ops; the incumbent is
    always included."""
    cur = list(ptrs[n])
    lo = cur[j - 1] if j > 0 else 0
    hi = cur[j + 1] if j + 1 < len(cur) else n_ops
    cand = set(range(lo, hi + 1, max(1, stride))) | {hi, cur[j]}
    out = []
    for v in sorted(cand):
        row = list(cur)
        row[j] = v
        out.append(tuple(tuple(r) if i != n else tuple(row) for i, r in enumerate(ptrs)))
    return out


def add_pointer(ptrs: Pointers, n_ops: Sequence[int]) -> Pointers:
    """Algorithm 1 "Add pointer in Matrix_P": one more slot per model (equal
    counts), placed at the midpoint of that model's largest segment."""
    out = []
    for cuts, n in zip(ptrs, n_ops):
        bounds = [0] + list(cuts) + [n]
        k = max(range(len(bounds) - 1), key=lambda i: (bounds[i + 1] - bounds[i], -i))
        mid = (bounds[k] + bounds[k + 1] + 1) // 2
        out.append(tuple(sorted(list(cuts) + [mid])))
    return tuple(out)


def equal_op_pointers(n_ops: Sequence[int], k: int) -> Pointers:
    return tuple(tuple(round(n * (j + 1) / (k + 1)) for j in range(k)) for n in n_ops)


@dataclass
class SearchConfig:
    rounds: int = 1                 # X: coordinate-descent rounds per pointer count
    max_pointers: int = 3
    stride: int = 1                 # pointer position subsampling
    spatial_chunks: Tuple[int, ...] = (2,)   # binary moves (then finer if listed)
    max_evals: int = 10_000


@dataclass
class SearchResult:
    pointers: Pointers
    decomposition: Decomp
    R: float
    evals: int
    history: List[Tuple[int, float]] = field(default_factory=list)
    records: Dict[int, float] = field(default_factory=dict)   # best R per pointer count (D)


class _Memo:
    def __init__(self, evaluate: Callable[[Pointers, Decomp], float], max_evals: int):
        self.f, self.cache, self.n, self.max = evaluate, {}, 0, max_evals
        self.history: List[Tuple[int, float]] = []

    def __call__(self, ptrs: Pointers, dec: Decomp) -> float:
        k = _key(ptrs, dec)
        if k not in self.cache:
            if self.n >= self.max:
                return math.inf
            self.cache[k] = float(self.f(ptrs, dec))
            self.n += 1
            self.history.append((self.n, self.cache[k]))
        return self.cache[k]


def granularity_aware_search(evaluate: Callable[[Pointers, Decomp], float], n_ops: Sequence[int],
                             cfg: Optional[SearchConfig] = None) -> SearchResult:
    """Algorithm 1: coordinate descent over Matrix_P with alternating spatial
    moves; escalate the pointer count while the best R keeps improving."""
    cfg = cfg or SearchConfig()
    T = len(n_ops)
    R = _Memo(evaluate, cfg.max_evals)
    by_n: Dict[int, Tuple[float, Pointers, Decomp]] = {}
    for n_ptr in range(0, cfg.max_pointers + 1):
        if n_ptr == 0:
            ptrs: Pointers = tuple(() for _ in range(T))
            dec: Decomp = tuple((t, 1) for t in range(T))
        else:
            _, ptrs, dec = by_n[n_ptr - 1]
            ptrs = add_pointer(ptrs, n_ops)          # "Add pointer in Matrix_P"
        cur = (R(ptrs, dec), ptrs, dec)
        for _ in range(cfg.rounds):
            # temporal: coordinate descent, one (model, slot) coordinate at a time
            for n in range(T):
                for j in range(n_ptr):
                    cands = coordinate_moves(cur[1], n, j, n_ops[n], cfg.stride)
                    r, _, c = min(((R(c, cur[2]), c[n][j], c) for c in cands), key=lambda z: (z[0], z[1]))
                    if r < cur[0]:
                        cur = (r, c, cur[2])
            # spatial: binary (then finer) batch split of one tenant's ops,
            # kept only when it strictly lowers R
            for n in range(T):
                for ch in cfg.spatial_chunks:
                    d2 = tuple((t, ch if t == n else c) for t, c in cur[2])
                    r = R(cur[1], d2)
                    if r < cur[0]:
                        cur = (r, cur[1], d2)
        by_n[n_ptr] = cur
        if n_ptr > 0 and cur[0] >= by_n[n_ptr - 1][0]:
            break                                    # stop rule: |P| is no better than |P| - 1
    best = min(by_n.values(), key=lambda z: z[0])
    return SearchResult(pointers=best[1], decomposition=best[2], R=best[0], evals=R.n,
                        history=R.history, records={k: v[0] for k, v in by_n.items()})


def all_pointer_matrices(n_ops: Sequence[int], k: int) -> List[Pointers]:
    """Every legal Matrix_P with k pointers per model (non-decreasing cuts)."""
    per = [list(itertools.combinations_with_replacement(range(n + 1), k)) for n in n_ops]
    return [tuple(tuple(c) for c in combo) for combo in itertools.product(*per)]


def brute_force_oracle(evaluate: Callable[[Pointers, Decomp], float], n_ops: Sequence[int], max_pointers: int,
                       chunk_options: Sequence[int] = (1,), guard: int = 200_000) -> Tuple[float, Pointers, Decomp]:
    """Exhaustive minimum of R over all Matrix_P with <= max_pointers pointers
    per model and all per-tenant chunk counts in chunk_options (tiny
    instances only)."""
    T = len(n_ops)
    decs = [tuple((t, c) for t, c in enumerate(cs)) for cs in itertools.product(chunk_options, repeat=T)]
    size = sum(math.prod(math.comb(n + k, k) for n in n_ops) for k in range(max_pointers + 1)) * len(decs)
    if size > guard:
        raise ValueError("InstanceTooLarge")
    spaces = [all_pointer_matrices(n_ops, k) for k in range(max_pointers + 1)]
    best = (math.inf, None, None)
    for space in spaces:
        for p in space:
            for d in decs:
                r = float(evaluate(p, d))
                if r < best[0]:
                    best = (r, p, d)
    return best


# ---------------------------------------------------------------- device glue
def measured_objective(G, sess, graphs, batches, torch, stream, flush=None, rounds: int = 5,
                       warmup: int = 2) -> Callable[[Pointers, Decomp], float]:
    """R = median executor makespan (ms) of the plan, CUDA events on `stream`
    (L2 flushed between rounds when `flush` is given)."""
    import numpy as np

    def plan_decomposition(dec: Decomp):
        out = []
        for t, ch in dec:
            if ch <= 1:
                continue
            g, B = graphs[t], batches[t]
            k = min(ch, B)
            sizes = [B // k + (1 if j < B % k else 0) for j in range(k)]
            for i, op in enumerate(g.ops):
                if op["kind"] in ("conv", "linear", "maxpool", "avgpool", "gap", "add", "relu", "relu6", "bn"):
                    out.append((t, i + 1, "batch", sizes))
        return out or None

    def evaluate(ptrs: Pointers, dec: Decomp) -> float:
        sess.set_regulation(plan_decomposition(dec), [list(p) for p in ptrs] if any(ptrs) else None)
        sess.set_mode("executor")
        for _ in range(warmup):
            G.gacer_run_round_async(stream.cuda_stream)
        ts = []
        for _ in range(rounds):
            if flush is not None:
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            G.gacer_run_round_async(stream.cuda_stream)
            b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        return float(np.median(ts))

    evaluate.plan_decomposition = plan_decomposition
    return evaluate
