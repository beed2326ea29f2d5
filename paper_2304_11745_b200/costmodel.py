"""Model-based regulation search: the paper's
own planner -- a profiled lookup table of W and T per operator, the residue
objective of Eq. 1-3 with the pointer penalty of Eq. 8, the largest-residue
spatial heuristic of §4.2 and Algorithm 1's coordinate descent -- on B200
numbers.  Host-side planning only (pure Python over a table); the plan it
returns is installed through ``gacer_set_regulation`` like any other.

* Lookup table (l.597-601, "we map the operator workload W(O^B) to the SM
  occupancy ... formulate a lookup table"): per (tenant, fused operator,
  batch b) the SM share W = min(1, items / #SMs) (or, w_mode
  "occupancy", the op's measured SM occupancy over its span) and the time T
  of the operator alone on the GPU, measured on the executor with op-level
  dependencies (``build_lut``: the device trace's span of each operator).
  NEXT-3 (l.269, l.817, "we can also extend this approach to other
  resources, such as GPU memory bandwidth"): W_bw = algorithmic bytes / T /
  the measured HBM bandwidth, a second resource pool.
* Deployment model (Eq. 1, l.613-624): every tenant issues its operators in
  order (one stream per tenant); an operator starts when its predecessor in
  the tenant has finished, its cluster is open (Eq. 6/7: clusters in order,
  a cluster opens when every operator of the previous one is done), and the
  running operators leave room for its W (Sum W <= S_GPU = 1; also
  Sum W_bw <= 1 when bandwidth-aware) -- otherwise "it is moved to the next
  cycle" (l.438-444).  Operators span as many cycles as their T.
* Objective (Eq. 2, 3, 8): R = Sum over cycles of (S_GPU - S_T) plus
  |P| * S_GPU * T_SW, with continuous time (a cycle = the interval between
  two events), T_SW the measured device pointer cost (D7).
* Spatial heuristic (l.688-695): take the cycle with the biggest residue
  (skipping the tail where one tenant runs alone), decompose the largest
  operator waiting for resources in it into a chunk that fits the residue
  and the rest (list_B), keep it when R drops.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

from .planner import add_pointer, coordinate_moves

NUM_SMS = 148


@dataclass
class OpCost:
    W: float          # SM occupancy share (S_GPU = 1)
    T: float          # us, alone on the GPU
    Wb: float = 0.0   # HBM bandwidth share (NEXT-3)


@dataclass
class TenantModel:
    """One tenant for the model: its fused operators in issue order."""
    batch: int
    n_orig: int
    last_member: List[int]          # per fused op: last original op (0-based), for pointer clusters
    first_member: List[int]         # per fused op: an original op (0-based) carrying its chunking
    decomposable: List[bool]        # batch chunks allowed (per-sample operators)
    cost: Dict[Tuple[int, int], OpCost] = field(default_factory=dict)   # (fused op, batch) -> cost

    def op_cost(self, f: int, b: int) -> OpCost:
        c = self.cost.get((f, b))
        if c is not None:
            return c
        # interpolate from the nearest profiled batch sizes (T linear in b
        # between profiled sizes, W rescaled by items ~ b)
        bs = sorted(bb for (ff, bb) in self.cost if ff == f)
        lo = max([x for x in bs if x <= b], default=bs[0])
        hi = min([x for x in bs if x >= b], default=bs[-1])
        a, z = self.cost[(f, lo)], self.cost[(f, hi)]
        if hi == lo:
            r = b / lo
            return OpCost(min(1.0, a.W * r), a.T * max(1.0, r), min(1.0, a.Wb * r))
        t = (b - lo) / (hi - lo)
        return OpCost(a.W + t * (z.W - a.W), a.T + t * (z.T - a.T), a.Wb + t * (z.Wb - a.Wb))


Plan = Tuple[Tuple[Tuple[int, ...], ...], Dict[Tuple[int, int], Tuple[int, ...]]]   # (Matrix_P, {(t, f): list_B})


@dataclass
class SimResult:
    R: float                      # Eq. 8 residue (GPU-us)
    makespan: float
    intervals: List[Tuple[float, float, float, List[Tuple[int, int, int]], int]]
    # (t0, t1, S_T, waiting-for-resources units (t, f, chunk), #tenants with work left)


def simulate(tenants: Sequence[TenantModel], ptrs, dec, t_sw: float, bandwidth: bool = False) -> SimResult:
    """Event-driven deployment of Eq. 1 under a plan; R of Eq. 8."""
    nt = len(tenants)
    units = []   # per tenant: list of (f, chunk_index, b, cost, cluster)
    n_clusters = (len(ptrs[0]) if ptrs and len(ptrs) else 0) + 1
    for t, tm in enumerate(tenants):
        cuts = ptrs[t] if ptrs and len(ptrs) else ()
        us = []
        for f in range(len(tm.last_member)):
            k = sum(1 for c in cuts if c <= tm.last_member[f])
            sizes = dec.get((t, f), (tm.batch,))
            for j, b in enumerate(sizes):
                us.append((f, j, b, tm.op_cost(f, b), k))
        units.append(us)
    nxt = [0] * nt                     # next unit per tenant
    busy_until = [0.0] * nt            # stream order: previous unit's end
    running: List[Tuple[float, float, float, int]] = []   # (end, W, Wb, cluster)
    left_in_cluster = [0] * n_clusters
    for us in units:
        for u in us:
            left_in_cluster[u[4]] += 1
    k_open = 0
    while k_open < n_clusters and left_in_cluster[k_open] == 0:
        k_open += 1
    now, R, intervals = 0.0, 0.0, []
    total = sum(len(us) for us in units)
    done = 0
    while done < total:
        # issue every eligible unit (tenants in order, greedy: l.438-444)
        S = sum(r[1] for r in running)
        Sb = sum(r[2] for r in running)
        waiting = []
        progressed = True
        while progressed:
            progressed = False
            for t in range(nt):
                if nxt[t] >= len(units[t]) or busy_until[t] > now + 1e-9:
                    continue
                f, j, b, c, k = units[t][nxt[t]]
                if k != k_open:
                    continue
                if S + c.W > 1.0 + 1e-9 or (bandwidth and Sb + c.Wb > 1.0 + 1e-9):
                    if S > 0:                                # moved to the next cycle
                        waiting.append((t, f, j))
                        continue
                running.append((now + c.T, c.W, c.Wb if bandwidth else 0.0, k, t))
                S += c.W
                Sb += c.Wb if bandwidth else 0.0
                busy_until[t] = now + c.T
                nxt[t] += 1
                progressed = True
        # advance to the next completion
        end = min(r[0] for r in running)
        active = sum(1 for t in range(nt) if nxt[t] < len(units[t]) or any(r[4] == t for r in running))
        S_T = min(1.0, sum(r[1] for r in running))
        intervals.append((now, end, S_T, waiting, active))
        R += (1.0 - S_T) * (end - now)
        now = end
        fin = [r for r in running if r[0] <= now + 1e-9]
        running = [r for r in running if r[0] > now + 1e-9]
        for r in fin:
            left_in_cluster[r[3]] -= 1
            done += 1
        while k_open < n_clusters and left_in_cluster[k_open] == 0:
            k_open += 1
    n_p = len(ptrs[0]) if ptrs and len(ptrs) else 0
    R += n_p * 1.0 * t_sw                                   # Eq. 8: |P_n| * S_GPU * T_SW
    return SimResult(R=R, makespan=now, intervals=intervals)


def largest_residue_split(tenants: Sequence[TenantModel], sim: SimResult, dec, tried=()) -> Optional[dict]:
    """§4.2 "Overall Spatial Regulation" (l.688-695): the cycle with the
    biggest residue R_{S_T} = S_GPU - S_T (Eq. 2), tail cycles with a single
    tenant left skipped; the largest operator waiting in it is decomposed
    into a chunk whose W fits the residue and the rest.  Returns the new
    decomposition, or None."""
    cands = []
    for (t0, t1, S, waiting, active) in sim.intervals:
        if active <= 1 or not waiting or t1 - t0 <= 0:
            continue
        cands.append((1.0 - S, t1 - t0, waiting))
    cands.sort(key=lambda z: (-z[0], -z[1]))
    for res, _, waiting in cands:
        # the largest waiting operator (W at its current chunk size)
        best = None
        for (t, f, j) in waiting:
            tm = tenants[t]
            if not tm.decomposable[f]:
                continue
            sizes = dec.get((t, f), (tm.batch,))
            b = sizes[j]
            if b < 2:
                continue
            w = tm.op_cost(f, b).W
            if best is None or w > best[0]:
                best = (w, t, f, j, sizes, b)
        if best is None:
            continue
        _, t, f, j, sizes, b = best
        tm = tenants[t]
        b1 = max((x for x in range(1, b) if tm.op_cost(f, x).W <= res + 1e-9), default=1)
        new_sizes = tuple(sizes[:j]) + (b1, b - b1) + tuple(sizes[j + 1:])
        if ((t, f), new_sizes) in tried:
            continue
        d2 = dict(dec)
        d2[(t, f)] = new_sizes
        return d2
    return None


@dataclass
class ModelSearchResult:
    pointers: Tuple[Tuple[int, ...], ...]
    decomposition: Dict[Tuple[int, int], Tuple[int, ...]]
    R: float
    makespan: float
    evals: int
    seconds: float
    records: Dict[int, float] = field(default_factory=dict)


def model_based_search(tenants: Sequence[TenantModel], t_sw: float, max_pointers: int = 3, rounds: int = 1,
                       stride: int = 1, spatial_steps: int = 8, bandwidth: bool = False,
                       max_evals: int = 100_000) -> ModelSearchResult:
    """Algorithm 1 (l.832-855) on the model objective: per pointer count,
    coordinate descent over Matrix_P alternated with largest-residue
    decompositions; add a pointer while the best R improves (stop rule)."""
    t_start = time.perf_counter()
    n_ops = [tm.n_orig for tm in tenants]
    cache: Dict = {}
    n_eval = [0]

    def R(ptrs, dec):
        key = (ptrs, tuple(sorted(dec.items())))
        if key not in cache:
            if n_eval[0] >= max_evals:
                return math.inf, None
            n_eval[0] += 1
            sim = simulate(tenants, ptrs, dec, t_sw, bandwidth)
            cache[key] = (sim.R, sim)
        return cache[key]

    by_n = {}
    for n_ptr in range(0, max_pointers + 1):
        if n_ptr == 0:
            ptrs = tuple(() for _ in tenants)
            dec: Dict = {}
        else:
            _, ptrs, dec, _ = by_n[n_ptr - 1]
            ptrs = add_pointer(ptrs, n_ops)
        r0, sim = R(ptrs, dec)
        if sim is None:                                    # evaluation budget spent
            break
        cur = (r0, ptrs, dec, sim)
        for _ in range(rounds):
            for n in range(len(tenants)):                  # temporal: coordinate descent
                for j in range(n_ptr):
                    for c in coordinate_moves(cur[1], n, j, n_ops[n], stride):
                        r, s = R(c, cur[2])
                        if r < cur[0]:
                            cur = (r, c, cur[2], s)
            tried = set()
            for _ in range(spatial_steps):                 # spatial: largest residue first
                if cur[3] is None:
                    break
                d2 = largest_residue_split(tenants, cur[3], cur[2], tried)
                if d2 is None:
                    break
                changed = [k for k in d2 if d2[k] != cur[2].get(k)]
                tried.update((k, d2[k]) for k in changed)
                r, s = R(cur[1], d2)
                if r < cur[0]:
                    cur = (r, cur[1], d2, s)
        by_n[n_ptr] = cur
        if n_ptr > 0 and cur[0] >= by_n[n_ptr - 1][0]:
            break                                          # |P| no better than |P| - 1
    best = min(by_n.values(), key=lambda z: z[0])
    return ModelSearchResult(pointers=best[1], decomposition=best[2], R=best[0], makespan=best[3].makespan,
                             evals=n_eval[0], seconds=time.perf_counter() - t_start,
                             records={k: v[0] for k, v in by_n.items()})


def plan_to_abi(tenants: Sequence[TenantModel], res: ModelSearchResult):
    """(decomposition list for gacer_set_regulation, pointer lists or None)."""
    dec = [(t, tenants[t].first_member[f] + 1, "batch", list(sizes))
           for (t, f), sizes in sorted(res.decomposition.items()) if len(sizes) > 1]
    ptrs = [list(p) for p in res.pointers] if any(res.pointers) else None
    return (dec or None), ptrs


# ---------------------------------------------------------------- device glue


def build_lut(G, Session, graphs, params, batches, dtypes, inputs, batch_sizes=None, hbm_gbs: float = 6451.2,
              rounds: int = 3, w_mode: str = "tiles"):
    """Profile the lookup table on the GPU: every tenant alone, at each batch
    size, executor with op-level dependencies and the device trace; T = the
    span of each fused op's items, W = min(1, items / #SMs)."""
    import numpy as np
    tenants = []
    for t, (g, p, B, dt, x) in enumerate(zip(graphs, params, batches, dtypes, inputs)):
        sizes = batch_sizes or sorted({1, 2, B // 2 if B > 1 else 1, B, max(1, B // 4)})
        tm = None
        for b in sizes:
            s = Session([(g, p, b, dt)], trace=True, coarse_deps=True)
            s.set_input(0, x[:b])
            for _ in range(rounds):
                s.run()
            st = G.gacer_get_stats()
            tr = G.gacer_get_trace(int(st["n_items"]))
            info = G.gacer_get_tenant_info(0)
            fused = G.gacer_query_op_fused(0, len(g.ops))
            if tm is None:
                nf = info["n_fused_ops"]
                last = [max(i for i, f in enumerate(fused) if f == ff) for ff in range(nf)]
                first = [min(i for i, f in enumerate(fused) if f == ff) for ff in range(nf)]
                tm = TenantModel(batch=B, n_orig=len(g.ops), last_member=last, first_member=first,
                                 decomposable=[True] * nf)
            base = info["op_base"]
            for ff in range(info["n_fused_ops"]):
                sel = tr[tr[:, 1] == base + ff]
                d = G.gacer_describe_op(base + ff)
                if len(sel) == 0:
                    continue
                T = (float(sel[:, 7].max()) - float(sel[:, 6].min())) / 1e3
                T = max(T, 1e-3)
                if w_mode == "occupancy":
                    # the op's measured SM occupancy over its span (Fig. 8's
                    # "SM occupancy", l.979): SM-time of its items / (T x #SMs)
                    W = min(1.0, float((sel[:, 7] - sel[:, 6]).sum()) / 1e3 / (T * NUM_SMS))
                else:   # Q10: the tile count's share of the SMs
                    W = min(1.0, d["items"] / NUM_SMS)
                Wb = min(1.0, d["bytes"] / (T * 1e-6) / (hbm_gbs * 1e9))
                tm.cost[(ff, b)] = OpCost(W=W, T=T, Wb=Wb)
            s.close()
        tenants.append(tm)
    return tenants
