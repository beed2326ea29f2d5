"""Offline / online plan cache (§4.4 l.860-863:
"In offline deployment, we can know all the multi-tenant deployment
scenarios and can store the searched strategies in the device and use them
directly when new requests appear.  For online deployment, GACER could yield
near-optimal schedule solutions within a short time").

A plan is everything ``gacer_set_regulation`` / ``gacer_set_partition`` /
``gacer_set_sm_shares`` take (mask + list_B [+ SM budgets], Matrix_P, the SM
partition policy and shares).  Plans are keyed by the tenant mix -- per
tenant, in registration order: model name, operator count, batch, dtype --
and the device name, and stored as JSON.  ``PlanCache.apply`` installs a
plan between rounds (the C ABI swaps plans atomically: a failed install
leaves the previous one in force), so a server can hot-swap the regulation
when the mix changes.  Online mode: on a miss, ``lookup_or_search`` runs the
given search (the measured Algorithm 1 of planner.py or the model-based one
of costmodel.py) once and stores its result.

Host-side bookkeeping only; it never touches tensors.
"""
from __future__ import annotations

import json
import os
import threading
import time
from dataclasses import asdict, dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple


@dataclass
class TenantKey:
    model: str
    n_ops: int
    batch: int
    dtype: str = "bf16"


@dataclass
class CachedPlan:
    decomposition: Optional[List[list]] = None    # [(tenant, op_index, axis, sizes[, sm_budget])]
    pointers: Optional[List[List[int]]] = None    # Matrix_P
    partition: str = "priority"
    shares: Optional[List[float]] = None
    ms: Optional[float] = None                    # measured makespan when stored
    source: str = "manual"                        # "measured_search", "model_search", "sweep", ...
    stored_at: float = field(default_factory=time.time)


def mix_key(tenants: Sequence[TenantKey], device: str = "") -> str:
    """Canonical key: order matters (tenant ids are registration order)."""
    parts = [f"{t.model}/{t.n_ops}/B{t.batch}/{t.dtype}" for t in tenants]
    return (device + "|" if device else "") + ";".join(parts)


def keys_for(graphs, batches, dtypes) -> List[TenantKey]:
    return [TenantKey(g.name, len(g.ops), int(b), d) for g, b, d in zip(graphs, batches, dtypes)]


class PlanCache:
    """JSON-backed {mix key -> CachedPlan} store (thread-safe, atomic writes)."""

    def __init__(self, path: Optional[str] = None):
        self.path = path
        self.lock = threading.Lock()
        self.plans: Dict[str, CachedPlan] = {}
        self.hits = self.misses = 0
        if path and os.path.exists(path):
            with open(path) as f:
                for k, v in json.load(f).items():
                    self.plans[k] = CachedPlan(**v)

    def get(self, key: str) -> Optional[CachedPlan]:
        with self.lock:
            p = self.plans.get(key)
            if p is None:
                self.misses += 1
            else:
                self.hits += 1
            return p

    def put(self, key: str, plan: CachedPlan, keep_best: bool = True) -> CachedPlan:
        """Store; with keep_best an existing plan with a lower measured ms wins."""
        with self.lock:
            old = self.plans.get(key)
            if keep_best and old is not None and old.ms is not None and plan.ms is not None and old.ms <= plan.ms:
                return old
            self.plans[key] = plan
            self._save()
            return plan

    def _save(self):
        if not self.path:
            return
        tmp = self.path + ".tmp"
        with open(tmp, "w") as f:
            json.dump({k: asdict(v) for k, v in self.plans.items()}, f, indent=1)
        os.replace(tmp, self.path)

    @staticmethod
    def apply(G, plan: CachedPlan, n_tenants: int):
        """Install between rounds through the C ABI (atomic per call)."""
        dec = [tuple(d[:4]) + ((list(d[4]),) if len(d) > 4 and d[4] is not None else ())
               for d in plan.decomposition] if plan.decomposition else None
        G.gacer_set_regulation(dec, plan.pointers, n_tenants=n_tenants)
        G.gacer_set_partition(plan.partition)
        G.gacer_set_sm_shares(plan.shares)

    def lookup_or_search(self, G, key: str, n_tenants: int,
                         search: Callable[[], CachedPlan]) -> Tuple[CachedPlan, bool]:
        """Online deployment: a hit installs the stored plan; a miss runs
        `search` once (it returns a CachedPlan), stores and installs it.
        Returns (plan, hit)."""
        p = self.get(key)
        hit = p is not None
        if not hit:
            p = self.put(key, search())
        self.apply(G, p, n_tenants)
        return p, hit
