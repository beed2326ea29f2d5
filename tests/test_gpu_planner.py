"""Algorithm 1 on the device (§4.4): the measured-objective search
installs every candidate plan through the C ABI and times executor rounds;
the plan it returns must give byte-identical outputs to the identity plan
(north_star: results do not depend on the regulation) and a makespan no
worse than the identity plan's measurement."""
import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu


def test_measured_search_returns_valid_invariant_plan():
    import torch

    from paper_2304_11745_b200 import gacer as G
    from paper_2304_11745_b200 import planner as P
    from paper_2304_11745_b200.runtime import Session

    specs = [("resnet18", 4, 64), ("mobilenet_v2", 4, 64)]
    tenants, xs = [], []
    for i, (name, B, hw) in enumerate(specs):
        g = workloads.build_model(name, hw)
        tenants.append((g, workloads.make_params(g, 70 + i, "bf16"), B, "bf16"))
        xs.append(workloads.make_input(g, B, 70 + i, "bf16"))
    s = Session(tenants)
    try:
        for t, x in enumerate(xs):
            s.set_input(t, x)
        s.run()
        ref = s.results()
        stream = torch.cuda.Stream()
        ev = P.measured_objective(G, s, [t[0] for t in tenants], [t[2] for t in tenants], torch, stream,
                                  rounds=3, warmup=1)
        n_ops = [len(t[0].ops) for t in tenants]
        res = P.granularity_aware_search(ev, n_ops, P.SearchConfig(max_pointers=2, stride=8, max_evals=40))
        assert res.evals <= 40
        assert res.R <= res.records[0] + 1e-9
        assert all(len(p) == len(res.pointers[0]) for p in res.pointers)      # equal counts
        assert all(list(p) == sorted(p) and (not p or 0 <= p[0] and p[-1] <= n) for p, n in zip(res.pointers, n_ops))
        s.set_regulation(ev.plan_decomposition(res.decomposition),
                         [list(p) for p in res.pointers] if any(res.pointers) else None)
        s.set_mode("executor")
        s.run()
        out = s.results()
        for a, b in zip(ref, out):
            assert np.asarray(a).tobytes() == np.asarray(b).tobytes()
    finally:
        s.close()
