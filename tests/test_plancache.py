"""NEXT-4 plan cache: keyed storage, keep-best,
persistence, and installing a cached plan through the C ABI (host-only
instance: plan compilation without a GPU)."""
import workloads
from paper_2304_11745_b200 import gacer as G
from paper_2304_11745_b200.plancache import CachedPlan, PlanCache, keys_for, mix_key


def test_keys_are_order_sensitive_and_canonical():
    a, b = workloads.build_model("resnet18"), workloads.build_model("vgg16")
    k1 = mix_key(keys_for([a, b], [8, 8], ["bf16", "bf16"]), "B200")
    k2 = mix_key(keys_for([b, a], [8, 8], ["bf16", "bf16"]), "B200")
    k3 = mix_key(keys_for([a, b], [8, 4], ["bf16", "bf16"]), "B200")
    assert len({k1, k2, k3}) == 3
    assert k1 == mix_key(keys_for([a, b], [8, 8], ["bf16", "bf16"]), "B200")


def test_put_keep_best_and_persistence(tmp_path):
    path = str(tmp_path / "plans.json")
    c = PlanCache(path)
    c.put("k", CachedPlan(pointers=[[3], [2]], ms=2.0, source="sweep"))
    kept = c.put("k", CachedPlan(pointers=[[5], [1]], ms=2.5, source="model_search"))
    assert kept.pointers == [[3], [2]]                      # the slower plan does not replace it
    c.put("k", CachedPlan(pointers=[[4], [1]], ms=1.5, source="measured_search"))
    c2 = PlanCache(path)                                     # offline store reloaded
    assert c2.get("k").pointers == [[4], [1]] and c2.get("k").source == "measured_search"
    assert c2.get("missing") is None and (c2.hits, c2.misses) == (2, 1)


def test_online_lookup_installs_and_searches_once():
    G.gacer_init(-1)
    try:
        gs = [workloads.build_model("resnet18"), workloads.build_model("mobilenet_v2")]
        for g in gs:
            G.gacer_register_tenant(g, workloads.make_params(g, 1, "bf16"), 4, "bf16")
        key = mix_key(keys_for(gs, [4, 4], ["bf16", "bf16"]))
        c = PlanCache()
        calls = []

        def search():
            calls.append(1)
            return CachedPlan(decomposition=[[0, 1, "batch", [2, 2], [20, 0]]], pointers=[[10], [20]],
                              partition="hybrid", ms=1.0, source="test")
        p, hit = c.lookup_or_search(G, key, 2, search)
        assert not hit and len(calls) == 1
        assert G.gacer_query_op_clusters(0, 11)[9:] == [0, 1]   # pointer after op 10 installed
        p, hit = c.lookup_or_search(G, key, 2, search)
        assert hit and len(calls) == 1                          # served from the cache
    finally:
        G.gacer_shutdown()
