"""Known-answer and property tests of the reference's own test suite
(/root/reference/proj/tests/test_{router,cache,balancer,prefetch}.cpp),
restated in Python and run against BOTH the CPU oracle and the device
implementation (the latter marked gpu). Test names cite the reference case."""
import itertools

import numpy as np
import pytest

import pyoracle as po
from impls import IMPLS, make_impl
from route_oracle import evaluate

BAND = [0.30, 0.25, 0.10, 0.09, 0.085, 0.07, 0.06, 0.05]  # test_router.cpp:14


@pytest.fixture(params=IMPLS)
def impl(request):
    return make_impl(request.param)


def mask_of(E, on):
    m = np.zeros(E, dtype=np.uint8)
    for e in on:
        m[e] = 1
    return m


def random_scores(rng, experts):
    """test_router.cpp:30-44 (quantised 1/3 of the time to force ties)."""
    quant = rng.below(3) == 0
    s = [float(rng.below(8)) if quant else rng.double() for _ in range(experts)]
    tot = sum(s)
    if tot > 0.0:
        s = [v / (tot * (1.0 + 1e-12)) for v in s]
    return s


# ------------------------------------------------------------- router
def test_classify_worked_band_example(impl):  # test_router.cpp:48-60
    c = impl.classify(BAND, 3, 0.2)
    assert c["beta"] == pytest.approx(0.09)
    assert c["T"] == pytest.approx(0.108)
    assert c["R"] == pytest.approx(0.072)
    assert c["actives"] == [0, 1, 2]
    assert c["top"] == [0, 1]
    assert c["low"] == [2]
    assert c["alt"] == [4]


def test_classify_alpha_zero_collapses_bands(impl):  # :62-67
    c = impl.classify(BAND, 3, 0.0)
    assert c["low"] == [] and c["alt"] == [] and c["top"] == [0, 1, 2]


def test_classify_all_equal_lowest_indices(impl):  # :69-75
    c = impl.classify([0.125] * 8, 3, 0.0)
    assert c["actives"] == [0, 1, 2] and c["top"] == [0, 1, 2] and c["alt"] == []


def test_classify_beta_zero_disables_substitution(impl):  # :77-84
    c = impl.classify([0.5, 0.3, 0.2, 0.0, 0.0, 0.0], 3, 0.5)
    assert c["beta"] == 0.0 and len(c["top"]) == 3 and c["low"] == [] and c["alt"] == []


def test_classify_beta_undefined(impl):  # :86-89 (ConfigError)
    with pytest.raises(Exception) as ei:
        impl.classify([0.5, 0.5], 2, 0.1)
    assert "beta undefined" in str(ei.value)


def test_route_resident_alternative_replaces_low(impl):  # :91-98
    r = impl.route(np.array([BAND]), mask_of(8, [4]), 3, 0.2)
    t = r["tok"][0]
    assert set(t["sel"]) == {0, 1, 4}
    assert t["sub"] == [[2, 4]]
    assert r["pending"] == []


def test_route_no_alternative_keeps_residue_pending(impl):  # :100-105
    r = impl.route(np.array([BAND]), mask_of(8, []), 3, 0.2)
    assert set(r["tok"][0]["sel"]) == {0, 1, 2}
    assert r["tok"][0]["sub"] == []
    assert r["pending"] == [2]


def test_route_other_tokens_top_score_is_a_substitute(impl):  # :107-118
    t0 = [0.05, 0.06, 0.07, 0.085, 0.30, 0.25, 0.10, 0.09]
    t1 = [0.30, 0.25, 0.10, 0.09, 0.080, 0.07, 0.06, 0.05]
    r = impl.route(np.array([t0, t1]), mask_of(8, []), 3, 0.2)
    assert r["C"] == [0, 1, 4, 5]
    assert len(r["tok"][1]["sub"]) == 1 and r["tok"][1]["sub"][0][1] == 4
    assert set(r["tok"][1]["sel"]) == {0, 1, 4}


def _random_batch(rng, tokens_max=3):
    k = 1 + rng.below(3)
    experts = k + 1 + rng.below(8 - k)
    tokens = 1 + rng.below(tokens_max)
    batch = [random_scores(rng, experts) for _ in range(tokens)]
    resident = [1 if rng.below(2) != 0 else 0 for _ in range(experts)]
    return k, experts, batch, resident


def test_route_exactly_k_and_top_score_retained(impl):  # :120-159 (seed 99, 200 cases)
    rng = po.Rng(99)
    for _ in range(200):
        k, E, batch, res = _random_batch(rng)
        alpha = rng.double() * 0.6
        b = np.array(batch)
        r = impl.route(b, np.array(res, dtype=np.uint8), k, alpha)
        c = impl.route(b, np.array(res, dtype=np.uint8), k, alpha, coalesce=True)
        for t in range(len(batch)):
            cls = po.classify(batch[t], k, alpha)
            for res_ in (r, c):
                sel = res_["tok"][t]["sel"]
                assert len(sel) == k and len(set(sel)) == k
                assert set(cls["top"]) <= set(sel)
                for d, ch in res_["tok"][t]["sub"]:
                    assert cls["R"] <= batch[t][ch] < cls["L"]


def test_route_matches_band_rule_oracle(impl):  # :161-197 (seed 20240401, 1000 cases)
    rng = po.Rng(20240401)
    alphas = [0.0, 0.1, 0.25, 0.5]
    for _ in range(1000):
        k, E, batch, res = _random_batch(rng)
        alpha = alphas[rng.below(4)]
        got = impl.route(np.array(batch), np.array(res, dtype=np.uint8), k, alpha)
        toks, shared, pending = evaluate(batch, res, k, alpha)
        assert set(got["C"]) == shared
        assert set(got["pending"]) == pending
        for t, want in enumerate(toks):
            g = got["tok"][t]
            assert set(g["sel"]) == want["selected"]
            assert set(g["kept"]) == want["kept_low"]
            assert {d for d, _ in g["sub"]} == want["dropped"]
            assert {c for _, c in g["sub"]} == want["chosen"]


def test_alpha_zero_routing_is_plain_top_k(impl):  # :199-213 (seed 7, 1000 cases)
    rng = po.Rng(7)
    for _ in range(1000):
        k = 1 + rng.below(3)
        E = k + 1 + rng.below(8 - k)
        s = random_scores(rng, E)
        res = [1 if rng.below(2) != 0 else 0 for _ in range(E)]
        r = impl.route(np.array([s]), np.array(res, dtype=np.uint8), k, 0.0)
        assert r["tok"][0]["sub"] == []
        top = sorted(range(E), key=lambda i: (-s[i], i))[:k]
        assert set(r["tok"][0]["sel"]) == set(top)


def test_coalesce_batch_size_example(impl):  # :215-244
    t0 = [0.09, 0.30, 0.25, 0.02, 0.10, 0.02, 0.01, 0.01]
    t1 = [0.09, 0.30, 0.01, 0.02, 0.10, 0.25, 0.02, 0.01]
    t2 = [0.01, 0.08, 0.30, 0.01, 0.07, 0.01, 0.09, 0.25]
    b = np.array([t0, t1, t2])
    base = impl.route(b, mask_of(8, []), 3, 0.5)
    assert [set(t["sel"]) for t in base["tok"]] == [{1, 2, 4}, {1, 5, 4}, {2, 6, 7}]
    assert base["tok"][2]["kept"] == [6]
    merged = impl.route(b, mask_of(8, []), 3, 0.5, coalesce=True)
    assert set(merged["tok"][2]["sel"]) == {2, 4, 7}
    assert merged["tok"][2]["sub"] == [[6, 4]]
    d0 = set().union(*[set(t["sel"]) for t in base["tok"]])
    d1 = set().union(*[set(t["sel"]) for t in merged["tok"]])
    assert len(d1) < len(d0)


def test_coalesce_nothing_without_low_score(impl):  # :246-254
    s = np.array([[0.5, 0.3, 0.2, 0.0, 0.0, 0.0]])
    base = impl.route(s, np.ones(6, dtype=np.uint8), 3, 0.4)
    merged = impl.route(s, np.ones(6, dtype=np.uint8), 3, 0.4, coalesce=True)
    assert base["tok"][0]["kept"] == [] and merged["tok"][0]["sel"] == base["tok"][0]["sel"]


def test_coalesce_single_token_stays_put(impl):  # :256-261
    m = mask_of(8, [4, 3])
    base = impl.route(np.array([BAND]), m, 3, 0.2)
    merged = impl.route(np.array([BAND]), m, 3, 0.2, coalesce=True)
    assert merged["tok"][0]["sel"] == base["tok"][0]["sel"]
    assert len(merged["tok"][0]["sub"]) == len(base["tok"][0]["sub"])


def test_coalesce_never_raises_nonresident_count(impl):  # :263-291 (seed 4242, 300 cases)
    rng = po.Rng(4242)
    for _ in range(300):
        k, E, batch, res = _random_batch(rng)
        alpha = rng.double() * 0.6
        b, m = np.array(batch), np.array(res, dtype=np.uint8)
        base = impl.route(b, m, k, alpha)
        merged = impl.route(b, m, k, alpha, coalesce=True)

        def nonres(r):
            return sum(1 for e in set().union(*[set(t["sel"]) for t in r["tok"]]) if not res[e])
        assert nonres(merged) <= nonres(base)
        assert len(merged["pending"]) <= len(base["pending"])


# -------------------------------------------------------------- cache
def make_cache(impl, experts, slots, window, policy):  # test_cache.cpp:14-19
    return impl.Cache(1, experts, slots, window, policy, 0, 0)


def test_ring_keeps_last_n(impl):  # test_cache.cpp:23-32
    c = make_cache(impl, 3, 3, 2, 0)
    c.record(0, [0.9, 0.0, 0.0])
    c.record(0, [0.0, 0.5, 0.0])
    c.record(0, [0.0, 0.1, 0.3])
    assert c.window_average(0, 0) == pytest.approx(0.0)
    assert c.window_average(0, 1) == pytest.approx(0.3)
    assert c.window_average(0, 2) == pytest.approx(0.15)


def test_empty_history_averages_zero(impl):  # :34-38
    c = make_cache(impl, 3, 3, 4, 0)
    assert c.window_average(0, 0) == 0.0 and c.window_average(0, 2) == 0.0


def test_score_window_eviction(impl):  # :40-57
    c = make_cache(impl, 3, 3, 2, 0)
    c.record(0, [0.3, 0.01, 0.1])
    c.record(0, [0.1, 0.03, 0.05])
    assert c.try_evict(0) == 1
    c.shield(0, 1)
    assert c.try_evict(0) == 2
    c.unshield(0)
    assert c.try_evict(0) == 1


def test_lru_eviction(impl):  # :59-67
    c = make_cache(impl, 3, 3, 2, 1)
    c.touch(0, 0, 5)
    c.touch(0, 1, 9)
    c.touch(0, 2, 7)
    assert c.try_evict(0) == 0
    c.shield(0, 0)
    assert c.try_evict(0) == 2


def test_all_shielded_no_candidate(impl):  # :69-75 (CacheError "no evictable expert")
    c = make_cache(impl, 2, 2, 2, 0)
    c.shield(0, 0)
    c.shield(0, 1)
    assert c.try_evict(0) is None
    c2 = impl.Cache(1, 3, 2, 2, 0, 0, 0)
    c2.shield(0, 0)
    c2.shield(0, 1)
    rc, ev = c2.admit(0, 2, 1)
    assert rc == 3


def test_admit_capacity(impl):  # :77-95
    cold = impl.Cache(1, 8, 2, 2, 0, 2, 0)
    assert cold.resident(0) == []
    assert cold.admit(0, 3, 1) == (0, None)
    assert cold.resident(0) == [3]
    c = impl.Cache(1, 8, 2, 2, 0, 0, 0)
    assert c.resident(0) == [0, 1]
    c.record(0, [0.5, 0.1, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0])
    assert c.admit(0, 5, 10) == (0, 1)
    assert c.resident(0) == [0, 5]


def test_admit_resident_is_caller_bug(impl):  # :97-100 (std::logic_error)
    c = make_cache(impl, 4, 2, 2, 0)
    rc, _ = c.admit(0, 0, 1)
    assert rc == 4


def test_window_one_behaves_like_lru(impl):  # :102-113
    s = make_cache(impl, 3, 3, 1, 0)
    lru = make_cache(impl, 3, 3, 1, 1)
    lru.touch(0, 2, 1)
    lru.touch(0, 0, 2)
    lru.touch(0, 1, 3)
    s.record(0, [0.2, 0.3, 0.1])
    assert s.try_evict(0) == lru.try_evict(0)


def test_cache_random_ops_match_oracle(impl):  # :115-188 (seed 123456), op stream replayed on both
    experts, slots = 12, 5
    dev = impl.Cache(2, experts, slots, 3, 0, 0, 1)
    ref = po.Cache(2, experts, slots, 3, 0, 0, 1)
    rng = po.Rng(123456)
    n_ops = 10000 if impl.name == "oracle" else 2000
    shielded = [set(), set()]
    for op in range(n_ops):
        layer = rng.below(2)
        kind = rng.below(5)
        if kind == 0:
            v = [rng.double() / experts for _ in range(experts)]
            dev.record(layer, v)
            ref.record(layer, v)
        elif kind == 1:
            res = ref.resident(layer)
            if res:
                pick = res[rng.below(len(res))]
                dev.shield(layer, pick)
                ref.shield(layer, pick)
                shielded[layer].add(pick)
        elif kind == 2:
            dev.unshield(layer)
            ref.unshield(layer)
            shielded[layer].clear()
        elif kind == 3:
            e = rng.below(experts)
            if e not in ref.resident(layer):
                assert dev.admit(layer, e, op) == ref.admit(layer, e, op)
        else:
            v = ref.try_evict(layer)
            assert dev.try_evict(layer) == v
            if v is not None:
                assert v not in shielded[layer]
                for o in ref.resident(layer):
                    if o not in shielded[layer]:
                        assert ref.window_average(layer, v) <= ref.window_average(layer, o)
        assert dev.resident(layer) == ref.resident(layer)
        assert len(ref.resident(layer)) <= slots


def test_seeded_fill_is_reproducible_prefix(impl):  # :210-226
    a = impl.Cache(3, 16, 6, 2, 0, 1, 9)
    b = impl.Cache(3, 16, 6, 2, 0, 1, 9)
    c = impl.Cache(3, 16, 6, 2, 0, 1, 10)
    snap = lambda x: [x.resident(l) for l in range(3)]  # noqa: E731
    assert snap(a) == snap(b) and snap(a) != snap(c)
    ref = po.Cache(3, 16, 6, 2, 0, 1, 9)
    assert snap(a) == [ref.resident(l) for l in range(3)]
    for l in range(3):
        r = a.resident(l)
        assert len(r) == 6 and len(set(r)) == 6 and all(e < 16 for e in r)


# ----------------------------------------------------------- balancer
def brute_force(items, t_cpu, t_load):  # balancer.cpp:40-59
    best = None
    for mask in range(1 << len(items)):
        cl = sum(t_load for i in range(len(items)) if mask >> i & 1)
        cc = sum(b * t_cpu for i, (_, b) in enumerate(items) if not mask >> i & 1)
        best = max(cl, cc) if best is None else min(best, max(cl, cc))
    return 0 if not items else best


def test_balance_hand_traced(impl):  # test_balancer.cpp:12-22
    ll, cl, c_load, c_cpu = impl.balance([(0, 4), (1, 2), (2, 1)], 1, 3)
    assert ll == [0] and cl == [2, 1] and c_load == 3 and c_cpu == 3
    assert brute_force([(0, 4), (1, 2), (2, 1)], 1, 3) == 3


def test_balance_empty_and_single(impl):  # :24-40
    assert impl.balance([], 1, 3) == ([], [], 0, 0)
    assert impl.balance([(7, 5)], 1, 3)[:2] == ([7], [])


def test_balance_sort_order(impl):  # :52-61
    ll, cl, _, _ = impl.balance([(9, 2), (3, 2), (5, 7)], 1, 100)
    assert len(ll) + len(cl) == 3 and ll[0] == 5 and cl[0] == 9


def test_balance_partition_and_quality(impl):  # :63-108 (seed 20240817)
    rng = po.Rng(20240817)
    optimal = 0
    n_inst = 500 if impl.name == "oracle" else 200
    for _ in range(n_inst):
        n = 1 + rng.below(10)
        items = [(j, 1 + rng.below(3)) for j in range(n)]
        t_cpu = 1 + rng.below(10)
        t_load = t_cpu + rng.below(t_cpu + 1)
        ll, cl, c_load, c_cpu = impl.balance(items, t_cpu, t_load)
        assert sorted(ll + cl) == list(range(n))
        assert c_cpu == sum(b * t_cpu for u, b in items if u in cl)
        assert c_load == len(ll) * t_load
        opt = brute_force(items, t_cpu, t_load)
        assert opt <= max(c_load, c_cpu) <= 2 * opt
        optimal += max(c_load, c_cpu) == opt
        assert (ll, cl) == po.balance(items, t_cpu, t_load)[:2]
    assert optimal >= n_inst * 60 // 100


# ----------------------------------------------------------- prefetch
TRUE = [0.30, 0.25, 0.10, 0.09, 0.085, 0.07, 0.06, 0.045]  # test_prefetch.cpp:16


def test_perfect_predictor(impl):  # test_prefetch.cpp:21-39
    rng = po.Rng(1)
    for _ in range(50):
        out, head, kind = impl.predict_scores(TRUE, None, 1.0, 0.95, 3, 0.2, rng)
        assert kind == 0
        top2 = sorted(range(8), key=lambda i: (-out[i], i))[:2]
        assert set(top2) == {0, 1}
        assert sorted(out) == sorted(TRUE)


def test_supplied_prediction_passthrough(impl):  # :41-53
    sup = [0.0] * 7 + [1.0]
    r1, r2 = po.Rng(5), po.Rng(5)
    before = r1.u64()
    out, head, kind = impl.predict_scores(TRUE, sup, 0.0, 0.0, 3, 0.2, r2)
    assert list(out) == sup and head == 7
    assert r2.u64() == before


def test_predictor_calibration(impl):  # :55-67 (seed 20250810)
    rng = po.Rng(20250810)
    n = 10000 if impl.name == "oracle" else 2000
    kinds = [impl.predict_scores(TRUE, None, 0.82, 0.95, 3, 0.2, rng)[2] for _ in range(n)]
    top = kinds.count(0) / n
    non_top = n - kinds.count(0)
    assert top == pytest.approx(0.82, rel=0.025 if n == 10000 else 0.05)
    assert kinds.count(1) / non_top == pytest.approx(0.95, rel=0.021 if n == 10000 else 0.06)


def test_predictor_matches_oracle_stream(impl):  # device vs oracle draw-by-draw
    r_dev, r_ref = po.Rng(33), po.Rng(33)
    for _ in range(300 if impl.name == "device" else 50):
        a = impl.predict_scores(TRUE, None, 0.5, 0.5, 3, 0.2, r_dev)
        b = po.predict_scores(TRUE, None, 0.5, 0.5, 3, 0.2, r_ref)
        assert list(a[0]) == list(b[0]) and a[1:] == b[1:]
        assert sum(a[0]) == pytest.approx(1.0, abs=1e-9)


def test_build_queue(impl):  # :84-105
    q = impl.build_queue([0.0, 0.2, 0.0, 0.3, 0.0, 0.4], np.array([0, 0, 0, 1, 0, 0], dtype=np.uint8), 2)
    assert q == [5, 1]
    assert impl.build_queue([0.5, 0.3, 0.2], np.array([1, 1, 1], dtype=np.uint8), 3) == []
    assert impl.build_queue([0.5, 0.3, 0.2], np.zeros(3, dtype=np.uint8), 0) == []


@pytest.mark.parametrize("seed", range(3))
def test_build_queue_ties_match_oracle(impl, seed):
    rng = np.random.RandomState(seed)
    for _ in range(50):
        E = rng.randint(2, 65)
        p = np.floor(rng.rand(E) * 4) / 4
        m = (rng.rand(E) < 0.3).astype(np.uint8)
        d = rng.randint(0, 8)
        assert impl.build_queue(p, m, d) == po.build_queue(p, m, d)


def test_all_subsets_of_small_band_example(impl):
    """Exhaustive residency masks on the band example (route vs band oracle)."""
    for bits in itertools.product([0, 1], repeat=8):
        r = impl.route(np.array([BAND]), np.array(bits, dtype=np.uint8), 3, 0.2)
        toks, shared, pending = evaluate([BAND], list(bits), 3, 0.2)
        assert set(r["tok"][0]["sel"]) == toks[0]["selected"] and set(r["pending"]) == pending
