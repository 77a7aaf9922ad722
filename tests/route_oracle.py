"""Independent band-rule evaluator restated from the reference's test-only
oracle (proj/tests/route_oracle.hpp:44-122), used as in test_router.cpp:161-197."""


def rank_desc(s):
    return sorted(range(len(s)), key=lambda i: -s[i])  # stable: index ascending on ties


def evaluate(batch, resident, k, alpha):
    toks = [dict(selected=set(), dropped=set(), chosen=set(), kept_low=set()) for _ in batch]
    shared_top, pending = set(), set()
    bands = []
    for t, s in enumerate(batch):
        order = rank_desc(s)
        actives = order[:k]
        beta = s[order[k]]
        top, low, alt = (1.0 + alpha) * beta, beta, (1.0 - alpha) * beta
        bands.append((beta, top, low, alt, actives))
        for e in actives:
            is_low = beta > 0.0 and s[e] >= low and s[e] < top
            if not is_low:
                toks[t]["selected"].add(e)
                shared_top.add(e)
    for t, s in enumerate(batch):
        beta, top, low, alt, actives = bands[t]
        b_low, alts = [], []
        for e in rank_desc(s):
            if e in actives and beta > 0.0 and low <= s[e] < top:
                if resident[e] or e in shared_top:
                    toks[t]["selected"].add(e)
                else:
                    b_low.append(e)
        for e in rank_desc(s):
            if e not in actives and beta > 0.0 and alt <= s[e] < low and (resident[e] or e in shared_top):
                alts.append(e)
        m, used = len(b_low), min(len(b_low), len(alts))
        for i in range(m - used):
            toks[t]["selected"].add(b_low[i])
            toks[t]["kept_low"].add(b_low[i])
            if not resident[b_low[i]]:
                pending.add(b_low[i])
        for i in range(used):
            toks[t]["selected"].add(alts[i])
            toks[t]["chosen"].add(alts[i])
            toks[t]["dropped"].add(b_low[m - used + i])
    return toks, shared_top, pending
