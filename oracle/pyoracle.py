"""ctypes front-end to the oracle — TEST INFRASTRUCTURE ONLY.

Loads oracle/liboracle.so (the C restatement) and, when present,
oracle/_ref/libmoesched_ref.so (the unmodified reference library compiled from
/root/reference). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs import this module.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, fields

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


class OrcConfig(C.Structure):
    """Layout of orc_config (moesched_oracle.h); mirrors SimConfig (core.hpp:94-106)."""

    _fields_ = [
        ("num_layers", C.c_uint32), ("experts", C.c_uint32), ("top_k", C.c_uint32),
        ("batch", C.c_uint32), ("alpha", C.c_double), ("slots", C.c_uint32),
        ("window", C.c_uint32), ("policy", C.c_int32), ("init_fill", C.c_int32),
        ("t_attn", C.c_uint64), ("t_gpu", C.c_uint64), ("t_cpu_token", C.c_uint64),
        ("t_load", C.c_uint64), ("t_route", C.c_uint64), ("p_top", C.c_double),
        ("p_active", C.c_double), ("queue_depth", C.c_uint32), ("ce", C.c_int32),
        ("er", C.c_int32), ("pre", C.c_int32), ("ba", C.c_int32), ("seed", C.c_uint64),
    ]


@dataclass
class SimCfg:
    """Python view of SimConfig with the reference defaults (core.hpp:40-106)."""

    num_layers: int = 4
    experts: int = 64
    top_k: int = 6
    batch: int = 1
    alpha: float = 0.25
    slots: int = 16
    window: int = 16
    policy: int = 0  # 0 ScoreWindow, 1 LRU
    init_fill: int = 0  # 0 FirstSlots, 1 SeededRandom, 2 Empty
    t_attn: int = 5
    t_gpu: int = 1
    t_cpu_token: int = 30
    t_load: int = 100
    t_route: int = 0
    p_top: float = 0.82
    p_active: float = 0.95
    queue_depth: int = 0
    ce: int = 1
    er: int = 1
    pre: int = 1
    ba: int = 1
    seed: int = 0

    def to_c(self) -> OrcConfig:
        return OrcConfig(**{f.name: getattr(self, f.name) for f in fields(self)})


def _load(path):
    return C.CDLL(path) if os.path.exists(path) else None


_orc = None
_ref = None


def orc():
    global _orc
    if _orc is None:
        lib = _load(os.path.join(HERE, "liboracle.so"))
        if lib is None:
            raise RuntimeError("oracle/liboracle.so missing: run `make -C oracle`")
        lib.orc_simulate_json.restype = C.c_void_p
        lib.orc_free.argtypes = [C.c_void_p]
        lib.orc_rng_double.restype = C.c_double
        lib.orc_rng_u64.restype = C.c_uint64
        lib.orc_rng_below.restype = C.c_uint64
        lib.orc_rng_below.argtypes = [C.c_void_p, C.c_uint64]
        lib.orc_rng_gamma.restype = C.c_double
        lib.orc_rng_gamma.argtypes = [C.c_void_p, C.c_double]
        lib.orc_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
        lib.orc_derive_seed.restype = C.c_uint64
        lib.orc_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        lib.orc_cache_window_average.restype = C.c_double
        lib.orc_cache_try_evict.restype = C.c_int64
        lib.orc_cache_new.restype = C.c_void_p
        lib.orc_cache_new.argtypes = [C.c_uint32] * 4 + [C.c_int32, C.c_int32, C.c_uint64]
        for n in ("orc_cache_free", "orc_cache_resident", "orc_cache_record", "orc_cache_window_average",
                  "orc_cache_try_evict", "orc_cache_shield", "orc_cache_unshield", "orc_cache_is_shielded",
                  "orc_cache_touch", "orc_cache_admit"):
            f = getattr(lib, n)
            if f.argtypes is None:
                f.argtypes = None
        _orc = lib
    return _orc


def ref():
    """The reference library (None when it was not built, e.g. on the GPU box)."""
    global _ref
    if _ref is None:
        lib = _load(os.path.join(HERE, "_ref", "libmoesched_ref.so"))
        if lib is None:
            return None
        lib.ref_simulate_json.restype = C.c_void_p
        lib.ref_route_json.restype = C.c_void_p
        lib.ref_free.argtypes = [C.c_void_p]
        lib.ref_time_simulate.restype = C.c_double
        if hasattr(lib, "ref_report_from_trace_file"):
            lib.ref_report_from_trace_file.restype = C.c_void_p
        _ref = lib
    return _ref


def _dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _u8ptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def _take_json(lib, freefn, p):
    s = C.string_at(p).decode()
    freefn(p)
    return json.loads(s)


def generate_trace(L, E, B, iters, seed, hot_fraction=0.125, hot_mass=0.8, persistence=0.92,
                   concentration=1.5, use_ref=False, k=6):
    """generate_trace (trace.cpp:106-151) -> float64 [iters, L, B, E]."""
    out = np.zeros((iters, L, B, E), dtype=np.float64)
    if use_ref:
        r = ref()
        r.ref_generate_trace(C.c_uint32(L), C.c_uint32(E), C.c_uint32(k), C.c_uint32(B),
                             C.c_double(hot_fraction), C.c_double(hot_mass), C.c_double(persistence),
                             C.c_double(concentration), C.c_uint64(iters), C.c_uint64(seed), _dptr(out))
    else:
        orc().orc_generate_trace(C.c_uint32(L), C.c_uint32(E), C.c_uint32(B), C.c_double(hot_fraction),
                                 C.c_double(hot_mass), C.c_double(persistence), C.c_double(concentration),
                                 C.c_uint64(iters), C.c_uint64(seed), _dptr(out))
    return out


def _pred_args(pred, has_pred):
    if pred is None:
        return None, None
    pred = np.ascontiguousarray(pred, dtype=np.float64)
    has_pred = np.ascontiguousarray(has_pred, dtype=np.uint8)
    return pred, has_pred


def simulate(cfg: SimCfg, scores, pred=None, has_pred=None, steps=False, timeline=True):
    """The C restatement of simulate() (pipeline.cpp:374-385)."""
    scores = np.ascontiguousarray(scores, dtype=np.float64)
    pred, has_pred = _pred_args(pred, has_pred)
    c = cfg.to_c()
    lib = orc()
    p = lib.orc_simulate_json(C.byref(c), _dptr(scores), _dptr(pred) if pred is not None else None,
                              _u8ptr(has_pred) if has_pred is not None else None,
                              C.c_uint64(scores.shape[0]), C.c_int32(int(steps)), C.c_int32(int(timeline)))
    return _take_json(lib, lib.orc_free, p)


def ref_simulate(cfg: SimCfg, scores, pred=None, has_pred=None, timeline=True):
    """The reference simulate() itself (oracle/_ref)."""
    scores = np.ascontiguousarray(scores, dtype=np.float64)
    pred, has_pred = _pred_args(pred, has_pred)
    c = cfg.to_c()
    lib = ref()
    p = lib.ref_simulate_json(C.byref(c), _dptr(scores), _dptr(pred) if pred is not None else None,
                              _u8ptr(has_pred) if has_pred is not None else None,
                              C.c_uint64(scores.shape[0]), C.c_int(int(timeline)))
    return _take_json(lib, lib.ref_free, p)


def ref_simulate_seconds(cfg: SimCfg, scores):
    """Wall time of the reference simulate() alone (oracle/_ref), seconds."""
    scores = np.ascontiguousarray(scores, dtype=np.float64)
    c = cfg.to_c()
    lib = ref()
    lib.ref_simulate_ns.restype = C.c_uint64
    ns = lib.ref_simulate_ns(C.byref(c), _dptr(scores), C.c_uint64(scores.shape[0]))
    if not ns:
        raise RuntimeError("reference simulate() failed")
    return ns * 1e-9


def ref_report_from_trace_file(cfg: SimCfg, path: str):
    """The reference's load_trace() + simulate() + build_report() on a JSONL file."""
    lib = ref()
    c = cfg.to_c()
    p = lib.ref_report_from_trace_file(C.byref(c), path.encode())
    return _take_json(lib, lib.ref_free, p)


def ref_route(scores, mask, k, alpha, coalesce=False):
    scores = np.ascontiguousarray(scores, dtype=np.float64)
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    B, E = scores.shape
    lib = ref()
    p = lib.ref_route_json(_dptr(scores), C.c_uint32(B), C.c_uint32(E), _u8ptr(mask), C.c_uint32(k),
                           C.c_double(alpha), C.c_int(int(coalesce)))
    return _take_json(lib, lib.ref_free, p)


# ---- per-function oracle entry points (KAT tests) ----

class OrcRng(C.Structure):
    _fields_ = [("s", C.c_uint64 * 4)]


MAXE = 256


class OrcCls(C.Structure):
    _fields_ = [("beta", C.c_double), ("thr_top", C.c_double), ("thr_low", C.c_double),
                ("thr_alt", C.c_double), ("n_act", C.c_uint32), ("n_top", C.c_uint32),
                ("n_low", C.c_uint32), ("n_alt", C.c_uint32), ("act", C.c_uint32 * MAXE),
                ("top", C.c_uint32 * MAXE), ("low", C.c_uint32 * MAXE), ("alt", C.c_uint32 * MAXE)]


class OrcTok(C.Structure):
    _fields_ = [("n_sel", C.c_uint32), ("n_sub", C.c_uint32), ("n_kept", C.c_uint32),
                ("sel", C.c_uint32 * MAXE), ("sub_dropped", C.c_uint32 * MAXE),
                ("sub_chosen", C.c_uint32 * MAXE), ("kept", C.c_uint32 * MAXE), ("cls", OrcCls)]


def classify(scores, k, alpha):
    s = np.ascontiguousarray(scores, dtype=np.float64)
    c = OrcCls()
    rc = orc().orc_classify(_dptr(s), C.c_uint32(len(s)), C.c_uint32(k), C.c_double(alpha), C.byref(c))
    if rc:
        raise ValueError("classify: beta undefined, need at least k+1 experts")
    return dict(beta=c.beta, T=c.thr_top, L=c.thr_low, R=c.thr_alt,
                actives=list(c.act[:c.n_act]), top=list(c.top[:c.n_top]),
                low=list(c.low[:c.n_low]), alt=list(c.alt[:c.n_alt]))


def route(scores, mask, k, alpha, coalesce=False):
    s = np.ascontiguousarray(scores, dtype=np.float64)
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    B, E = s.shape
    toks = (OrcTok * B)()
    cset = (C.c_uint32 * MAXE)()
    nc = C.c_uint32()
    pend = (C.c_uint32 * (MAXE * 8))()
    npend = C.c_uint32()
    lib = orc()
    rc = lib.orc_route(_dptr(s), C.c_uint32(B), C.c_uint32(E), _u8ptr(m), C.c_uint32(k), C.c_double(alpha),
                       toks, cset, C.byref(nc), pend, C.byref(npend))
    if rc:
        raise ValueError("classify: beta undefined, need at least k+1 experts")
    if coalesce:
        lib.orc_coalesce(toks, _dptr(s), C.c_uint32(B), C.c_uint32(E), _u8ptr(m), cset, nc, pend, C.byref(npend))
    return {
        "C": list(cset[:nc.value]), "pending": list(pend[:npend.value]),
        "tok": [{"sel": list(t.sel[:t.n_sel]),
                 "sub": [[t.sub_dropped[i], t.sub_chosen[i]] for i in range(t.n_sub)],
                 "kept": list(t.kept[:t.n_kept])} for t in toks],
    }


def balance(items, t_cpu_token, t_load):
    n = len(items)
    uid = (C.c_uint32 * max(n, 1))(*[u for u, _ in items])
    bat = (C.c_uint32 * max(n, 1))(*[b for _, b in items])
    ll = (C.c_uint32 * max(n, 1))()
    cl = (C.c_uint32 * max(n, 1))()
    nl, nc = C.c_uint32(), C.c_uint32()
    c_load, c_cpu = C.c_uint64(), C.c_uint64()
    orc().orc_balance(uid, bat, C.c_uint32(n), C.c_uint64(t_cpu_token), C.c_uint64(t_load), ll, C.byref(nl),
                      cl, C.byref(nc), C.byref(c_load), C.byref(c_cpu))
    return list(ll[:nl.value]), list(cl[:nc.value]), c_load.value, c_cpu.value


class Rng:
    """xoshiro256** via the oracle (rng.cpp)."""

    def __init__(self, seed):
        self.st = OrcRng()
        orc().orc_rng_seed(C.byref(self.st), C.c_uint64(seed))

    def u64(self):
        return orc().orc_rng_u64(C.byref(self.st))

    def double(self):
        return orc().orc_rng_double(C.byref(self.st))

    def below(self, n):
        return orc().orc_rng_below(C.byref(self.st), C.c_uint64(n))

    def gamma(self, shape):
        return orc().orc_rng_gamma(C.byref(self.st), C.c_double(shape))


def derive_seed(seed, tag):
    return orc().orc_derive_seed(C.c_uint64(seed), C.c_uint64(tag))


def predict_scores(true_next, supplied, p_top, p_active, k, alpha, rng: Rng):
    tn = np.ascontiguousarray(true_next, dtype=np.float64)
    sup = None if supplied is None else np.ascontiguousarray(supplied, dtype=np.float64)
    out = np.zeros_like(tn)
    head = C.c_uint32()
    kind = C.c_int32()
    rc = orc().orc_predict_scores(_dptr(tn), _dptr(sup) if sup is not None else None, C.c_uint32(len(tn)),
                                  C.c_double(p_top), C.c_double(p_active), C.c_uint32(k), C.c_double(alpha),
                                  C.byref(rng.st), _dptr(out), C.byref(head), C.byref(kind))
    if rc:
        raise ValueError("classify: beta undefined, need at least k+1 experts")
    return out, head.value, kind.value


def build_queue(pred, mask, depth):
    p = np.ascontiguousarray(pred, dtype=np.float64)
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    ent = (C.c_uint32 * MAXE)()
    n = C.c_uint32()
    orc().orc_build_queue(_dptr(p), _u8ptr(m), C.c_uint32(len(p)), C.c_uint32(depth), ent, C.byref(n))
    return list(ent[:n.value])


class Cache:
    """CacheState restated (cache.cpp:10-156)."""

    def __init__(self, L, E, slots, window, policy=0, init_fill=0, seed=0):
        self.lib = orc()
        self.E = E
        self.h = self.lib.orc_cache_new(L, E, slots, window, policy, init_fill, seed)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.orc_cache_free(C.c_void_p(self.h))
            self.h = None

    def resident(self, layer):
        out = (C.c_uint32 * MAXE)()
        n = self.lib.orc_cache_resident(C.c_void_p(self.h), C.c_uint32(layer), out)
        return list(out[:n])

    def record(self, layer, scores):
        s = np.ascontiguousarray(scores, dtype=np.float64)
        return self.lib.orc_cache_record(C.c_void_p(self.h), C.c_uint32(layer), _dptr(s), C.c_uint32(len(s)))

    def window_average(self, layer, e):
        return self.lib.orc_cache_window_average(C.c_void_p(self.h), C.c_uint32(layer), C.c_uint32(e))

    def try_evict(self, layer):
        v = self.lib.orc_cache_try_evict(C.c_void_p(self.h), C.c_uint32(layer))
        return None if v < 0 else v

    def shield(self, layer, e):
        self.lib.orc_cache_shield(C.c_void_p(self.h), C.c_uint32(layer), C.c_uint32(e))

    def unshield(self, layer):
        self.lib.orc_cache_unshield(C.c_void_p(self.h), C.c_uint32(layer))

    def touch(self, layer, e, now):
        self.lib.orc_cache_touch(C.c_void_p(self.h), C.c_uint32(layer), C.c_uint32(e), C.c_uint64(now))

    def admit(self, layer, e, now):
        ev = C.c_int64()
        rc = self.lib.orc_cache_admit(C.c_void_p(self.h), C.c_uint32(layer), C.c_uint32(e), C.c_uint64(now),
                                      C.byref(ev))
        return rc, (None if ev.value < 0 else ev.value)
