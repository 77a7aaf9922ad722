"""ctypes binding of the C-ABI in include/moesched_b200.h (libmoeb.so).

Used by tests/ and bench.py to drive the CUDA product path exactly as a
foreign caller of the reference's decision path would. There is no Python
fallback: if libmoeb.so is missing or no GPU is present the calls fail.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MOEB_LIB") or os.path.join(HERE, "libmoeb.so")  # MOEB_LIB: an alternative build (e.g. make PROFILE=1), diagnostics

MAXE, MAXK, MAXB = 64, 16, 32


class MoebError(RuntimeError):
    """Status != 0 from the C-ABI; .code mirrors the reference exception type."""

    KINDS = {1: "ConfigError", 2: "IoError", 3: "CacheError", 4: "logic_error", 5: "CudaError"}

    def __init__(self, code, msg):
        super().__init__(f"{self.KINDS.get(code, code)}: {msg}")
        self.code = code
        self.msg = msg


class Config(C.Structure):
    """moeb_config == SimConfig (core.hpp:94-106) with the reference defaults."""

    _fields_ = [
        ("num_layers", C.c_uint32), ("experts", C.c_uint32), ("top_k", C.c_uint32),
        ("batch", C.c_uint32), ("alpha", C.c_double), ("slots", C.c_uint32),
        ("window", C.c_uint32), ("policy", C.c_int32), ("init_fill", C.c_int32),
        ("t_attn", C.c_uint64), ("t_gpu", C.c_uint64), ("t_cpu_token", C.c_uint64),
        ("t_load", C.c_uint64), ("t_route", C.c_uint64), ("p_top", C.c_double),
        ("p_active", C.c_double), ("queue_depth", C.c_uint32), ("ce", C.c_int32),
        ("er", C.c_int32), ("pre", C.c_int32), ("ba", C.c_int32), ("seed", C.c_uint64),
    ]

    DEFAULTS = dict(num_layers=4, experts=64, top_k=6, batch=1, alpha=0.25, slots=16, window=16,
                    policy=0, init_fill=0, t_attn=5, t_gpu=1, t_cpu_token=30, t_load=100, t_route=0,
                    p_top=0.82, p_active=0.95, queue_depth=0, ce=1, er=1, pre=1, ba=1, seed=0)

    @classmethod
    def make(cls, **kw):
        d = dict(cls.DEFAULTS)
        d.update(kw)
        return cls(**d)

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class Model(C.Structure):
    _fields_ = [
        ("d_model", C.c_uint32), ("ffn", C.c_uint32), ("shared_ffn", C.c_uint32),
        ("shared_gate", C.c_int32), ("renormalize", C.c_int32), ("routed_scale", C.c_float),
        ("weight_seed", C.c_uint64), ("max_batch", C.c_uint32), ("flags", C.c_uint32),
    ]


class Metrics(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("tpot", "hit_rate", "substitution_ratio")] + [
        (n, C.c_uint64) for n in (
            "demand_loads", "prefetch_loads", "cpu_computed", "hits", "misses", "substitutions",
            "low_score_kept", "selections", "iterations", "total_time", "draws", "trace_supplied",
            "head_top", "head_active", "head_inactive", "issued", "cancelled")]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class IoStats(C.Structure):
    _fields_ = [("h2d_bytes", C.c_uint64), ("h2d_copies", C.c_uint64), ("d2d_copies", C.c_uint64),
                ("steps", C.c_uint64), ("copy_ms", C.c_double), ("spec_jobs", C.c_uint64),
                ("spec_promoted", C.c_uint64), ("spec_chunks", C.c_uint64), ("spec_bytes", C.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() (make -C paper_2508_18983_b200/csrc)")
        L = C.CDLL(LIB_PATH)
        L.moeb_last_error.restype = C.c_char_p
        L.moeb_free.argtypes = [C.c_void_p]
        L.moeb_result_free.argtypes = [C.c_void_p]
        L.moeb_cache_destroy.argtypes = [C.c_void_p]
        if hasattr(L, "moeb_destroy"):
            L.moeb_destroy.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def check(rc):
    if rc != 0:
        raise MoebError(rc, lib().moeb_last_error().decode())


def _d(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _u8(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def _u32buf(n):
    return (C.c_uint32 * max(int(n), 1))()


def _take_str(p):
    s = C.string_at(p).decode()
    lib().moeb_free(p)
    return s


# ----------------------------------------------------------------- policies

def classify(scores, k, alpha):
    s = np.ascontiguousarray(scores, dtype=np.float64)
    E = len(s)
    thr = (C.c_double * 4)()
    act, top, low, alt = _u32buf(E), _u32buf(E), _u32buf(E), _u32buf(E)
    nt, nl, na = C.c_uint32(), C.c_uint32(), C.c_uint32()
    check(lib().moeb_classify(_d(s), C.c_uint32(E), C.c_uint32(k), C.c_double(alpha), thr, act, top,
                              C.byref(nt), low, C.byref(nl), alt, C.byref(na)))
    return dict(beta=thr[0], T=thr[1], L=thr[2], R=thr[3], actives=list(act[:k]),
                top=list(top[:nt.value]), low=list(low[:nl.value]), alt=list(alt[:na.value]))


def plain_top_k(scores, k):
    s = np.ascontiguousarray(scores, dtype=np.float64)
    out, n = _u32buf(len(s)), C.c_uint32()
    check(lib().moeb_plain_top_k(_d(s), C.c_uint32(len(s)), C.c_uint32(k), out, C.byref(n)))
    return list(out[:n.value])


def _route_out(B, k, sel, nsel, sub, nsub, kept, nkept):
    return [{"sel": list(sel[t * k:t * k + nsel[t]]),
             "sub": [[sub[(t * k + i) * 2], sub[(t * k + i) * 2 + 1]] for i in range(nsub[t])],
             "kept": list(kept[t * k:t * k + nkept[t]])} for t in range(B)]


def route(scores, mask, k, alpha, coalesce=False):
    s = np.ascontiguousarray(scores, dtype=np.float64)
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    B, E = s.shape
    sel, sub, kept = _u32buf(B * k), _u32buf(2 * B * k), _u32buf(B * k)
    nsel, nsub, nkept = _u32buf(B), _u32buf(B), _u32buf(B)
    cset, pend = _u32buf(E), _u32buf(E)
    nc, npd = C.c_uint32(), C.c_uint32()
    check(lib().moeb_route(_d(s), C.c_uint32(B), C.c_uint32(E), _u8(m), C.c_uint32(k), C.c_double(alpha),
                           C.c_int32(int(coalesce)), sel, nsel, sub, nsub, kept, nkept, cset, C.byref(nc),
                           pend, C.byref(npd)))
    return {"C": list(cset[:nc.value]), "pending": list(pend[:npd.value]),
            "tok": _route_out(B, k, sel, nsel, sub, nsub, kept, nkept)}


def balance(items, t_cpu_token, t_load):
    n = len(items)
    uid = (C.c_uint32 * max(n, 1))(*[u for u, _ in items])
    bat = (C.c_uint32 * max(n, 1))(*[b for _, b in items])
    ll, cl = _u32buf(n), _u32buf(n)
    nl, nc = C.c_uint32(), C.c_uint32()
    c_load, c_cpu = C.c_uint64(), C.c_uint64()
    check(lib().moeb_balance(uid, bat, C.c_uint32(n), C.c_uint64(t_cpu_token), C.c_uint64(t_load), ll,
                             C.byref(nl), cl, C.byref(nc), C.byref(c_load), C.byref(c_cpu)))
    return list(ll[:nl.value]), list(cl[:nc.value]), c_load.value, c_cpu.value


def predict_scores(true_next, supplied, p_top, p_active, k, alpha, rng_state):
    """rng_state: list of 4 uint64 words, advanced in place."""
    tn = np.ascontiguousarray(true_next, dtype=np.float64)
    sup = None if supplied is None else np.ascontiguousarray(supplied, dtype=np.float64)
    st = (C.c_uint64 * 4)(*rng_state)
    out = np.zeros_like(tn)
    head, kind = C.c_uint32(), C.c_int32()
    check(lib().moeb_predict_scores(_d(tn), _d(sup) if sup is not None else None, C.c_uint32(len(tn)),
                                    C.c_double(p_top), C.c_double(p_active), C.c_uint32(k), C.c_double(alpha),
                                    st, _d(out), C.byref(head), C.byref(kind)))
    rng_state[:] = list(st)
    return out, head.value, kind.value


def build_queue(pred, mask, depth):
    p = np.ascontiguousarray(pred, dtype=np.float64)
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    ent, n = _u32buf(len(p)), C.c_uint32()
    check(lib().moeb_build_queue(_d(p), _u8(m), C.c_uint32(len(p)), C.c_uint32(depth), ent, C.byref(n)))
    return list(ent[:n.value])


class Cache:
    """CacheState (cache.hpp:25-78) living on the device."""

    def __init__(self, L, E, slots, window, policy=0, init_fill=0, seed=0):
        h = C.c_void_p()
        check(lib().moeb_cache_create(C.c_uint32(L), C.c_uint32(E), C.c_uint32(slots), C.c_uint32(window),
                                      C.c_int32(policy), C.c_int32(init_fill), C.c_uint64(seed), C.byref(h)))
        self.h, self.E = h, E

    def close(self):
        if self.h:
            lib().moeb_cache_destroy(self.h)
            self.h = None

    __del__ = close

    def resident(self, layer):
        out, n = _u32buf(self.E), C.c_uint32()
        check(lib().moeb_cache_resident(self.h, C.c_uint32(layer), out, C.byref(n)))
        return list(out[:n.value])

    def record(self, layer, scores):
        s = np.ascontiguousarray(scores, dtype=np.float64)
        check(lib().moeb_cache_record(self.h, C.c_uint32(layer), _d(s), C.c_uint32(len(s))))

    def window_average(self, layer, e):
        v = C.c_double()
        check(lib().moeb_cache_window_average(self.h, C.c_uint32(layer), C.c_uint32(e), C.byref(v)))
        return v.value

    def try_evict(self, layer):
        v = C.c_int64()
        check(lib().moeb_cache_try_evict(self.h, C.c_uint32(layer), C.byref(v)))
        return None if v.value < 0 else v.value

    def shield(self, layer, e):
        check(lib().moeb_cache_shield(self.h, C.c_uint32(layer), C.c_uint32(e)))

    def unshield(self, layer):
        check(lib().moeb_cache_unshield_layer(self.h, C.c_uint32(layer)))

    def is_shielded(self, layer, e):
        v = C.c_int32()
        check(lib().moeb_cache_is_shielded(self.h, C.c_uint32(layer), C.c_uint32(e), C.byref(v)))
        return bool(v.value)

    def touch(self, layer, e, now):
        check(lib().moeb_cache_touch(self.h, C.c_uint32(layer), C.c_uint32(e), C.c_uint64(now)))

    def admit(self, layer, e, now):
        """Returns (status, evicted) with status 0 ok / 3 CacheError / 4 logic_error."""
        ev = C.c_int64(-1)
        rc = lib().moeb_cache_admit(self.h, C.c_uint32(layer), C.c_uint32(e), C.c_uint64(now), C.byref(ev))
        return rc, (None if ev.value < 0 else ev.value)


def simulate(cfg: Config, scores, pred=None, has_pred=None, steps=False):
    """simulate() (pipeline.hpp:97) on the device; JSON dict in the oracle's schema."""
    s = np.ascontiguousarray(scores, dtype=np.float64)
    p = hp = None
    if pred is not None:
        p = np.ascontiguousarray(pred, dtype=np.float64)
        hp = np.ascontiguousarray(has_pred, dtype=np.uint8)
    r = C.c_void_p()
    check(lib().moeb_simulate(C.byref(cfg), _d(s), _d(p) if p is not None else None,
                              _u8(hp) if hp is not None else None, C.c_uint64(s.shape[0]),
                              C.c_int32(int(steps)), C.byref(r)))
    try:
        j = C.c_void_p()
        check(lib().moeb_result_json(r, C.byref(j)))
        return json.loads(_take_str(j))
    finally:
        lib().moeb_result_free(r)


MODEL_LOG_STEPS = 1
MODEL_PREDICTOR = 128  # the partial-forward predictor (include/moesched_b200.h)

# Model presets (dimensions of the BASELINE.json configs)
DSV2_LITE = dict(d_model=2048, ffn=1408, shared_ffn=2816, shared_gate=0, renormalize=0, routed_scale=1.0)
QWEN15_MOE = dict(d_model=2048, ffn=1408, shared_ffn=5632, shared_gate=1, renormalize=0, routed_scale=1.0)
MIXTRAL_8X7B = dict(d_model=4096, ffn=14336, shared_ffn=0, shared_gate=0, renormalize=1, routed_scale=1.0)


class Stack:
    """The MoE decode stack (moeb_create / moeb_step): bf16 device tensors in/out."""

    def __init__(self, cfg: Config, d_model, ffn, shared_ffn=0, shared_gate=0, renormalize=0,
                 routed_scale=1.0, weight_seed=7, log_steps=False, device=0, weights_host=None,
                 time_kernels=False, trace_timeline=False, deterministic=False, fill_pool=False, pool_flags=0,
                 predictor=False):
        flags = (MODEL_LOG_STEPS if log_steps else 0) | (2 if time_kernels else 0) | (4 if trace_timeline else 0) | \
            (16 if deterministic else 0) | (32 if fill_pool else 0) | pool_flags | (MODEL_PREDICTOR if predictor else 0)
        m = Model(d_model=d_model, ffn=ffn, shared_ffn=shared_ffn, shared_gate=shared_gate,
                  renormalize=renormalize, routed_scale=routed_scale, weight_seed=weight_seed,
                  max_batch=cfg.batch, flags=flags)
        h = C.c_void_p()
        self._weights = weights_host  # keep alive (numpy array, or (int pointer, owner))
        if weights_host is None:
            wp = None
        elif isinstance(weights_host, tuple):
            wp = C.c_void_p(weights_host[0])
            owner = weights_host[1] if len(weights_host) > 1 else None
            if isinstance(owner, Stack):  # a pool shared from another stack: same layout
                fl = C.c_uint32(0)
                check(lib().moeb_host_pool_flags(owner.h, C.byref(fl)))
                m.flags |= fl.value
        else:
            wp = C.c_void_p(weights_host.ctypes.data)
        check(lib().moeb_create(C.byref(cfg), C.byref(m), wp, C.c_int(device), C.byref(h)))
        self.h, self.cfg, self.model = h, cfg, m

    def pool_flags(self):
        """Layout flags of this stack's host pool (MOEB_MODEL_DOWN_T / MOEB_MODEL_TILED)."""
        fl = C.c_uint32(0)
        check(lib().moeb_host_pool_flags(self.h, C.byref(fl)))
        return fl.value

    def close(self):
        if getattr(self, "h", None):
            lib().moeb_destroy(self.h)
            self.h = None

    __del__ = close

    def set_logits_trace(self, logits, total_iterations=0):
        """logits: float32 [n_steps, L, B, E] numpy array or torch tensor (host or device)."""
        if hasattr(logits, "data_ptr"):
            ptr, n = logits.data_ptr(), logits.shape[0]
        else:
            logits = np.ascontiguousarray(logits, dtype=np.float32)
            self._trace = logits
            ptr, n = logits.ctypes.data, logits.shape[0]
        check(lib().moeb_set_logits_trace(self.h, C.c_void_p(ptr), C.c_uint64(n), C.c_uint64(total_iterations)))

    def step(self, x_ptr, y_ptr, B, stream=0):
        check(lib().moeb_step(self.h, C.c_void_p(x_ptr), C.c_void_p(y_ptr), C.c_uint32(B), C.c_void_p(stream)))

    def sync(self):
        check(lib().moeb_sync(self.h))

    def prefill(self, x_ptr, y_ptr, n_tokens, stream=0):
        """Prompt pass of n_tokens tokens (moeb_prefill): bf16 [n_tokens, d] device
        pointers; returns the bytes uploaded from the pinned pool."""
        b = C.c_uint64(0)
        check(lib().moeb_prefill(self.h, C.c_void_p(x_ptr), C.c_void_p(y_ptr), C.c_uint32(n_tokens),
                                 C.c_void_p(stream), C.byref(b)))
        return b.value

    def set_expert_sources(self, ptrs):
        """Upload each (layer, expert) from a device pointer (a peer GPU's HBM or
        this one's) instead of the pinned host pool; None restores the pool."""
        if ptrs is None:
            check(lib().moeb_set_expert_sources(self.h, None, C.c_size_t(0)))
            return
        arr = (C.c_void_p * len(ptrs))(*[int(p) for p in ptrs])
        check(lib().moeb_set_expert_sources(self.h, arr, C.c_size_t(len(ptrs))))

    def prefill_log(self, layer):
        """The last prefill's layer `layer` (MOEB_MODEL_LOG_STEPS): input hidden (bf16 bits
        [N, d]), router scores [N, E], selections [N, k] and the fp32 layer output [N, d]."""
        n = C.c_uint32(0)
        check(lib().moeb_get_prefill_log(self.h, C.c_uint32(layer), C.byref(n), None, None, None, None))
        N, d, E, k = n.value, self.model.d_model, self.cfg.experts, self.cfg.top_k
        x = np.zeros((N, d), dtype=np.uint16)
        sc = np.zeros((N, E), dtype=np.float32)
        sel = np.zeros((N, k), dtype=np.uint8)
        y = np.zeros((N, d), dtype=np.float32)
        check(lib().moeb_get_prefill_log(self.h, C.c_uint32(layer), C.byref(n), C.c_void_p(x.ctypes.data),
                                         C.c_void_p(sc.ctypes.data), C.c_void_p(sel.ctypes.data),
                                         C.c_void_p(y.ctypes.data)))
        return x, sc, sel, y


    def metrics(self):
        m = Metrics()
        check(lib().moeb_get_metrics(self.h, C.byref(m)))
        return m.as_dict()

    def decisions(self):
        j = C.c_void_p()
        check(lib().moeb_get_decisions_json(self.h, C.byref(j)))
        return json.loads(_take_str(j))

    def scores(self):
        n = C.c_size_t()
        check(lib().moeb_get_scores(self.h, None, C.c_size_t(0), C.byref(n)))
        out = np.zeros(n.value, dtype=np.float32)
        check(lib().moeb_get_scores(self.h, out.ctypes.data_as(C.POINTER(C.c_float)), C.c_size_t(n.value),
                                    C.byref(n)))
        return out

    def pred_scores(self):
        """Predicted scores each step's prefetch used ([steps*B*E] fp32; NaN: none)."""
        n = C.c_size_t()
        check(lib().moeb_get_pred_scores(self.h, None, C.c_size_t(0), C.byref(n)))
        out = np.zeros(n.value, dtype=np.float32)
        check(lib().moeb_get_pred_scores(self.h, out.ctypes.data_as(C.POINTER(C.c_float)), C.c_size_t(n.value),
                                         C.byref(n)))
        return out

    def copy_times(self):
        """Per-upload durations (ms) on the copy stream."""
        n = C.c_size_t()
        check(lib().moeb_get_copy_times(self.h, None, C.c_size_t(0), C.byref(n)))
        out = np.zeros(n.value, dtype=np.float32)
        check(lib().moeb_get_copy_times(self.h, out.ctypes.data_as(C.POINTER(C.c_float)), C.c_size_t(n.value),
                                        C.byref(n)))
        return out

    def io_stats(self):
        s = IoStats()
        check(lib().moeb_get_io_stats(self.h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in IoStats._fields_}

    def layer_outputs(self):
        L, B, d = self.cfg.num_layers, self.cfg.batch, self.model.d_model
        out = np.zeros(L * B * d, dtype=np.float32)
        check(lib().moeb_get_layer_outputs(self.h, out.ctypes.data_as(C.POINTER(C.c_float)), C.c_size_t(out.size)))
        return out.reshape(L, B, d)

MODEL_TIME_KERNELS = 2


class KernelStats(C.Structure):
    _fields_ = [("route_ms", C.c_double), ("ffn_ms", C.c_double),
                ("route_launches", C.c_uint64), ("ffn_launches", C.c_uint64),
                ("route_bytes", C.c_uint64), ("ffn_bytes", C.c_uint64), ("ffn_planned", C.c_uint64),
                ("prof_ns", C.c_uint64 * 32)]


def generate_trace(L, E, B, iters, seed, hot_fraction=0.125, hot_mass=0.8, persistence=0.92, concentration=1.5):
    """generate_trace (trace.cpp:106-151) via the product library -> float64 [iters, L, B, E]."""
    out = np.zeros((iters, L, B, E), dtype=np.float64)
    check(lib().moeb_generate_trace(C.c_uint32(L), C.c_uint32(E), C.c_uint32(B), C.c_double(hot_fraction),
                                    C.c_double(hot_mass), C.c_double(persistence), C.c_double(concentration),
                                    C.c_uint64(iters), C.c_uint64(seed), _d(out)))
    return out


def trace_logits(scores):
    """Router logits whose softmax reproduces a score trace: ln(s) in fp32."""
    with np.errstate(divide="ignore"):
        return np.log(scores).astype(np.float32)


def _stack_extra():
    L = lib()
    L.moeb_stream.restype = C.c_void_p


class _StackExt:
    def reset(self):
        check(lib().moeb_reset(self.h))

    def stream(self):
        lib().moeb_stream.restype = C.c_void_p
        return lib().moeb_stream(self.h) or 0

    def kernel_stats(self):
        s = KernelStats()
        check(lib().moeb_get_kernel_stats(self.h, C.byref(s)))
        d = {f: getattr(s, f) for f, _ in KernelStats._fields_}
        d["prof_ns"] = list(s.prof_ns)
        return d

    def timeline(self):
        """Device-clock (ns) timeline, one row of 16 words per layer-step (word table: moeb_get_timeline in include/moesched_b200.h)."""
        n = C.c_size_t(0)
        check(lib().moeb_get_timeline(self.h, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=np.uint64)
        check(lib().moeb_get_timeline(self.h, out.ctypes.data_as(C.POINTER(C.c_uint64)), n.value, C.byref(n)))
        return out.reshape(-1, 16)

    def reset_kernel_stats(self):
        check(lib().moeb_reset_kernel_stats(self.h))

    def host_pool(self):
        p, n = C.c_void_p(), C.c_size_t()
        check(lib().moeb_get_host_pool(self.h, C.byref(p), C.byref(n)))
        return p.value, n.value


for _n, _f in vars(_StackExt).items():
    if not _n.startswith("__"):
        setattr(Stack, _n, _f)
