"""Two implementations of the reference policy API behind one interface:
  * "oracle": the CPU restatement (oracle/, test infrastructure)
  * "device": the product — CUDA kernels through the C-ABI (libmoeb.so)
so every known-answer test runs unchanged against both."""
import pytest

import pyoracle as po


class OracleImpl:
    name = "oracle"
    classify = staticmethod(po.classify)
    route = staticmethod(po.route)
    balance = staticmethod(po.balance)
    build_queue = staticmethod(po.build_queue)
    Cache = po.Cache

    @staticmethod
    def predict_scores(true_next, supplied, p_top, p_active, k, alpha, rng):
        return po.predict_scores(true_next, supplied, p_top, p_active, k, alpha, rng)

    @staticmethod
    def simulate(kw, scores, pred=None, has_pred=None, steps=False):
        return po.simulate(po.SimCfg(**kw), scores, pred, has_pred, steps=steps)


class DeviceImpl:
    name = "device"

    def __init__(self):
        from paper_2508_18983_b200 import capi
        self.capi = capi
        self.classify = capi.classify
        self.route = capi.route
        self.balance = capi.balance
        self.build_queue = capi.build_queue
        self.Cache = capi.Cache

    def predict_scores(self, true_next, supplied, p_top, p_active, k, alpha, rng):
        # rng: a pyoracle.Rng whose xoshiro state is advanced exactly as the device does
        st = list(rng.st.s)
        out = self.capi.predict_scores(true_next, supplied, p_top, p_active, k, alpha, st)
        for i in range(4):
            rng.st.s[i] = st[i]
        return out

    def simulate(self, kw, scores, pred=None, has_pred=None, steps=False):
        return self.capi.simulate(self.capi.Config.make(**kw), scores, pred, has_pred, steps=steps)


IMPLS = ["oracle", pytest.param("device", marks=pytest.mark.gpu)]


def make_impl(name):
    if name == "oracle":
        return OracleImpl()
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return DeviceImpl()
