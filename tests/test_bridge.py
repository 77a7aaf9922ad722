"""Wire-format bridge (paper_2508_18983_b200/bridge.py):
a decode run exported as the reference's GateTrace JSONL is read back by the
reference's own load_trace() (oracle/_ref, compiled from /root/reference) and
replayed by its simulate(); the reference's build_report() must then agree
with our report() of the run — metrics, predictor statistics and the trace
fingerprint.

CPU: the run is the oracle's (a stand-in stack object). GPU: the real stack.
"""
import numpy as np
import pytest

import pyoracle as po
from paper_2508_18983_b200 import bridge

needs_ref = pytest.mark.skipif(po.ref() is None, reason="reference library not built (oracle/_ref)")


def test_fingerprint_is_fnv1a():
    assert bridge.fingerprint_bytes(b"") == "cbf29ce484222325"
    assert bridge.fingerprint_bytes(b"a") == "af63dc4c8601ec8c"


def test_stage_labels():  # core.cpp:11-24
    assert bridge.stage_label(dict(ce=0, er=0, pre=0, ba=0)) == "baseline"
    assert bridge.stage_label(dict(ce=1, er=1, pre=0, ba=1)) == "CE+ER+BA"
    assert bridge.stage_label({}) == "CE+ER+Pre+BA"


class OracleRun:
    """A finished run with the stack's read-out interface, produced by the oracle."""

    def __init__(self, kw, scores):
        self._scores = scores.astype(np.float32)
        out = po.simulate(po.SimCfg(**kw), self._scores.astype(np.float64))
        self._m = dict(out["metrics"], **out["stats"])

    def scores(self):
        return self._scores.reshape(-1)

    def metrics(self):
        return self._m


def _check(run, kw, tmp_path):
    path = str(tmp_path / "run.jsonl")
    n = bridge.export_trace(run, kw, path)
    assert n > 0
    mine = bridge.report(run, kw, path)
    theirs = po.ref_report_from_trace_file(po.SimCfg(**kw), path)
    assert "error" not in theirs, theirs
    assert theirs["trace_fingerprint"] == mine["trace_fingerprint"]
    for key, v in mine["metrics"].items():
        assert theirs["metrics"][key] == v, key
    for key, v in mine["prefetch_stats"].items():
        assert theirs["prefetch_stats"][key] == v, key


@needs_ref
@pytest.mark.parametrize("B", [1, 3])
def test_oracle_run_round_trips_through_reference(tmp_path, B):
    kw = dict(num_layers=3, experts=32, top_k=4, batch=B, slots=8, alpha=0.25, seed=7)
    scores = po.generate_trace(3, 32, B, 12, 7)
    _check(OracleRun(kw, scores), kw, tmp_path)


@pytest.mark.gpu
@needs_ref
def test_device_run_round_trips_through_reference(gpu, tmp_path):
    import torch
    from test_stack_gpu import run_stack
    st, kw, xs, _ = run_stack(gpu, torch, 2, 64, 6, 2, 256, 128, 256, 16, 20)
    _check(st, kw, tmp_path)
    st.close()
