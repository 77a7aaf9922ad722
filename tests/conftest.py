"""Test configuration. `-m gpu` tests need a B200 (they call the CUDA path
through the C-ABI); everything else runs on CPU (oracle checks, ABI/export
checks, host logic, multi-process gloo)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device; runs the product kernels")


def _ensure_oracle():
    lib = os.path.join(REPO, "oracle", "liboracle.so")
    cpu = os.path.join(REPO, "oracle", "libcpumoe.so")
    if not (os.path.exists(lib) and os.path.exists(cpu)):
        subprocess.run(["make", "-C", os.path.join(REPO, "oracle"), "liboracle.so", "libcpumoe.so"], check=True,
                       capture_output=True)


_ensure_oracle()

GOLDEN_CASES = sorted(f[:-5] for f in os.listdir(GOLDEN) if f.endswith(".json") and f not in
                      ("index.json", "route_cases.json"))


def load_golden(name):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        meta = json.load(f)
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    pred = z["pred"] if "pred" in z.files else None
    has_pred = z["has_pred"] if "has_pred" in z.files else None
    return meta["config"], z["scores"], pred, has_pred, meta["expected"]


def load_route_cases():
    with open(os.path.join(GOLDEN, "route_cases.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def gpu():
    """Skip GPU tests when there is no device; fail loudly if the product
    library is missing on a GPU box."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2508_18983_b200 import capi
    capi.lib()
    return capi
