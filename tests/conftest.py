import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


class GoldenCase:
    def __init__(self, path):
        z = np.load(path)
        self.name = os.path.basename(path)[:-4]
        self.spec = json.loads(str(z["spec"]))
        self.fixture, self.fn = self.spec["fixture"], self.spec["fn"]
        self.ret, self.fault = self.spec["ret"], self.spec["fault"]
        self.args, self.outs = [], {}
        for i, a in enumerate(self.spec["args"]):
            if a["kind"] == "array":
                self.args.append(z[a["key"]].copy())
                if f"out{i}" in z:
                    self.outs[i] = z[f"out{i}"].copy()
            else:
                self.args.append(a["value"] if a["kind"] == "float" else int(a["value"]))

    def __repr__(self):
        return self.name


def golden_cases(prefix=""):
    return [GoldenCase(p) for p in sorted(glob.glob(os.path.join(GOLDEN, prefix + "*.npz")))]


def normwise_err(got, ref, scale):
    """max_i |got_i - ref_i| / scale_i (scale_i = sum_j |terms_ij|, the reduction's magnitude);
    entries with scale 0 must match exactly."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    scale = np.asarray(scale, np.float64)
    d = np.abs(got - ref)
    z = scale == 0
    if np.any(d[z] != 0):
        return np.inf
    if np.all(z):
        return 0.0
    return float(np.max(d[~z] / scale[~z]))


@pytest.fixture(scope="session")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1302_5586_b200 as pb
    pb.load()
    return torch
