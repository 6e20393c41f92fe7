import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    # the C restatement is test infrastructure; (re)build it when its sources changed
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "liboracle.so"], check=True)


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


@pytest.fixture(scope="session")
def instances(golden):
    names = sorted({k.split("/")[1] for k in golden.files if k.startswith("inst/")})
    out = {}
    for nm in names:
        p = f"inst/{nm}/"
        m, n = (int(v) for v in golden[p + "shape"])
        out[nm] = dict(m=m, n=n, row_ptr=golden[p + "row_ptr"], col_idx=golden[p + "col_idx"],
                       values=golden[p + "values"], row_norm=golden[p + "row_norm"], b=golden[p + "b"],
                       x_star=golden[p + "x_star"])
    return out


def triplets(inst):
    rows = np.repeat(np.arange(inst["m"]), np.diff(inst["row_ptr"]))
    return rows, inst["col_idx"], inst["values"]
