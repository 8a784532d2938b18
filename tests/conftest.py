import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


def golden_cases():
    return sorted(os.path.basename(p)[len("hodlr_"):-len(".npz")]
                  for p in glob.glob(os.path.join(GOLDEN, "hodlr_*.npz")))


def load_case(name):
    """(H in the package's flat model, vectors dict, summary dict)."""
    from paper_2407_21637_b200.model import load_hodlr

    H = load_hodlr(os.path.join(GOLDEN, f"hodlr_{name}.npz"))
    with np.load(os.path.join(GOLDEN, f"vec_{name}.npz")) as z:
        vec = {k: z[k] for k in z.files if k != "summary"}
        summ = json.loads(str(z["summary"][()]))
    return H, vec, summ


def matvec_bound(depth, eps):
    """Thm 3.5 constant."""
    return 2 * (2 ** 0.5 + 1) * (2 ** (depth + 1) + 2 ** (depth - 1)) ** 0.5 * eps


@pytest.fixture(scope="session")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch
