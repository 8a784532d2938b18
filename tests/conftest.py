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


def random_hodlr(n, depth, fmts, ranks, working="fp64", seed=0, scale_levels=True):
    """A HODLR matrix with random factors already rounded to their formats
    (oracle.round_matrix), for exercising layouts the golden cases lack."""
    from oracle.fpsim import round_matrix
    from paper_2407_21637_b200 import NAMED_FORMATS, model

    rng = np.random.default_rng(seed)
    T = model.build_tree(n, depth)
    W = NAMED_FORMATS[working]
    leaves = [round_matrix(rng.standard_normal((b - a, b - a)), working) for a, b in T.ranges[depth]]
    blocks = []
    for k in range(1, depth + 1):
        F = NAMED_FORMATS[fmts[k - 1]]
        r = ranks[k - 1]
        lvl = []
        for i in range(2 ** (k - 1)):
            pair = []
            for rr, cc in ((T.ranges[k][2 * i], T.ranges[k][2 * i + 1]),
                           (T.ranges[k][2 * i + 1], T.ranges[k][2 * i])):
                rk = int(r if np.isscalar(r) else rng.integers(r[0], r[1] + 1))
                sc = 0.5 ** k if scale_levels else 1.0
                U = round_matrix(rng.standard_normal((rr[1] - rr[0], rk)) / np.sqrt(rr[1] - rr[0]), F)
                V = np.asfortranarray(round_matrix(rng.standard_normal((cc[1] - cc[0], rk)) * sc, F))
                pair.append(model.LowRankFactor(U, V, F))
            lvl.append(tuple(pair))
        blocks.append(lvl)
    return model.HodlrMatrix(T, leaves, blocks, 1e-6, model.PrecisionPlan([NAMED_FORMATS[f] for f in fmts]), W)
