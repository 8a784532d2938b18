"""The matrix-free builders pinned to the reference's
``build_adaptive`` (hodlr.py:227-265) and ``_truncation_rank`` (lowrank.py:80-99):
on dense instances the reference can build (tests/golden/builder_golden.json,
written by tests/golden/make_golden_r2.py from /root/reference), the GPU
sources must reproduce the plan (formats, xi), every block's rank and
``storage_bits``.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLDEN, "builder_golden.json")) as f:
        return json.load(f)


def compare(H, want):
    from paper_2407_21637_b200 import model

    assert [f.name for f in H.plan.chosen] == want["formats"]
    assert np.allclose(H.plan.xi, want["xi"], rtol=1e-12, atol=0)
    assert np.allclose(H.plan.thresholds, want["thresholds"], rtol=1e-12, atol=0)
    assert list(H.plan.fallback) == want["fallback"]
    ranks = [[up.rank, lo.rank] for _, _, _, _, up, lo in H.offdiag_blocks()]
    assert ranks == want["ranks"]
    assert model.storage_bits(H) == want["storage_bits"]
    assert (H.n, H.depth, H.eps, H.working_format.name) == (want["n"], want["depth"], want["eps"], want["working"])


def test_toeplitz_source_matches_reference_n8192(cuda, golden):
    from paper_2407_21637_b200 import FP64, problems

    H, _, _ = problems.toeplitz_config(8192, 5, 1e-6, FP64, 0)
    compare(H, golden["toeplitz_inv_8192"])


def test_toeplitz_source_fft_path_matches_reference(cuda, golden):
    """Same instance through the never-formed (FFT-applied) range finder that
    cfg5's top levels use."""
    from paper_2407_21637_b200 import FP64, problems
    from paper_2407_21637_b200.construct import build_adaptive
    from paper_2407_21637_b200.model import build_tree

    src = problems.ToeplitzInvSource(8192)
    src.dense_max = 1024  # levels 1-2 (4096 / 2048 rows) go through the FFT path
    H = build_adaptive(src, build_tree(8192, 5), 1e-6, FP64, problems.ALL_FORMATS,
                       same_blocks_per_level=True, symmetric=True)
    compare(H, golden["toeplitz_inv_8192"])


def test_toeplitz_source_narrow_plan_matches_reference(cuda, golden):
    from paper_2407_21637_b200 import FP32, problems

    H, _, _ = problems.toeplitz_config(4096, 4, 1e-2, FP32, 0)
    compare(H, golden["toeplitz_inv_4096_e2"])


def test_point_source_2d_exponential_matches_reference(cuda, golden):
    """cfg3's source (2-D exponential kernel, Morton order) at n = 4096."""
    from paper_2407_21637_b200 import problems

    H, _, _ = problems.cfg3(4096, 4, 1)
    compare(H, golden["exp2d_morton_4096"])


def test_point_source_2d_randomized_path_matches_reference(cuda, golden):
    """Same instance with the blocks forced through the tiled randomized range
    finder (what cfg3's 131072-row blocks use)."""
    import torch

    from paper_2407_21637_b200 import FP32, problems
    from paper_2407_21637_b200.construct import build_adaptive
    from paper_2407_21637_b200.model import build_tree

    P = np.random.default_rng(0).random((4096, 2))
    src = problems.PointKernelSource(P[problems.morton_order(P)], lambda r: torch.exp(-r / 0.2))
    src.dense_max, src.tile, src.dense_svd_max = 256, 512, 256
    H = build_adaptive(src, build_tree(4096, 4), 1e-4, FP32, problems.ALL_FORMATS, symmetric=True)
    compare(H, golden["exp2d_morton_4096"])


def test_point_source_1d_gaussian_matches_reference(cuda, golden):
    """cfg4's source (1-D Gaussian, sigma 0.01, cutoff tiles) at n = 8192."""
    from paper_2407_21637_b200 import problems

    H, _, _ = problems.cfg4(8192, 5, 1)
    compare(H, golden["gauss1d_8192"])
