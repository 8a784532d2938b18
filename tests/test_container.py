"""Containers either side of the path (hodlr.py:297-363): v1 (the reference's
schema, binary64 payloads) and v2 (same keys, narrow payloads), and the
reference's own recursive HodlrMatrix driven through the drop-in.
"""

import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, golden_cases, load_case, random_hodlr
from oracle.matvec import matvec_oracle


def same_bits(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def same_matrix(H, G):
    if (H.n, H.depth) != (G.n, G.depth) or H.working_format.name != G.working_format.name:
        return False
    for (_, _, D), (_, _, E) in zip(H.leaves(), G.leaves()):
        if not same_bits(D, E):
            return False
    for a, b in zip(H.offdiag_blocks(), G.offdiag_blocks()):
        for f, g in zip(a[4:], b[4:]):
            if f.fmt.name != g.fmt.name or not same_bits(f.U, g.U) or not same_bits(f.V, g.V):
                return False
            if np.asarray(f.V).flags.f_contiguous != np.asarray(g.V).flags.f_contiguous:
                return False
    return True


def _reference():
    """The reference package: /root/reference in the build container, the
    offline install under baseline/_ref on the GPU box."""
    for p in ("/root/reference/pkg/src", os.path.join(ROOT, "baseline", "_ref")):
        if os.path.isdir(os.path.join(p, "hodlrmp")):
            if p not in sys.path:
                sys.path.insert(0, p)
            import hodlrmp.hodlr  # noqa: F401

            return sys.modules["hodlrmp"]
    pytest.skip("reference package not available")


# ---------------------------------------------------------------- CPU
@pytest.mark.parametrize("name", golden_cases())
def test_container_v2_roundtrip_bit_exact(tmp_path, name):
    """v2 stores every payload in its own format and decodes to the same bits;
    its payload is never larger than v1's and shrinks by the formats' widths."""
    from paper_2407_21637_b200 import model

    H = model.load_hodlr(os.path.join(GOLDEN, f"hodlr_{name}.npz"))
    p2 = str(tmp_path / "v2.npz")
    model.save_hodlr(H, p2, narrow=True)
    assert same_matrix(H, model.load_hodlr(p2))
    E = model.load_encoded(p2)
    assert E.encoded and E.payload_bytes() * 8 == model.storage_bits(H)
    p1 = str(tmp_path / "v1.npz")
    model.save_hodlr(H, p1)
    E1 = model.load_encoded(p1)
    assert not E1.encoded and E1.payload_bytes() >= E.payload_bytes()
    assert same_matrix(H, model.load_hodlr(p1))


def test_container_v2_all_formats_and_errors(tmp_path):
    from paper_2407_21637_b200 import model

    H = random_hodlr(600, 3, ["q52", "bf16", "fp16"], [3, 4, 5], "fp32", seed=4)
    p = str(tmp_path / "m.npz")
    model.save_hodlr(H, p, narrow=True)
    E = model.load_encoded(p)
    assert [a.dtype for a in E.blocks[0][0][0]] == [np.uint8, np.uint8]
    assert E.blocks[1][0][0][0].dtype == np.uint16 and E.blocks[2][0][1][1].dtype == np.float16
    assert E.leaf_blocks[0].dtype == np.float32
    assert same_matrix(H, model.load_hodlr(p))
    # a corrupted version tag is rejected like the reference does (hodlr.py:335-337)
    import json

    with np.load(p) as z:
        arrays = {k: z[k] for k in z.files}
    meta = json.loads(str(arrays["__meta__"][()]))
    meta["container_version"] = 7
    arrays["__meta__"] = np.array(json.dumps(meta))
    np.savez(p, **arrays)
    with pytest.raises(ValueError):
        model.load_hodlr(p)


def test_reference_container_interchange(tmp_path):
    """Files written by either package load in the other, bit for bit (v1)."""
    ref = _reference()
    from paper_2407_21637_b200 import model

    src = os.path.join(GOLDEN, "hodlr_toep1024_e2_fp32.npz")  # written by the reference's save_hodlr
    Hr = ref.hodlr.load_hodlr(src)
    H = model.load_hodlr(src)
    assert same_matrix(Hr, H)
    p = str(tmp_path / "ours.npz")
    model.save_hodlr(H, p)
    assert same_matrix(ref.hodlr.load_hodlr(p), H)
    assert ref.hodlr.storage_bits(Hr) == model.storage_bits(H)


def test_reference_hodlrmatrix_descriptor_identical():
    """The drop-in takes the reference's recursive HodlrMatrix (hodlr.py:95-135):
    its descriptor (shapes, formats, strides, values) equals the flat model's."""
    ref = _reference()
    from paper_2407_21637_b200 import linops, model

    for name in ("g2000_fp32", "toep1024_e4_fp64", "depth0_fp32"):
        src = os.path.join(GOLDEN, f"hodlr_{name}.npz")
        dr, df = linops.descriptor(ref.hodlr.load_hodlr(src)), linops.descriptor(model.load_hodlr(src))
        assert (dr.desc.n, dr.desc.depth, dr.desc.leaf_fmt) == (df.desc.n, df.desc.depth, df.desc.leaf_fmt)
        nf = 2 * (2 ** dr.desc.depth - 1)
        for i in range(nf):
            a, b = dr.desc.factors[i], df.desc.factors[i]
            assert (a.fmt, a.rank, a.rows, a.cols) == (b.fmt, b.rank, b.rows, b.cols)
            assert (a.u_rs, a.u_cs, a.v_rs, a.v_cs) == (b.u_rs, b.u_cs, b.v_rs, b.v_cs)
            for pa, pb, rows, rs, cs in ((a.U, b.U, a.rows, a.u_rs, a.u_cs), (a.V, b.V, a.cols, a.v_rs, a.v_cs)):
                for r, c in ((0, 0), (rows - 1, a.rank - 1)):
                    if a.rank:
                        assert pa[r * rs + c * cs] == pb[r * rs + c * cs]
        nl = 2 ** dr.desc.depth
        assert [dr.desc.leaf_bounds[i] for i in range(nl + 1)] == [df.desc.leaf_bounds[i] for i in range(nl + 1)]


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("name", ["g2000_fp32", "toep1024_e4_fp64", "g600_bf16"])
def test_gpu_loader_from_narrow_container(cuda, tmp_path, name):
    """from_container on a v2 file packs the narrow payloads directly: the
    packed factors and leaves unpack to the original bits and the matvec equals
    the one of the operator built from the binary64 model."""
    from paper_2407_21637_b200 import linops, model

    src = os.path.join(GOLDEN, ("nwhodlr_" if name == "g600_bf16" else "hodlr_") + name + ".npz")
    H = model.load_hodlr(src)
    p = str(tmp_path / "v2.npz")
    model.save_hodlr(H, p, narrow=True)
    op = linops.HodlrOperator.from_container(p, device=0)
    for idx, blk in enumerate(H.offdiag_blocks()):
        for lo, f in enumerate(blk[4:]):
            U, V = op.unpack_factor(2 * idx + lo, f.rows, f.cols, f.rank)
            assert same_bits(U, f.U) and same_bits(V, np.ascontiguousarray(f.V))
    for i, (a, b), D in H.leaves():
        assert same_bits(op.unpack_leaf(i, b - a), D)
    w = H.working_format if H.working_format.name != "bf16" else None
    x = np.random.default_rng(1).standard_normal((H.n, 2))
    ref_op = linops.HodlrOperator(H, device=0)
    assert same_bits(op.matvec_host(x, w), ref_op.matvec_host(x, w))
    assert op.matrix_bytes * 8 == model.storage_bits(H)
    # v1 files take the binary64 route to the same packed matrix
    op1 = linops.HodlrOperator.from_container(src, device=0)
    assert same_bits(op1.matvec_host(x, w), ref_op.matvec_host(x, w))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["g2000_fp32", "toep1024_e4_fp64", "rand96_fp32"])
def test_gpu_reference_hodlrmatrix_through_dropin(cuda, name):
    """linops.matvec(H_ref, x) with H_ref the reference's own object equals the
    flat model's result bit for bit and the oracle within tolerance."""
    ref = _reference()
    from paper_2407_21637_b200 import linops

    Hr = ref.hodlr.load_hodlr(os.path.join(GOLDEN, f"hodlr_{name}.npz"))
    H, vec, _ = load_case(name)
    x = vec["x"]
    b_ref_obj = linops.matvec(Hr, x)
    assert same_bits(b_ref_obj, linops.matvec(H, x))
    want = matvec_oracle(H, x)
    tol = 1e-12 if H.working_format.name == "fp64" else 1e-5
    assert np.linalg.norm(b_ref_obj - want) <= tol * np.linalg.norm(want)
