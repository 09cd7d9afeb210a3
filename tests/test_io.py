"""Instance / candidate files (csrc/io.cpp) against the reference's io.hpp (tests/unit/test_io.cpp).

* our writer produces the SAME BYTES as femsched::save_instance (oracle/_ref) on the acceptance /
  unit tuples, the benchmark mesh forms and a non-affine instance;
* our reader loads reference-written files bit-exactly, and the reference loads ours;
* the committed fixture tests/golden/instance_laplace_2d_p2.txt (written by the reference,
  tests/golden/make_golden.py) loads without the reference and reproduces the golden y;
* malformed documents are rejected with context (test_io.cpp:126-152);
* candidate files round-trip (test_io.cpp:104-124)."""
import os

import numpy as np
import pytest

import paper_2506_17471_b200 as fg
from paper_2506_17471_b200 import abi
from tests.helpers import ACCEPTANCE, UNIT, preset_problem

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def same_problem(a, b):
    assert a.signature.dim == b.signature.dim and a.signature.quad_points == b.signature.quad_points
    assert [(s.dofs, s.deriv_terms) for s in a.signature.scalar_spaces] == \
        [(s.dofs, s.deriv_terms) for s in b.signature.scalar_spaces]
    assert [(v.dofs, v.deriv_terms, list(v.components)) for v in a.signature.vector_spaces] == \
        [(v.dofs, v.deriv_terms, list(v.components)) for v in b.signature.vector_spaces]
    ta, tb = a.tabulations, b.tabulations
    for x, y in zip(list(ta.scalar_phi) + list(ta.vector_phi) + [ta.psi, ta.weights],
                    list(tb.scalar_phi) + list(tb.vector_phi) + [tb.psi, tb.weights]):
        assert np.array_equal(np.asarray(x).view(np.uint64), np.asarray(y).view(np.uint64))  # bit-exact
    ca, cb = a.connectivity, b.connectivity
    for x, y in zip(ca.scalar_maps + ca.vector_maps + [ca.test_map], cb.scalar_maps + cb.vector_maps + [cb.test_map]):
        assert np.array_equal(x.indices, y.indices) and x.global_count == y.global_count
    if a.signature.affine_geometry:
        assert np.array_equal(ca.coord_map.indices, cb.coord_map.indices)
        assert np.array_equal(np.asarray(ca.coords).view(np.uint64), np.asarray(cb.coords).view(np.uint64))
    for x, y in zip(list(a.scalar_inputs) + list(a.vector_inputs), list(b.scalar_inputs) + list(b.vector_inputs)):
        assert np.array_equal(np.asarray(x).view(np.uint64), np.asarray(y).view(np.uint64))
    assert list(a.map.nodes) == list(b.map.nodes) and list(a.map.outputs) == list(b.map.outputs)
    assert a.output_size == b.output_size


def non_affine_problem():
    """non_affine_sig / non_affine_map of test_io.cpp:10-42 (coordinates as a vector trial space)."""
    sig = fg.FormSignature(dim=2, scalar_spaces=[fg.ScalarSpace(3, 2)], vector_spaces=[fg.VectorSpace(3, 4, [0, 0, 1, 1])],
                           test_dofs=3, test_deriv_terms=2, quad_points=4, coord_dofs=0, affine_geometry=False,
                           coordinate_space=0)
    m = fg.PointwiseMap()
    g = lambda r, c: m.vector_deriv(0, r * 2 + c)  # noqa: E731
    det = m.add(m.mul(g(0, 0), g(1, 1)), m.mul(m.constant(-1.0), m.mul(g(0, 1), g(1, 0))))
    wdet = m.mul(m.weight(), det)
    for r in range(2):
        terms = []
        for c in range(2):
            metric = m.add(m.mul(g(0, r), g(0, c)), m.mul(g(1, r), g(1, c)))
            terms.append(m.mul(metric, m.scalar_deriv(0, c)))
        m.add_output(m.mul(wdet, m.sum(terms)))
    return fg.make_problem(sig, m, 5, 17)


CASES = [(op, d, p, q, 16, 7) for op, d, p, q in ACCEPTANCE] + list(UNIT)


@pytest.mark.parametrize("case", CASES[:8], ids=str)
def test_writer_matches_reference_bytes(tmp_path, oracle, case):
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    p = preset_problem(*case)
    ours, theirs = tmp_path / "ours.txt", tmp_path / "ref.txt"
    fg.save_instance(p, ours)
    oracle.ref_save_instance(p, theirs)
    assert ours.read_bytes() == theirs.read_bytes()
    assert ours.read_text().startswith("format_version: 1\n")


@pytest.mark.parametrize("form,dim,deg,Q,n", [("laplace", 3, 2, 4, 2), ("elasticity", 3, 2, 4, 2),
                                              ("hyperelastic", 3, 2, 14, 1), ("advection", 3, 3, 24, 1)])
def test_mesh_forms_round_trip_both_ways(tmp_path, oracle, form, dim, deg, Q, n):
    p = fg.mesh_problem(form, dim, deg, Q, n)
    f = tmp_path / "inst.txt"
    fg.save_instance(p, f)
    q = fg.load_instance(f)
    same_problem(p, q)
    if oracle.ref_available():
        same_problem(p, oracle.ref_load_instance(f))  # the reference reads our file
        g = tmp_path / "ref.txt"
        oracle.ref_save_instance(p, g)
        same_problem(p, fg.load_instance(g))  # we read the reference's file
        assert f.read_bytes() == g.read_bytes()
    # a second round trip reproduces the same document bytes (test_io.cpp:57-63)
    f2 = tmp_path / "inst2.txt"
    fg.save_instance(q, f2)
    assert f2.read_bytes() == f.read_bytes()
    np.testing.assert_array_equal(oracle.reference_action(q), oracle.reference_action(p))


def test_non_affine_round_trip(tmp_path, oracle):
    p = non_affine_problem()
    f = tmp_path / "na.txt"
    fg.save_instance(p, f)
    q = fg.load_instance(f)
    same_problem(p, q)
    assert np.array_equal(oracle.reference_action(q), oracle.reference_action(p))
    if oracle.ref_available():
        g = tmp_path / "na_ref.txt"
        oracle.ref_save_instance(p, g)
        assert g.read_bytes() == f.read_bytes()


def test_golden_fixture_loads_without_reference(oracle):
    p = fg.load_instance(os.path.join(GOLDEN, "instance_laplace_2d_p2.txt"))
    gold = np.load(os.path.join(GOLDEN, "reference_outputs.npz"))
    y = oracle.reference_action(p)
    assert np.array_equal(y, gold["y:laplace|2|2|6|16|7"])


@pytest.mark.parametrize("text,match", [
    ("format_version: 9\n", "unsupported format version"),
    ("format_version: 1\nnot_a_signature: 2\n", "signature_begin"),
    ("format_version: 1\nsignature_begin:\ndim: 2\n", "unexpected end of input"),
])
def test_malformed_documents_are_rejected(tmp_path, text, match):
    f = tmp_path / "bad.txt"
    f.write_text(text)
    with pytest.raises(ValueError, match=match):
        fg.load_instance(f)


def test_truncated_document_is_rejected(tmp_path):
    p = preset_problem("mass", 2, 1, 2, 2, 3)
    f = tmp_path / "full.txt"
    fg.save_instance(p, f)
    text = f.read_text()
    g = tmp_path / "trunc.txt"
    g.write_text(text[: len(text) // 2])
    with pytest.raises(ValueError):
        fg.load_instance(g)


def test_candidate_files_round_trip(tmp_path):
    sig = fg.preset_signature("laplace", 2, 2, 6)
    t = fg.TilingParams.untiled(sig, 64, 2)
    t.quad_tile, t.eval_row_tile, t.quad_col_tile = 3, 3, 3
    f = tmp_path / "mlt.txt"
    fg.save_schedule(t, f)
    assert f.read_text() == ("format_version: 1\nkind: mlt\nquad_tile: 3\neval_row_tile: 3\neval_col_tiles_scalar: 6\n"
                             "eval_col_tiles_vector:\nquad_row_tile: 6\nquad_col_tile: 3\ncells_per_group: 64\n"
                             "lanes_per_cell: 2\n")
    q = fg.load_schedule(f)
    assert q.order_key() == t.order_key() and q.kind == abi.MLT
    f2 = tmp_path / "scpt.txt"
    fg.save_schedule(fg.TilingParams(kind=abi.SCPT), f2)
    assert f2.read_text() == "format_version: 1\nkind: scpt\n"
    assert fg.load_schedule(f2).kind == abi.SCPT
    d = fg.TilingParams.dmma(cells_per_group=16, quad_tile=8, eval_row_tile=2, block_cells=128)
    f3 = tmp_path / "dmma.txt"
    fg.save_schedule(d, f3)
    e = fg.load_schedule(f3)
    assert (e.kind, e.cells_per_group, e.quad_tile, e.eval_row_tile, e.block_cells) == (abi.DMMA, 16, 8, 2, 128)
    g = tmp_path / "warp.txt"
    g.write_text("format_version: 1\nkind: warp\n")
    with pytest.raises(ValueError, match="unknown kind"):
        fg.load_schedule(g)


def test_candidate_files_keep_b200_knobs(tmp_path):
    """strict (bitwise) SCPT, register targets, kernel variants and zeroing decisions must
    survive a save/load round trip; an MLT candidate with the strict flag keeps it too."""
    cases = [fg.TilingParams.scpt(strict=True),
             fg.TilingParams.scpt(reg_target=200, min_blocks=3),
             fg.TilingParams.scpt(scatter=abi.SCATTER_MACRO, group_cells=6, block_cells=32, stage_smem=3,
                                  qmopt=16, reg_target=232, fused_zero=True, zero_slabs=4)]
    sig = fg.preset_signature("laplace", 2, 2, 6)
    m = fg.TilingParams.untiled(sig, 64, 2)
    m.strict = True
    cases.append(m)
    for i, t in enumerate(cases):
        f = tmp_path / ("c%d.txt" % i)
        fg.save_schedule(t, f, n_scalar=len(sig.scalar_spaces))
        q = fg.load_schedule(f)
        assert q.to_c().reserved[:] == t.to_c().reserved[:], (i, f.read_text())
        assert (q.kind, q.scatter, q.group_cells, q.block_cells, q.strict) == (t.kind, t.scatter, t.group_cells,
                                                                               t.block_cells, t.strict)
    assert "b200_mlt" in (tmp_path / "c3.txt").read_text()


@pytest.mark.parametrize("name", ["mesh_helmholtz_coef_2d_p3", "mesh_elasticity_3d_p2"])
def test_reference_written_mesh_instances_load_to_the_golden_y(oracle, name):
    """Mesh instance files written by the reference (make_golden.py): our reader + the C oracle
    reproduce the reference's own output bit for bit (no reference needed on this host)."""
    p = fg.load_instance(os.path.join(GOLDEN, name + ".txt"))
    gold = np.load(os.path.join(GOLDEN, "mesh_instance_outputs.npz"))["y:" + name]
    assert np.array_equal(oracle.reference_action(p), gold)
