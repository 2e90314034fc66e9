"""Matrix Market IO (reference sparse.py:484-502) and solve_file
(SPEC.md:589-597): round trips on the host, the solve on the GPU."""

import json
import os

import numpy as np
import pytest

from paper_1904_05960_b200 import problems, sparse


def export(tmp_path, pb):
    A = sparse.CsrMatrix(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
    sparse.write_matrix_market(tmp_path / "A.mtx", A)
    sparse.write_vector(tmp_path / "b.mtx", pb.rhs)
    from paper_1904_05960_b200 import solve

    solve.write_layout(tmp_path / "L.json", pb.field_of, pb.entity_of)
    return A


def test_matrix_market_round_trip_is_bitwise(tmp_path):
    pb = problems.make_c2(seed=3, n=3)
    A = export(tmp_path, pb)
    B = sparse.read_matrix_market(tmp_path / "A.mtx")
    assert np.array_equal(A.row_offsets, B.row_offsets)
    assert np.array_equal(A.col_indices, B.col_indices)
    assert np.array_equal(A.values, B.values)
    assert np.array_equal(sparse.read_vector(tmp_path / "b.mtx"), pb.rhs)
    from paper_1904_05960_b200 import solve

    lay = solve.read_layout(tmp_path / "L.json")
    assert np.array_equal(lay.field_of, pb.field_of) and np.array_equal(lay.entity_of, pb.entity_of)


def test_explicit_zeros_survive(tmp_path):
    A = sparse.CsrMatrix.from_dense(np.array([[2.0, 0.0], [0.0, 1.0]]), keep_zeros=True)
    sparse.write_matrix_market(tmp_path / "z.mtx", A)
    assert sparse.read_matrix_market(tmp_path / "z.mtx").nnz == 4


def test_solve_file_input_errors(tmp_path):
    from paper_1904_05960_b200 import solve

    pb = problems.make_c1(seed=1, n=3)
    export(tmp_path, pb)
    solve.write_layout(tmp_path / "short.json", pb.field_of[:-1], pb.entity_of[:-1])
    with pytest.raises(ValueError, match="layout covers"):
        solve.solve_file(tmp_path / "A.mtx", tmp_path / "b.mtx", tmp_path / "short.json")
    sparse.write_vector(tmp_path / "short.mtx", pb.rhs[:-2])
    with pytest.raises(ValueError, match="rhs length"):
        solve.solve_file(tmp_path / "A.mtx", tmp_path / "short.mtx", tmp_path / "L.json")
    with open(tmp_path / "bad.json", "w") as f:
        json.dump({"field_of": ["u", "q"]}, f)
    with pytest.raises(ValueError, match="unknown field tag"):
        solve.read_layout(tmp_path / "bad.json")
    with pytest.raises(OSError):
        solve.solve_file(tmp_path / "missing.mtx", tmp_path / "b.mtx", tmp_path / "L.json")
    # the CLI turns input errors into exit code 2
    assert solve.main(["--matrix", str(tmp_path / "A.mtx"), "--rhs", str(tmp_path / "short.mtx"),
                       "--layout", str(tmp_path / "L.json")]) == 2


@pytest.mark.gpu
def test_solve_file_matches_in_process(tmp_path):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1904_05960_b200 import amg, krylov, mgr, solve

    pb = problems.make_c2(seed=5, n=8)
    A = export(tmp_path, pb)
    with open(tmp_path / "S.json", "w") as f:
        json.dump({"gmres": {"restart": 100, "max_iters": 500}}, f)
    rep = solve.solve_file(tmp_path / "A.mtx", tmp_path / "b.mtx", tmp_path / "L.json", str(tmp_path / "S.json"))
    F = sparse.Field
    cfg = mgr.MgrConfig(levels=(mgr.MgrLevelSpec({F.U}, {F.S, F.P}, f_relax="amg", n_max=4),
                                mgr.MgrLevelSpec({F.S}, {F.P}, f_relax="jacobi")),
                        amg_f_relax=amg.AmgConfig(strength_threshold=0.5, num_functions=3, npartitions=10 ** 9),
                        amg_terminal=amg.AmgConfig(strength_threshold=0.25, npartitions=10 ** 9))
    h = mgr.mgr_setup(A, sparse.FieldLayout(pb.field_of, pb.entity_of), cfg)
    x, st = krylov.gmres(A, h.apply, pb.rhs, cfg=krylov.GmresConfig(restart=100, max_iters=500))
    assert rep["converged"] and rep["iterations"] == st.iterations
    assert np.array_equal(rep["x"], x)
    assert rep["true_residual"] <= 1e-6 * rep["rhs_norm"] * (1 + 1e-9)
    # the CLI writes the solution
    assert solve.main(["--matrix", str(tmp_path / "A.mtx"), "--rhs", str(tmp_path / "b.mtx"), "--layout",
                       str(tmp_path / "L.json"), "--solver", str(tmp_path / "S.json"), "--solution",
                       str(tmp_path / "x.mtx")]) == 0
    assert np.array_equal(sparse.read_vector(tmp_path / "x.mtx"), x)


@pytest.mark.gpu
def test_solve_file_identity_one_iteration(tmp_path):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1904_05960_b200 import solve

    n = 50
    sparse.write_matrix_market(tmp_path / "I.mtx", sparse.CsrMatrix.identity(n))
    sparse.write_vector(tmp_path / "b.mtx", np.linspace(1.0, 2.0, n))
    solve.write_layout(tmp_path / "L.json", [2] * n, range(n))
    rep = solve.solve_file(tmp_path / "I.mtx", tmp_path / "b.mtx", tmp_path / "L.json")
    assert rep["converged"] and rep["iterations"] == 1
