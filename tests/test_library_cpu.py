"""CPU-side checks: the C ABI library loads and exports every symbol that
include/pmgr.h declares; host containers mirror the reference's validation."""

import os
import re

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(REPO, "include", "pmgr.h")).read()
    return sorted(set(re.findall(r"^PMGR_API\s+[\w\s\*]+?\b(pmgr_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_api():
    syms = header_symbols()
    assert "pmgr_gmres" in syms and "pmgr_mgr_setup" in syms and "pmgr_spmv" in syms
    assert len(syms) >= 25


def test_library_exports_every_header_symbol():
    from paper_1904_05960_b200 import _lib

    L = _lib.lib()  # loading needs no GPU (static cudart)
    for name in header_symbols():
        assert hasattr(L, name), name
    assert set(_lib.SIGNATURES) == set(header_symbols())
    assert L.pmgr_version() == 1


def test_library_missing_fails_loudly(monkeypatch):
    from paper_1904_05960_b200 import _lib

    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", "/nonexistent/libpmgr.so")
    with pytest.raises(_lib.LibraryMissing):
        _lib.lib()


def test_csr_validation_messages():
    from paper_1904_05960_b200.sparse import CsrMatrix

    with pytest.raises(ValueError, match="expected nrows\\+1"):
        CsrMatrix(2, 2, [0, 1], [0], [1.0])
    with pytest.raises(ValueError, match="endpoints"):
        CsrMatrix(2, 2, [0, 1, 3], [0, 1], [1.0, 2.0])
    with pytest.raises(ValueError, match="non-decreasing"):
        CsrMatrix(2, 2, [0, 2, 1], [0], [1.0])
    with pytest.raises(ValueError, match="out of range"):
        CsrMatrix(1, 2, [0, 1], [2], [1.0])
    with pytest.raises(ValueError, match="strictly increasing"):
        CsrMatrix(1, 3, [0, 2], [1, 1], [1.0, 2.0])
    m = CsrMatrix(2, 3, [0, 2, 3], [0, 2, 1], [1.0, 0.0, 3.0])  # explicit zeros legal
    assert m.nnz == 3 and np.array_equal(m.to_dense(), [[1, 0, 0], [0, 3, 0]])
    assert np.array_equal(CsrMatrix.from_dense([[0.0, 2.0], [3.0, 0.0]]).col_indices, [1, 0])


def test_level_spec_validation():
    from paper_1904_05960_b200.mgr import MgrConfig, MgrLevelSpec
    from paper_1904_05960_b200.sparse import Field

    with pytest.raises(ValueError, match="disjoint"):
        MgrLevelSpec({Field.U}, {Field.U})
    with pytest.raises(ValueError, match="interp"):
        MgrLevelSpec({Field.U}, {Field.P}, interp="bogus")
    with pytest.raises(ValueError, match="n_max"):
        MgrLevelSpec({Field.U}, {Field.P}, n_max=-1)
    with pytest.raises(ValueError):
        MgrLevelSpec({7}, {Field.P})
    with pytest.raises(ValueError, match="f_relax_position"):
        MgrConfig(levels=(), f_relax_position="mid")
    c = MgrConfig.default_three_level()
    assert c.levels[0].n_max == 4 and c.levels[1].global_smoother == "ilu"
    spec = MgrLevelSpec({Field.U}, {Field.S, Field.P}, f_relax="amg", n_max=4).to_c()
    assert spec.f_mask == 1 and spec.c_mask == 0b110 and spec.amg_num_functions == 3 and spec.n_max == 4


def test_field_layout_restrict_downgrades_interleaving():
    from paper_1904_05960_b200.sparse import FieldLayout, Ordering

    lay = FieldLayout.interleaved_flow(4)
    sub = lay.restrict(np.array([1, 3, 5, 7]))  # pressure only: reference raises here (mgr.py:359)
    assert sub.ordering == Ordering.FIELD_BLOCKED and sub.ndofs == 4


def test_generator_layout_and_symmetry():
    from paper_1904_05960_b200 import problems

    pb = problems.make_c2(seed=2, n=4)
    assert pb.n == 3 * 125 + 2 * 64
    ci = pb.col_indices.astype(np.int64)
    for i in range(pb.n):
        row = ci[pb.row_offsets[i]:pb.row_offsets[i + 1]]
        assert np.all(np.diff(row) > 0)
    assert set(np.unique(pb.field_of)) == {0, 1, 2}
    again = problems.make_c2(seed=2, n=4)
    assert np.array_equal(pb.values, again.values) and np.array_equal(pb.rhs, again.rhs)
