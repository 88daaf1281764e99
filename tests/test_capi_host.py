"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/dg.h declares,
validates arguments before touching CUDA, and its 1-D tables (product path, closed-form D)
agree with closed forms and with the independent oracle tables.  No compute call needs a GPU.
"""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dg.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_2112_04167_b200 as dg

    lib = ctypes.CDLL(dg.library_path())
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    # and the Python binding carries the same names
    for s in syms:
        assert hasattr(dg, s), s


@pytest.mark.parametrize("kw", [
    dict(dim=4, N=(2, 2, 2), P=3), dict(dim=3, N=(2, 2, 2), P=0), dict(dim=3, N=(2, 2, 2), P=11),
    dict(dim=3, N=(2, 0, 2), P=3), dict(dim=3, N=(2, 2, 3), P=3, nranks=2, uid=b"\0" * 128),
    dict(dim=2, N=(2, 5), P=3, nranks=2, uid=b"\0" * 128), dict(dim=3, N=(2, 2, 2), P=3, nranks=2),
    dict(dim=3, N=(2, 2, 2), P=3, rank=2, nranks=2, uid=b"\0" * 128),
])
def test_mesh_create_rejects_invalid(kw):
    import paper_2112_04167_b200 as dg

    with pytest.raises(dg.DGError) as e:
        dg.dg_mesh_create(kw["dim"], kw["N"], (1.0, 1.0, 1.0), kw["P"], rank=kw.get("rank", 0),
                          nranks=kw.get("nranks", 1), nccl_uid=kw.get("uid"))
    assert e.value.status == dg.DG_EINVAL


@pytest.mark.parametrize("P", range(1, 11))
def test_product_tables(P):
    import oracle
    import paper_2112_04167_b200 as dg

    xi, w, D = dg.dg_gll_tables(P)
    xo, wo = oracle.gll(P)
    np.testing.assert_allclose(xi, xo, atol=2e-16 * 4)
    np.testing.assert_allclose(w, wo, atol=2e-16 * 4)
    # D against the oracle's product-formula derivatives and closed forms
    for i in range(P + 1):
        _, dl = oracle.lagrange(P, xo, xo[i])
        np.testing.assert_allclose(D[i], dl, atol=1e-12 * P * P)
    assert D[0, 0] == -P * (P + 1) / 4 and D[P, P] == P * (P + 1) / 4
    for k in range(P + 1):
        np.testing.assert_allclose(D @ xi ** k, k * xi ** max(k - 1, 0) if k else 0 * xi, atol=1e-11 * P * P)


def test_tables_reject_bad_degree():
    import paper_2112_04167_b200 as dg

    with pytest.raises(dg.DGError):
        dg.dg_gll_tables(0)
    with pytest.raises(dg.DGError):
        dg.dg_gll_tables(11)
