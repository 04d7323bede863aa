"""Host-side checks of the C-ABI library (no GPU compute): it loads, exports every
symbol include/far.h declares, its tree tables agree with the oracle's, argument
errors are synchronous, and compute calls fail loudly without a device."""
import ctypes as C

import numpy as np
import pytest

from paper_2507_13601_b200 import far


def test_exports_every_declared_symbol():
    L = far.lib()
    names = far.declared_functions()
    assert len(names) >= 14 and "far_concat_streams" in names
    for name in names:
        assert hasattr(L, name), name


@pytest.mark.parametrize("profile", ["A30", "A100", "H100"])
def test_tree_matches_oracle(O, profile):
    F = far.Far(profile)
    lo, hi, par = F.node_table()
    olo, ohi, opar = O.nodes(profile)
    assert (lo == olo).all() and (hi == ohi).all() and (par == opar).all()
    assert F.sizes == list({"A30": (1, 2, 4)}.get(profile, (1, 2, 3, 4, 7)))
    assert F.nslices == {"A30": 4}.get(profile, 7)


def test_create_errors():
    with pytest.raises(far.FarError) as e:
        far.Far(9)
    assert e.value.status == 2
    with pytest.raises(far.FarError) as e:
        far.Far("A30", np.array([[1, 1, -1], [0, 0, 0]]))
    assert e.value.status == 3


def test_argument_errors_are_synchronous():
    F = far.Far("A30")
    L = far.lib()
    o = far.Opts(100, 0, 0)
    ms = np.zeros(4, np.int32)
    assert L.far_solve_many(F._h, None, 4, -1, C.byref(o), ms.ctypes.data_as(C.c_void_p), None, None, None) == 1
    assert L.far_solve_many(F._h, None, 4, 2000, C.byref(o), ms.ctypes.data_as(C.c_void_p), None, None, None) == 4
    bad = far.Opts(-1, 0, 0)
    assert L.far_solve_many_host(F._h, None, 0, 3, C.byref(bad), None, None, None) == 1


def test_compute_without_gpu_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    F = far.Far("A100")
    with pytest.raises(far.FarError) as e:
        F.schedule_batch(np.ones((3, 5), np.int32))
    assert e.value.status == 5
    with pytest.raises(far.FarError):
        F.solve_many_host(np.ones((2, 3, 5), np.int32))
