"""Host-only checks of the C-ABI library: it loads, exports every symbol include/taccel.h declares,
and sizes a workspace (template preparation runs on the host; no compute calls without a GPU)."""
import ctypes

import pytest

from paper_2504_12908_b200 import scenes as S
from paper_2504_12908_b200 import taccel as T
from paper_2504_12908_b200.build import build


@pytest.fixture(scope="module")
def lib():
    build()
    return T.load()


def test_exports_every_header_symbol(lib):
    names = T.header_symbols()
    assert "tac_step" in names and "tac_debug_eval" in names and len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_workspace_size(lib, name):
    sc = S.make_scene(name)
    one = T.workspace_size(sc, 1)
    many = T.workspace_size(sc, 8)
    assert one > 0 and many > 4 * one


def test_validation_errors(lib):
    sc = S.make_scene("C1")
    sc.soft[0].rest_pos = sc.soft[0].rest_pos.copy()
    t = sc.soft[0].tets[0]
    sc.soft[0].rest_pos[t[3]] = sc.soft[0].rest_pos[t[0]]      # collapse a tet
    with pytest.raises(T.TaccelError) as e:
        T.workspace_size(sc, 1)
    assert e.value.code == 2 and "degenerate tet" in str(e.value)
    sc = S.make_scene("C1")
    sc.config.dt = -1.0
    with pytest.raises(T.TaccelError) as e:
        T.workspace_size(sc, 1)
    assert e.value.code == 1


def test_no_cpu_fallback_without_cuda(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        T.Batch(S.make_scene("C1"), 1)
