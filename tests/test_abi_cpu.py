"""Host-side checks of the boundary (no GPU): the C-ABI library loads, exports every symbol that
include/gs.h declares, and the ctypes struct layouts match the header."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gs.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gs_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def gslib():
    from paper_2311_11700_b200 import build
    build.build()
    import paper_2311_11700_b200 as g
    return g


def test_header_declares_the_survey_boundary():
    fns = declared_functions()
    for name in ("gs_project", "gs_bin_sort", "gs_render_fwd", "gs_render_bwd", "gs_pose_grad", "gs_densify_prune",
                 "gs_loss_l1", "gs_adam_step", "gs_pose_step", "gs_workspace_bytes", "gs_status_string"):
        assert name in fns


def test_library_exports_every_declared_symbol(gslib):
    lib = ctypes.CDLL(gslib.LIB_PATH)
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing
    assert set(declared_functions()) == set(gslib.EXPORTED)


def test_struct_layouts(gslib):
    assert ctypes.sizeof(gslib.gs_ws) == 1024
    assert ctypes.sizeof(gslib.gs_camera) == 4 * 4 + 2 * 4 + 4 + 12 + 4
    assert ctypes.sizeof(gslib.gs_densify_cfg) == 4 * 8 + 8 + 2 * 4 + 4 + 4   # + rows, padded to 8


def test_workspace_sizing_and_argument_errors(gslib):
    lib = gslib._lib
    a = lib.gs_workspace_bytes(1000, 10_000, 64, 48)
    b = lib.gs_workspace_bytes(2000, 10_000, 64, 48)
    c = lib.gs_workspace_bytes(1000, 20_000, 64, 48)
    assert 0 < a < b and a < c
    assert lib.gs_workspace_bytes(-1, 0, 64, 48) == 0
    assert lib.gs_status_string(gslib.GS_ERR_STALE) == b"GS_ERR_STALE"
    # host-side argument checks happen before any launch (no GPU needed)
    ws = gslib.gs_ws()
    assert lib.gs_ws_init(ctypes.byref(ws), None, 0, 10, 10, 64, 48) == gslib.GS_ERR_INVALID_ARG
    assert lib.gs_ws_init(ctypes.byref(ws), ctypes.c_void_p(256), 10, 10, 10, 64, 48) == gslib.GS_ERR_INVALID_ARG
    cam = gslib.gs_camera()
    assert lib.gs_project(None, 0, 0, None, None, ctypes.byref(cam), ctypes.byref(ws), None) == \
        gslib.GS_ERR_INVALID_ARG
    assert lib.gs_ws_launch_count(ctypes.byref(ws)) == -1


def test_product_does_not_import_oracle():
    """The product package never imports, links or executes anything under oracle/."""
    pkg = os.path.join(ROOT, "paper_2311_11700_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "liboracle" not in txt, f


def test_flag_and_status_values_match_the_header(gslib):
    """Every GS_FLAG_* / GS_DENSIFY_* / GS_OK / GS_ERR_* value the binding exports equals the header's."""
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    vals = {name: int(v) for name, v in re.findall(r"\b((?:GS_FLAG|GS_DENSIFY|GS_ERR|GS_OK)[A-Z0-9_]*)\s*=\s*(\d+)u?", src)}
    assert len(vals) >= 10
    for name, v in vals.items():
        if hasattr(gslib, name):
            assert getattr(gslib, name) == v, name
    for name in ("GS_FLAG_BWD_SCREEN_ONLY", "GS_FLAG_BWD_CHAIN_ONLY", "GS_FLAG_GRAD_ASSIGN", "GS_FLAG_NO_HOST_SYNC"):
        assert name in vals and getattr(gslib, name) == vals[name]
    flags = [v for k, v in vals.items() if k.startswith("GS_FLAG")]
    assert all(f & (f - 1) == 0 for f in flags) and len(set(flags)) == len(flags)   # distinct single bits
