"""The C-ABI library loads and exports every symbol include/gsr.h declares, and its
host-side argument validation works without a GPU (-m "not gpu")."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gsr.h")


@pytest.fixture(scope="module")
def libs():
    from paper_2408_12677_b200 import _build
    _build.build()
    from paper_2408_12677_b200 import gsr
    return gsr.load(False), gsr.load(True)


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gs_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_five_calls():
    names = declared_functions()
    for fn in ("gs_project", "gs_bin_tiles", "gs_render_fwd", "gs_render_bwd", "gs_adam_step"):
        assert fn in names


def test_every_declared_symbol_is_exported(libs):
    for lib in libs:
        for fn in declared_functions():
            assert hasattr(lib.lib, fn), f"{lib.path} does not export {fn}"


def test_versions_and_flags(libs):
    fast, exact = libs
    assert fast.lib.gs_version() == 2 and exact.lib.gs_version() == 2
    assert fast.lib.gs_exact_exp() == 0 and exact.lib.gs_exact_exp() == 1
    assert fast.launch_count() >= 0


def test_host_validation_without_gpu(libs):
    from paper_2408_12677_b200 import gsr
    import scenegen
    lib = libs[0]
    cam = gsr.camera(scenegen.identity_camera(64, 48, 60.0, 32.0, 24.0))
    proj = gsr.GsProj(None, None, None, None)
    # NULL camera / bad scene / misalignment are rejected before any CUDA call
    st = lib.lib.gs_project(None, C.byref(gsr.scene_desc(4, 4, 0)), None, proj, None)
    assert st == gsr.GS_ERR_ARG and "camera" in lib.last_error()
    st = lib.lib.gs_project(C.byref(cam), C.byref(gsr.scene_desc(4, 4, 7)), None, proj, None)
    assert st == gsr.GS_ERR_ARG
    st = lib.lib.gs_project(C.byref(cam), C.byref(gsr.scene_desc(5, 6, 0)), None, proj, None)
    assert st == gsr.GS_ERR_ALIGN
    st = lib.lib.gs_project(C.byref(cam), C.byref(gsr.scene_desc(4, 4, 0)), C.c_void_p(0x1003), proj, None)
    assert st == gsr.GS_ERR_ALIGN
    # P == 0 is a valid no-op projection; Adam on P == 0 is GS_ERR_EMPTY (SPEC NoGaussians)
    assert lib.lib.gs_project(C.byref(cam), C.byref(gsr.scene_desc(0, 0, 0)), None, proj, None) == gsr.GS_OK
    lr = (C.c_float * 14)(*([1e-3] * 14))
    st = lib.lib.gs_adam_step(C.byref(gsr.scene_desc(0, 0, 0)), None, None, None, None, lr, 0.9, 0.999, 1e-15, 1,
                              1, None)
    assert st == gsr.GS_ERR_EMPTY
    big = gsr.camera(scenegen.identity_camera(8192, 4096, 60.0, 32.0, 24.0))  # 131072 tiles > 65536
    assert lib.lib.gs_project(C.byref(big), C.byref(gsr.scene_desc(0, 0, 0)), None, proj, None) == gsr.GS_ERR_ARG


def test_workspace_queries(libs):
    from paper_2408_12677_b200 import gsr
    import scenegen
    lib = libs[0]
    cam = gsr.camera(scenegen.identity_camera(1752, 1168, 1100.0, 875.5, 583.5))
    a = lib.bin_tiles_workspace(cam, 1_000_000, 8_000_000)
    b = lib.bin_tiles_workspace(cam, 1_000_000, 16_000_000)
    assert 0 < a < b
    assert lib.render_bwd_workspace(gsr.scene_desc(1000, 1000, 3)) == 1000 * 12 * 4


def test_product_package_does_not_import_oracle():
    import subprocess
    import sys
    code = ("import sys; import paper_2408_12677_b200.pipeline, paper_2408_12677_b200.gsr; "
            "bad=[m for m in sys.modules if m.startswith('oracle')]; assert not bad, bad")
    subprocess.check_call([sys.executable, "-c", code], cwd=ROOT)
    for f in os.listdir(os.path.join(ROOT, "paper_2408_12677_b200")):
        if f.endswith(".py"):
            src = open(os.path.join(ROOT, "paper_2408_12677_b200", f)).read()
            assert "oracle" not in re.sub(r'""".*?"""|#.*', "", src, flags=re.S), f


def test_state_mismatch_detected_on_host(libs):
    """GS_ERR_STATE (SPEC.md:349 StateMismatch) is decided on the host before any launch:
    a never-written state, another image size, or buffers that are not the forward's."""
    from paper_2408_12677_b200 import gsr
    import scenegen
    lib = libs[0]
    cam = gsr.camera(scenegen.identity_camera(64, 48, 60.0, 32.0, 24.0))
    sc = gsr.scene_desc(4, 4, 0)
    A = [C.c_void_p(0x10000 * (k + 1)) for k in range(8)]  # fake, aligned, never dereferenced
    proj = gsr.GsProj(A[0], A[1], A[2], A[3])
    st = gsr.GsFwdState()  # id 0: never written by a forward
    opts = gsr.bwd_opts(fwd=st)

    def call(o):
        return lib.lib.gs_render_bwd_screen(C.byref(cam), C.byref(sc), proj, A[4], A[5], None, A[6], A[7], A[4],
                                            None, None, A[5], C.byref(o), None)
    assert call(opts) == gsr.GS_ERR_STATE and "never written" in lib.last_error()
    st.id, st.width, st.height = 12345, 64, 40
    assert call(opts) == gsr.GS_ERR_STATE and "size" in lib.last_error()
    st.height = 48
    st.rec, st.sorted_ids, st.tile_ranges, st.T_final, st.n_contrib = 0x10000, 0x50000, 0x60000, 0x70000, 0x80000
    assert call(opts) == gsr.GS_ERR_STATE and "n_contrib" in lib.last_error()  # no forward wrote A[7]: stale
    st.sorted_ids = 0x90000
    assert call(opts) == gsr.GS_ERR_STATE and "sorted_ids" in lib.last_error()
    # the deterministic workspace is validated too; the K13 port rejects the mode
    o2 = gsr.GsBwdOpts()
    o2.det_ws, o2.det_keys = 0x10004, 16
    assert call(o2) == gsr.GS_ERR_ALIGN
    o2.det_ws = 0x10000
    st2 = lib.lib.gs_naive_render_bwd_screen(C.byref(cam), C.byref(sc), proj, A[4], A[5], A[6], A[7], A[4], None,
                                             A[5], C.byref(o2), None)
    assert st2 == gsr.GS_ERR_ARG and "deterministic" in lib.last_error()


def test_render_rows_switch_host_only(libs):
    """gs_set_render_rows / gs_render_rows: a host-side, process-wide switch (no GPU)."""
    for lib in libs:
        was = lib.render_rows()
        try:
            for v in (1, 0, 7):
                lib.set_render_rows(v)
                assert lib.render_rows() == bool(v)
        finally:
            lib.set_render_rows(was)


def test_project_bwd_views_adam_dev_host_validation(libs):
    """gs_project_bwd_views_adam_dev rejects bad arguments before any CUDA call."""
    from paper_2408_12677_b200 import gsr
    import scenegen
    lib = libs[0]
    sc = gsr.scene_desc(4, 4, 0)
    lr = (C.c_float * 14)(*([1e-3] * 14))
    fn = lib.lib.gs_project_bwd_views_adam_dev
    # n_views < 1
    st = fn(0, None, C.byref(sc), None, None, None, None, 0, None, None, lr, 0.9, 0.999, 1e-15, None, None, None)
    assert st == gsr.GS_ERR_ARG and "gs_project_bwd_views_adam_dev" in lib.last_error()
    cam = (gsr.GsCamera * 1)(gsr.camera(scenegen.identity_camera(64, 48, 60.0, 32.0, 24.0)))
    fl = (C.c_void_p * 1)(C.c_void_p(0x1000))
    sg = (C.c_void_p * 1)(C.c_void_p(0x1000))
    step = C.c_void_p(0x1000)
    # step_dev NULL; beta outside [0, 1)
    st = fn(1, cam, C.byref(sc), None, fl, sg, None, 0, None, None, lr, 0.9, 0.999, 1e-15, None, None, None)
    assert st == gsr.GS_ERR_ARG
    st = fn(1, cam, C.byref(sc), None, fl, sg, None, 0, None, None, lr, 1.5, 0.999, 1e-15, step, None, None)
    assert st == gsr.GS_ERR_ARG
