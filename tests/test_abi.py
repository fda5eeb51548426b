"""CPU-side checks of the C ABI: libtvprox.so builds for sm_100a, loads, exports every
symbol include/tvprox.h declares, and rejects bad arguments before any launch."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tvprox.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2204_03643_b200 import build, _lib
    build.build()
    return _lib.load()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b([a-z_0-9]+)\s*\(", src)
    skip = {"if", "defined", "sizeof"}
    return sorted({n for n in names if n.startswith(("tv1d_", "tv2d_", "tvp_")) and n not in skip})


def test_header_functions_exported(lib):
    from paper_2204_03643_b200 import _lib
    decl = declared_functions()
    assert set(decl) == set(_lib.EXPORTS), (decl, _lib.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    syms = {line.split()[-1] for line in out.splitlines() if line.strip()}
    for name in decl:
        assert name in syms, name
        assert hasattr(lib, name)


def test_sm100a_cubin_present():
    from paper_2204_03643_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_size_queries(lib):
    assert lib.tv1d_mask_words(1) == 0
    assert lib.tv1d_mask_words(2) == 1
    assert lib.tv1d_mask_words(17) == 1
    assert lib.tv1d_mask_words(18) == 2
    assert lib.tv1d_mask_words(1024) == 64
    assert lib.tvp_max_line(0) >= 1024
    assert lib.tvp_max_line_1d(0) == 65536 and lib.tvp_max_line_1d(1) == 65536
    # saved = K * planes * (H * ceil((W-1)/16) + W * ceil((H-1)/16)) words
    assert lib.tv2d_saved_bytes(2, 3, 56, 56, 4) == 4 * 6 * (56 * 4 + 56 * 4) * 4
    assert lib.tv2d_workspace_bytes(0, 2, 3, 56, 56, 4) >= 3 * 6 * 56 * 56 * 4
    assert lib.tv1d_bwd_workspace_bytes(0, 100, 0) >= 400
    assert lib.tv1d_bwd_workspace_bytes(0, 100, 1) == 0
    assert lib.tvp_version() >= 100
    assert lib.tvp_max_line(1) >= 1024


def test_invalid_arguments_rejected_before_launch(lib):
    from paper_2204_03643_b200 import _lib
    fake = ctypes.c_void_p(16)    # never dereferenced: validation fails first
    E = _lib.TVP_EINVAL
    assert lib.tv1d_prox_fwd(0, fake, fake, 4, 0, 4, None, 0, 0.5, None, None, None) == E      # n < 1
    assert lib.tv1d_prox_fwd(0, fake, fake, 4, 8, 4, None, 0, 0.5, None, None, None) == E      # stride < n
    assert lib.tv1d_prox_fwd(0, fake, fake, -1, 8, 8, None, 0, 0.5, None, None, None) == E     # batch < 0
    assert lib.tv1d_prox_fwd(0, fake, fake, 4, 8, 8, None, 0, -0.5, None, None, None) == E     # lam < 0
    assert lib.tv1d_prox_fwd(0, fake, fake, 4, 8, 8, None, 0, float("nan"), None, None, None) == E
    assert lib.tv1d_prox_fwd(0, fake, fake, 4, 8, 8, None, 1, 0.0, None, None, None) == E      # NULL lam
    assert lib.tv1d_prox_fwd(0, fake, fake, 4, 8, 8, fake, 3, 0.0, None, None, None) == E      # 2D mode
    assert lib.tv1d_prox_fwd(7, fake, fake, 4, 8, 8, None, 0, 0.5, None, None, None) == E      # dtype
    assert lib.tv1d_prox_fwd(0, None, fake, 4, 8, 8, None, 0, 0.5, None, None, None) == E      # NULL y
    assert lib.tv1d_prox_fwd(0, fake, fake, 0, 8, 8, None, 0, 0.5, None, None, None) == _lib.TVP_OK  # empty
    assert lib.tv1d_prox_fwd(0, fake, fake, 4, 65537, 65537, None, 0, 0.5, None, None, None) == _lib.TVP_EUNSUPPORTED
    assert lib.tv1d_prox_fwd(1, fake, fake, 4, 65537, 65537, None, 0, 0.5, None, None, None) == _lib.TVP_EUNSUPPORTED
    assert lib.tv2d_prox_fwd(0, fake, fake, 1, 1, 4, 1025, None, 0, 0.5, 4, None, fake, None, None) \
        == _lib.TVP_EUNSUPPORTED
    assert lib.tv1d_prox_bwd(0, fake, None, fake, None, 4, 8, 8, 1, None, None) == E            # NULL mask
    assert lib.tv2d_prox_fwd(0, fake, fake, 1, 1, 0, 4, None, 0, 0.5, 4, None, fake, None, None) == E  # H < 1
    assert lib.tv2d_prox_fwd(0, fake, fake, 1, 1, 4, 4, None, 0, 0.5, 0, None, fake, None, None) == E  # iters
    assert lib.tv2d_prox_fwd(0, fake, fake, 1, 1, 4, 4, None, 1, 0.5, 4, None, fake, None, None) == E  # row mode
    assert lib.tv2d_prox_fwd(0, fake, fake, 1, 1, 4, 4, None, 0, 0.5, 4, None, None, None, None) == E  # no ws
    assert lib.tv2d_prox_bwd(0, fake, None, fake, None, 1, 1, 4, 4, 0, 4, fake, None) == E          # no saved
    msg = lib.tvp_last_error().decode()
    assert "tv2d_prox_bwd" in msg
    assert b"EINVAL" in lib.tvp_status_string(E)


def test_options_validated_and_defaulted(lib):
    """tvp_options_t (per-call options): defaults, and invalid values rejected before any launch."""
    import ctypes as ct
    from paper_2204_03643_b200 import _lib
    o = _lib.Options(7, 7, 7, None, None)
    lib.tvp_options_default(ct.byref(o))
    assert (o.fused2d, o.line_search, o.ls_after, o.diag, o.iter_hist) == (-1, _lib.LS_BACKTRACK, 0, None, None)
    fake = ct.c_void_p(16)
    E = _lib.TVP_EINVAL
    for bad in (_lib.Options(2, 0, 0, None, None), _lib.Options(-2, 0, 0, None, None),
                _lib.Options(-1, 2, 0, None, None), _lib.Options(-1, 0, -1, None, None)):
        assert lib.tv1d_prox_fwd_ex(0, fake, fake, 4, 8, 8, None, 0, 0.5, None, None, None, ct.byref(bad), None) == E
        assert lib.tv2d_prox_fwd_ex(0, fake, fake, 1, 1, 4, 4, None, 0, 0.5, 4, None, fake, None, ct.byref(bad),
                                    None) == E
        assert lib.tv2d_prox_bwd_ex(0, fake, fake, fake, None, 1, 1, 4, 4, 0, 4, fake, ct.byref(bad), None) == E
    assert "tvp_options_t" in lib.tvp_last_error().decode()
    ok = _lib.Options(1, 1, 2, None, None)
    # valid options, empty batch: OK without touching the (fake) buffers
    assert lib.tv1d_prox_fwd_ex(0, fake, fake, 0, 8, 8, None, 0, 0.5, None, None, None, ct.byref(ok), None) == 0
    assert lib.tv2d_prox_fwd_ex(0, fake, fake, 0, 3, 4, 4, None, 0, 0.5, 4, None, fake, None, ct.byref(ok), None) == 0


def test_fused2d_default_is_thread_local(lib):
    """tvp_set_fused2d sets the CALLING thread's default only (no process-global state)."""
    import threading
    prev = lib.tvp_set_fused2d(0)
    seen = []
    t = threading.Thread(target=lambda: seen.append(lib.tvp_set_fused2d(1)))
    t.start()
    t.join()
    assert seen == [1]                         # the other thread still had the initial default
    assert lib.tvp_set_fused2d(prev) == 0      # ours was not changed by the other thread
