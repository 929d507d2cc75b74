"""CPU checks of the C-ABI library: it loads without a GPU and exports every symbol that
include/ttcross.h declares; argument validation fails loudly before any device work."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ttcross.h")


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__ as g
    g.build()
    from paper_1903_11554_b200 import binding
    return binding.load()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tt_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("tt_cross_init", "tt_cross_sweep", "tt_integrate"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    from paper_1903_11554_b200 import binding
    names = declared_functions()
    assert sorted(binding.EXPORTS) == names
    for n in names:
        assert hasattr(lib, n), n


def test_build_info_and_error_string(lib):
    assert b"sm_100a" in lib.tt_build_info()
    assert isinstance(lib.tt_last_error(), bytes)


def good_config(binding):
    # family, d, n, rank_cap, n_samples, rook_iters, tol, seed, rank, world
    return binding.TtcConfig(0, 4, 9, 4, 16, 4, 1e-12, 1, 0, 1, 0)


@pytest.mark.parametrize("field,value", [("d", 1), ("d", 2001), ("n", 1), ("n", 4097), ("rank_cap", 0),
                                         ("rank_cap", 65), ("family", 7), ("n_samples", 0),
                                         ("n_samples", 1025), ("rook_iters", -1), ("rook_iters", 65),
                                         ("tol", 1.5), ("tol", -1.0), ("world", 0), ("rank", 1),
                                         ("fold_weights", 1), ("fold_weights", 2), ("family", 5)])
def test_invalid_arguments_rejected_without_gpu(lib, field, value):
    from paper_1903_11554_b200 import binding
    cfg = good_config(binding)
    setattr(cfg, field, value)
    u = np.ones((4, 9))
    h = ctypes.c_void_p()
    rc = lib.tt_cross_init(ctypes.byref(h), ctypes.byref(cfg), u.ctypes.data_as(ctypes.c_void_p),
                           u.ctypes.data_as(ctypes.c_void_p), 0, None)
    assert rc == binding.TTC_OK + 1  # TTC_ERR_ARG
    assert not h.value


def test_nonpositive_nodes_rejected(lib):
    from paper_1903_11554_b200 import binding
    cfg = binding.TtcConfig(0, 3, 5, 4, 16, 4, 1e-12, 1, 0, 1, 0)
    u = np.ones((3, 5))
    u[1, 2] = -1.0
    h = ctypes.c_void_p()
    rc = lib.tt_cross_init(ctypes.byref(h), ctypes.byref(cfg), u.ctypes.data_as(ctypes.c_void_p),
                           u.ctypes.data_as(ctypes.c_void_p), 0, None)
    # argument validation happens before any CUDA call, so this is ERR_ARG even on a CPU box
    assert rc == 1


def test_config_struct_layout_matches_header():
    """The ctypes mirror of ttc_config / ttc_stats has the C layout (offsets from the header's
    field order and natural alignment)."""
    from paper_1903_11554_b200 import binding
    assert ctypes.sizeof(binding.TtcConfig) == 6 * 4 + 8 + 8 + 3 * 4 + 4  # trailing pad to 8
    assert binding.TtcConfig.tol.offset == 24 and binding.TtcConfig.seed.offset == 32
    assert ctypes.sizeof(binding.TtcStats) == 8 + 8 + 4 + 4 + 4 * 8 + 7 * 8


def test_c_demo_links_against_the_library(lib):
    """examples/ttcross_demo.c uses the C-ABI from plain C; build() links it against the
    in-tree libttcross.so."""
    import subprocess
    demo = os.path.join(ROOT, "examples", "ttcross_demo")
    assert os.path.exists(demo)
    out = subprocess.run(["ldd", demo], capture_output=True, text=True).stdout
    assert "libttcross.so" in out and "not found" not in out.split("libttcross.so")[1].split("\n")[0]
