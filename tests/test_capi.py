"""C-ABI library (no GPU needed): loads, exports every symbol include/gi.h declares,
struct layouts agree with the binding, and error paths return statuses without compute."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gi.h")


@pytest.fixture(scope="module")
def gi():
    from paper_1911_07260_b200 import _build
    _build.build_lib()
    from paper_1911_07260_b200 import gi as m
    return m


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gi_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    fns = _declared_functions()
    for f in ("gi_graph_create", "gi_sssp_delta", "gi_sssp_batch"):
        assert f in fns


def test_library_exports_every_declared_symbol(gi):
    so = os.path.join(ROOT, "paper_1911_07260_b200", "libgi.so")
    out = subprocess.check_output(["nm", "-D", "--defined-only", so], text=True)
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    for f in _declared_functions():
        assert f in exported, f
        assert hasattr(gi.lib(), f)
    assert sorted(gi.EXPORTS) == sorted(_declared_functions())


def test_sm100a_code_only(gi):
    so = os.path.join(ROOT, "paper_1911_07260_b200", "libgi.so")
    out = subprocess.check_output(["cuobjdump", "--list-elf", so], text=True)
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_version_status_strings_and_struct_layout(gi):
    assert gi.version() == 201
    lib = gi.lib()
    for code, name in gi.STATUS.items():
        assert lib.gi_status_string(code).decode() == name
    o = gi.gi_options()
    lib.gi_options_default(ctypes.byref(o))
    assert o.struct_size == ctypes.sizeof(gi.gi_options)
    assert o.fusion == 1 and o.fusion_threshold == 0 and o.max_ctas == 0 and o.window == 0


def test_error_paths_without_gpu(gi):
    """No GPU here: argument errors are reported before any device work; device
    errors come back as GI_ERR_CUDA with a message, never a crash."""
    lib = gi.lib()
    off = np.array([0, 1], np.int64)
    cols = np.array([0], np.int32)
    w = np.array([1], np.uint32)
    h = ctypes.c_void_p()
    # invalid n
    rc = lib.gi_graph_create(0, 0, off.ctypes.data, None, None, 0, ctypes.byref(h))
    assert rc == 3 and b"GI_ERR_INVALID_GRAPH" in lib.gi_last_error()
    # NULL out
    assert lib.gi_graph_create(1, 1, off.ctypes.data, cols.ctypes.data, w.ctypes.data, 0, None) == 1
    # NULL graph for queries / info
    d = np.zeros(1, np.uint32)
    assert lib.gi_sssp_delta(None, 0, 1, d.ctypes.data) == 1
    assert lib.gi_graph_info(None, None, None, None) == 1
    lib.gi_graph_destroy(None)  # NULL-safe
    # the fused-gather batch and the IPC helpers: argument errors before any device work
    peers = (ctypes.c_void_p * 2)(None, None)
    assert lib.gi_sssp_batch_peers(None, None, 0, 1, None, peers, 2, 0, None) == 1  # NULL peer rows
    assert lib.gi_sssp_batch_peers(None, None, 0, 1, None, peers, 0, 0, None) == 1  # npeers < 1
    assert lib.gi_sssp_batch_peers(None, None, 0, 1, None, peers, 2, 2, None) == 1  # self out of range
    hbuf = (ctypes.c_uint8 * 64)()
    off64 = ctypes.c_uint64()
    assert lib.gi_ipc_get_handle(None, hbuf, ctypes.byref(off64)) == 1
    assert lib.gi_ipc_open_handle(None, 0, 0, None) == 1
    assert lib.gi_ipc_close_handle(None, 0, 0) == 1
    import torch
    if not torch.cuda.is_available():
        rc = lib.gi_graph_create(1, 1, off.ctypes.data, cols.ctypes.data, w.ctypes.data, 0, ctypes.byref(h))
        assert rc == 5 and lib.gi_last_error().startswith(b"GI_ERR_CUDA")


def test_fastdiv_formula_matches_floor_division():
    """The kernels divide by Δ with the Granlund–Montgomery round-up method
    (gi_internal.h make_fastdiv / fdiv). Re-derive it here and check it against //."""
    def make(d):
        l = 0
        while l < 32 and (1 << l) < d:
            l += 1
        mul = ((((1 << l) - d) << 32) // d + 1) & 0xFFFFFFFF
        return mul, (1 if l > 0 else 0), (l - 1 if l > 0 else 0)

    def fdiv(x, f):
        mul, s1, s2 = f
        t = (x * mul) >> 32
        return (t + ((x - t) >> s1)) >> s2

    rng = np.random.default_rng(0)
    ds = [1, 2, 3, 7, 1000, 1 << 10, (1 << 16) + 1, 10000, 0x7FFFFFFF, 0xFFFFFFFE, 0xFFFFFFFF]
    ds += [int(x) for x in rng.integers(1, 2**32, 200)]
    xs = [0, 1, 2**31, 2**32 - 2, 2**32 - 1] + [int(x) for x in rng.integers(0, 2**32, 300)]
    for d in ds:
        f = make(d)
        for x in xs + [d - 1, d, d + 1 if d < 2**32 - 1 else d, 2 * d - 1 if 2 * d - 1 < 2**32 else d]:
            assert fdiv(x, f) == x // d, (x, d)
