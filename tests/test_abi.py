"""CPU: the C-ABI library loads and exports exactly what include/ttg.h declares
(no compute calls without a GPU); the Python host mirror's pure-host logic."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ttg.h")
LIB = os.path.join(ROOT, "paper_2211_12487_b200", "libttg.so")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ttg_[a-z_0-9]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        import __graft_entry__

        __graft_entry__.build()
    return ctypes.CDLL(LIB)


def test_header_declares_the_path(lib):
    syms = declared_symbols()
    for must in ["ttg_bootstrap", "ttg_tt_ice_update", "ttg_tt_ice_update_with_tolerances", "ttg_tt_ice_star_update",
                 "ttg_project", "ttg_reconstruct", "ttg_per_obs_errors", "ttg_tt_upload", "ttg_ctx_create"]:
        assert must in syms


def test_library_exports_every_declared_symbol(lib):
    for s in declared_symbols():
        assert hasattr(lib, s), f"libttg.so does not export {s}"


def test_exports_are_c_linkage():
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    for s in declared_symbols():
        assert s in exported


def test_ctypes_binding_covers_header():
    from paper_2211_12487_b200 import _lib

    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert bound == set(declared_symbols())


def test_struct_layouts_match_header():
    from paper_2211_12487_b200 import _lib

    # ttg_report: 3 int64 + 2 int32 + 2*(33 int64) + 3 double + 5 int32 (+ tail padding to 8)
    assert ctypes.sizeof(_lib.Report) == 3 * 8 + 2 * 4 + 2 * 33 * 8 + 3 * 8 + 5 * 4 + 4
    assert ctypes.sizeof(_lib.Heuristics) == 8 + 4 * 4
    # and the C compiler agrees with the ctypes mirror, field by field
    import subprocess
    import tempfile

    fields = [f for f, _ in _lib.Report._fields_]
    prog = "#include <stdio.h>\n#include <stddef.h>\n#include \"ttg.h\"\nint main(void){printf(\"%zu\", sizeof(ttg_report));"
    prog += "".join(f'printf(" %zu", offsetof(ttg_report, {f}));' for f in fields) + "return 0;}\n"
    with tempfile.TemporaryDirectory() as td:
        src, exe = os.path.join(td, "s.c"), os.path.join(td, "s")
        with open(src, "w") as f:
            f.write(prog)
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", exe, src], check=True)
        got = [int(v) for v in subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()]
    assert got[0] == ctypes.sizeof(_lib.Report)
    assert got[1:] == [getattr(_lib.Report, f).offset for f in fields]


def test_heuristics_default_from_library(lib):
    from paper_2211_12487_b200 import _lib

    L = _lib.load()
    h = _lib.Heuristics()
    L.ttg_heuristics_default(ctypes.byref(h))
    assert h.occupancy_threshold == 0.8 and h.skip_enabled == 1 and h.subselect_enabled == 1
    assert h.skip_statistic == 0 and h.use_approx_tolerance == 0


def test_null_arguments_return_status_without_gpu(lib):
    from paper_2211_12487_b200 import _lib

    L = _lib.load()
    assert L.ttg_ctx_create(0, None) == 10  # TTG_E_ARGUMENT
    assert L.ttg_tt_num_cores(None) == -1
    assert L.ttg_ctx_wait_stream(None, None) == 10
    assert L.ttg_ctx_join_stream(None, None) == 10
    # ctx NULL: the message of the calling thread's last context-free call (TTB1)
    import ctypes

    nd, cnt = ctypes.c_int(), ctypes.c_int64()
    assert L.ttg_read_batch(b"/nonexistent/x.ttb", None, ctypes.byref(nd), None, 0, ctypes.byref(cnt)) == 4
    assert L.ttg_last_error(None).startswith(b"cannot open")


def test_host_mirror_pure_helpers():
    from paper_2211_12487_b200 import ConfigError, HeuristicConfig, occupancy, relaxed_tolerance_approx, subselect

    assert subselect([0.2, 0.05, 0.1], 0.1) == ([0], [1, 2])
    assert relaxed_tolerance_approx(10, 5, 0.05, 0.1) == pytest.approx(0.15)
    with pytest.raises(ConfigError):
        relaxed_tolerance_approx(3, 3, 0.0, 0.1)
    assert occupancy(np.zeros((1, 4, 2))) == 0.5
    h = HeuristicConfig(skip_statistic="full")._to()
    assert h.skip_statistic == 1
    with pytest.raises(ValueError):
        HeuristicConfig(skip_statistic="median")._to()


def test_status_codes_map_to_reference_exceptions():
    from paper_2211_12487_b200 import errors

    assert errors.STATUS_TO_ERROR[1] is errors.DimensionError
    assert errors.STATUS_TO_ERROR[2] is errors.NumericError
    assert errors.STATUS_TO_ERROR[3] is errors.StateError
    assert errors.STATUS_TO_ERROR[6] is errors.ConfigError
    for cls in errors.STATUS_TO_ERROR.values():
        assert issubclass(cls, errors.Error)


def test_sass_uses_fp64_tensor_cores():
    """The fused Gram / projection kernels are DMMA (FP64 tensor core) code."""
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in out


def test_loading_the_library_before_torch_keeps_torch_importable():
    """libttg.so depends on libnccl.so.2; loading it before torch must not bind
    the process to the older system NCCL (libtorch_cuda then fails with an
    undefined ncclDevCommCreate).  _lib.load() loads torch first."""
    import subprocess
    import sys

    code = "from paper_2211_12487_b200 import _lib; _lib.load(); import torch; print('ok')"
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
