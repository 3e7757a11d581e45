"""Negative control for tests/test_gpu_parity.py::test_device_io_ordered_against_torch_stream:
with either stream-ordering call stubbed out, the test must fail -- the
update reads an increment torch has not finished writing (its bytes are
written only by a copy queued behind large torch kernels, so an early read
sees zeros), or torch reads the reconstruction before it is written.  Each
stub is tried separately.  Run on a GPU box:
    PYTHONPATH=. python tools/probe/ordering_negative_control.py"""
import subprocess
import sys

CHILD = r"""
import sys, pytest
from paper_2211_12487_b200 import _lib
L = _lib.load()
setattr(L, sys.argv[1], lambda *a: 0)
sys.exit(pytest.main(["-x", "-q", "tests/test_gpu_parity.py", "-k", "ordered", "-p", "no:cacheprovider"]))
"""

ok = True
for name in ("ttg_ctx_wait_stream", "ttg_ctx_join_stream"):
    rc = subprocess.run([sys.executable, "-c", CHILD, name]).returncode
    print(f"negative control, {name} stubbed:", "test FAILED as expected" if rc == 1 else f"unexpected pytest rc {rc}")
    ok &= rc == 1
sys.exit(0 if ok else 1)
