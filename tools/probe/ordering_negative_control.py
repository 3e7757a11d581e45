"""Negative control for tests/test_gpu_parity.py::test_device_io_ordered_against_torch_stream:
with the stream-ordering calls stubbed out, the test must fail (the update
reads increments torch has not finished writing, or torch reads the
reconstruction before it is written).  Run on a GPU box:
    PYTHONPATH=. python tools/probe/ordering_negative_control.py"""
import sys

import pytest

from paper_2211_12487_b200 import _lib

L = _lib.load()
L.ttg_ctx_wait_stream = lambda *a: 0
L.ttg_ctx_join_stream = lambda *a: 0
rc = pytest.main(["-x", "-q", "tests/test_gpu_parity.py", "-k", "ordered", "-p", "no:cacheprovider"])
print("negative control:", "test FAILED as expected" if rc == 1 else f"unexpected pytest rc {rc}")
sys.exit(0 if rc == 1 else 1)
