"""The ctypes stub INTEGRATION.md §2 shows a maintainer binds the same
bsim_layout_t the library exports (field names and order of
_native.LAYOUT_INTS / LAYOUT_PTRS, which tests/test_abi.py probes against
include/batchsim_b200.h with gcc).  CPU only."""

import os
import re

from paper_2108_10470_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_integration_layout_stub_matches_abi():
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = doc[doc.index("class Layout(C.Structure):"):]
    block = block[:block.index("\n\n")]
    ints_part, ptrs_part = block.split("C.c_int32) for n in (", 1)[1].split("C.c_void_p) for n in (", 1)
    ints = re.findall(r'"(\w+)"', ints_part)
    ptrs = re.findall(r'"(\w+)"', ptrs_part)
    assert tuple(ints) == N.LAYOUT_INTS
    assert tuple(ptrs) == N.LAYOUT_PTRS
