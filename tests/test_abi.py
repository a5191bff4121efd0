"""The C-ABI boundary without a GPU: the in-tree library loads, exports every
function include/batchsim_b200.h declares, and the ctypes mirrors of the
header's structs have exactly the C layout (size and every field offset,
checked against a gcc-compiled probe of the header)."""

import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "batchsim_b200.h")


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    src = re.sub(r"//[^\n]*", "", src)
    return sorted(set(re.findall(r"\b(bsim_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2108_10470_b200 import build
    return build.build()


def test_library_exports_every_declared_function(lib_path):
    names = _declared_functions()
    assert len(names) >= 30
    lib = C.CDLL(lib_path)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    lib.bsim_abi_version.restype = C.c_int
    assert lib.bsim_abi_version() == 2


def test_loader_declares_every_function(lib_path):
    """_native.lib() sets argtypes/restype for every exported entry point."""
    from paper_2108_10470_b200 import _native as N
    lib = N.lib()
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    void = set(re.findall(r"\bvoid\s+(bsim_\w+)\s*\(", src))
    for n in _declared_functions():
        fn = getattr(lib, n)
        assert fn.argtypes is not None, n
        assert (fn.restype is None) == (n in void), n


def _struct_pairs():
    from paper_2108_10470_b200 import _native as N
    from paper_2108_10470_b200.envs import Task
    from paper_2108_10470_b200.randomize import DR, Force
    return [(N.Joint, "bsim_joint_t"), (N.Joint64, "bsim_joint64_t"), (N.Tendon, "bsim_tendon_t"),
            (N.Tendon64, "bsim_tendon64_t"), (N.TendonElem, "bsim_tendon_elem_t"),
            (N.TendonElem64, "bsim_tendon_elem64_t"), (N.Params, "bsim_params_t"),
            (N.Params64, "bsim_params64_t"), (N.Layout, "bsim_layout_t"), (N.State, "bsim_state_t"),
            (N.Actions, "bsim_actions_t"), (DR, "bsim_dr_t"), (Task, "bsim_task_t"),
            (Force, "bsim_force_t")]


def test_ctypes_structs_match_c_layout(tmp_path):
    pairs = _struct_pairs()
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "batchsim_b200.h"', "int main(void) {"]
    for cls, cname in pairs:
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f in cls._fields_:
            lines.append(f'printf("{cname} {f[0]} %zu\\n", offsetof({cname}, {f[0]}));')
    lines += ["return 0;", "}"]
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.check_call(["gcc", "-std=c99", "-I", os.path.dirname(HEADER), str(src), "-o", str(exe)])
    got = {}
    for line in subprocess.check_output([str(exe)], text=True).splitlines():
        cname, field, val = line.split()
        got[(cname, field)] = int(val)
    for cls, cname in pairs:
        assert got[(cname, "size")] == C.sizeof(cls), cname
        for f in cls._fields_:
            assert got[(cname, f[0])] == getattr(cls, f[0]).offset, (cname, f[0])


def test_product_has_no_cpu_fallback(monkeypatch):
    """Without the built library the product raises instead of computing."""
    from paper_2108_10470_b200 import _native as N
    monkeypatch.setattr(N, "_lib", None)
    monkeypatch.setattr(N, "LIB_PATH", "/nonexistent/libbsim_b200.so")
    with pytest.raises(N.NativeError):
        N.lib()
