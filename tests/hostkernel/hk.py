"""TEST-ONLY: drive the host build of the step kernel body (host_step.cu)."""

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2108_10470_b200 import tables
from paper_2108_10470_b200 import _native as N

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "libhk.so")
ROOT = os.path.dirname(os.path.dirname(HERE))


def build():
    extra = os.environ.get("BSIM_HK_EXTRA", "").split()      # dev experiments (tools/fp32_error_probe.py)
    so = SO if not extra else SO.replace(".so", "_" + "_".join(x.strip("-D").replace("=", "") for x in extra) + ".so")
    srcs = [os.path.join(HERE, "host_step.cu")] + [
        os.path.join(ROOT, "paper_2108_10470_b200", "csrc", f)
        for f in ("bsim_step.cuh", "bsim_math.cuh", "bsim_topologies.cuh")]
    if os.path.exists(so) and os.path.getmtime(so) >= max(os.path.getmtime(s) for s in srcs):
        return so
    os.makedirs(os.path.dirname(so), exist_ok=True)
    subprocess.check_call(["nvcc", "-O2", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
                           "-Wno-deprecated-gpu-targets", *extra, srcs[0], "-o", so])
    return so


class HostKernel:
    def __init__(self, layout, num_envs, params, env_origins, fp64=False, specialize=True):
        from paper_2108_10470_b200.codegen import topology_id
        self.topo = topology_id(layout) if specialize else 0
        self.L = layout
        self.E = num_envs
        self.params = params
        self.fp64 = fp64
        self.tab = tables.pack_tables(layout, fp64)
        self.arr = tables.init_state_arrays(layout, num_envs, params, env_origins, fp64)
        self.lib = C.CDLL(build())
        self.lib.hk_step.argtypes = [C.POINTER(N.Layout), C.POINTER(N.Params), C.POINTER(N.State), C.c_int]
        self.lib.hk_step_f64.argtypes = [C.POINTER(N.Layout), C.POINTER(N.Params64), C.POINTER(N.State), C.c_int]

    def step(self, n=1):
        lay = tables.layout_struct(self.L, self.E, {k: v.ctypes.data for k, v in self.tab.items()},
                                   topology_id=self.topo)
        st = tables.state_struct({k: v.ctypes.data for k, v in self.arr.items()})
        par = tables.params_struct(self.params, self.fp64)
        fn = self.lib.hk_step_f64 if self.fp64 else self.lib.hk_step
        fn(C.byref(lay), C.byref(par), C.byref(st), n)
