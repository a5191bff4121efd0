"""ctypes declarations of the task-layer entry points (bsim_tasks.cu)."""

import ctypes as C


def declare(lib):
    vp = C.c_void_p
    for suffix in ("", "_f64"):
        f = getattr(lib, "bsim_task_step" + suffix)
        f.argtypes, f.restype = [vp, vp, vp, vp], C.c_int
        f = getattr(lib, "bsim_task_reset" + suffix)
        f.argtypes, f.restype = [vp, vp, vp, vp, vp], C.c_int
    lib.bsim_task_last_error.argtypes, lib.bsim_task_last_error.restype = [], C.c_char_p
    return lib
