"""ctypes declarations of the task-layer entry points (bsim_tasks.cu)."""

import ctypes as C


def declare(lib):
    vp = C.c_void_p
    for suffix in ("", "_f64"):
        f = getattr(lib, "bsim_task_step" + suffix)
        f.argtypes, f.restype = [vp, vp, vp, vp], C.c_int
        f = getattr(lib, "bsim_task_reset" + suffix)
        f.argtypes, f.restype = [vp, vp, vp, vp, vp], C.c_int
        f = getattr(lib, "bsim_task_step_range" + suffix)
        f.argtypes, f.restype = [vp, vp, vp, C.c_int32, C.c_int32, vp], C.c_int
    lib.bsim_task_last_error.argtypes, lib.bsim_task_last_error.restype = [], C.c_char_p
    for suffix in ("", "_f64"):
        f = getattr(lib, "bsim_randomize" + suffix)
        f.argtypes, f.restype = [vp, vp, vp, vp, C.c_int64, vp], C.c_int
    i = C.c_int
    lib.bsim_force_resample.argtypes, lib.bsim_force_resample.restype = [vp, vp, vp], C.c_int
    lib.bsim_random_object_force.argtypes = [vp, vp, C.c_double, vp, C.c_int32, C.c_int32, vp]
    lib.bsim_random_object_force.restype = C.c_int
    lib.bsim_reward_locomotion.argtypes = [i, i, i] + [vp] * 11 + [vp, vp, vp, vp]
    lib.bsim_reward_anymal.argtypes = [i, i, i, i, i] + [vp] * 9 + [vp, i, vp, vp]
    lib.bsim_reward_cube.argtypes = [i, i, i] + [vp] * 5 + [vp, vp, vp, vp, vp]
    lib.bsim_reward_franka.argtypes = [i, i] + [vp] * 5 + [vp, vp, vp]
    lib.bsim_reward_trifinger.argtypes = [i, i, i] + [vp] * 9 + [vp, vp, vp]
    lib.bsim_reward_ingenuity.argtypes = [i, i, i] + [vp] * 4 + [vp, vp]
    lib.bsim_reward_amp.argtypes = [i, i, vp, vp, vp]
    for n in ("bsim_reward_locomotion", "bsim_reward_anymal", "bsim_reward_cube", "bsim_reward_franka",
              "bsim_reward_trifinger", "bsim_reward_ingenuity", "bsim_reward_amp"):
        getattr(lib, n).restype = C.c_int
    return lib
