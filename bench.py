"""Throughput benchmark of the batched control step (physics + task layer).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--envs E] [--precision fp32|fp64]
                    [--workload ant|humanoid|anymal]
    python bench.py --impl reference ...          # the CPU reference arm

One "step" = one control step of the Ant-analog locomotion task for every
env: fused action mapping + 2 physics substeps (TGS, 8 position / 1 velocity
iterations) + reward / done / observation / auto-reset (reference
`EnvBatch.step`, envs.py:178-200).  Workload = BASELINE.json north-star
configuration: Ant at 16384 envs per GPU, control dt 1/60, 2 substeps,
uniform random actions (`--workload` selects another BASELINE.json config;
the line's `other_configs` carries the humanoid / ANYmal analogs and PPO
rollout steps -- policy inference + env step -- measured the same way).  Multi-GPU: one process per GPU (torchrun), each
rank owns a contiguous global env range (weak scaling, no data-path
collective); timing is the max over ranks.  `--gpus N` outside torchrun
re-launches itself under `torch.distributed.run` with N ranks (NCCL, LOCAL_RANK
-> device); with fewer GPUs than ranks (a 1-GPU smoke test of the multi-rank
path) the ranks share the device over gloo.

Timed-region rules: W untimed warm-up steps; K timed steps, each bracketed by
CUDA events on the launching stream, an L2 flush (256 MiB write) between
steps outside the events; barrier + synchronize on both sides.  `value` uses
device-resident inputs; `e2e` repeats the run through the public EnvBatch API
(step_host) with the actions copied from pinned host memory and obs / reward / done
copied back every step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "env-steps/sec (whole box) at 1/2/4/8 B200 vs host-CPU ref; % of HBM roofline"
UNIT = "env-steps/s"


def dist_info():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu):
        self.gpu, self.samples, self.proc = gpu, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons}


def kernel_src_sha():
    """The kernel-source hash tools/ncu_summary.py stamps into a summary."""
    import glob
    import hashlib
    h = hashlib.sha256()
    for f in sorted(glob.glob(os.path.join(ROOT, "paper_2108_10470_b200", "csrc", "*.cu*"))) + [
            os.path.join(ROOT, "include", "batchsim_b200.h")]:
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def ncu_traffic(envs):
    """dram__bytes_read.sum + dram__bytes_write.sum per step-kernel launch from
    the newest committed `ncu --set full` summary of this workload
    (profiles/r*_step_*_ncu.json, written by tools/ncu_summary.py), else None.
    Returns (bytes, file, flop/env, fresh): `fresh` is False when the summary
    was captured from other kernel sources than the ones built now."""
    import glob
    import re

    def version(path):      # r01_step_v13_ncu.json -> (1, 13): newest round, then kernel version
        m = re.search(r"r(\d+)_step_v(\d+)", os.path.basename(path))
        return (int(m.group(1)), int(m.group(2))) if m else (-1, -1)

    best = None
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_step_*_ncu.json")), key=version):
        try:
            with open(path) as f:
                j = json.load(f)
        except (OSError, ValueError):
            continue
        if j.get("envs") != envs:
            continue
        for l in j.get("launches", []):
            if "step_kernel<float" in l.get("kernel", "") and "dram_bytes_per_launch" in l:
                best = (l["dram_bytes_per_launch"], os.path.basename(path), l.get("fp32_flop_per_env_launch"),
                        j.get("src_sha") == kernel_src_sha())
    return best


def kernel_bytes(env):
    """Compulsory HBM bytes of one fused step-kernel launch (reads + writes of
    every array the launch touches, counted once), per env."""
    s = env.scene
    E = s.num_envs
    read = ("body_q", "friction_anchor", "inv_mass", "inv_inertia_local", "gravity", "mu_static",
            "mu_dynamic", "joint_stiffness", "joint_damping", "joint_armature", "joint_friction",
            "joint_limit_lo", "joint_limit_hi", "plane_off", "plane_rad", "ctrl_dof_vel_target",
            "ctrl_dof_force", "ctrl_body_force", "ctrl_body_torque", "dof_mode", "env_origins",
            "nonfinite")
    write = ("body_q", "friction_anchor", "body_state", "root_state", "dof_state", "net_contact",
             "dof_force", "sensor_forces", "ctrl_dof_pos_target")
    def nb(name):
        t = s._friction_anchor if name == "friction_anchor" else getattr(s, name)
        return t.numel() * t.element_size()
    total = sum(nb(n) for n in read) + sum(nb(n) for n in write)
    total += 2 * env.actions.numel() * env.actions.element_size()   # actions in, clipped out
    return total / E


WORKLOADS = {
    # name: (task, model builder name, rest height attr, description)
    "ant": ("quadruped", "quadruped", "QUADRUPED_REST_HEIGHT",
            "ant-quadruped locomotion, {E} envs/GPU, control dt 1/60 (2 substeps), random actions"),
    "humanoid": ("humanoid", "humanoid", "HUMANOID_REST_HEIGHT",
                 "humanoid (authored 21-DOF) locomotion, {E} envs/GPU, control dt 1/60 (2 substeps), random actions"),
    "anymal": ("quadruped-anymal-obs", "quadruped12", "QUADRUPED12_REST_HEIGHT",
               "anymal-analog velocity tracking (12 DOF, PD targets), {E} envs/GPU, 2 substeps, random actions"),
}


def measure(task, E, args, rank, world, clocks=None, policy=False, kernel=True, e2e=True):
    """Device-timed control steps of `task` (CUDA events per step, L2 flushed
    between steps, max over ranks); optionally the fused physics launch alone
    and the end-to-end run through EnvBatch.step with host buffers."""
    import torch
    import torch.distributed as dist

    from paper_2108_10470_b200.envs import make_env
    env = make_env(task, num_envs=E, seed=args.seed, precision=args.precision,
                   env_offset=rank * E, total_envs=world * E)
    dev = env.scene.device
    stream = torch.cuda.current_stream()
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    acts = [torch.rand((E, env.act_dim), generator=gen, device=dev, dtype=env.scene.dtype) * 2 - 1
            for _ in range(8)]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    agent = None
    if policy:      # PPO rollout step: policy inference (reference MLP sizes) + env step
        from paper_2108_10470_b200.ppo import PPO
        agent = PPO(env.obs_dim, env.act_dim, device=dev)

    policy_graph = None
    if agent is not None:     # the policy as one CUDA graph (ppo.PolicyGraph): ~25 small kernels -> 1 launch
        from paper_2108_10470_b200.ppo import PolicyGraph
        policy_graph = PolicyGraph(agent.net, agent.gen, env.obs)

    def control_step(i):
        if agent is not None:
            a, _, _ = policy_graph(env.obs)
            return env.step(a)
        return env.step(acts[i % len(acts)])

    def maxr(ms):
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    out = {"task": task, "envs_per_gpu": E, "launches_per_step": 1 if env.fused else 2}
    if clocks is not None:      # nvidia-smi sampler running through warm-up and the timed steps
        clocks.__enter__()
    for i in range(args.warmup):
        control_step(i)
    torch.cuda.synchronize()
    if clocks is not None:      # the first sample lands before the timed region starts
        t_wait = time.time()
        while not clocks.samples and time.time() - t_wait < 3.0:
            control_step(0)
            torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.zero_()                       # L2 flush between timed steps (outside the events)
        ev[i][0].record(stream)
        control_step(i)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    if clocks is not None:      # keep sampling until one sample postdates the timed region
        n0, t_wait = len(clocks.samples), time.time()
        while len(clocks.samples) == n0 and time.time() - t_wait < 3.0:
            control_step(0)
            torch.cuda.synchronize()
        clocks.__exit__(None, None, None)
    if world > 1:
        dist.barrier()
    ms_total = maxr(sum(a.elapsed_time(b) for a, b in ev))
    out["ms_total"] = ms_total
    out["value"] = world * E * args.steps / (ms_total / 1e3)

    if kernel:      # dominant kernel alone: the fused physics launch
        kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        for i in range(args.steps):
            flush.zero_()
            kev[i][0].record(stream)
            env.scene.step(env.config.decimation, actions=acts[i % len(acts)], action_scale=env.action_scale,
                           actions_clipped=env.actions)
            kev[i][1].record(stream)
        torch.cuda.synchronize()
        out["kernel_ms"] = sum(a.elapsed_time(b) for a, b in kev) / args.steps
        out["bytes_per_env"] = kernel_bytes(env)
        env.reset()

    if e2e:         # end to end through the public API with host buffers (EnvBatch.step_host:
        # pinned actions in, pinned obs / reward / done / info out, the host
        # consumes each step's results before issuing the next)
        h_act = [a.cpu().pin_memory() for a in acts]
        for i in range(args.warmup):
            env.step_host(h_act[i % len(h_act)])
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(args.steps):
            o = env.step_host(h_act[i % len(h_act)])
        e1.record(stream)
        torch.cuda.synchronize()
        d2h = sum(t.numel() * t.element_size() for t in (o.obs, o.reward, o.done, *o.info.values()))
        out["e2e"] = {"value": world * E * args.steps / (maxr(e0.elapsed_time(e1)) / 1e3), "unit": UNIT,
                      "h2d_bytes_per_step": h_act[0].numel() * h_act[0].element_size(),
                      "d2h_bytes_per_step": d2h,
                      "api": "EnvBatch.step_host, zero-copy: one fused launch whose CTAs read the pinned host "
                             "actions and write obs / reward / done / info to pinned host memory over PCIe"
                      if env.host_zero_copy else
                      f"EnvBatch.step_host, {env.host_chunk_count()} wave-sized env chunks with the copies "
                      "overlapped on a copy stream"}
    env.close()
    del flush
    torch.cuda.empty_cache()
    return out


def measure_franka(E, args, rank, world):
    """Franka cube-stack (BASELINE.json config 4): FrankaCubeStackEnv -- the
    authored arm + gripper and two cubes with box / capsule pair contacts
    (shape_pairs="all"), 2 substeps, and the fused stacking task tail
    (franka_stack_reward, stacked / timeout, 54-dim obs, auto-reset) per
    control step, uniform random actions.  The reference has the reward but
    no env for this config: the env layer is ours."""
    import torch
    import torch.distributed as dist

    from paper_2108_10470_b200.envs import make_env
    env = make_env("franka-cube-stack", num_envs=E, seed=0, env_offset=rank * E, total_envs=world * E)
    gen = torch.Generator(device=env.obs.device).manual_seed(99 + rank)
    s = env.scene

    def step():
        a = torch.rand((E, env.act_dim), generator=gen, device=env.obs.device, dtype=s.dtype) * 2 - 1
        return env.step(a).reward

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        r = step()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], device=s.device, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ok = bool(torch.isfinite(r).all()) and int(s.nonfinite.sum()) == 0
    env.close()
    return world * E * args.steps / (float(t.item()) / 1e3), ok


def measure_shadow_hand(E, args, rank, world):
    """Shadow Hand cube reorientation (BASELINE.json config 5): ShadowHandEnv
    -- the authored 24-DOF hand with coupling tendons and a cube (box pair
    contacts), Table-12 domain randomisation at every reset, 2 substeps, and
    the fused cube task tail (cube_reorientation_reward, fall / timeout,
    goal resets on success, 96-dim obs, auto-reset) per control step, uniform
    random actions.  The reference has the reward but no env for this config
    (SURVEY.md 8(d)): the env layer is ours (envs.ShadowHandEnv)."""
    import torch
    import torch.distributed as dist

    from paper_2108_10470_b200.envs import make_env
    env = make_env("shadow-hand", num_envs=E, seed=0, randomize=True, env_offset=rank * E, total_envs=world * E)
    gen = torch.Generator(device=env.obs.device).manual_seed(77 + rank)
    s = env.scene

    def step():
        a = torch.rand((E, env.act_dim), generator=gen, device=env.obs.device, dtype=s.dtype) * 2 - 1
        return env.step(a).reward

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        r = step()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], device=s.device, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ok = bool(torch.isfinite(r).all()) and int(s.nonfinite.sum()) == 0
    env.close()
    return world * E * args.steps / (float(t.item()) / 1e3), ok


def config_dict(args, world, E):
    """The workload description both arms print (identical dicts)."""
    task, _, _, desc = WORKLOADS[args.workload]
    return {"workload": desc.format(E=E), "task": task, "envs_per_gpu": E, "global_envs": world * E,
            "substeps": 2, "position_iterations": 8, "velocity_iterations": 1,
            "actions": "uniform(-1, 1) per env per control step", "parallelism": f"env-shard x{world}",
            "l2": "flushed between timed GPU steps (256 MiB write)"}


def cpu_info(threads):
    """CPU model, physical / logical core counts and the threads a CPU leg used."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            model = next((l.split(":", 1)[1].strip() for l in f if l.startswith("model name")), None)
    except OSError:
        pass
    try:
        import psutil
        physical = psutil.cpu_count(logical=False)
    except ImportError:
        physical = None
    return {"cpu_model": model, "physical_cores": physical, "logical_cpus": os.cpu_count(), "threads": threads}


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def measure_ant_fp64(E, args, rank, world):
    import copy
    a2 = copy.copy(args)
    a2.precision = "fp64"
    return measure("quadruped", E, a2, rank, world, kernel=False, e2e=False)


def run_gpu(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_info()
    ndev = torch.cuda.device_count()
    # one GPU per rank (LOCAL_RANK); ranks sharing a device (fewer GPUs than
    # ranks: a 1-GPU smoke test of the multi-rank path) must use gloo
    torch.cuda.set_device(local % ndev)
    backend = os.environ.get("BENCH_DIST_BACKEND") or ("nccl" if world <= ndev else "gloo")
    if world > 1:
        dist.init_process_group(backend)
    if args.gpus != world and rank == 0:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; reporting n_gpus={world}\n")
    E = args.envs
    clocks = ClockSampler(local % ndev)
    m = measure(WORKLOADS[args.workload][0], E, args, rank, world, clocks=clocks)
    others = {}
    if not args.no_other_configs:
        # the other BASELINE.json configs (fewer steps, device-resident inputs)
        import copy
        a2 = copy.copy(args)
        a2.steps = args.other_steps
        for name in WORKLOADS:
            if name == args.workload:
                continue
            r = measure(WORKLOADS[name][0], E, a2, rank, world, kernel=False, e2e=False)
            others[name] = {"value": r["value"], "unit": UNIT, "envs_per_gpu": E, "steps": a2.steps}
        if args.workload == "ant":
            # BASELINE.json config 1: Ant at 4096 envs (single-GPU step vs the CPU reference step)
            r = measure("quadruped", 4096, a2, rank, world, kernel=False, e2e=True)
            others["ant_4096"] = {"value": r["value"], "unit": UNIT, "envs_per_gpu": 4096, "steps": a2.steps,
                                  "e2e": r["e2e"]}
            # the exact-parity path: the same kernels in float64 (parity 1e-8 vs the reference)
            r = measure_ant_fp64(E, a2, rank, world)
            others["ant_fp64"] = {"value": r["value"], "unit": UNIT, "envs_per_gpu": E, "steps": a2.steps,
                                  "dtype": "f64", "note": "float64 exact-parity path (1e-8 vs the reference)"}
        fv, fok = measure_franka(8192, a2, rank, world)
        others["franka_cube_stack"] = {"value": fv, "unit": UNIT, "envs_per_gpu": 8192, "steps": a2.steps,
                                       "finite": fok,
                                       "note": "FrankaCubeStackEnv: physics (arm + 2 cubes, box pair contacts) + "
                                               "fused stacking task tail (reward, stacked / timeout, obs, "
                                               "auto-reset); the reference has the reward but no env"}
        hv, hok = measure_shadow_hand(16384, a2, rank, world)
        others["shadow_hand"] = {"value": hv, "unit": UNIT, "envs_per_gpu": 16384, "steps": a2.steps,
                                 "finite": hok,
                                 "note": "ShadowHandEnv: physics (24-DOF hand, tendons, cube, box pair contacts) "
                                         "+ domain randomisation at resets + fused cube task tail (reward, fall / "
                                         "timeout, goal resets, obs, auto-reset); the reference has the reward "
                                         "but no env for this config"}
        for name in ("ant", "humanoid"):   # PPO-rollout steps: policy inference + env step
            r = measure(WORKLOADS[name][0], E, a2, rank, world, policy=True, kernel=False, e2e=False)
            others[f"{name}_ppo_rollout"] = {"value": r["value"], "unit": UNIT, "envs_per_gpu": E,
                                             "steps": a2.steps,
                                             "note": "ActorCritic 256-128-64 act() (one CUDA graph) + env.step per step"}
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    pk, src = peaks()
    k_ms, bytes_env = m["kernel_ms"], m["bytes_per_env"]
    achieved = bytes_env * E / (k_ms / 1e3) / 1e9
    tr = ncu_traffic(E) if (args.precision == "fp32" and args.workload == "ant") else None
    fresh = bool(tr and tr[3])
    # FP32 view: flop per env per launch measured by ncu (ffma*2 + fadd + fmul), else the
    # SURVEY.md 8(d) estimate of 9.3e4 flop per env-sim-step x 2 substeps (Ant)
    flop_env = tr[2] if tr and tr[2] else 9.3e4 * 2
    flops = flop_env * E
    props = torch.cuda.get_device_properties(torch.cuda.current_device())
    fp32_peak = props.multi_processor_count * 128 * 2 * pk.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
    line = {
        "metric": METRIC, "value": m["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": m["ms_total"] / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32" if args.precision == "fp32" else "f64",
        "data": "synthetic (uniform random actions, bundled/authored models, no checkpoints)",
        "config": config_dict(args, world, E),
        "gpu_launches": m["launches_per_step"] * args.steps,
        "clocks": clocks.summary(),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / pk["hbm_gbs"], "traffic": tr[0] if fresh else None,
                     "traffic_unit": "bytes per launch (ncu dram__bytes_read+write, cold L2)",
                     "traffic_source": (f"profiles/{tr[1]}" if fresh else
                                        f"stale: profiles/{tr[1]} was captured from other kernel sources"
                                        if tr else None),
                     "peak_source": src, "kernel": "step_kernel (fused 2 substeps + task tail)", "kernel_ms": k_ms,
                     "bytes_per_env": bytes_env,
                     "fp32": {"achieved_tflops": flops / (k_ms / 1e3) / 1e12, "peak_tflops": fp32_peak,
                              "frac": flops / (k_ms / 1e3) / 1e12 / fp32_peak,
                              "flop_per_env_launch": flop_env,
                              "source": "ncu-measured flop count" if tr and tr[2] else "SURVEY 8(d) estimate"},
                     "note": "compulsory bytes; the fused kernel is latency/FP32-issue bound, not HBM bound "
                             "(DESIGN.md)"},
        "e2e": m["e2e"],
    }
    if world > 1:
        line["dist_backend"] = backend
    if others:
        line["other_configs"] = others
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, bounded=True)
        if others:
            cpu_baseline_others(args, others)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _oracle_env(workload, n_envs, threads, seed=0):
    """The oracle restatement of the reference env (C physics + NumPy task layer)."""
    from oracle.oracle import build
    from oracle.tasks import OracleEnv
    build()
    return OracleEnv(WORKLOADS[workload][0], n_envs, seed=seed, threads=threads)


def _time_oracle_env(env, warmup, steps=None, seconds=None, max_steps=None, seed=0):
    """Control steps of uniform random actions (cli.py:129-140); returns (steps, seconds)."""
    import numpy as np
    rng = np.random.default_rng(seed)
    for _ in range(warmup):
        env.step(rng.uniform(-1, 1, (env.num_envs, env.act_dim)))
    n, t0 = 0, time.perf_counter()
    while True:
        env.step(rng.uniform(-1, 1, (env.num_envs, env.act_dim)))
        n += 1
        dt = time.perf_counter() - t0
        if steps is not None and n >= steps:
            break
        if steps is None and (dt > seconds or n >= max_steps):
            break
    return n, dt


ORACLE_DESC = ("C oracle float64 physics (oracle/bso.c, OpenMP {t} threads) + the NumPy restatement of the "
               "reference env layer (oracle/tasks.py: obs, reward, done, timeout, auto-reset with FK)")


def cpu_baseline(args, bounded=True):
    """The reference's algorithm (oracle restatement, physics + task layer) on
    this host's cores, on a bounded sample of the same workload."""
    threads = host_threads()
    sample = min(args.envs, args.cpu_sample_envs)
    env = _oracle_env(args.workload, sample, threads)
    n, dt = _time_oracle_env(env, 1, seconds=args.cpu_seconds, max_steps=args.cpu_max_steps)
    return {"value": sample * n / dt, "unit": UNIT, "cores": threads, "kind": "port",
            **cpu_info(threads),
            "sample": f"{sample} envs x {n} control steps (2 substeps each + obs / reward / done / auto-reset) "
                      f"of the same {args.workload} workload, " + ORACLE_DESC.format(t=threads)}


def cpu_baseline_others(args, others):
    """A bounded CPU-reference sample beside each other config: the oracle env
    for the configs with a reference task (ANYmal, humanoid, Ant 4096), the
    oracle physics alone for Franka / Shadow Hand (the reference has no env)."""
    import numpy as np
    threads = host_threads()
    secs = args.cpu_seconds / 2
    for name, wl, n in (("anymal", "anymal", 1024), ("humanoid", "humanoid", 512), ("ant_4096", "ant", 4096)):
        if name not in others:
            continue
        env = _oracle_env(wl, n, threads)
        k, dt = _time_oracle_env(env, 1, seconds=secs, max_steps=200)
        others[name]["cpu_baseline"] = {"value": n * k / dt, "unit": UNIT, "cores": threads, "kind": "port",
                                        "sample": f"{n} envs x {k} control steps, " + ORACLE_DESC.format(t=threads)}
    from oracle.oracle import OracleScene
    from paper_2108_10470_b200.params import SimParams
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import pair_scenes as PS
    for name, scene, n in (("franka_cube_stack", "franka_cube_stack", 512), ("shadow_hand", "shadow_hand_cube", 256)):
        if name not in others:
            continue
        s = OracleScene(PS.SCENES[scene][0](), n, SimParams(dt=1 / 120), threads=threads, shape_pairs="all")
        PS.setup(scene, s)
        rng = np.random.default_rng(0)
        base = s.ctrl_dof_pos_target.copy()
        k, t0 = 0, time.perf_counter()
        while True:
            s.ctrl_dof_pos_target[:] = base + 0.3 * rng.uniform(-1, 1, s.num_dofs)
            s.step()
            s.step()
            k += 1
            dt = time.perf_counter() - t0
            if dt > secs or k >= 200:
                break
        others[name]["cpu_baseline"] = {"value": n * k / dt, "unit": UNIT, "cores": threads, "kind": "port",
                                        "sample": f"{n} envs x {k} control steps (2 substeps, random PD "
                                                  f"targets), C oracle float64 physics only, OpenMP {threads} "
                                                  f"threads (no reference env exists for this config)"}


def run_reference(args):
    """The reference arm: the reference's algorithm on the host cores, the
    SAME work as the GPU arm's `value` (physics + obs / reward / done /
    auto-reset of every env of the job).  The reference is pure Python/NumPy
    and cannot travel to the GPU box, so this times its restatement: the
    float64 C port of Scene.step (oracle/bso.c, ~7x faster per core than the
    NumPy reference) on all host threads plus the NumPy port of
    the env layer (oracle/tasks.py, pinned to the reference's env traces).
    Under torchrun rank 0 alone runs it, on the whole job's envs."""
    rank, world, _ = dist_info()
    if rank != 0:
        return
    threads = host_threads()
    n_envs = args.envs * world
    env = _oracle_env(args.workload, n_envs, threads)
    n, dt = _time_oracle_env(env, args.warmup, steps=args.steps)
    value = n_envs * n / dt
    base = {"value": value, "unit": UNIT, "cores": threads, "kind": "port", **cpu_info(threads),
            "sample": f"{n_envs} envs x {n} timed control steps (after {args.warmup} warm-up; 2 substeps each + "
                      "obs / reward / done / auto-reset), " + ORACLE_DESC.format(t=threads)}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / n,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (uniform random actions, bundled/authored models, no checkpoints)",
            "impl": "reference", "config": config_dict(args, world, args.envs),
            "cpu_baseline": base,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def spawn(args):
    """`--gpus N` outside torchrun: re-launch this script under
    torch.distributed.run with N ranks on this node (127.0.0.1)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--envs", type=int, default=16384)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="ant", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true")
    ap.add_argument("--other-steps", type=int, default=10)
    ap.add_argument("--cpu-sample-envs", type=int, default=2048)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--cpu-max-steps", type=int, default=400)
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
