"""Dev tool: condense one `ncu --set full` report into a JSON summary under
profiles/ (bench.py reads `dram_bytes_per_launch` from it for roofline.traffic).

    python tools/ncu_summary.py REPORT.ncu-rep profiles/rNN_step_ncu.json --envs 16384 --note "..."
"""
import argparse, csv, glob, hashlib, json, os, subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def kernel_src_sha():
    """sha256 (16 hex) over the CUDA sources + the ABI header: bench.py only
    uses a summary's traffic when it was captured from the current kernels."""
    h = hashlib.sha256()
    for f in sorted(glob.glob(os.path.join(ROOT, "paper_2108_10470_b200", "csrc", "*.cu*"))) + [
            os.path.join(ROOT, "include", "batchsim_b200.h")]:
        h.update(open(f, "rb").read())
    return h.hexdigest()[:16]

KEYS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__shared_mem_per_block_dynamic": "dyn_smem_per_block",
    "launch__occupancy_limit_registers": "occ_limit_registers",
    "launch__occupancy_limit_shared_mem": "occ_limit_smem",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__cycles_elapsed.avg": "cycles",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum.per_cycle_elapsed": "ffma_per_cycle",
    "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum.per_cycle_elapsed": "fadd_per_cycle",
    "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum.per_cycle_elapsed": "fmul_per_cycle",
    "smsp__cycles_active.avg": "smsp_cycles_active",
}
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "nsecond": 1e-3, "msecond": 1e3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report"); ap.add_argument("out")
    ap.add_argument("--envs", type=int, required=True)
    ap.add_argument("--note", default="")
    ap.add_argument("--command", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        m = {"kernel": d.get("Kernel Name", "")[:120]}
        for k, name in KEYS.items():
            if k in d and d[k] not in ("", "n/a"):
                try:
                    v = float(d[k].replace(",", ""))
                except ValueError:
                    continue
                v *= UNITS.get(u.get(k, "").split("/")[0], 1)
                m[name] = v
        st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in k
              and v.replace(".", "").isdigit()}
        tot = sum(st.values()) or 1.0
        m["stall_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:8]}
        if "dram_read" in m:
            m["dram_bytes_per_launch"] = m["dram_read"] + m.get("dram_write", 0.0)
            m["dram_bytes_per_env"] = m["dram_bytes_per_launch"] / a.envs
        if "ffma_per_cycle" in m and "cycles" in m:
            fl = (2 * m["ffma_per_cycle"] + m.get("fadd_per_cycle", 0) + m.get("fmul_per_cycle", 0)) * m["cycles"]
            m["fp32_flop_per_launch"] = fl
            m["fp32_flop_per_env_launch"] = fl / a.envs
        launches.append(m)
    json.dump({"envs": a.envs, "command": a.command, "note": a.note, "src_sha": kernel_src_sha(),
               "launches": launches},
              open(a.out, "w"), indent=1)
    print(json.dumps(launches, indent=1)[:3000])


if __name__ == "__main__":
    main()
