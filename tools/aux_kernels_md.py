"""DEV TOOL: markdown table of the non-step kernels from an ncu summary JSON
(tools/ncu_summary.py) and the algorithmic bytes printed by
tools/aux_kernels_drive.py.

    python tools/aux_kernels_md.py profiles/r02_aux_kernels_ncu.json gpurun_out/aux_drive.log > profiles/r02_aux_kernels.md
"""
import json
import re
import sys

PEAK = 6538.3          # MEASURED_PEAKS.json hbm_gbs (copy bandwidth, burst)


def main(summary, drive_log):
    s = json.load(open(summary))
    algo = {}
    for line in open(drive_log):
        if line.startswith("AUX_ALGO_BYTES "):
            algo = json.loads(line[len("AUX_ALGO_BYTES "):])["bytes_per_launch"]
    print(f"# Non-step kernels at {s['envs']} Ant-analog envs (fp32), one ncu --set full capture each\n")
    print(f"Command: `{s.get('command', '')}`.  Peak = {PEAK} GB/s (MEASURED_PEAKS.json, copy bandwidth).")
    print("`dram GB/s` = ncu dram bytes read + written / duration; `algo GB/s` = the bytes the launch must")
    print("move by its array shapes (tools/aux_kernels_drive.py) / duration.  ncu replays each kernel with")
    print("a cold L2 and serialised, so short launches are latency-bound: the duration, grid and occupancy")
    print("columns say why.\n")
    print("| kernel | duration us | grid x block | regs | achieved occupancy % | dram MB | dram GB/s | frac | "
          "algo MB | algo GB/s | frac | top stalls |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for m in s["launches"]:
        name = re.sub(r"^void |\(.*$|<.*?>|bsim::|\(anonymous namespace\)::", "", m["kernel"])
        name = name.split("::")[-1]
        us = m.get("duration_us", 0.0)
        dram = m.get("dram_bytes_per_launch", 0.0)
        key = next((k for k in algo if k.startswith(name) or name.startswith(k.replace("_kernel", ""))), None)
        ab = algo.get(key, 0.0) if key else 0.0
        g = lambda b: b / (us * 1e-6) / 1e9 if us else 0.0  # noqa: E731
        stalls = ", ".join(f"{k} {v}" for k, v in list(m.get("stall_pct", {}).items())[:3])
        print(f"| {name} | {us:.1f} | {int(m.get('grid', 0))} x {int(m.get('block', 0))} | "
              f"{int(m.get('registers_per_thread', 0))} | {m.get('achieved_occupancy_pct', 0):.1f} | "
              f"{dram / 1e6:.2f} | {g(dram):.0f} | {g(dram) / PEAK:.3f} | {ab / 1e6:.2f} | {g(ab):.0f} | "
              f"{g(ab) / PEAK:.3f} | {stalls} |")


if __name__ == "__main__":
    main(*sys.argv[1:3])
