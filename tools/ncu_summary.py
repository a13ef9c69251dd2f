"""Summarise an ncu report (--set full) into profiles/: key pipe/DRAM metrics and top stalls.

usage: python tools/ncu_summary.py gpurun_out/prof_gauss.ncu-rep profiles/r01_ncu_gauss.md [--config C5]
With --config, the DRAM read+write bytes per launch are recorded in profiles/ncu_traffic.json
(bench.py's roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size",
    "launch__block_size", "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    cfg = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else None
    raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    lines = [f"# ncu summary: {os.path.basename(rep)}", ""]
    traffic = []
    for r in data:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        lines.append(f"## {d.get('Kernel Name', '?')[:120]}")
        lines.append("| metric | value | unit |\n|---|---|---|")
        for k in KEYS[1:]:
            if k in d:
                lines.append(f"| {k} | {d[k]} | {u.get(k, '')} |")
        stalls = []
        for k, v in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        lines.append("")
        lines.append("top stalls (warps per issue): " + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:8]))
        lines.append("")

        def to_bytes(k):
            v = float(d[k].replace(",", ""))
            un = u.get(k, "byte").lower()
            mult = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(un, 1)
            return v * mult
        if "dram__bytes_read.sum" in d:
            traffic.append(to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum"))
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if cfg and traffic:
        p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
        d = json.load(open(p)) if os.path.exists(p) else {}
        d[cfg] = traffic[0]
        d[cfg + "_source"] = os.path.basename(out)
        json.dump(d, open(p, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
