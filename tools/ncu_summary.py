"""Summarise an ncu report (raw page) into the metrics this project tracks.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [out.txt]
"""
import csv
import io
import re
import subprocess
import sys

KEYS = [
    r"^gpu__time_duration.sum$", r"^launch__grid_size$", r"^launch__block_size$",
    r"^launch__registers_per_thread$", r"^launch__occupancy_limit_(registers|shared_mem|warps)$",
    r"^sm__warps_active.avg.pct_of_peak_sustained_active$",
    r"^sm__inst_executed.avg.per_cycle_active$",
    r"^smsp__issue_active.avg.pct_of_peak_sustained_active$",
    r"^sm__inst_executed_pipe_(alu|fma|xu|lsu|adu|fmaheavy|fmalite)\.avg\.pct_of_peak_sustained_active$",
    r"^sm__pipe_(alu|fma|shared|xu)_cycles_active.avg.pct_of_peak_sustained_active$",
    r"^l1tex__data_pipe_lsu_wavefronts_mem_shared(_op_atom)?.sum$",
    r"^l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed$",
    r"^l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum$",
    r"^smsp__inst_executed_op_shared_atom.sum$", r"^smsp__inst_executed.sum$",
    r"^dram__bytes_(read|write).sum$", r"^sm__cycles_elapsed.avg$",
    r"^smsp__average_warp_latency_issue_stalled_.*_per_warp_active.ratio$",
    r"^smsp__pcsamp_warps_issue_stalled_(lg_throttle|mio_throttle|short_scoreboard|wait|math_pipe_throttle|not_selected|selected|long_scoreboard|no_instructions|dispatch_stall|barrier|membar|branch_resolving|drain|sleeping|tex_throttle|imc_miss|misc)$",
]


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        out.append(f"kernel: {name}")
        for h, u, v in zip(hdr, units, vals):
            if any(re.search(k, h) for k in KEYS):
                out.append(f"  {h} [{u}] = {v}")
    text = "\n".join(out) + "\n"
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(text)
    print(text)


if __name__ == "__main__":
    main()
