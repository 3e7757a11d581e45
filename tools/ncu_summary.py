"""Summarise one `ncu --set full` capture (.ncu-rep) into markdown: key raw
metrics (duration, DRAM bytes, DMMA pipe, shared-memory wavefronts) and the
Speed-of-Light / memory / scheduler / occupancy rows of the details page.

usage: python tools/ncu_summary.py capture.ncu-rep out.md "title" "command"
"""
import csv
import io
import json
import subprocess
import sys

RAW = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "launch__grid_size", "launch__block_size",
       "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic"]
SECTIONS = ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Scheduler Statistics",
            "Warp State Statistics", "Occupancy", "Compute Workload Analysis")


def ncu(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True, check=True).stdout


def main():
    rep, out, title, cmd = sys.argv[1:5]
    raw = list(csv.reader(io.StringIO(ncu([rep, "--page", "raw", "--csv", "--metrics", ",".join(RAW)]))))
    h, units, row = raw[0], raw[1], raw[2]
    vals = {k: (row[i], units[i]) for i, k in enumerate(h)}
    lines = [f"# {title}", "", "Command (after the same command exited 0 without ncu):", "", "    " + cmd, "",
             f"Kernel: `{vals.get('Kernel Name', ('?', ''))[0]}`", "", "| metric | value |", "|---|---|"]
    for k in RAW:
        if k in vals:
            lines.append(f"| {k} | {vals[k][0]} {vals[k][1]} |")
    det = list(csv.reader(io.StringIO(ncu([rep, "--page", "details", "--csv"]))))
    dh = {k: i for i, k in enumerate(det[0])}
    lines += ["", "## Details page", "", "| section | metric | value |", "|---|---|---|"]
    for r in det[1:]:
        if r[dh["Section Name"]] in SECTIONS and r[dh["Metric Name"]]:
            lines.append(f"| {r[dh['Section Name']]} | {r[dh['Metric Name']]} | {r[dh['Metric Value']]} "
                         f"{r[dh['Metric Unit']]} |")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    rd = float(vals["dram__bytes_read.sum"][0].replace(",", "")) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[vals["dram__bytes_read.sum"][1]]
    wr = float(vals["dram__bytes_write.sum"][0].replace(",", "")) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[vals["dram__bytes_write.sum"][1]]
    print(json.dumps({"dram_bytes_per_launch": rd + wr}))


if __name__ == "__main__":
    main()
