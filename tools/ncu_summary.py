"""Summarise an ncu report (--set full) into markdown: key throughput metrics,
DRAM traffic per launch and the top warp-stall reasons. Usage:
    python tools/ncu_summary.py report.ncu-rep [label] >> profiles/rNN_ncu.md
Also prints a one-line JSON {kernel: dram_bytes} for profiles/ncu_traffic.json."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg.per_second"]


def main(path, label=""):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    traffic = {}
    print(f"\n### {label or path}\n")
    for d in data:
        rec = dict(zip(hdr, d))
        name = rec.get("Kernel Name", "?")
        print(f"**{name[:110]}**\n")
        print("| metric | value | unit |\n|---|---|---|")
        for k in KEYS:
            if k in rec:
                print(f"| {k} | {rec[k]} | {units[hdr.index(k)]} |")
        st = [(float(rec[n]), n) for n in hdr if n.startswith("smsp__pcsamp_warps_issue_stalled") and
              not n.endswith("not_issued") and rec[n].replace(".", "").isdigit()]
        tot = sum(x for x, _ in st) or 1.0
        st.sort(reverse=True)
        print("\nTop stall reasons (share of PC samples): " +
              ", ".join(f"{n.replace('smsp__pcsamp_warps_issue_stalled_', '')} {x / tot * 100:.1f}%" for x, n in st[:6]) + "\n")
        try:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd = float(rec["dram__bytes_read.sum"]) * scale[units[hdr.index("dram__bytes_read.sum")]]
            wr = float(rec["dram__bytes_write.sum"]) * scale[units[hdr.index("dram__bytes_write.sum")]]
            traffic[name.split("(")[0].split("::")[-1].split("<")[0]] = rd + wr
        except (KeyError, ValueError):
            pass
    print("<!-- traffic " + json.dumps(traffic) + " -->")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
