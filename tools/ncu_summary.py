"""Summarise ncu reports (run here, no GPU): key metrics + top stall reasons.
Usage: python tools/ncu_summary.py gpurun_out/prof_X.ncu-rep [...] > profiles/rNN_summary.md"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes.sum.per_second", "DRAM throughput"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tc pipe active %"),
    ("sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active", "UMMA issue %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__cycles_active.avg", "SMSP active cycles (avg)"),
    ("sm__cycles_elapsed.max", "SM elapsed cycles (max)"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sass__inst_executed_local_loads", "local loads"),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return None, {}
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    name = d.get("Kernel Name", ("?", ""))[0]
    return name, d


def main(paths):
    for p in paths:
        name, d = raw(p)
        if name is None:
            print(f"## {p}: no data\n")
            continue
        print(f"## {p.split('/')[-1]} -- kernel `{name[:90]}`\n")
        print("| metric | value |\n|---|---|")
        for k, label in KEYS:
            if k in d:
                v, u = d[k]
                print(f"| {label} (`{k}`) | {v} {u} |")
        st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v[0]) for k, v in d.items()
              if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")
              and v[0].replace(".", "", 1).isdigit()}
        tot = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda kv: -kv[1])[:6]
        print("\nTop warp stall reasons (pc sampling): " +
              ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in top) + "\n")


if __name__ == "__main__":
    main(sys.argv[1:])
