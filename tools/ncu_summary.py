"""Summarise ncu outputs into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py report  gpurun_out/prof.ncu-rep  > profiles/X.txt
    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/Y.txt
"""

import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("lts__t_sector_hit_rate.pct", "L2_hit_%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2_%peak"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2_read_sectors"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM_%peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "inst"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_%"),
    ("sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active", "tc_inst_%"),
]


def _csv(args):
    out = subprocess.run(["ncu"] + args, capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def report(path):
    rows = _csv(["-i", path, "--page", "raw", "--csv"])
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    for d in data:
        print(f"== {d[col['Kernel Name']][:110]}")
        for m, name in METRICS:
            if m in col and d[col[m]] not in ("", "n/a"):
                print(f"   {name:16s} {d[col[m]]:>18s} {units[col[m]]}")
        st = {}
        for h, i in col.items():
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    st[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(d[i])
                except ValueError:
                    pass
        top = sorted(st.items(), key=lambda kv: -kv[1])[:5]
        print("   stalls/issue    " + ", ".join(f"{k} {v:.2f}" for k, v in top))


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    tot, cnt = {}, {}
    n = 0
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            k = d["Kernel Name"]
            v = float(d["Metric Value"])
            unit = d.get("Metric Unit", "")
            if unit == "usecond":
                v *= 1e3
            elif unit == "msecond":
                v *= 1e6
            tot[k] = tot.get(k, 0.0) + v
            cnt[k] = cnt.get(k, 0) + 1
            n += 1
    all_ns = sum(tot.values())
    print(f"{n} launches, {all_ns / 1e6:.3f} ms total (cold-cache, serialised)")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{v / 1e6:10.3f} ms  {100 * v / all_ns:5.1f}%  x{cnt[k]:<4d} {k[:100]}")


if __name__ == "__main__":
    {"report": report, "launches": launches}[sys.argv[1]](sys.argv[2])
