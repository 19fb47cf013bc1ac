"""Record ncu DRAM bytes per launch into profiles/ncu_dram_bytes.json (run here, on the CPU box,
on the .ncu-rep files a gpurun call brought back), stamped with the sha256 of the kernel source
they were taken on, so bench.py can tell whether the record matches the benched kernel.

    python tools/ncu_dram.py KEY=gpurun_out/x.ncu-rep [KEY=...]

Each report must hold exactly one launch (ncu -k ... --launch-skip S --launch-count 1).
"""

import csv
import hashlib
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_dram_bytes.json")
# the gather kernel's sources: the record is valid for the build these hash to
SRCS = [os.path.join(ROOT, "paper_1810_08403_b200", "csrc", f) for f in ("propagate.cu", "vecio.cuh")]


def source_sha():
    h = hashlib.sha256()
    for f in SRCS:
        h.update(open(f, "rb").read())
    return h.hexdigest()[:16]


def dram_bytes(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    assert len(data) == 1, f"{rep}: {len(data)} launches (want 1)"
    col = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        tot += float(data[0][col[m]].replace(",", "")) * scale[units[col[m]]]
    t_unit = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}[units[col["gpu__time_duration.sum"]]]
    ms = float(data[0][col["gpu__time_duration.sum"]].replace(",", "")) * t_unit
    return int(tot), ms, data[0][col["Kernel Name"]]


def main():
    rec = json.load(open(OUT)) if os.path.exists(OUT) else {}
    sha = source_sha()
    if rec.get("kernel_source_sha256") != sha:
        rec = {"records": {}, "launch_ms_under_ncu": {}, "kernels": {}}
    rec["kernel_source_sha256"] = sha
    rec["source"] = ("ncu --clock-control none (dram__bytes_read.sum + dram__bytes_write.sum, one "
                     "launch per key), tools/gpu_r2_final.sh; summarised by tools/ncu_dram.py")
    for arg in sys.argv[1:]:
        key, rep = arg.split("=", 1)
        b, ms, name = dram_bytes(rep)
        rec["records"][key] = b
        rec["launch_ms_under_ncu"][key] = ms
        rec["kernels"][key] = name[:120]
        print(f"{key}: {b / 1e9:.2f} GB DRAM, {ms:.3f} ms under ncu ({name[:60]})")
    json.dump(rec, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main()
