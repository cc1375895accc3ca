"""Summarise an `ncu --set full` report of the sweep kernels: per launch duration, DRAM bytes,
issue activity; writes the per-launch DRAM traffic that bench.py reports as roofline.traffic.

    python tools/ncu_report_summary.py gpurun_out/prof_r01.ncu-rep C4_c64 \
        > profiles/r01_ncu_sweep.txt   (also updates profiles/ncu_sweep_summary.json)
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size"]


def main():
    rep, key = sys.argv[1], sys.argv[2]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ix = {m: hdr.index(m) for m in METRICS if m in hdr}
    kn = hdr.index("Kernel Name")
    print(f"# {rep}  (ncu --set full --clock-control none; cold-cache, serialised replays)")
    print(f"{'kernel':44s} {'ms':>8s} {'DRAM rd GB':>10s} {'DRAM wr GB':>10s} {'GB/s':>8s} {'issue%':>7s} {'regs':>5s}")
    sweep_bytes, n = 0.0, 0
    for r in rows[2:]:
        name = r[kn].replace("void ", "").split("(")[0]
        ms = float(r[ix["gpu__time_duration.sum"]])
        if units[ix["gpu__time_duration.sum"]] == "us":
            ms /= 1e3
        rd = float(r[ix["dram__bytes_read.sum"]]) * (1e-9 if units[ix["dram__bytes_read.sum"]] == "byte" else 1.0)
        wr = float(r[ix["dram__bytes_write.sum"]]) * (1e-9 if units[ix["dram__bytes_write.sum"]] == "byte" else 1.0)
        if units[ix["dram__bytes_read.sum"]] == "Mbyte":
            rd, wr = rd / 1e3, wr / 1e3
        gbs = (rd + wr) / (ms / 1e3)
        print(f"{name[:44]:44s} {ms:8.3f} {rd:10.3f} {wr:10.3f} {gbs:8.0f} "
              f"{float(r[ix['smsp__issue_active.avg.pct_of_peak_sustained_active']]):7.1f} "
              f"{r[ix['launch__registers_per_thread']]:>5s}")
        if "tile_sweep" in name:
            sweep_bytes += (rd + wr) * 1e9
            n += 1
    if n:
        path = os.path.join(ROOT, "profiles", "ncu_sweep_summary.json")
        d = json.load(open(path)) if os.path.exists(path) else {}
        d[key] = {"dram_bytes_per_launch": sweep_bytes / n, "launches": n, "report": os.path.basename(rep)}
        json.dump(d, open(path, "w"), indent=1)
        print(f"# mean DRAM traffic per sweep launch: {sweep_bytes / n / 1e9:.3f} GB over {n} launches")


if __name__ == "__main__":
    main()
