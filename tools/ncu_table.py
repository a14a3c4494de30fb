"""Table of ncu --set full captures: per launch time, DRAM bytes and GB/s
(against MEASURED_PEAKS hbm_gbs), tensor-pipe / SM / L2 / DRAM utilisation.
usage: python tools/ncu_table.py <dir-or-reps...> [--md]"""
import csv
import glob
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3,
         "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "%": 1.0, "": 1.0}


def metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]

    def get(name):
        if name not in h:
            return None
        i = h.index(name)
        try:
            return float(v[i].replace(",", "")) * SCALE.get(u[i], 1.0)
        except ValueError:
            return None
    return {"kernel": v[h.index("Kernel Name")],
            "us": get("gpu__time_duration.sum"),
            "rd": get("dram__bytes_read.sum"), "wr": get("dram__bytes_write.sum"),
            "tensor": get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
            "sm": get("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
            "l2": get("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
            "dram": get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "grid": get("launch__grid_size"), "regs": get("launch__registers_per_thread")}


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    reps = []
    for a in args:
        reps += sorted(glob.glob(os.path.join(a, "*.ncu-rep"))) if os.path.isdir(a) else [a]
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = 6650.0
    print(f"{'capture':24s} {'kernel':34s} {'us':>8s} {'DRAM MB':>9s} {'GB/s':>7s} "
          f"{'of HBM':>6s} {'tensor%':>7s} {'SM%':>5s} {'L2%':>5s} {'DRAM%':>5s}")
    for rep in reps:
        m = metrics(rep)
        mb = ((m["rd"] or 0) + (m["wr"] or 0)) / 1e6
        gbs = mb * 1e6 / (m["us"] * 1e3) if m["us"] else 0.0
        k = m["kernel"].split("(")[0].replace("void ", "")[:34]
        f = lambda x: f"{x:5.1f}" if x is not None else "  -  "
        print(f"{os.path.basename(rep)[:-8]:24s} {k:34s} {m['us']:8.1f} {mb:9.2f} {gbs:7.0f} "
              f"{gbs / peak:6.2f} {f(m['tensor']):>7s} {f(m['sm'])} {f(m['l2'])} {f(m['dram'])}")
    print(f"(HBM peak {peak:.0f} GB/s, MEASURED_PEAKS.json; per-launch values, one ncu "
          "--set full capture each, --clock-control none)")


if __name__ == "__main__":
    main()
