"""Record the DRAM traffic of one ncu --set full capture for bench.py's
roofline.traffic: python tools/ncu_traffic.py <rep.ncu-rep> "<layer> <op>" [tag]
-> merges {"<layer> <op>": {dram_read, dram_write, traffic, time_us, kernel,
source}} into profiles/dominant_traffic.json (per launch)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rep, key = sys.argv[1], sys.argv[2]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]

    def get(name):
        i = h.index(name)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1,
                 "us": 1, "ms": 1e3, "msecond": 1e3, "ns": 1e-3, "nsecond": 1e-3}[u[i]]
        return float(v[i].replace(",", "")) * scale

    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    rec = {"dram_read": rd, "dram_write": wr, "traffic": rd + wr,
           "time_us": get("gpu__time_duration.sum"), "kernel": v[h.index("Kernel Name")],
           "tensor_pipe_pct": float(v[h.index(
               "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")]),
           "source": os.path.basename(rep)}
    path = os.path.join(ROOT, "profiles", "dominant_traffic.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    data[key] = rec
    with open(path, "w") as fh:
        json.dump(data, fh, indent=1, sort_keys=True)
    print(key, rec)


if __name__ == "__main__":
    main()
