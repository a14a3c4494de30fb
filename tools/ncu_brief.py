"""One-paragraph summary of ncu --set full captures (key roofline metrics).
usage: python tools/ncu_brief.py a.ncu-rep [b.ncu-rep ...]"""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "time"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
        ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
         "LSU smem wavefronts %"),
        ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("launch__registers_per_thread", "regs")]


def main():
    for rep in sys.argv[1:]:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        h, u, v = rows[0], rows[1], rows[2]
        print(f"== {rep.split('/')[-1]}: {v[h.index('Kernel Name')][:100]}")
        for k, label in KEYS:
            if k in h:
                i = h.index(k)
                print(f"   {label:24s} {v[i]:>14s} {u[i]}")


if __name__ == "__main__":
    main()
