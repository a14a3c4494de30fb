"""Hot SASS lines of an ncu --set full capture (source page): top stall
samples, shared-memory excess wavefronts, instruction counts.
usage: python tools/ncu_src.py rep.ncu-rep [topN]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    data = rows[2:]
    ix = {k: h.index(k) for k in h}

    def f(r, k):
        try:
            return float(r[ix[k]])
        except (ValueError, KeyError):
            return 0.0
    tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
    ex = sum(f(r, "L1 Wavefronts Shared Excessive") for r in data)
    ins = sum(f(r, "Instructions Executed") for r in data)
    print(f"samples {tot:.0f}  smem excess wavefronts {ex:.0f}  instructions {ins:.0f}")
    print("-- top stall lines")
    for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:top]:
        s = f(r, "Warp Stall Sampling (All Samples)")
        stalls = sorted(((f(r, k), k[6:]) for k in h if k.startswith("stall_") and "Not" not in k),
                        reverse=True)[:2]
        print(f"{r[0]:>6s} {100 * s / tot:5.1f}%  {r[1][:60]:60s} "
              + " ".join(f"{k}:{v:.0f}" for v, k in stalls))
    print("-- excess shared wavefronts")
    for r in sorted(data, key=lambda r: -f(r, "L1 Wavefronts Shared Excessive"))[:8]:
        if f(r, "L1 Wavefronts Shared Excessive") > 0:
            print(f"{r[0]:>6s} {r[1][:70]:70s} excess {f(r, 'L1 Wavefronts Shared Excessive'):.0f} "
                  f"of {f(r, 'L1 Wavefronts Shared'):.0f}")


if __name__ == "__main__":
    main()
