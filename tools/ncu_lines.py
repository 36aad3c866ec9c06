"""Per-CUDA-source-line warp-stall samples and executed instructions of the
kernels in an ncu report (captured with --import-source on, built -lineinfo).
usage: python tools/ncu_lines.py REPORT [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    names = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", "launch__grid_size"],
                           capture_output=True, text=True).stdout
    nk = max(0, len(list(csv.reader(io.StringIO(names)))) - 2)
    for blk in range(nk):
        out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                              "--launch-skip", str(blk), "--launch-count", "1"],
                             capture_output=True, text=True).stdout
        fname, hdr, agg, kname = None, None, [], ""
        for r in csv.reader(io.StringIO(out)):
            if not r:
                continue
            if r[0] == "Function Name":
                kname = r[1][:90]
            if r[0] == "File Path":
                fname = r[1].split("/")[-1]
                continue
            if r[0] == "Line No":
                hdr = r
                continue
            if hdr and r[0].isdigit():
                try:
                    s, i = float(r[4]), float(r[7])
                except ValueError:
                    continue
                st = sorted(((float(r[j]), hdr[j][6:]) for j in range(len(hdr))
                             if hdr[j].startswith("stall_") and "Not Issued" not in hdr[j] and r[j] not in ("", "-")),
                            reverse=True)[:3]
                agg.append((s, i, f"{fname}:{r[0]}", r[1].strip()[:64], st))
        ts = sum(a[0] for a in agg) or 1
        ti = sum(a[1] for a in agg) or 1
        print(f"=== {kname}  samples {ts:.0f}  instructions {ti:.3g}")
        for a in sorted(agg, key=lambda a: -a[0])[:top]:
            print(f"{100 * a[0] / ts:5.1f}%s {100 * a[1] / ti:5.1f}%i {a[2]:24s} {a[3]:64s} "
                  + " ".join(f"{n}:{v:.0f}" for v, n in a[4]))


if __name__ == "__main__":
    main()
