"""Per-source-line warp-stall samples and instruction counts from an ncu report.

    python tools/ncu_src.py report.ncu-rep [kernel-substring] [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    kern = sys.argv[2] if len(sys.argv) > 2 else None
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kern:
        cmd += ["--kernel-name-base", "demangled", "-k", f"regex:{kern}"]
    txt = subprocess.run(cmd, capture_output=True, text=True).stdout
    f = None
    out = []
    tot = tot_i = 0
    for r in csv.reader(io.StringIO(txt)):
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0].isdigit() and len(r) > 7 and r[2] == "-":
            v, ins = int(r[4]), int(r[7] or 0)
            tot += v
            tot_i += ins
            out.append((v, ins, f"{f}:{r[0]}", r[1][:90]))
    out.sort(reverse=True)
    print(f"total stall samples {tot}, warp instructions {tot_i}")
    for v, ins, loc, s in out[:top]:
        print(f"{v:6d} {ins:10d}  {loc:22s} {s}")


if __name__ == "__main__":
    main()
