"""Per-source-line warp-stall samples from an ncu report (--import-source on,
-lineinfo build):  python tools/ncu_lines.py <report.ncu-rep> [launch_index] [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    skip = sys.argv[2] if len(sys.argv) > 2 else "0"
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass", "--launch-skip", skip, "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    cur, hdr, rows = None, None, []
    for r in csv.reader(io.StringIO(out)):
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            hdr = r
        elif hdr and len(r) == len(hdr) and r[0].isdigit():
            try:
                s = int(r[hdr.index("# Samples")])
                ls = int(r[hdr.index("stall_long_sb")])
                w = int(r[hdr.index("stall_wait")])
                sh = int(r[hdr.index("stall_short_sb")])
            except ValueError:
                continue
            rows.append((s, ls, w, sh, f"{cur}:{r[0]}", r[1].strip()[:80]))
    tot = sum(x[0] for x in rows)
    print(f"total samples {tot}; columns: samples long_sb wait short_sb")
    for x in sorted(rows, reverse=True)[:top]:
        print(f"{x[0]:8d} {x[1]:7d} {x[2]:7d} {x[3]:7d}  {x[4]:<24} {x[5]}")


if __name__ == "__main__":
    main()
