"""Dynamic opcode mix and per-source-line instruction counts of one launch
in an ncu report (--set full --import-source on, -lineinfo build):

    python tools/ncu_opmix.py <report.ncu-rep> [launch_index] [top]

Prints warp-level instructions executed per SASS opcode (first mnemonic
token, predicate stripped) and per CUDA source line (inclusive over inline chains), both as shares of
the launch total.
"""
import collections
import csv
import io
import subprocess
import sys


def rows(rep, skip):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass", "--launch-skip", str(skip), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    cur, hdr, line = None, None, None
    for r in csv.reader(io.StringIO(out)):
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            hdr = r
        elif hdr and len(r) >= len(hdr) - 1:
            if r[0].isdigit():
                line = (cur, int(r[0]), r[1].strip())
            elif r[2].startswith("0x") and line is not None:
                try:
                    n = int(r[hdr.index("Instructions Executed")])
                except ValueError:
                    continue
                yield line, r[2], r[3].strip(), n


def opcode(sass):
    t = sass.split()
    if t and t[0].startswith("@"):
        t = t[1:]
    return t[0] if t else "?"


def main():
    rep = sys.argv[1]
    skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    ops, lines = collections.Counter(), collections.Counter()
    src = {}
    seen = set()
    for (f, ln, s), addr, sass, n in rows(rep, skip):
        # an inlined instruction is listed under every file of its inline
        # chain: opcodes count each address once, lines are inclusive
        if addr not in seen:
            seen.add(addr)
            ops[opcode(sass)] += n
        lines[(f, ln)] += n
        src[(f, ln)] = s
    tot = sum(ops.values())
    print(f"total warp instructions {tot:,}")
    print("-- opcodes")
    for k, v in ops.most_common(top):
        print(f"{v:14,d} {100 * v / tot:6.2f}%  {k}")
    print("-- source lines")
    for k, v in lines.most_common(top):
        print(f"{v:14,d} {100 * v / tot:6.2f}%  {k[0]}:{k[1]:<5} {src[k][:90]}")


if __name__ == "__main__":
    main()
