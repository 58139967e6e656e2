"""Executed-instruction mix per opcode from an ncu report's source page (per unit of work)."""
import collections
import csv
import subprocess
import sys


def mix(path, units):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    ia, isrc = h.index("Instructions Executed"), h.index("Source")
    iss = h.index("Warp Stall Sampling (All Samples)")
    ops, stall, tot = collections.Counter(), collections.Counter(), 0
    for r in rows[2:]:
        try:
            n = int(r[ia])
        except (ValueError, IndexError):
            continue
        tok = r[isrc].strip().split()
        if not tok:
            continue
        o = tok[1] if tok[0].startswith("@") else tok[0]
        o = o.split(".")[0]
        ops[o] += n
        tot += n
        stall[o] += int(r[iss] or 0)
    print(f"== {path}: {tot / units:.1f} instructions per unit")
    for o, n in ops.most_common(22):
        print(f"   {o:10s} {n / units:7.2f}   stall samples {stall[o]}")


if __name__ == "__main__":
    units = float(sys.argv[1])
    for p in sys.argv[2:]:
        mix(p, units)
