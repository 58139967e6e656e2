"""Per-basic-block view of an ncu source page (SASS): consecutive instructions with the same
execution count form a block; prints blocks sorted by total executed instructions, with the
count per unit of work and the opcode mix.  Usage: sass_blocks.py <src.csv> <units>"""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
units = float(sys.argv[2])
h = rows[1]
ia, isrc, iss = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
blocks = []
cur = None
for r in rows[2:]:
    try:
        n = int(r[ia])
    except (ValueError, IndexError):
        continue
    src = r[isrc].strip()
    tok = src.split()
    op = (tok[1] if tok and tok[0].startswith("@") else (tok[0] if tok else "?")).split(".")[0]
    if cur is None or cur["n"] != n:
        cur = {"n": n, "ops": collections.Counter(), "first": src, "addr": r[0], "len": 0, "stall": 0}
        blocks.append(cur)
    cur["ops"][op] += 1
    cur["len"] += 1
    cur["stall"] += int(r[iss] or 0)
tot = sum(b["n"] * b["len"] for b in blocks)
print(f"total {tot / units:.1f} instr/unit")
for b in sorted(blocks, key=lambda b: -b["n"] * b["len"])[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]:
    if b["n"] == 0:
        continue
    print(f"{b['n'] * b['len'] / units:6.2f}/unit  exec/unit {b['n'] / units:6.3f} len {b['len']:4d} stall {b['stall']:7d}  "
          f"{b['addr'][-5:]} {dict(b['ops'].most_common(8))}")
