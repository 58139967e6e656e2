"""Records per-launch ncu counters of the profiled passes in profiles/ncu_traffic.json (read by bench.py
for the physical roofline): DRAM bytes (read + write), L2 bytes (lts__t_bytes), executed warp
instructions, issue / DRAM / L2 / L1 utilisation, and the sha256 of the kernel sources the report was
taken from (bench.py flags the numbers as stale when the sources changed since).

Usage: python tools/make_traffic.py [--out PATH] <workload> stage=report.ncu-rep|raw.csv ...
"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import summary  # noqa: E402

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "inst": 1, "%": 1}
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KERNEL_SOURCES = ("paper_2604_16715_b200/csrc/attn_pipe.cu",)   # the three pass kernels


def code_of(text: str) -> str:
    """The source without // comments and blank lines (comment edits do not change the kernels)."""
    out = []
    for line in text.splitlines():
        i = line.find("//")
        line = (line[:i] if i >= 0 else line).rstrip()
        if line:
            out.append(line)
    return "\n".join(out)


def kernel_sha(root=ROOT, texts=None):
    h = hashlib.sha256()
    for i, f in enumerate(KERNEL_SOURCES):
        if texts is not None:
            t = texts[i]
        else:
            with open(os.path.join(root, f)) as fh:
                t = fh.read()
        h.update(code_of(t).encode())
    return h.hexdigest()[:16]


def val(r, k):
    if k not in r:
        return None
    v, u = r[k]
    try:
        return float(v.replace(",", "")) * UNIT.get(u, 1)
    except ValueError:
        return None


def ms(r):
    v, u = r["gpu__time_duration.sum"]
    return float(v.replace(",", "")) * {"msecond": 1.0, "ms": 1.0, "usecond": 1e-3, "us": 1e-3, "nsecond": 1e-6,
                                        "ns": 1e-6, "second": 1e3}.get(u, 1.0)


def main(argv):
    out = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if argv and argv[0] == "--out":
        out, argv = argv[1], argv[2:]
    data = json.load(open(out)) if os.path.exists(out) else {}
    wl = argv[0]
    for arg in argv[1:]:
        stage, rep = arg.split("=", 1)
        r = summary(rep)
        rec = {
            "dram_bytes": (val(r, "dram__bytes_read.sum") or 0) + (val(r, "dram__bytes_write.sum") or 0),
            # bytes the SMs requested from L2 (L1TEX-sourced sectors x 32 B): the L2 -> SM roofline's numerator
            "l2_bytes": (val(r, "lts__t_sectors_srcunit_tex.sum") or 0) * 32 or val(r, "lts__t_bytes.sum"),
            "l2_fabric_bytes": (val(r, "lts__t_sectors_srcunit_ltcfabric.sum") or 0) * 32,
            "inst": val(r, "smsp__inst_executed.sum"),
            "ncu_ms": ms(r),
            "issue_active_pct": val(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "dram_pct": val(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "l2_pct": val(r, "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
            "l1_pct": val(r, "l1tex__throughput.avg.pct_of_peak_sustained_active"),
            "l2_hit_pct": val(r, "lts__t_sector_hit_rate.pct"),
            "warps_active_pct": val(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
            "kernel": r["kernel"][:120],
            "kernel_sha": kernel_sha(),
            "report": os.path.basename(rep),
        }
        data.setdefault(wl, {})[stage] = rec
        print(wl, stage, f"dram {rec['dram_bytes'] / 1e9:.2f} GB, l2 {(rec['l2_bytes'] or 0) / 1e9:.2f} GB, "
                         f"issue {rec['issue_active_pct']} %")
    json.dump(data, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
