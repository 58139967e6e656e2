"""Prints the key metrics of .ncu-rep files (run here, no GPU needed)."""
import csv
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem', 'launch__grid_size',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'lts__t_bytes.sum', 'sm__cycles_elapsed.avg.per_second', 'lts__t_sectors_srcunit_tex.sum',
        'lts__t_sectors_srcunit_ltcfabric.sum', 'lts__t_sectors.sum.pct_of_peak_sustained_elapsed']


def summary(path):
    """path: an .ncu-rep, or its `--page raw --csv` export (*.csv)."""
    if path.endswith(".csv"):
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = [r for r in csv.reader(out.splitlines()) if r and not r[0].startswith("==")]
    h, units, v = rows[0], rows[1], rows[2]
    res = {"kernel": v[h.index("Kernel Name")]}
    for k in KEYS:
        if k in h:
            res[k] = (v[h.index(k)], units[h.index(k)])
    stalls = {}
    for i, k in enumerate(h):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                x = float(v[i])
            except ValueError:
                continue
            if x >= 0.05:
                stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = x
    res["stalls"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
    return res


if __name__ == "__main__":
    for p in sys.argv[1:]:
        r = summary(p)
        print("==", p, r.pop("kernel")[:90])
        st = r.pop("stalls")
        for k, (val, u) in r.items():
            print(f"  {k:62s} {val:>18s} {u}")
        print("  stalls/issue:", ", ".join(f"{k}={x:.2f}" for k, x in st.items()))
