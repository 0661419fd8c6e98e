"""Summaries for profiles/: (1) a per-kernel share table from an ncu launch-list CSV
(--metrics gpu__time_duration.sum), (2) the key counters of one `ncu --set full`
capture (.ncu-rep, read with `ncu -i ... --page raw --csv`).

  python tools/ncu_summary.py launches gpurun_out/launches.csv
  python tools/ncu_summary.py full gpurun_out/k_solve_pp.ncu-rep
"""
import collections, csv, io, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum",
        "l1tex__t_sector_hit_rate.pct"]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot = collections.Counter(); cnt = collections.Counter(); seq = []
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[h.index("Metric Unit")] if "Metric Unit" in h else "ns"
        us = v * {"ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(unit, 1e-3)
        tot[r[ki]] += us; cnt[r[ki]] += 1
        if "k_solve" in r[ki]:
            seq.append(us)
    T = sum(tot.values())
    for k, v in tot.most_common():
        print(f"{cnt[k]:5d} launches {v:11.1f} us {100 * v / T:5.1f}%  {k[:90]}")
    print("\nk_solve per-launch us (in order): " + ", ".join(f"{x:.0f}" for x in seq))


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"{k:60s} {r[i]:>16s} {units[i]}")
        print()


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
