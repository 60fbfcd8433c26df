"""Summarise ncu output into profiles/*.md (run here, on the CPU box).

    python tools/summarize_ncu.py launches gpurun_out/launches.csv  > profiles/rNN_launches.md
    python tools/summarize_ncu.py full gpurun_out/prof.ncu-rep      > profiles/rNN_k2_full.md
"""
import collections
import csv
import io
import subprocess
import sys

MINE = ("cs::", "pack_kernel", "unpack_sgd", "p2p_reduce", "stats_kernel")


def launches(path: str) -> None:
    lines = [ln for ln in open(path) if ln.startswith('"')]
    r = csv.reader(lines)
    hdr = next(r)
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for row in r:
        v = float(row[vi].replace(",", ""))
        v *= {"usecond": 1e3, "msecond": 1e6, "nsecond": 1.0}.get(row[ui], 1.0)
        name = row[ki]
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    n = sum(a[0] for a in agg.values())
    print(f"# ncu launch list summary (`{path}`)\n")
    print(f"{n} kernel launches, {tot / 1e6:.3f} ms summed device time "
          "(ncu: serialised, cold-cache -- compare shares, not absolutes).\n")
    print("| share | total ms | launches | avg us | kernel |\n|---:|---:|---:|---:|---|")
    rows = sorted(agg.items(), key=lambda x: -x[1][1])
    for name, (cnt, t) in rows[:25]:
        print(f"| {100 * t / tot:.1f}% | {t / 1e6:.3f} | {cnt} | {t / cnt / 1e3:.1f} | `{name[:110]}` |")
    mine = [(k, v) for k, v in agg.items() if any(m in k for m in MINE)]
    mt = sum(v[1] for _, v in mine)
    print(f"\n## our kernels (libcrossover.so): {100 * mt / tot:.2f}% of device time\n")
    print("| total ms | launches | avg us | kernel |\n|---:|---:|---:|---|")
    for name, (cnt, t) in sorted(mine, key=lambda x: -x[1][1]):
        print(f"| {t / 1e6:.4f} | {cnt} | {t / cnt / 1e3:.2f} | `{name[:110]}` |")


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum"]


def full(path: str) -> None:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary (`{path}`)\n")
    for row in rows[2:]:
        name = row[hdr.index("Kernel Name")]
        print(f"## `{name[:120]}`\n\n| metric | value | unit |\n|---|---:|---|")
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                print(f"| {w} | {row[i]} | {units[i]} |")
        print()


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
