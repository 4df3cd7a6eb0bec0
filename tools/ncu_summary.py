"""Summarise ncu outputs into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py launches <launches.csv> <out.txt> [title]
    python tools/ncu_summary.py full <report.ncu-rep> <out.txt> [title]
"""
import collections
import csv
import io
import subprocess
import sys

FULL_KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size",
]


def launches(path, out, title):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[i], rows[i + 1:]
    ki, mi, vi, idi = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    by = collections.OrderedDict()
    for r in data:
        by.setdefault(r[idi], {"name": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
    seq = list(by.values())
    idx = [j for j, s in enumerate(seq) if "k_prep" in s["name"] and "finish" not in s["name"]]
    if len(idx) >= 2:
        st, en = idx[-2], idx[-1]
    else:  # one profiled iteration (tools/ncu_iteration.py): up to the cone step
        st = idx[0]
        tail = [j for j, s in enumerate(seq) if j > st and "k_cone_apply" in s["name"]]
        en = (tail[0] + 1) if tail else len(seq)
        while en < len(seq) and "k_psd" in seq[en]["name"]:  # PSD kernels after k_cone_apply
            en += 1
    lines = [f"# {title}", "# one ADMM iteration (the last complete one in the capture);",
             "# ncu per-launch times are cold-cache and serialised: compare shares",
             f"{'kernel':64s} {'us':>9s} {'share':>6s} {'DRAM rd GB':>10s} {'wr GB':>7s} {'L2 hit %':>8s}"]
    tot = sum(s["gpu__time_duration.sum"] for s in seq[st:en])
    for s in seq[st:en]:
        t = s["gpu__time_duration.sum"]
        lines.append(f"{s['name'][:64]:64s} {t / 1e3:9.1f} {100 * t / tot:5.1f}% "
                     f"{s.get('dram__bytes_read.sum', 0) / 1e9:10.3f} "
                     f"{s.get('dram__bytes_write.sum', 0) / 1e9:7.3f} "
                     f"{s.get('lts__t_sector_hit_rate.pct', 0):8.1f}")
    lines.append(f"{'total':64s} {tot / 1e3:9.1f}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(path, out, title):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    lines = [f"# {title}", f"# source: {path} (ncu --set full --clock-control none)", ""]
    for r in rows[2:]:
        for k in FULL_KEYS:
            if k in hdr:
                j = hdr.index(k)
                lines.append(f"{k:75s} {r[j]} {units[j]}")
        stall = [(float(r[j] or 0), hdr[j]) for j in range(len(hdr))
                 if hdr[j].startswith("smsp__average_warps_issue_stalled_")
                 and hdr[j].endswith("_per_issue_active.ratio")]
        for v, h in sorted(stall, reverse=True)[:5]:
            lines.append(f"  stall {h[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:30s} {v:.2f}")
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:40]))


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    title = sys.argv[4] if len(sys.argv) > 4 else src
    (launches if mode == "launches" else full)(src, dst, title)
