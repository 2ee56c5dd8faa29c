"""Build profiles/rNN_summary.md from an ncu launch list (--csv --metrics
gpu__time_duration.sum) and `ncu --set full` reports of the top kernels.
Usage: python tools/profile_report.py RND launches.csv rep1.ncu-rep|raw1.csv [...]"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %peak"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %peak"), ("lts__t_sector_hit_rate.pct", "L2 hit %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("smsp__thread_inst_executed_per_inst_executed.ratio", "lanes/warp-inst"),
        ("launch__registers_per_thread", "regs/thread"), ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long-sb/issue"),
        ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier/issue"),
        ("smsp__inst_executed.sum", "warp insts")]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                out.append((d["Kernel Name"], float(d["Metric Value"]), d["Metric Unit"]))
    starts = [i for i, (k, _, _) in enumerate(out) if k.startswith("lcc::<unnamed>::k_bin")]
    return out[starts[-1]:] if starts else out


def main():
    rnd, lpath, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    seg = launches(lpath)
    tot = sum(v for _, v, _ in seg)
    agg = collections.OrderedDict()
    for k, v, _ in seg:
        name = k[:k.index("(")] if "(" in k else k
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    lines = [f"# Round {rnd} profile summary (B200, bench.py default: R-MAT s24 round 1, async)", "",
             "## Launch list of one step (ncu --metrics gpu__time_duration.sum --clock-control none;",
             "cold-cache, serialised: compare shares, not absolutes)", "",
             f"total {tot/1e6:.3f} ms over {len(seg)} launches", "", "| kernel | launches | ms | share |",
             "|---|---:|---:|---:|"]
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k[-90:]}` | {c} | {v/1e6:.3f} | {100*v/tot:.1f}% |")
    for rep in reps:
        if rep.endswith(".csv"):  # raw-page export made on the GPU box
            rows = list(csv.reader(open(rep)))
        else:
            raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
            rows = list(csv.reader(io.StringIO(raw)))
        if len(rows) < 3:
            continue
        hdr, units = rows[0], rows[1]
        lines += ["", f"## `ncu --set full` — {rep.split('/')[-1]}", ""]
        head = "| metric | " + " | ".join(f"launch {i}" for i in range(len(rows) - 2)) + " |"
        lines += [head, "|---|" + "---:|" * (len(rows) - 2)]
        kn = hdr.index("Kernel Name")
        lines.append("| kernel | " + " | ".join(r[kn].split("(")[0].replace("unnamed>::", "")[-60:] for r in rows[2:]) + " |")
        for key, label in KEYS:
            if key in hdr:
                i = hdr.index(key)
                lines.append(f"| {label} ({units[i]}) | " + " | ".join(r[i] for r in rows[2:]) + " |")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
