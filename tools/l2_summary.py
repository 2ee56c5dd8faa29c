"""Summarise tools/prof_l2.sh's ncu CSV: per kernel (summed over its
launches) DRAM bytes, L2 read sectors and hit rate, write / atomic traffic,
fabric sectors, and bytes per scanned entry when the entry count is known.
Usage: python tools/l2_summary.py CSV"""
import collections
import csv
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "ID")
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    seen = set()
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("lcc::<unnamed>::", "").replace("lcc::", "")
        try:
            v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
        except ValueError:
            continue
        per[name][d["Metric Name"]] += v
        if (d["ID"], name) not in seen:
            seen.add((d["ID"], name))
            cnt[name] += 1
    cols = ["launches", "ms", "DRAM rd GB", "DRAM wr GB", "L2 rd sectors G", "rd hit %", "rd req G",
            "wr sectors G", "atom req G", "red req G", "fabric sectors G", "fill sectors G",
            "evict_last hit %", "evict_normal hit %", "evict_first hit %", "inst G"]
    print("| kernel | " + " | ".join(cols) + " |")
    print("|---|" + "---:|" * len(cols))
    for name, m in per.items():
        g = lambda k: m.get(k, 0.0)
        pct = lambda a, b: 100.0 * g(a) / g(b) if g(b) else float("nan")
        vals = [cnt[name], g("gpu__time_duration.sum"), g("dram__bytes_read.sum") / 1e9, g("dram__bytes_write.sum") / 1e9,
                g("lts__t_sectors_srcunit_tex_op_read.sum") / 1e9,
                pct("lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum", "lts__t_sectors_srcunit_tex_op_read.sum"),
                g("lts__t_requests_srcunit_tex_op_read.sum") / 1e9, g("lts__t_sectors_srcunit_tex_op_write.sum") / 1e9,
                g("lts__t_requests_srcunit_tex_op_atom.sum") / 1e9, g("lts__t_requests_srcunit_tex_op_red.sum") / 1e9,
                g("lts__t_sectors_srcunit_ltcfabric.sum") / 1e9, g("lts__d_sectors_fill_device.sum") / 1e9,
                pct("lts__t_requests_srcunit_tex_evict_last_lookup_hit.sum", "lts__t_requests_srcunit_tex_evict_last.sum"),
                pct("lts__t_requests_srcunit_tex_evict_normal_lookup_hit.sum", "lts__t_requests_srcunit_tex_evict_normal.sum"),
                pct("lts__t_requests_srcunit_tex_evict_first_lookup_hit.sum", "lts__t_requests_srcunit_tex_evict_first.sum"),
                g("smsp__inst_executed.sum") / 1e9]
        print(f"| {name[:70]} | " + " | ".join(f"{v:.3g}" if isinstance(v, float) else str(v) for v in vals) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
