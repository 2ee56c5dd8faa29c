"""DRAM traffic of one bench step's best-move kernels, from an ncu metrics
CSV (tools/prof_round.sh): every best-move kernel launch of the step with
gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum.
Usage: python tools/traffic_step.py CSV CFG TAG -> profiles/TAG_traffic_CFG.json"""
import collections
import csv
import json
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
         "ns": 1e-6, "us": 1e-3, "ms": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "second": 1e3}
BEST = ("k_group", "k_small", "k_tiny", "k_isolated", "k_hub_", "k_large_", "k_window")


def main(path, cfg, tag):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "ID")
    i0 = rows.index(hdr)
    per = collections.defaultdict(dict)
    for r in rows[i0 + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"]
        if not any(b in name for b in BEST):
            continue
        v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
        per[(int(d["ID"]), name)][d["Metric Name"]] = v
    kernels = collections.OrderedDict()
    tot_b = tot_ms = 0.0
    for (lid, name), m in sorted(per.items()):
        short = name.split("(")[0].replace("lcc::<unnamed>::", "")
        k = kernels.setdefault(short, {"launches": 0, "dram_bytes": 0.0, "ms": 0.0})
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        k["launches"] += 1
        k["dram_bytes"] += b
        k["ms"] += m.get("gpu__time_duration.sum", 0.0)
        tot_b += b
        tot_ms += m.get("gpu__time_duration.sum", 0.0)
    out = {"config": cfg, "dram_bytes_per_step": tot_b, "kernel_ms_cold_serialised": tot_ms,
           "dram_gbs_while_running": tot_b / (tot_ms / 1e3) / 1e9 if tot_ms else None,
           "kernels": kernels,
           "source": f"{path} (ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                     f"--clock-control none, one bench step)"}
    json.dump(out, open(f"profiles/{tag}_traffic_{cfg}.json", "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "kernels"}))


if __name__ == "__main__":
    main(*sys.argv[1:4])
