"""DRAM traffic of the best-move kernel group per bench step, from the raw
CSV exports of tools/refresh_profiles.sh (groups capture = every group /
small / isolated kernel of one step; hubs capture = the first of the step's
hub batches, scaled by the batch count from the launch list).
Usage: python tools/traffic.py RND  -> profiles/rRND_traffic.json"""
import csv
import json
import sys


def rows(path):
    r = list(csv.reader(open(path)))
    hdr = r[0]
    out = []
    for x in r[2:]:
        if len(x) != len(hdr):
            continue
        d = dict(zip(hdr, x))
        out.append(d)
    return out, r[1]


def val(d, units, key):
    v = float(d[key])
    u = units.get(key, "")
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]


def main(rnd):
    out = {"kernels": {}, "source": f"gpurun_out/r{rnd}_groups_raw.csv + r{rnd}_hubs_raw.csv (ncu --set full)"}
    total = 0.0
    kern_ms = 0.0
    for rep, scale in (("groups", 1), ("hubs", None)):
        rs, unit_row = rows(f"gpurun_out/r{rnd}_{rep}_raw.csv")
        hdr = list(rs[0].keys()) if rs else []
        units = dict(zip(hdr, unit_row))
        if scale is None:  # hub batches per step (global-table path), from the launch list; 1 for buckets
            n = sum(1 for line in open(f"gpurun_out/launches_r{rnd}.csv") if "k_large_insert" in line and
                    "gpu__time_duration" in line)
            scale = max(n, 1)
        for d in rs:
            name = d["Kernel Name"].split("(")[0]
            b = val(d, units, "dram__bytes_read.sum") + val(d, units, "dram__bytes_write.sum")
            t = float(d["gpu__time_duration.sum"]) * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3,
                                                        "ms": 1.0, "msecond": 1.0}[units["gpu__time_duration.sum"]]
            k = out["kernels"].setdefault(name, {"dram_bytes": 0.0, "ms": 0.0, "launches_captured": 0, "scale": scale})
            k["dram_bytes"] += b * scale
            k["ms"] += t * scale
            k["launches_captured"] += 1
            total += b * scale
            kern_ms += t * scale
    out["dram_bytes_per_step"] = total
    out["kernel_ms_per_step_ncu"] = kern_ms
    json.dump(out, open(f"profiles/r{rnd}_traffic.json", "w"), indent=1)
    print(json.dumps({"dram_GB_per_step": total / 1e9, "ncu_kernel_ms": kern_ms}))


if __name__ == "__main__":
    main(sys.argv[1])
