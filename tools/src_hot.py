"""Summarise an `ncu --page source --csv --print-source cuda,sass` export:
per CUDA source line, instructions executed and stall samples (top N)."""
import csv
import sys
from collections import defaultdict


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    hdr = rows[hdr_i]
    # the cuda,sass view repeats: cuda lines first (Line No, Source ...), then
    # sass rows with Address; we aggregate the cuda-line rows
    iL, iS = 0, 1
    iX = hdr.index("Instructions Executed")
    iW = hdr.index("Warp Stall Sampling (All Samples)")
    agg = []
    for r in rows[hdr_i + 1:]:
        if len(r) < len(hdr) or not r[0].strip().isdigit():
            continue
        try:
            x = float(r[iX] or 0)
            w = float(r[iW] or 0)
        except ValueError:
            continue
        agg.append((w, x, int(r[iL]), r[iS].strip()[:110]))
    tw = sum(a[0] for a in agg) or 1
    tx = sum(a[1] for a in agg) or 1
    print(f"total stall samples {tw:.0f}, warp insts {tx:.3g}")
    for w, x, ln, src in sorted(agg, reverse=True)[:top]:
        print(f"{100*w/tw:5.1f}% stall {100*x/tx:5.1f}% inst  L{ln:<5} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
