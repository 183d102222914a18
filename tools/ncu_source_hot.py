"""Aggregate an ncu source page (--print-source cuda,sass --csv) by CUDA source line:
instructions executed and stall samples per line, hottest first."""
import csv
import sys
from collections import defaultdict


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    hdr = rows[hi]
    col = {h: i for i, h in enumerate(hdr)}
    src_lines = {}
    agg = defaultdict(lambda: [0.0, 0.0])
    fname = ""
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        if len(r) < len(hdr) or not r[0].isdigit():
            continue  # SASS rows (empty line number) and section headers
        cur = (fname, int(r[0]))
        src_lines[cur] = r[1]
        try:
            ie = float(r[col["Instructions Executed"]] or 0)
            st = float(r[col["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        agg[cur][0] += ie
        agg[cur][1] += st
    tot_i = sum(v[0] for v in agg.values()) or 1
    tot_s = sum(v[1] for v in agg.values()) or 1
    print(f"total instructions {tot_i:.3e}, stall samples {tot_s:.0f}")
    for ln, (ie, st) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{ln[0][:10]}:{ln[1]:<5d} inst {100*ie/tot_i:5.1f}%  stall {100*st/tot_s:5.1f}%  {src_lines.get(ln,'')[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
