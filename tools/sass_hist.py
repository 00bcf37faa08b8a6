"""Per-opcode histogram of executed SASS instructions from an ncu report:
    ncu -i rep.ncu-rep --page source --csv --print-source sass > src.csv
    python tools/sass_hist.py src.csv [top]"""
import csv
import re
import sys
from collections import Counter


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    cut = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
    rows = rows[: cut[1]] if len(cut) > 1 else rows  # first kernel only
    hdr = rows[1]
    ia, ie, ist = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    ops, stalls, total, seq = Counter(), Counter(), 0, []
    for r in rows[2:]:
        if len(r) <= ie:
            continue
        src = r[ia].strip()
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", src)
        if not m:
            continue
        if not (r[ie] or "0").isdigit():
            continue
        n = int(r[ie] or 0)
        op = m.group(2)
        ops[op] += n
        stalls[op] += int(r[ist] or 0)
        total += n
        seq.append((r[0], src, n, int(r[ist] or 0)))
    print(f"total warp instructions {total:.4g}")
    for op, n in ops.most_common(top):
        print(f"{op:14s} {n:12d} {100 * n / total:6.2f}%  stall samples {stalls[op]}")
    return seq


if __name__ == "__main__":
    seq = main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
    if len(sys.argv) > 3:
        thr = float(sys.argv[3])
        mx = max(n for _, _, n, _ in seq)
        for a, s, n, st in seq:
            if n >= thr * mx:
                print(f"{a[-5:]} {n:11d} {st:6d}  {s}")
