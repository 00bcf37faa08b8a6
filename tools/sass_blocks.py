"""Basic-block view of an ncu source page (SASS): consecutive instructions
with the same execution count, ranked by their share of issued instructions.
    ncu -i rep.ncu-rep --page source --csv --print-source sass > src.csv
    python tools/sass_blocks.py src.csv [top] [--dump ADDR_HEX]"""
import collections
import csv
import re
import sys


def blocks(path):
    rows = list(csv.reader(open(path)))
    cut = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
    rows = rows[: cut[1]] if len(cut) > 1 else rows
    hdr = rows[1]
    ia, isrc, ie = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
    ist = hdr.index("Warp Stall Sampling (All Samples)")
    seq = []
    for r in rows[2:]:
        if len(r) <= ie:
            continue
        try:
            seq.append((int(r[ia], 16), r[isrc].strip(), int(r[ie] or 0), int(r[ist] or 0)))
        except ValueError:
            continue
    seq.sort()
    out, cur = [], None
    for a, src, n, st in seq:
        if cur and cur["n"] == n:
            cur["ins"].append(src)
            cur["st"] += st
        else:
            cur = {"a": a, "n": n, "ins": [src], "st": st}
            out.append(cur)
    return out


def main():
    bl = blocks(sys.argv[1])
    top = int(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else 16
    tot = sum(b["n"] * len(b["ins"]) for b in bl)
    print("issued warp instructions", tot)
    for b in sorted(sorted(bl, key=lambda b: -b["n"] * len(b["ins"]))[:top], key=lambda b: b["a"]):
        ops = collections.Counter(m.group(2) for m in (re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", s) for s in b["ins"]) if m)
        dp = sum(v for k, v in ops.items() if k in ("DFMA", "DMUL", "DADD"))
        print(f"{b['a'] & 0xfffff:05x} n={b['n']:>9} len={len(b['ins']):3d} share={100 * b['n'] * len(b['ins']) / tot:5.1f}% "
              f"dp={dp:2d} stall={b['st']:6d} {dict(ops.most_common(5))}")


if __name__ == "__main__":
    main()
