"""Aggregate an `ncu --page source --csv` SASS dump: executed instructions and
stall samples per opcode, plus the top stalled instructions."""
import csv
import re
import sys
from collections import Counter


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
    hdr = rows[hdr_i]
    ci, cs, cx = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    ops, stalls, lines = Counter(), Counter(), []
    for r in rows[hdr_i + 1:]:
        if len(r) <= cx:
            continue
        src = r[ci].strip()
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", src)
        if not m:
            continue
        op = m.group(2)
        try:
            n = int(float(r[cx] or 0))
            s = int(float(r[cs] or 0))
        except ValueError:
            continue
        ops[op] += n
        stalls[op] += s
        lines.append((s, n, r[0], src))
    tot = sum(ops.values())
    print(f"total warp-instructions executed: {tot:.3e}; stall samples {sum(stalls.values())}")
    for op, n in ops.most_common(top):
        print(f"{op:12s} {n:12d} {100 * n / tot:5.1f}%  stalls {stalls[op]}")
    print("--- most stalled instructions")
    for s, n, a, src in sorted(lines, reverse=True)[:top]:
        print(f"{s:6d} {n:10d} {a} {src[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
