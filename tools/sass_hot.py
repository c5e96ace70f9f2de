"""Summarise an `ncu --page source --csv --print-source sass` dump: stall samples and executed
instructions per opcode, and the hottest SASS lines. Usage: python tools/sass_hot.py dump.csv [N]"""
import csv
import sys
from collections import Counter


def main(path, n=30):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if "Source" in r and "Address" in r)
    iS, iE, iSrc = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"), hdr.index("Source")
    data = [r for r in rows if len(r) == len(hdr) and r[iS].isdigit()]
    tot = sum(int(r[iS]) for r in data)
    c, e = Counter(), Counter()
    for r in data:
        t = r[iSrc].split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        c[op] += int(r[iS])
        e[op] += int(r[iE] or 0)
    print("total stall samples", tot)
    for op, v in c.most_common(22):
        print(f"{op:12s} samples {v:6d} ({100 * v / max(tot, 1):4.1f}%) executed {e[op]}")
    print()
    for r in sorted(data, key=lambda r: -int(r[iS]))[:n]:
        print(r[0][-5:], r[iS], r[iE], r[iSrc][:100])


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
