"""Reads the FATRACE lines a DCAT_FA_TRACE build of attn_fa.cu prints (CTA 0 timeline) and shows
one launch's events and per-chunk softmax durations. Usage: python tools/fa_trace.py log [launch] [n]"""
import sys
from collections import defaultdict

NAMES = {10: 'P0kv', 11: 'P1kv', 20: 'M0pfull', 21: 'M1pfull', 30: 'M0kvfull', 31: 'M1kvfull', 40: 'S0wait',
         41: 'S1wait', 50: 'S0got', 51: 'S1got', 60: 'S0pdone', 61: 'S1pdone', 70: 'S0qwait', 71: 'S1qwait',
         80: 'S0qgot', 81: 'S1qgot'}


def main(path, launch=3, n=80):
    blocks = open(path).read().split("FATRACE begin")[1:]
    for li, blk in enumerate(blocks):
        ev = sorted(tuple(map(int, l.split()[1:])) for l in blk.split("\n")[1:] if l.startswith("FATRACE"))
        if not ev:
            continue
        t0 = ev[0][0]
        print(f"launch {li}: {blk.splitlines()[0].strip()} events {len(ev)} span {ev[-1][0] - t0}")
        if li != launch:
            continue
        got, dur, gap = {}, defaultdict(list), defaultdict(list)
        last_done = {}
        for t, c, v in ev:
            if c in (50, 51):
                got[(c - 50, v)] = t
                if (c - 50) in last_done:
                    gap[c - 50].append(t - last_done[c - 50])
            if c in (60, 61) and (c - 60, v) in got:
                dur[c - 60].append(t - got[(c - 60, v)])
                last_done[c - 60] = t
        for g in (0, 1):
            if dur[g]:
                print(f"  pipeline {g}: softmax per chunk mean {sum(dur[g]) / len(dur[g]):.0f} cycles; "
                      f"p_done -> next S mean {sum(gap[g]) / max(1, len(gap[g])):.0f}")
        for t, c, v in ev[:n]:
            print(f"{t - t0:8d} {NAMES.get(c, c):10s} {v}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 3, int(sys.argv[3]) if len(sys.argv) > 3 else 80)
