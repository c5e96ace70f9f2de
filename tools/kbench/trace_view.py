"""Print the clock64 event trace written by kbench_trace (DCAT_FFN_TRACE build).

Event code = 16 * role + kind; role = 4 * cta + (0 producer, 1 MMA issuer, 2 epilogue warp 0,
3 epilogue warp 15). Usage: trace_view.py trace.txt [max_events] [skip_kinds, e.g. 11,12]"""
import sys

NAMES = {1: 'F1iss', 2: 'F2iss', 3: 'G.start', 4: 'G.done', 5: 'fin.start', 6: 'fin.rel', 7: 'G.done',
         9: 'tile.end', 10: 'prod.A', 11: 'slot.iss', 12: 'slot.rdy'}
ROLES = ['prod', 'mma', 'epi0', 'epi15']
txt = open(sys.argv[1]).read()
line = [l for l in txt.split('\n') if l.startswith('TRACE')][0]
ev = sorted(tuple(map(int, x.split(':'))) for x in line.split()[1:])
t0 = ev[0][0]
lim = int(sys.argv[2]) if len(sys.argv) > 2 else 200
skip = {int(x) for x in sys.argv[3].split(',')} if len(sys.argv) > 3 else set()
n = 0
for t, c, j in ev:
    role, kind = c >> 4, c & 15
    if kind in skip:
        continue
    print(f"{t - t0:8d} cta{role // 4} {ROLES[role % 4]:6s} {NAMES.get(kind, str(kind)):9s} {j}")
    n += 1
    if n >= lim:
        break
