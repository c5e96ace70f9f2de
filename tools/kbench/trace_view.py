"""Print the clock64 event trace written by kbench_trace (DCAT_FFN_TRACE build)."""
import sys

NAMES = {1: 'F1iss', 2: 'F2iss', 3: 'G.start', 4: 'G.done0', 5: 'fin.start', 6: 'fin.rel', 7: 'G.done15',
         9: 'tile.end', 10: 'prod.A'}
txt = open(sys.argv[1]).read()
line = [l for l in txt.split('\n') if l.startswith('TRACE')][0]
ev = sorted(tuple(map(int, x.split(':'))) for x in line.split()[1:])
t0 = ev[0][0]
lim = int(sys.argv[2]) if len(sys.argv) > 2 else 200
for t, c, j in ev[:lim]:
    print(f"{t - t0:8d} {str(NAMES.get(c, c)):10s} {j}")
