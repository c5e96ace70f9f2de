"""clock64 timeline of the fused layer tail inside a real PinFM-base scoring call (kernel
investigation, not the product). Needs a DCAT_FFN_TRACE build of the library:
    tools/build_variant.sh trace "-DDCAT_FFN_TRACE=1"
    DCAT_LIB_PATH=build_variants/lib_trace.so python tools/tail_trace.py [users] [max_events]
Prints the events of the last tail launch (CTAs 0 and 1, first 4 tiles) and per-phase spans."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import pyoracle  # noqa: E402
from paper_2507_12704_b200 import api  # noqa: E402
from paper_2507_12704_b200.abi import FinetuneSpec  # noqa: E402
from paper_2507_12704_b200.synth import CONFIGS, make_batch  # noqa: E402

NAMES = {1: 'F1iss', 2: 'F2iss', 3: 'G.start', 4: 'G.done', 5: 'fin.start', 6: 'fin.rel', 7: 'G.done15',
         8: 'LN2.start', 9: 'tile.end', 10: 'prod.A', 11: 'slot.iss', 12: 'slot.rdy', 13: 'O.issued', 14: 'a2'}
ROLES = ['prod', 'mma', 'epi0', 'epi15']


def main():
    U = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
    lim = int(sys.argv[2]) if len(sys.argv) > 2 else 400
    cfg = CONFIGS["pinfm-base"]
    spec, Cn, L = cfg["spec"], cfg["C"], cfg["L"]
    orc = pyoracle.oracle()
    w = orc.init_weights(spec, 42, table=(8, 4096, spec.d_emb // 8, 7, 0.05), head_seed=11)
    m = api.DcatModel(w)
    ft = FinetuneSpec(max_events=L)
    host = make_batch(U, Cn, L, seed=1)
    dev = host.to(lambda a: torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).cuda())
    for _ in range(2):
        m.rank_forward_batch(dev, ft)
    torch.cuda.synchronize()
    lib = api.lib()
    lib.dcat_ffn_trace_reset()
    m.rank_forward_batch(dev, ft)
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 8192)()
    n = lib.dcat_ffn_trace_read(buf, 8192)
    ev = sorted(((v >> 16), (v >> 8) & 0xFF, v & 0xFF) for v in buf[:n])
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    np.save(os.path.join(ROOT, "gpurun_out", "tail_trace_raw.npy"), np.array(ev, dtype=np.int64))
    t0 = ev[0][0]
    skip = {11, 12}
    k = 0
    for t, c, j in ev:
        role, kind = c >> 4, c & 15
        if kind in skip or role // 4 != 0:
            continue
        print(f"{t - t0:8d} cta{role // 4} {ROLES[role % 4]:6s} {NAMES.get(kind, str(kind)):9s} {j}")
        k += 1
        if k >= lim:
            break
    # ring slots of cta 0: producer issue (after its empty wait) -> MMA issuer sees it full
    iss = [t for t, c, j in ev if c == 0 * 16 + 11]
    rdy = [t for t, c, j in ev if c == 1 * 16 + 12]
    n2 = min(len(iss), len(rdy))
    if n2 > 8:
        lat = np.array(rdy[:n2]) - np.array(iss[:n2])
        print(f"slot issue->seen-full: median={np.median(lat):.0f} p10={np.percentile(lat, 10):.0f} "
              f"p90={np.percentile(lat, 90):.0f} clk over {n2} slots")
        stages = int(os.environ.get("TAIL_RING_SLOTS", "6"))  # DCAT_FFN_STAGES256 of the traced build
        free = np.array(iss[stages:n2]) - np.array(rdy[:n2 - stages])
        print(f"slot seen-full -> re-issued (MMA consume + commit + producer): median={np.median(free):.0f} clk")
    if len(rdy) > 2:
        d = np.diff(rdy)
        print(f"slot.rdy gaps: n={len(d)} median={np.median(d):.0f} p90={np.percentile(d, 90):.0f} clk")


if __name__ == "__main__":
    main()
