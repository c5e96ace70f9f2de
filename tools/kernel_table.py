"""profiles/r01_kernels.md from a `ncu --set full` raw CSV of one PinFM-base call (tool, not the
product):

    ncu --set full --clock-control none -o call python tools/profile_step.py --calls 1
    ncu -i call.ncu-rep --page raw --csv > call_raw.csv
    python tools/kernel_table.py call_raw.csv > profiles/r01_kernels.md

With `--calls 3` the last complete call is tabulated (the second one: captured into the cached
graph and launched from it).

One row per launch: ncu duration (serialised, cold L2: compare shares, not absolutes), DRAM bytes,
achieved DRAM GB/s and its fraction of the measured HBM peak, tensor-pipe utilisation, issue
utilisation. Launch labels follow run_dcat's order (PinFM-base, 4 layers)."""
import csv
import json
import os
import re
import sys

raw = list(csv.reader(open(sys.argv[1])))
i = 0
while "Kernel Name" not in raw[i]:
    i += 1
h = raw[i]
rows = [r for r in raw[i + 2:] if len(r) == len(h) and r[h.index("Kernel Name")]]
col = {n: k for k, n in enumerate(h)}
# several calls in the capture: keep the last one (calls start at the dedup's first kernel, k_span;
# a steady-state call replays the cached graphs)
starts = [k for k, r in enumerate(rows) if "k_span(" in r[col["Kernel Name"]]] + [len(rows)]
calls = [rows[a:b] for a, b in zip(starts[:-1], starts[1:])]
complete = [c for c in calls if any("k_scatter" in r[col["Kernel Name"]] for r in c)]
if complete:  # the last call that ran to its end (a capture can stop mid-call)
    rows = complete[-1]
peaks = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
hbm_peak = 6545.6
try:
    pk = json.load(open(peaks))
    for k, v in pk.items():
        if "hbm" in k.lower() and isinstance(v, (int, float)):
            hbm_peak = float(v)
except (OSError, ValueError):
    pass


def f(r, name):
    try:
        return float(r[col[name]].replace(",", ""))
    except (KeyError, ValueError):
        return None


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = name.replace("void ", "").replace("__nv_bfloat16", "bf16")
    name = re.sub(r"^.*?::(?=k_)", "", name)  # "dcat::<unnamed>::" / "unnamed>::" (ncu versions)
    return name.strip()


n_layers = 4
ctx = ["gather_ctx", "phi_in1", "phi_in2"]
for l in range(n_layers - 1):
    ctx += [f"qkv{l}", f"attn{l}", f"tail{l}"]
ctx += ["kv"]
cross = ["gather_cand", "phi_in1", "phi_in2"]
for l in range(n_layers):
    cross += [f"qkv{l}", f"attn{l}", f"tail{l}"]
cross += ["phi_out1", "phi_out2", "head", "scatter"]
labels = iter(["ctx." + x for x in ctx] + ["cross." + x for x in cross])

print("# Round 1 — every kernel of one PinFM-base call under `ncu --set full`\n")
print("B200, 1000 users x 128 candidates, L = 256, 4 layers, d = 256, 8 heads; "
      "`tools/profile_step.py --calls 3` (the last complete call, launched from the cached graph), `--clock-control none`. ncu serialises launches and runs "
      "each one cold, so the durations are per-launch and the step's real time is in `bench.py`; "
      f"DRAM % is against the measured HBM peak {hbm_peak:.1f} GB/s (MEASURED_PEAKS.json).\n")
print("| # | stage | kernel | us | DRAM MB (r+w) | DRAM GB/s | % HBM peak | tensor pipe % | issue % |")
print("|---|---|---|---|---|---|---|---|---|")
tot_us = 0.0
dedup_us = 0.0
for k, r in enumerate(rows):
    name = short(r[col["Kernel Name"]])
    us = f(r, "gpu__time_duration.sum") or 0.0
    rd, wr = f(r, "dram__bytes_read.sum") or 0.0, f(r, "dram__bytes_write.sum") or 0.0
    unit = raw[i + 1][col["dram__bytes_read.sum"]]
    scale = {"Mbyte": 1.0, "Kbyte": 1e-3, "Gbyte": 1e3, "byte": 1e-6}.get(unit, 1.0)
    mb = (rd + wr) * scale
    gbs = mb / us * 1e3 if us else 0.0  # MB/us = TB/s
    tp = f(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")
    iss = f(r, "smsp__issue_active.avg.pct_of_peak_sustained_active")
    if name.startswith("at::") or "reduce_kernel" in name or "elementwise" in name:
        continue  # the tool's own torch reductions
    if not name.startswith(("k_gather", "k_gemm", "k_ffn", "k_flash", "k_attn", "k_scatter")):
        dedup_us += us
        tot_us += us
        continue
    label = next(labels, "")
    tot_us += us
    print(f"| {k} | {label} | `{name}` | {us:.1f} | {mb:.1f} | {gbs:.0f} | {100 * gbs / hbm_peak:.1f} | "
          f"{tp if tp is not None else float('nan'):.1f} | {iss if iss is not None else float('nan'):.1f} |")
print(f"\nDedup / plan kernels (dedup.cu, {sum(1 for r in rows if not short(r[col['Kernel Name']]).startswith(('k_gather', 'k_gemm', 'k_ffn', 'k_flash', 'k_attn', 'k_scatter', 'at::')))} launches): "
      f"{dedup_us:.1f} us serialised; integer / byte work, each launch a few us.\n")
print(f"Sum of all launches (serialised): {tot_us / 1e3:.3f} ms.")
