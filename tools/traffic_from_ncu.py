"""profiles/gemm_traffic.json from an ncu --set full capture of the tcgen05 GEMM-class launches
of one PinFM-base call (tool, not part of the product):

    ncu --set full --clock-control none -k "regex:k_gemm_tc|k_ffn_tc" -o step_gemms \
        python tools/profile_step.py --calls 1
    python tools/traffic_from_ncu.py step_gemms.ncu-rep > profiles/gemm_traffic.json

Launch labels follow run_dcat's order: context phi_in1, phi_in2, (qkv, tail) x (L-1), kv;
crossing phi_in1, phi_in2, (qkv, tail) x L, phi_out1, phi_out2, head."""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
n_layers = int(sys.argv[2]) if len(sys.argv) > 2 else 4
if rep.endswith(".csv"):  # an exported `ncu -i ... --page raw --csv` (any launches; non-GEMM ones are skipped)
    raw = open(rep).read()
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
while rows and "Kernel Name" not in rows[0]:
    rows = rows[1:]
h = rows[0]
col = {n: i for i, n in enumerate(h)}
labels = ["ctx.phi_in1", "ctx.phi_in2"]
for l in range(n_layers - 1):
    labels += [f"ctx.qkv{l}", f"ctx.tail{l}"]
labels += ["ctx.kv", "cross.phi_in1", "cross.phi_in2"]
for l in range(n_layers):
    labels += [f"cross.qkv{l}", f"cross.tail{l}"]
labels += ["cross.phi_out1", "cross.phi_out2", "head"]


def f(r, name, scale=1.0):
    try:
        return float(r[col[name]].replace(",", "")) * scale
    except (KeyError, ValueError):
        return None


body = rows[2:]
# several calls in the capture: keep the last complete one (it starts at the dedup's k_span and ends
# with k_scatter; a capture can stop mid-call)
starts = [k for k, r in enumerate(body) if len(r) == len(h) and "k_span(" in r[col["Kernel Name"]]] + [len(body)]
calls = [body[a:b] for a, b in zip(starts[:-1], starts[1:])]
complete = [c for c in calls if any(len(r) == len(h) and "k_scatter" in r[col["Kernel Name"]] for r in c)]
if complete:
    body = complete[-1]
launches = []
for k, r in enumerate(body):
    if not r or len(r) != len(h) or not r[col["Kernel Name"]]:
        continue
    if not any(x in r[col["Kernel Name"]] for x in ("k_gemm_tc", "k_ffn_tc")):
        continue
    rd, wr = f(r, "dram__bytes_read.sum"), f(r, "dram__bytes_write.sum")
    launches.append({
        "launch": labels[len(launches)] if len(launches) < len(labels) else f"launch{len(launches)}",
        "kernel": r[col["Kernel Name"]][:60], "us": f(r, "gpu__time_duration.sum"),
        "dram_read_MB": rd, "dram_write_MB": wr,
        "dram_pct": f(r, "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
        "tensor_pct": f(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_pct": f(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "regs": f(r, "launch__registers_per_thread"), "grid": f(r, "launch__grid_size"),
    })
mb = 1e6
tail = [x for x in launches if ".tail" in x["launch"]]
out = {
    "source": "ncu --set full --clock-control none, tools/profile_step.py --calls 1 (PinFM-base 1000x128, L=256), "
              "k_gemm_tc + k_ffn_tc launches of one call",
    "units": "dram_*_MB in MB (1e6 B), us = per-launch duration under ncu (serialised, cold cache)",
    "launches": len(launches),
    "dram_bytes_per_step": sum((x["dram_read_MB"] or 0) + (x["dram_write_MB"] or 0) for x in launches) * mb,
    "sum_us_serialized": round(sum(x["us"] or 0 for x in launches), 2),
    "tail": {"launches": len(tail),
             "dram_bytes_ctx_launch": ((tail[0]["dram_read_MB"] or 0) + (tail[0]["dram_write_MB"] or 0)) * mb
             if tail else None,
             "dram_bytes_per_step": sum((x["dram_read_MB"] or 0) + (x["dram_write_MB"] or 0) for x in tail) * mb,
             "us_serialized": round(sum(x["us"] or 0 for x in tail), 2)},
    "per_launch": launches,
}
json.dump(out, sys.stdout, indent=1)
print()
