"""DCAT scoring benchmark (BASELINE.json metric: candidates scored / s).

One step = one rank_forward_batch over one request batch of synthetic input:
dedup -> context pass -> crossing pass -> ranking head, per GPU the PinFM-base
workload (BASELINE.json configs[1]: 4 layers, d=256, 8 heads, L=256, 1000 unique
users x 128 candidates). Multi-GPU (torchrun): every rank scores its own
user-disjoint batch (weak scaling), scores are gathered to rank 0 over NCCL
inside the timed region, time = max over ranks.

  value : device-resident inputs (CUDA events around each step; L2 flushed
          between steps), candidates/s summed over ranks.
  e2e   : the same call through the public API with pinned HOST buffers:
          H2D of the batch and D2H of the logits inside the timed region.
  --impl reference : the reference's own CPU implementation (oracle/_ref, the
          unmodified reference sources; rank_forward_batch fanned out over all
          host threads) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2507_12704_b200.abi import Batch, FinetuneSpec  # noqa: E402
from paper_2507_12704_b200.synth import CONFIGS, init_weights, make_batch  # noqa: E402

METRIC = "candidates scored/sec (seq len L, C cands/user) at 1/2/4/8 B200; vs CPU ref"
UNIT = "candidates/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p["bf16_tflops_sustained"], "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


def gemm_flops(cfg, U, C, L):
    """Algorithmic GEMM flops per batch: per unique user
    L*(2*de*d + 2*d^2) + (l-1)*L*24d^2 + L*4d^2, per candidate
    (2*de*d + 2d^2) + l*24d^2 + 4d^2 + 2(2d+8)*64 (head; the 64x3 tail is epilogue FFMA)."""
    s = cfg["spec"]
    d, de, nl = s.d_model, s.d_emb, s.n_layers
    per_user = L * (2 * de * d + 2 * d * d) + (nl - 1) * L * 24 * d * d + L * 4 * d * d
    per_cand = (2 * de * d + 2 * d * d) + nl * 24 * d * d + 4 * d * d + 2 * (d + de + 8) * 64
    return U * per_user + U * C * per_cand


def gemm_bytes(cfg, U, C, L):
    """Algorithmic HBM bytes of all tcgen05 GEMM-class launches of one step, as the fused
    kernels move them (bf16 activations, fp32 residual stream; weights are L2-resident):
    per row phi_in1 (E in, h1 out) + phi_in2 (h1 in, x + LN1 rows out); per full layer
    qkv (2d in, 6d out) + the fused layer tail (attention rows 2d + x 4d in, x 4d + next-LN
    rows 2d out; x_mid, LN2 rows and the d_ff-wide hidden never reach HBM); last context
    layer kv (2d in, 4d out); per candidate phi_out and the ranking head."""
    s = cfg["spec"]
    d, de, nl = s.d_model, s.d_emb, s.n_layers
    b2, b4 = 2, 4
    phi_in = (de * b2 + d * b2) + (d * b2 + d * b4 + d * b2)
    layer = (d * b2 + 3 * d * b2) + tail_row_bytes(cfg)
    kv = d * b2 + 2 * d * b2
    kh = (d + de + 8 + 63) // 64 * 64
    per_user = L * (phi_in + (nl - 1) * layer + kv)
    per_cand = phi_in + nl * layer + (d * b2 + d * b2) + (d * b2 + d * b2 + 12) + (kh * b2 + 12)
    return U * per_user + U * C * per_cand


def tail_row_bytes(cfg):
    """Fused layer tail, HBM bytes per row: attention output (bf16) and x (fp32) in, x and the
    next LN1 rows (bf16) out = 12 d."""
    d = cfg["spec"].d_model
    return d * 2 + d * 4 + d * 4 + d * 2


def tail_rows(cfg, U, C, L):
    """Rows through the layer tail per step: L - 1 full context layers per unique user, L
    crossing layers per candidate (valid = L synthetic sequences)."""
    nl = cfg["spec"].n_layers
    return U * L * (nl - 1) + U * C * nl


def tail_flops(cfg, U, C, L):
    """Fused layer tail FLOPs per step: output projection 2 d^2 + FFN 4 d d_ff per row."""
    s = cfg["spec"]
    return tail_rows(cfg, U, C, L) * (2 * s.d_model * s.d_model + 4 * s.d_model * s.d_ff)


def attn_flops(cfg, U, C, L):
    s = cfg["spec"]
    d, nl = s.d_model, s.n_layers
    ctx = (nl - 1) * 2 * d * L * (L + 1) * U
    cross = nl * 4 * d * (L + 1) * U * C
    return ctx, cross


class Clocks:
    """nvidia-smi sampling during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            try:
                a, b, r = [x.strip() for x in line.split(",")]
                self.samples.append((float(a), float(b), int(r, 16) if r.startswith("0x") else int(r)))
            except Exception:
                pass

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        busy = [s for s in self.samples if not (s[2] & 0x1)] or self.samples
        reasons = set()
        for s in busy:
            for bit, name in self.REASONS.items():
                if s[2] & bit and bit != 0x1:
                    reasons.add(name)
        return {"sm_mhz": float(np.median([s[0] for s in busy])), "sm_max_mhz": float(max(s[1] for s in busy)),
                "reasons": sorted(reasons), "samples": len(busy)}


def to_torch(a, device):
    import torch
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    t = torch.from_numpy(np.ascontiguousarray(a))
    return t.to(device) if device != "pinned" else t.pin_memory()


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2507_12704_b200 import api

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = CONFIGS[args.config]
    U, C, L = cfg["U"], cfg["C"], cfg["L"]
    if args.users:
        U = args.users
    spec = cfg["spec"]
    w = init_weights(spec, seed=42)
    ft = FinetuneSpec(max_events=L)
    # the request batch of the whole job: U users per GPU; each rank keeps the
    # user-disjoint shard of its content hash (sharding.py), scores it, and the
    # scores are gathered to rank 0 in the global row order (one NCCL gather)
    from paper_2507_12704_b200.sharding import ScoreGather
    from paper_2507_12704_b200.sharding import local_batch, shard_rows
    glob = make_batch(U * world, C, L, seed=1, layout="interleaved", shared_storage=not args.private_rows)
    shards = shard_rows(glob, world, spec.n_layers, spec.d_model, spec.n_heads, spec.d_emb)
    host = local_batch(glob, shards[rank]) if world > 1 else glob
    B = host.n_rows
    B_total = glob.n_rows
    model = api.DcatModel(w, device=local_rank)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    dbatch = host.to(lambda a: to_torch(a, dev))
    out_dev = (torch.empty((B, 3), device=dev), torch.empty((B, 3), device=dev), None)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    sg = ScoreGather(shards, B_total, (3, 3), dev) if world > 1 else None

    def gather_scores(lg, ml):
        if world == 1:
            return
        sg(lg, ml)

    def step_device(profile=False):
        lg, ml, _ = model.rank_forward_batch(dbatch, ft, stream=sp, out=out_dev, profile=profile)
        gather_scores(lg, ml)

    clocks = Clocks(local_rank)  # sampled from warm-up through the e2e steps (>= 100 ms of load)
    clocks.start()
    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    stage_tot = {}
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.zero_()  # L2 flush (256 MB > 126 MB L2), outside the timed span
        ev[k][0].record(stream)
        step_device()
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_dev = sum(a.elapsed_time(b) for a, b in ev)
    stats = model.last_stats()
    # per-stage device times (roofline / kernels / stages_ms) from a separate, untimed pass of the
    # same steps with the library's stage events on: the markers and their read-back are
    # instrumentation, not part of a scoring call
    for k in range(args.steps):
        flush.zero_()
        step_device(profile=True)
        for n, v in model.stage_times().items():
            stage_tot[n] = stage_tot.get(n, 0.0) + v
    torch.cuda.synchronize()

    # ---- e2e through the public API with pinned host buffers
    pinned = host.to(lambda a: to_torch(a, "pinned"))
    hbatch = pinned.to(lambda t: t.numpy())
    hbatch.ev_ts = hbatch.ev_ts.view(np.uint64)
    hbatch.ev_item = hbatch.ev_item.view(np.uint64)
    hbatch.candidate = hbatch.candidate.view(np.uint64)
    h_out = tuple(torch.empty((B, 3), dtype=torch.float32).pin_memory().numpy() for _ in range(2)) + (None,)
    h2d = sum(int(getattr(host, f).nbytes) for f in ("row_offset", "row_valid", "ev_ts", "ev_action", "ev_surface",
                                                     "ev_item", "candidate", "age_seconds"))
    d2h = 2 * B * 3 * 4

    def step_host():
        lg, ml, _ = model.rank_forward_batch(hbatch, ft, stream=sp, out=h_out)
        if world > 1:
            gather_scores(torch.from_numpy(lg).to(dev), torch.from_numpy(ml).to(dev))

    for _ in range(max(1, args.warmup)):
        step_host()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2e_ms = 0.0
    for k in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        ev[k][0].record(stream)
        step_host()
        ev[k][1].record(stream)
        torch.cuda.synchronize()
        e2e_ms += ev[k][0].elapsed_time(ev[k][1])

    clk = clocks.stop()

    # ---- private-rows variant (every row its own event copy, like std::vector<RankingExample>):
    # device-resident, and end to end from pinned host buffers (the whole event pool crosses PCIe)
    priv = priv_e2e = None
    priv_h2d = 0
    if not args.private_rows and not args.no_private and world == 1:
        pb = make_batch(U, C, L, seed=1 + 1000 * rank, layout="interleaved", shared_storage=False)
        pbd = pb.to(lambda a: to_torch(a, dev))
        model.rank_forward_batch(pbd, ft, stream=sp, out=out_dev)
        torch.cuda.synchronize()
        pms = 0.0
        for k in range(max(1, args.steps // 2)):
            flush.zero_()
            ev[k][0].record(stream)
            model.rank_forward_batch(pbd, ft, stream=sp, out=out_dev)
            ev[k][1].record(stream)
            torch.cuda.synchronize()
            pms += ev[k][0].elapsed_time(ev[k][1])
        priv = pms / max(1, args.steps // 2)
        del pbd
        ppin = pb.to(lambda a: to_torch(a, "pinned"))
        phb = ppin.to(lambda t: t.numpy())
        for f in ("ev_ts", "ev_item", "candidate"):
            setattr(phb, f, getattr(phb, f).view(np.uint64))
        priv_h2d = sum(int(getattr(pb, f).nbytes) for f in ("row_offset", "row_valid", "ev_ts", "ev_action",
                                                            "ev_surface", "ev_item", "candidate", "age_seconds"))
        model.rank_forward_batch(phb, ft, stream=sp, out=h_out)
        torch.cuda.synchronize()
        pe = 0.0
        for k in range(max(1, args.steps // 2)):
            flush.zero_()
            torch.cuda.synchronize()
            ev[k][0].record(stream)
            model.rank_forward_batch(phb, ft, stream=sp, out=h_out)
            ev[k][1].record(stream)
            torch.cuda.synchronize()
            pe += ev[k][0].elapsed_time(ev[k][1])
        priv_e2e = pe / max(1, args.steps // 2)
        del ppin, phb

    # N > 1 diagnostics: every rank's own device ms per step, and the score gather timed alone
    per_rank = [ms_dev / args.steps]
    gather_ms = None
    if world > 1:
        lg0, ml0 = out_dev[0], out_dev[1]
        dist.barrier()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            gather_scores(lg0, ml0)
        g1.record(stream)
        torch.cuda.synchronize()
        gather_ms = g0.elapsed_time(g1) / args.steps
        pr = torch.zeros(world, device=dev, dtype=torch.float64)
        pr[rank] = ms_dev / args.steps
        dist.all_reduce(pr)
        per_rank = [round(float(x), 4) for x in pr.tolist()]
    t = torch.tensor([ms_dev, e2e_ms, priv or 0.0, gather_ms or 0.0], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        gather_ms = float(t[3])
    ms_dev, e2e_ms, priv = float(t[0]), float(t[1]), (float(t[2]) if priv is not None else None)
    if rank != 0:
        return None

    K = args.steps
    ms_step = ms_dev / K
    value = B_total / (ms_step / 1e3)
    hbm, tf_burst, tf_sus, peak_kind = peaks()
    # GEMM class: every tcgen05 GEMM-class launch (k_gemm_tc + the fused layer tail)
    gemm_ms = sum(v for n, v in stage_tot.items() if n.startswith("gemm.")) / K
    U_loc = B // C  # unique users of this rank (rank 0 reports)
    gf = gemm_flops(cfg, U_loc, C, L)
    gb = gemm_bytes(cfg, U_loc, C, L)
    achieved = gf / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else None
    # dominant kernel: the fused layer tail (k_ffn_tc<d, 1, true>), all its launches of a step
    tail_ms = sum(v for n, v in stage_tot.items() if n.endswith(".tail")) / K
    n_tail = 2 * cfg["spec"].n_layers - 1  # tail launches per step: L - 1 context + L crossing layers
    tf_tail = tail_flops(cfg, U_loc, C, L)
    tb_tail = tail_rows(cfg, U_loc, C, L) * tail_row_bytes(cfg)
    ctx_f, cross_f = attn_flops(cfg, U, C, L)
    attn_ctx_ms = stage_tot.get("attn.ctx", 0.0) / K
    attn_cross_ms = stage_tot.get("attn.cross", 0.0) / K
    s = spec
    kv_bytes = s.n_layers * 4 * U * L * s.d_model + B * s.n_layers * 8 * s.d_model
    # measured DRAM bytes (dram__bytes_read + write) of the same launches from the committed
    # ncu --set full capture (profiles/gemm_traffic.json, tools/traffic_from_ncu.py), per step
    traffic = tail_traffic = None
    tp = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(tp) and args.config == "pinfm-base" and U_loc == CONFIGS["pinfm-base"]["U"]:
        try:
            tj = json.load(open(tp))
            traffic = tj.get("dram_bytes_per_step")
            tail_traffic = tj.get("tail", {}).get("dram_bytes_per_step")
        except Exception:
            traffic = tail_traffic = None
    stages = {n: round(v / K, 4) for n, v in sorted(stage_tot.items())}
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (seeded run_bench recipe, dcat.cpp:493-521; random-init weights)",
        "config": {"workload": f"{args.config}: {s.n_layers} layers, d={s.d_model}, {s.n_heads} heads, L={L}, "
                               f"{U} unique users x {C} candidates per GPU",
                   "unique_users_per_gpu": U, "cands_per_user": C, "seq_len": L, "rows_per_gpu": B, "rows_total": B_total,
                   "input": "private per-row event copies" if args.private_rows else
                            "CSR event pool, rows of one user share one event span: dedup content-hashes one row "
                            "per distinct span and settles the other rows by span identity (offset, valid); "
                            "e2e_private_rows gives every row its own event copy",
                   "l2": "256 MB buffer written between timed steps; per-step working set ~3 GB > 126 MB L2",
                   "parallelism": f"user-sharded x{world}, NCCL score gather"},
        "e2e": {"value": round(B_total / (e2e_ms / K / 1e3), 1), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms / K, 4)},
        "gpu_launches": int(stats["kernel_launches"]) * K,
        # dominant kernel: the fused layer tail (output projection + residual + LN2 + FFN +
        # residual + next LN1), ~45 % of the step. Per HBM byte it does 2 d^2 + 4 d d_ff flops over
        # 12 d bytes (~380 flop/B at d = 256), above the B200 ridge (1348.6 TF/s / 6545.6 GB/s
        # ~ 206 flop/B): tensor bound by the roofline. What binds it in practice is the per-SM
        # L2 -> SM interface that streams the 1.1 MB of weights per 128-row tile
        # (profiles/r01_ffn.md: ~27 B/clk per SM, loads and stores together).
        "roofline": {"bound": "tensor", "kernel": "k_ffn_tc<d, 1, TAIL> (fused layer tail, all launches of a step)",
                     "achieved": round(tf_tail / (tail_ms / 1e3) / 1e12, 1) if tail_ms else None,
                     "peak": tf_sus, "unit": "TFLOP/s",
                     "frac": round(tf_tail / (tail_ms / 1e3) / 1e12 / tf_sus, 4) if tail_ms else None,
                     "peak_kind": "sustained dense bf16 (MEASURED_PEAKS.json)",
                     "traffic": round(tail_traffic / n_tail) if tail_traffic else None,
                     "traffic_note": "ncu dram bytes per launch, mean over the step's tail launches",
                     "algorithmic_bytes_per_launch": round(tb_tail / n_tail), "flops_per_step": tf_tail,
                     "ms_per_step": round(tail_ms, 4), "share_of_step": round(tail_ms / ms_step, 3),
                     "hbm": {"achieved_gbs": round(tb_tail / (tail_ms / 1e3) / 1e9, 1) if tail_ms else None,
                             "frac": round(tb_tail / (tail_ms / 1e3) / 1e9 / hbm, 4) if tail_ms else None}},
        "gemm_class": {"kernels": "k_gemm_tc + layer tail (all tcgen05 GEMM launches of a step, fused epilogues)",
                       "ms_per_step": round(gemm_ms, 4), "share_of_step": round(gemm_ms / ms_step, 3),
                       "hbm_achieved_gbs": round(gb / (gemm_ms / 1e3) / 1e9, 1) if gemm_ms else None,
                       "hbm_frac": round(gb / (gemm_ms / 1e3) / 1e9 / hbm, 4) if gemm_ms else None,
                       "algorithmic_bytes_per_step": gb, "dram_traffic_per_step": traffic,
                       "tensor_achieved_tflops": round(achieved, 1) if achieved else None,
                       "tensor_frac": round(achieved / tf_sus, 4) if achieved else None, "flops_per_step": gf},
        "kernels": {
            "attn.ctx": {"ms": round(attn_ctx_ms, 4), "tflops": round(ctx_f / (attn_ctx_ms / 1e3) / 1e12, 1)
                         if attn_ctx_ms else None},
            "attn.cross": {"ms": round(attn_cross_ms, 4),
                           "tflops": round(cross_f / (attn_cross_ms / 1e3) / 1e12, 1) if attn_cross_ms else None,
                           "hbm_gbs": round(kv_bytes / (attn_cross_ms / 1e3) / 1e9, 1) if attn_cross_ms else None,
                           "hbm_frac": round(kv_bytes / (attn_cross_ms / 1e3) / 1e9 / hbm, 4) if attn_cross_ms else None},
        },
        "stages_ms": stages,
        "clocks": clk,
    }
    if priv:
        line["value_private_rows"] = round(B_total / (priv / 1e3), 1)
    if priv_e2e:
        line["e2e_private_rows"] = {"value": round(B_total / (priv_e2e / 1e3), 1), "unit": UNIT,
                                    "h2d_bytes_per_step": priv_h2d, "d2h_bytes_per_step": d2h,
                                    "ms_per_step": round(priv_e2e, 4),
                                    "input": "every row its own event copy in pinned host memory (the layout a "
                                             "std::vector<RankingExample> packs to); H2D of all of it inside the timed region"}
    if world == 1 and not args.no_shim:
        shim = bench_shim(args, U, C, L, spec)
        if shim:
            line["e2e_shim"] = shim
    if world > 1:
        line["per_rank_ms_per_step"] = per_rank
        line["score_gather_ms"] = round(gather_ms, 4)
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"], line["parity"] = cpu_baseline(args, w, host, ft, model)
    return line


def bench_shim(args, U, C, L, spec):
    """The drop-in C++ API end to end: tests/cpp/build/bench_shim (built against the reference
    headers) scores std::vector<RankingExample> batches with private Segments through
    seqfm::b200::Scorer::rank_forward_batch; host wall clock around the whole call."""
    exe = os.path.join(ROOT, "tests", "cpp", "build", "bench_shim")
    if not os.path.exists(exe):
        return None
    try:
        r = subprocess.run([exe, str(U), str(C), str(L), str(spec.n_layers), str(spec.d_model), str(spec.n_heads),
                            str(max(3, args.steps // 2)), "2"], capture_output=True, text=True, timeout=600)
        return json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else {"error": r.stderr[-300:]}
    except Exception as e:  # reported, not fatal: the headline numbers do not depend on it
        return {"error": str(e)[:300]}


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(args, w, host: Batch, ft, model):
    """The reference's CPU path (oracle/_ref, the unmodified sources) on bounded samples of the same
    workload: (i) rank_forward_batch as shipped, one thread, on 2 users with all
    their candidates; (ii) the same fanned out over all host threads on 2 users per thread. Each is
    the median of 3 timed runs; `value` is (ii)."""
    from oracle import pyoracle
    kind = "reference" if pyoracle.have_reference() else "port"
    impl = pyoracle.reference() if kind == "reference" else pyoracle.oracle()
    threads = os.cpu_count() or 1
    U = CONFIGS[args.config]["U"] if not args.users else args.users

    def sample(S):
        rows = np.nonzero(np.isin(np.arange(host.n_rows) % U, np.arange(S)))[0]
        return rows, host.take(rows)

    def median_rate(sub, n_threads):
        ts = []
        out = None
        for _ in range(3):
            t0 = time.perf_counter()
            if kind == "reference" and n_threads > 1:
                out = impl.rank_forward_batch(w, ft, sub, n_threads=n_threads)
            else:
                out = impl.rank_forward_batch(w, ft, sub)
            ts.append(time.perf_counter() - t0)
        return sub.n_rows / float(np.median(ts)), float(np.median(ts)), out

    rows1, sub1 = sample(min(U, 2))
    v1, t1, _ = median_rate(sub1, 1)
    S = min(U, max(2, args.cpu_users or 2 * threads)) if kind == "reference" else 2
    rows, sub = sample(S)
    vn, tn, (rl, rm, _, _) = median_rate(sub, threads if kind == "reference" else 1)
    cores = min(threads, S) if kind == "reference" else 1
    lg, ml, _ = model.rank_forward_batch(sub, ft)
    scale = max(1e-3, float(np.abs(rl).max()))
    parity = {"rows": int(len(rows)), "max_rel_err_logits": float(np.abs(lg - rl).max() / scale),
              "max_rel_err_module_logits": float(np.abs(ml - rm).max() / max(1e-3, float(np.abs(rm).max()))),
              "tolerance": 1e-2, "vs": kind}
    return ({"value": round(vn, 2), "unit": UNIT, "cores": cores, "kind": kind, "cpu_model": cpu_model(),
             "nproc": threads, "statistic": "median of 3",
             "sample": f"{S} users x {host.n_rows // U} candidates ({len(rows)} rows) of the same batch, "
                       f"{tn:.2f} s median wall on {cores} threads",
             "single_thread_as_shipped": {"value": round(v1, 2), "unit": UNIT, "cores": 1,
                                          "sample": f"{min(U, 2)} users x {host.n_rows // U} candidates "
                                                    f"({len(rows1)} rows), {t1:.2f} s median wall"}}, parity)


def run_reference(args):
    from oracle import pyoracle
    cfg = CONFIGS[args.config]
    U, C, L = cfg["U"], cfg["C"], cfg["L"]
    w = init_weights(cfg["spec"], seed=42)
    ft = FinetuneSpec(max_events=L)
    if not pyoracle.have_reference():
        kind, impl, threads = "port", pyoracle.oracle(), 1
    else:
        kind, impl, threads = "reference", pyoracle.reference(), os.cpu_count() or 1
    S = min(U, args.cpu_users or max(2, threads))  # users per step: one user per thread
    host = make_batch(U, C, L, seed=1, layout="interleaved")
    rows = np.nonzero(np.isin(np.arange(host.n_rows) % U, np.arange(S)))[0]
    sub = host.take(rows)
    run = (lambda: impl.rank_forward_batch(w, ft, sub, n_threads=threads)) if kind == "reference" else \
        (lambda: impl.rank_forward_batch(w, ft, sub))
    for _ in range(args.warmup):
        run()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run()
    dt = (time.perf_counter() - t0) / args.steps
    v = round(len(rows) / dt, 2)
    s = cfg["spec"]
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 2), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
            "config": {"workload": f"{args.config}: {s.n_layers} layers, d={s.d_model}, {s.n_heads} heads, L={L}, "
                                   f"{U} users x {C} candidates (each step: a {S}-user sample)"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": min(threads, S), "kind": kind,
                             "cpu_model": cpu_model(), "nproc": os.cpu_count() or 1,
                             "sample": f"{S} users x {C} candidates per step ({len(rows)} rows)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="pinfm-base", choices=sorted(CONFIGS))
    ap.add_argument("--users", type=int, default=0, help="override unique users per GPU")
    ap.add_argument("--cpu-users", type=int, default=0)
    ap.add_argument("--private-rows", action="store_true", help="every row carries its own event copy")
    ap.add_argument("--no-private", action="store_true", help="skip the private-rows side measurement")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-shim", action="store_true", help="skip the C++ drop-in API e2e leg")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    line = run_ours(args, rank, world, local_rank)
    if rank == 0 and line:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
